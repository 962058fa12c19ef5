#!/usr/bin/env python
"""Eager vs graph-replayed fused rounds at P ranks: per-CTA %globaltimer trace of one
round in each form (kernel span, entry wait, CTA start skew) and the device time of a
run of rounds, to locate where the graph form spends its extra time.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/graph_trace_probe.py
"""

import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200 as L  # noqa: E402
from paper_2203_13085_b200 import _native as N  # noqa: E402


def summary(tr):
    t0 = min(t[0] for t in tr)
    out = {"span_us": (max(t[3] for t in tr) - t0) / 1e3,
           "start_skew_us": (max(t[0] for t in tr) - t0) / 1e3,
           "entry_wait_us_median": statistics.median((t[1] - t[0]) / 1e3 for t in tr),
           "entry_passed_last_us": (max(t[1] for t in tr) - t0) / 1e3}
    mids = [t for t in tr if t[2] > t[1]]
    if mids:  # phase A (own chunk, until the mid barrier passed) and phase B
        out["mid_passed_first_us"] = (min(t[2] for t in mids) - t0) / 1e3
        out["mid_passed_last_us"] = (max(t[2] for t in mids) - t0) / 1e3
        out["phase_b_us_median"] = statistics.median((t[3] - t[2]) / 1e3 for t in mids)
        out["first_end_us"] = (min(t[3] for t in tr) - t0) / 1e3
    return out


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    n = 25_557_032
    algo = int(os.environ.get("ALGO", N.ALGO_AUTO))
    comm = L.P2PCommunicator(n, timeout_s=60.0)
    gen = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(n, device="cuda", generator=gen) * 0.02
    grads = [torch.randn(n, device="cuda", generator=gen) * 1e-2 for _ in range(2)]
    compute = torch.cuda.Stream()
    out = {"rank": rank, "world": world}
    with torch.cuda.stream(compute):
        w = L.LASGDWorker(x, grads[0], comm=comm, sync_period=1, pipeline="fused", lr=0.1, algo=algo,
                          sgd=L.SgdConfig(0.9, 0.0, 1e-4, True), compute_stream=compute)
        for t in range(4):
            w.g = grads[t % 2]
            w.step()
        torch.cuda.synchronize()
        dist.barrier()
        comm.set_trace(True)
        w.g = grads[0]
        w.step()
        comm.set_trace(False)
        torch.cuda.synchronize()
        out["eager_round"] = summary(comm.read_trace())
        w.g = grads[1]
        w.step()
        # a run of 20 rounds, eager vs graph, device time
        for name in ("eager", "graph"):
            torch.cuda.synchronize()
            dist.barrier()
            if name == "graph":
                comm.set_trace(True)
                g = w.capture([grads[t % 2] for t in range(20)])
                comm.set_trace(False)
                g.replay()
                torch.cuda.synchronize()
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(compute)
            if name == "graph":
                g.replay()
            else:
                for t in range(20):
                    w.g = grads[t % 2]
                    w.step()
            b.record(compute)
            torch.cuda.synchronize()
            out[f"{name}_ms_per_round"] = a.elapsed_time(b) / 20
            if name == "graph":
                out["graph_round"] = summary(comm.read_trace())
    res = [None] * world
    dist.all_gather_object(res, out)
    if rank == 0:
        for r in res:
            print(json.dumps(r), flush=True)
    w.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

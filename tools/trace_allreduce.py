#!/usr/bin/env python
"""Per-CTA timeline of the P2P mean all-reduce (globaltimer stamps written by the
kernel when tracing is on).  Summarises launch span, CTA start skew, barrier wait and
per-CTA data-phase time distribution on every rank.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/trace_allreduce.py
"""

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200 as L  # noqa: E402


def summarise(tr):
    t0 = [t[0] for t in tr]
    base = min(t0)
    span = (max(t[3] for t in tr) - base) / 1e3
    wait = [(t[1] - t[0]) / 1e3 for t in tr]
    data = [(t[3] - t[1]) / 1e3 for t in tr]
    mid = [(t[2] - t[1]) / 1e3 for t in tr if t[2] > t[1]]
    return {"span_us": span, "start_skew_us": (max(t0) - base) / 1e3,
            "entry_wait_us": [min(wait), statistics.median(wait), max(wait)],
            "cta_work_us": [min(data), statistics.median(data), max(data)],
            "first_end_us": (min(t[3] for t in tr) - base) / 1e3,
            "rs_plus_midwait_us": [min(mid), statistics.median(mid), max(mid)] if mid else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="16,102.228128,1024")
    ap.add_argument("--nblocks", default="64,128")
    ap.add_argument("--fused", action="store_true", help="trace the fused round kernel (K7) instead of K2/K3")
    ap.add_argument("--algos", default="1,2", help="1 one-shot, 2 two-shot, 3 push (fused only)")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    s = torch.cuda.Stream(device=dev)
    for mb in [float(v) for v in a.sizes_mb.split(",")]:
        n = int(mb * 1e6 / 4)
        comm = L.P2PCommunicator(n, timeout_s=60.0)
        comm.snapshots[0].normal_()
        comm.snapshots[1].normal_()
        xs, gs, ms = (torch.randn(n, device=dev) for _ in range(3))
        slot = [0]

        def launch(algo, nb):
            if not a.fused:
                return comm.allreduce(slot[0], algo, stream=s)
            r = comm.fused_round(slot[0], xs, gs, 0.01, m=ms, momentum=0.9, weight_decay=1e-4, nesterov=True,
                                 algo=algo, nblocks=nb, stream=s)
            slot[0] ^= 1
            return r
        for nb in [int(v) for v in a.nblocks.split(",")]:
            comm.set_nblocks(nb)
            for algo in [int(v) for v in a.algos.split(",")]:
                with torch.cuda.stream(s):
                    for i in range(4):
                        launch(algo, nb)
                    torch.cuda.synchronize()
                    dist.barrier()
                    comm.set_trace(True)
                    launch(algo, nb)
                    torch.cuda.synchronize()
                    comm.set_trace(False)
                tr = comm.read_trace()
                out = [None] * world
                dist.all_gather_object(out, summarise(tr))
                if rank == 0:
                    for r, sm in enumerate(out):
                        print(json.dumps({"MB": mb, "nblocks": nb, "algo": algo, "rank": r, **sm}), flush=True)
        dist.barrier()
        comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

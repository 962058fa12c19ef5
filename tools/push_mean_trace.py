#!/usr/bin/env python
"""Per-CTA %globaltimer trace of one push mean (ALGO_PUSH all-reduce) at P ranks:
start, contributions landed everywhere (end-signal wait passed), own means issued, end.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/push_mean_trace.py
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


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    n = int(float(os.environ.get("MB", "102.228128")) * 1e6 / 4)
    comm = L.P2PCommunicator(n, nblocks=int(os.environ.get("NB", "128")), timeout_s=60.0)
    comm.snapshots[0].normal_()
    s = torch.cuda.Stream()
    out = {"rank": rank, "world": world, "MB": 4 * n / 1e6}
    for _ in range(5):
        comm.allreduce(0, N.ALGO_PUSH, stream=s)
    torch.cuda.synchronize()
    dist.barrier()
    comm.set_trace(True)
    comm.device_barrier(s)
    comm.allreduce(0, N.ALGO_PUSH, stream=s)
    comm.set_trace(False)
    torch.cuda.synchronize()
    tr = [t for t in comm.read_trace() if t[0]]
    t0 = min(t[0] for t in tr)
    us = lambda v: round((v - t0) / 1e3, 1)  # noqa: E731
    out.update({"ctas": len(tr), "start_last_us": us(max(t[0] for t in tr)),
                "landed_first_us": us(min(t[1] for t in tr)), "landed_last_us": us(max(t[1] for t in tr)),
                "means_issued_first_us": us(min(t[2] for t in tr)), "means_issued_last_us": us(max(t[2] for t in tr)),
                "end_first_us": us(min(t[3] for t in tr)), "end_last_us": us(max(t[3] for t in tr)),
                "reduce_us_median": round(statistics.median((t[2] - t[1]) / 1e3 for t in tr), 1)})
    res = [None] * world
    dist.all_gather_object(res, out)
    if rank == 0:
        for r in res:
            print(json.dumps(r), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

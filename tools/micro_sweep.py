#!/usr/bin/env python
"""Param-sync microbenchmark (BASELINE.json configs[4]): snapshot + mean all-reduce +
elastic pull over 1 MB .. 1 GB flat fp32 buffers at P ranks, CUDA-event timed,
max over ranks.  Also sweeps the all-reduce algorithm and the CTA budget.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/micro_sweep.py --sizes-mb 1,16,128,1024 --nblocks 16,32,64,128

Prints one JSON line per (size, algo, nblocks) on rank 0.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200 as L  # noqa: E402
from paper_2203_13085_b200 import _native as N  # noqa: E402
from paper_2203_13085_b200 import kernels as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,102.228128,256,1024")
    ap.add_argument("--nblocks", default="32")
    ap.add_argument("--algos", default="oneshot,twoshot")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--threads", type=int, default=256)
    ap.add_argument("--fused-algos", default="auto,oneshot,push",
                    help="fused-round algorithms to time per size ('' to skip)")
    ap.add_argument("--nvls-nblocks", default="",
                    help="also time the in-switch (NVLS, tolerance-mode) mean with these CTA counts")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    s = torch.cuda.Stream(device=dev, priority=-1)
    codes = {"oneshot": N.ALGO_ONESHOT, "twoshot": N.ALGO_TWOSHOT, "ce": N.ALGO_CE, "push": N.ALGO_PUSH}

    def tmax(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for mb in [float(x) for x in a.sizes_mb.split(",")]:
        n = int(mb * 1e6 / 4) // 4 * 4 + (1 if world > 1 else 0)  # ragged on purpose
        comm = L.P2PCommunicator(n, nblocks=32, threads=a.threads, timeout_s=60.0)
        x = torch.randn(n, device=dev)
        comm.snapshots[0].copy_(x)
        comm.snapshots[1].copy_(x)
        torch.cuda.synchronize()
        for nb in [int(v) for v in a.nblocks.split(",")]:
            comm.set_nblocks(nb)
            for alg in a.algos.split(","):
                code = codes[alg]
                with torch.cuda.stream(s):
                    for i in range(a.warmup):
                        comm.allreduce(i % 2, code, stream=s)
                    torch.cuda.synchronize()
                    dist.barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    for i in range(a.reps):
                        comm.allreduce(i % 2, code, stream=s)
                    e1.record(s)
                    torch.cuda.synchronize()
                    ar_ms = tmax(e0.elapsed_time(e1) / a.reps)
                    # full round: snapshot (K1) -> all-reduce (K2/K3) -> pull (K4)
                    dist.barrier()
                    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    f0.record(s)
                    for i in range(a.reps):
                        K.snapshot(comm.snapshots[i % 2], x, stream=s)
                        comm.allreduce(i % 2, code, stream=s)
                        K.elastic_pull(x, comm.snapshots[i % 2], comm.xbar, 0.5, stream=s)
                    f1.record(s)
                    torch.cuda.synchronize()
                    round_ms = tmax(f0.elapsed_time(f1) / a.reps)
                nv = comm.bytes_per_node(code)
                if rank == 0:
                    print(json.dumps({"P": world, "MB": 4 * n / 1e6, "n": n, "algo": alg, "nblocks": nb,
                                      "threads": a.threads, "allreduce_ms": ar_ms, "nvlink_bytes": nv,
                                      "nvlink_gbs": nv / (ar_ms * 1e-3) / 1e9,
                                      "busbw_gbs": 2 * (world - 1) / world * 4 * n / (ar_ms * 1e-3) / 1e9,
                                      "round_ms": round_ms}), flush=True)
        # the fused round (K7 / K8: local step + mean + pull + next snapshot in one kernel)
        # against the same work as separate kernels (K5, K1, K2/K3, K4)
        if a.fused_algos:
            g = torch.randn(n, device=dev) * 1e-3
            m = torch.zeros(n, device=dev)
            fk = dict(m=m, momentum=0.9, weight_decay=1e-4, nesterov=True, alpha=0.5, stream=s)
            fcodes = {"auto": N.ALGO_AUTO, "oneshot": N.ALGO_ONESHOT, "twoshot": N.ALGO_TWOSHOT, "push": N.ALGO_PUSH}
            for alg in a.fused_algos.split(","):
                code = fcodes[alg]
                with torch.cuda.stream(s):
                    for i in range(a.warmup):
                        comm.fused_round(i % 2, x, g, 1e-3, algo=code, **fk)
                    torch.cuda.synchronize()
                    dist.barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    for i in range(a.reps):
                        comm.fused_round(i % 2, x, g, 1e-3, algo=code, **fk)
                    e1.record(s)
                    torch.cuda.synchronize()
                    f_ms = tmax(e0.elapsed_time(e1) / a.reps)
                    dist.barrier()
                    e0.record(s)
                    for i in range(a.reps):
                        K.sgd_step(x, g, 1e-3, m=m, momentum=0.9, weight_decay=1e-4, nesterov=True, stream=s)
                        K.snapshot(comm.snapshots[i % 2], x, stream=s)
                        comm.allreduce(i % 2, N.ALGO_AUTO, stream=s)
                        K.elastic_pull(x, comm.snapshots[i % 2], comm.xbar, 0.5, stream=s)
                    e1.record(s)
                    torch.cuda.synchronize()
                    sep_ms = tmax(e0.elapsed_time(e1) / a.reps)
                if rank == 0:
                    print(json.dumps({"P": world, "MB": 4 * n / 1e6, "n": n, "fused_algo": alg,
                                      "resolved": comm.resolve_fused_algo(code), "fused_round_ms": f_ms,
                                      "separate_kernels_ms": sep_ms, "speedup": sep_ms / f_ms,
                                      "busbw_equiv_gbs": 2 * (world - 1) / world * 4 * n / (f_ms * 1e-3) / 1e9}),
                          flush=True)
            del g, m
        if a.nvls_nblocks:
            nc = L.P2PCommunicator(n, nblocks=32, threads=a.threads, timeout_s=60.0, nvls=True)
            nc.snapshots[0].copy_(x)
            nc.snapshots[1].copy_(x)
            torch.cuda.synchronize()
            for nb in [int(v) for v in a.nvls_nblocks.split(",")]:
                nc.set_nblocks(nb)
                with torch.cuda.stream(s):
                    for i in range(a.warmup):
                        nc.allreduce(i % 2, N.ALGO_NVLS, stream=s)
                    torch.cuda.synchronize()
                    dist.barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    for i in range(a.reps):
                        nc.allreduce(i % 2, N.ALGO_NVLS, stream=s)
                    e1.record(s)
                    torch.cuda.synchronize()
                    ar_ms = tmax(e0.elapsed_time(e1) / a.reps)
                if rank == 0:
                    print(json.dumps({"P": world, "MB": 4 * n / 1e6, "n": n, "algo": "nvls", "nblocks": nb,
                                      "allreduce_ms": ar_ms,
                                      "busbw_gbs": 2 * (world - 1) / world * 4 * n / (ar_ms * 1e-3) / 1e9}),
                          flush=True)
            dist.barrier()
            nc.close()
        # NCCL all-reduce (sum) of the same buffer, for context (not on the product path)
        y = x.clone()
        for _ in range(a.warmup):
            dist.all_reduce(y)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            dist.all_reduce(y)
        e1.record()
        torch.cuda.synchronize()
        nccl_ms = tmax(e0.elapsed_time(e1) / a.reps)
        if rank == 0:
            print(json.dumps({"P": world, "MB": 4 * n / 1e6, "algo": "nccl_allreduce_sum", "allreduce_ms": nccl_ms,
                              "busbw_gbs": 2 * (world - 1) / world * 4 * n / (nccl_ms * 1e-3) / 1e9}), flush=True)
        del y
        comm.close()
        del x
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Timeline of one overlap-pipeline training step (the all-reduce of the
snapshot runs while the next minibatches compute): the side-stream mean all-reduce's
per-CTA %globaltimer stamps (start, entry barrier passed, mid barrier passed, end) next
to compute-stream stamps around the forward/backward it overlaps, on every rank.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/overlap_timeline.py > profiles/r02/overlap_timeline_p2.jsonl

Step t closes a round: the pull writes the next snapshot and launches its mean on the
side stream (traced).  Step t+1's forward/backward (one CUDA graph) runs meanwhile; its
local step then waits for the mean only at the next boundary.  All times are ns
relative to the start of step t+1's forward on that rank's GPU.
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
from paper_2203_13085_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--warm", type=int, default=6)
    ap.add_argument("--repeats", type=int, default=3)
    args = ap.parse_args()
    import torchvision

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    torch.backends.cudnn.benchmark = True
    classes, hw = (1000, 224) if args.model != "resnet18" else (10, 32)
    model = getattr(torchvision.models, args.model)(num_classes=classes).to(dev).to(memory_format=torch.channels_last)
    flat = L.FlatParams(model, channels_last=True, align_bytes=256)
    dist.broadcast(flat.x, 0)
    comm = L.P2PCommunicator(flat.numel, timeout_s=60.0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    images = torch.randn(args.batch, 3, hw, hw, device=dev, generator=gen).to(memory_format=torch.channels_last)
    labels = torch.randint(0, classes, (args.batch,), device=dev, generator=gen)
    lossf = torch.nn.CrossEntropyLoss()

    def fb():
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            lossf(model(images), labels).backward()

    step = L.GraphedStep(flat, fb)
    compute = torch.cuda.Stream(device=dev, priority=-1)
    stamps = torch.zeros(8, dtype=torch.int64, device=dev)

    def stamp(i):
        N.check(N.lib().lasgd_stamp(ctypes_ptr(stamps, i), ctypes_stream(compute)))

    with torch.cuda.stream(compute):
        w = L.LASGDWorker(flat.x, flat.g, comm=comm, sync_period=1, pipeline="overlap", lr=0.1,
                          sgd=L.SgdConfig(0.9, 0.0, 1e-4, True), compute_stream=compute)
        for _ in range(args.warm):
            step()
            w.step()
    torch.cuda.synchronize()
    for rep in range(args.repeats):
        dist.barrier()
        with torch.cuda.stream(compute):
            step()
            comm.set_trace(True)
            w.step()  # closes round t: pull + next snapshot, launches its mean (traced)
            comm.set_trace(False)
            stamp(0)
            step()  # step t+1 forward/backward: the mean runs under it
            stamp(1)
            w.step()  # next boundary: waits for the mean, pulls, launches the next one
            stamp(2)
        torch.cuda.synchronize()
        st = stamps.cpu().tolist()
        tr = comm.read_trace()
        base = st[0]
        starts = [t[0] - base for t in tr]
        entries = [t[1] - base for t in tr]
        ends = [t[3] - base for t in tr]
        rec = {"rank": rank, "world": world, "repeat": rep, "model": args.model, "n": flat.numel,
               "allreduce_algo": {1: "oneshot", 2: "twoshot"}.get(comm.resolve_algo(N.ALGO_AUTO)),
               "ctas": len(tr),
               "fwd_bwd_start_ns": 0, "fwd_bwd_end_ns": st[1] - base, "next_boundary_end_ns": st[2] - base,
               "allreduce_first_cta_start_ns": min(starts), "allreduce_last_cta_start_ns": max(starts),
               "allreduce_entry_passed_ns": [min(entries), int(statistics.median(entries)), max(entries)],
               "allreduce_last_cta_end_ns": max(ends),
               "allreduce_hidden": max(ends) <= st[1] - base,
               "allreduce_span_ns": max(ends) - min(starts)}
        out = [None] * world
        dist.all_gather_object(out, rec)
        if rank == 0:
            for r in out:
                print(json.dumps(r), flush=True)
    w.drain()
    torch.cuda.synchronize()
    w.close()
    comm.close()
    dist.destroy_process_group()


def ctypes_ptr(t, i):
    import ctypes

    return ctypes.c_void_p(t.data_ptr() + 8 * i)


def ctypes_stream(s):
    import ctypes

    return ctypes.c_void_p(s.cuda_stream)


if __name__ == "__main__":
    main()

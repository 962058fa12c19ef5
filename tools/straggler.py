#!/usr/bin/env python
"""Straggler / skew runs: LASGD's dynamic rate vs lock-step schedules on real training
(the shape of the paper's Table 3).

Real fwd/bwd (torchvision model, bf16 autocast, channels_last, synthetic data) on every
rank, with an injected per-step delay on the compute stream:

* ``none``   — no delay;
* ``slow``   — the last rank is slower by ``--slow-frac`` of the measured step time;
* ``jitter`` — every rank, every step, an exponential delay with mean
  ``--jitter-frac`` of the step time (seeded per rank and step).

Variants: ``sgd_ar`` (SGDARWorker: gradient mean every step), ``lasgd_fused`` /
``lasgd_overlap`` (deterministic, one round per step), ``lasgd_adaptive_t{T}``
(adaptive completion, tau_max = T).  Lock-step variants run ``--steps`` steps; the
adaptive ones run for the same wall time as ``lasgd_overlap`` and every rank takes as
many local steps as it can (ranks then drain unequal launch counts).  images/s =
(sum over ranks of local steps) x batch / (max over ranks of the device time).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/straggler.py
"""

import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200 as L  # noqa: E402

MODELS = {"resnet18": (32, 10), "resnet50": (224, 1000), "mobilenet_v2": (224, 1000)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=sorted(MODELS), default="resnet18")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--scenarios", default="none,slow,jitter")
    ap.add_argument("--slow-frac", type=float, default=0.5)
    ap.add_argument("--jitter-frac", type=float, default=0.25)
    ap.add_argument("--tau-max", default="2,4")
    ap.add_argument("--max-host-lead", type=int, default=2, help="adaptive: steps the host may run ahead of the GPU")
    ap.add_argument("--no-graphs", action="store_true", help="eager fwd/bwd instead of CUDA-graph replay")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)

    import torchvision

    hw, classes = MODELS[a.model]
    torch.backends.cudnn.benchmark = True
    torch.manual_seed(0)
    model = getattr(torchvision.models, a.model)(num_classes=classes).to(dev).to(memory_format=torch.channels_last)
    flat = L.FlatParams(model, channels_last=True)
    own_g = flat.g
    x0 = flat.x.clone()
    comm = L.P2PCommunicator(flat.numel, timeout_s=120.0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    images = torch.randn(a.batch, 3, hw, hw, device=dev, generator=gen).to(memory_format=torch.channels_last)
    labels = torch.randint(0, classes, (a.batch,), device=dev, generator=gen)
    lossf = torch.nn.CrossEntropyLoss()
    sgd = L.SgdConfig(0.9, 0.0, 1e-4, True)
    compute = torch.cuda.Stream(device=dev, priority=-1)

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t.item())

    # clock calibration for torch.cuda._sleep (cycles per ms) and the bare step time
    with torch.cuda.stream(compute):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1000)
        e0.record(compute)
        torch.cuda._sleep(20_000_000)
        e1.record(compute)
    torch.cuda.synchronize()
    cycles_per_ms = 20_000_000 / e0.elapsed_time(e1)

    def fwd_bwd_eager():
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            loss = lossf(model(images), labels)
        loss.backward()

    if a.no_graphs:
        def fwd_bwd():
            flat.zero_grad()
            fwd_bwd_eager()
    else:
        fwd_bwd = L.GraphedStep(flat, fwd_bwd_eager)

    with torch.cuda.stream(compute):
        for _ in range(a.warmup):
            fwd_bwd()
        e0.record(compute)
        for _ in range(20):
            fwd_bwd()
        e1.record(compute)
    torch.cuda.synchronize()
    step_ms = max_over_ranks(e0.elapsed_time(e1) / 20)

    def delay_fn(scenario):
        if scenario == "none":
            return lambda t: 0.0
        if scenario == "slow":
            d = a.slow_frac * step_ms if rank == world - 1 else 0.0
            return lambda t: d
        if scenario == "jitter":
            import random

            def f(t):
                return random.Random(1_000_003 * rank + t).expovariate(1.0 / (a.jitter_frac * step_ms))
            return f
        raise ValueError(scenario)

    def make(variant):
        flat.x.copy_(x0)
        flat.bind_grads(own_g)
        if variant == "sgd_ar":
            return L.SGDARWorker(flat.x, comm=comm, sgd=sgd, lr=0.01, compute_stream=compute, flat=flat)
        kw = dict(comm=comm, sync_period=1, alpha=1.0, mode="pull", sgd=sgd, lr=0.01, compute_stream=compute)
        if variant == "lasgd_fused":
            return L.LASGDWorker(flat.x, flat.g, pipeline="fused", **kw)
        if variant == "lasgd_overlap":
            return L.LASGDWorker(flat.x, flat.g, pipeline="overlap", **kw)
        tm = int(variant.rsplit("_t", 1)[1])
        return L.LASGDWorker(flat.x, flat.g, pipeline="overlap", adaptive=True, tau_max=tm,
                             max_host_lead=a.max_host_lead, **kw)

    def run(variant, scenario, steps=None, budget_s=None):
        delay = delay_fn(scenario)
        with torch.cuda.stream(compute):
            w = make(variant)

            def one(t):
                fwd_bwd()
                d = delay(t)
                if d > 0:
                    torch.cuda._sleep(int(d * cycles_per_ms))
                w.step()

            for t in range(a.warmup):
                one(t)
            if hasattr(w, "drain"):
                w.drain()
        torch.cuda.synchronize()
        dist.barrier()
        if hasattr(w, "reset_records"):
            w.reset_records()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        with torch.cuda.stream(compute):
            b0.record(compute)
            h0 = time.perf_counter()
            while (steps is not None and n < steps) or (budget_s is not None and time.perf_counter() - h0 < budget_s):
                one(a.warmup + n)
                n += 1
            if hasattr(w, "drain"):
                w.drain()
            b1.record(compute)
        torch.cuda.synchronize()
        ms = max_over_ranks(b0.elapsed_time(b1))
        total = sum_over_ranks(n)
        counts = [None] * world
        dist.all_gather_object(counts, n)
        hist = {str(k): v for k, v in sorted(dict(getattr(w, "tau_hist", {})).items())}
        if hasattr(w, "close"):
            w.close()
        dist.barrier()
        return {"images_per_s": total * a.batch / (ms / 1e3), "ms": ms, "steps_per_rank": counts,
                "tau_histogram": hist or None}

    taus = [int(v) for v in a.tau_max.split(",") if v]
    rows = []
    for scenario in a.scenarios.split(","):
        res = {}
        for variant in ("sgd_ar", "lasgd_fused", "lasgd_overlap"):
            res[variant] = run(variant, scenario, steps=a.steps)
        budget = res["lasgd_overlap"]["ms"] / 1e3
        for tm in taus:
            res[f"lasgd_adaptive_t{tm}"] = run(f"lasgd_adaptive_t{tm}", scenario, budget_s=budget)
        base = res["sgd_ar"]["images_per_s"]
        for variant, r in res.items():
            row = {"model": a.model, "batch_per_gpu": a.batch, "n_gpus": world, "scenario": scenario,
                   "fwd_bwd": "eager" if a.no_graphs else "cuda_graph", "max_host_lead": a.max_host_lead,
                   "bare_step_ms": step_ms, "variant": variant, "speedup_vs_sgd_ar": r["images_per_s"] / base, **r}
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
    if rank == 0 and a.out:
        with open(a.out, "w") as f:
            for row in rows:
                f.write(json.dumps(row) + "\n")
    comm.close()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

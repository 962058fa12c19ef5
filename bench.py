#!/usr/bin/env python
"""Benchmark of the LASGD parameter-synchronisation hot path (BASELINE.json metric).

Workload (BASELINE.json configs[2], the metric's config): ResNet-50 LASGD,
batch 256 per GPU, parameters in one contiguous fp32 flat buffer of
n = 25,557,032 (torchvision resnet50); `--model resnet18|mobilenet_v2` selects
the other BASELINE configs.  A "step" is one pass of the hot path over one
minibatch's synthetic gradient under the deterministic schedule (sync period 1,
the paper's tau_max = 1): the local step (Nesterov momentum 0.9, weight decay
1e-4 — PAPER.md:229) and the round boundary — mean of every rank's snapshot
over NVLink, elastic pull, next snapshot.  Default `--pipeline fused`: one
kernel per boundary step (P=1: K5 + snapshot; P=2: K8 mirror push; P>=3: K8 staged
push — `--algo` overrides); `--pipeline overlap`: K5, then K4 with the K2/K3 all-reduce on a
low-priority side stream.  images/s = images whose gradients the sync path
consumed per second over all ranks.

Also reported (not the headline): the real training step (forward/backward in
PyTorch, bf16 autocast, channels_last) with the sync path under each pipeline,
adaptive completion (tau histogram), the SGD-AR baseline (gradient mean every
step, on the same P2P all-reduce and on NCCL), and sync disabled (the no-sync
ceiling) -> exposed sync ms/step.

`--impl reference` times the reference's own CPU algorithm (f64, delta
bookkeeping, ring-order mean; the C restatement in oracle/, all host threads,
P workers in-process like LoopbackTransport) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResNet-50 LASGD images/sec at 1/2/4/8 B200; exposed sync ms/step; sync GB/s vs roofline"
# BASELINE.json configs: ResNet-50 / ImageNet 224 (the metric's config), ResNet-18 / CIFAR 32 (10 classes),
# MobileNetV2 / ImageNet 224.  params = torchvision parameter counts (flat fp32 buffer length).
MODELS = {
    "resnet50": {"params": 25_557_032, "image": 224, "classes": 1000, "ctor": "resnet50"},
    "resnet18": {"params": 11_181_642, "image": 32, "classes": 10, "ctor": "resnet18"},
    "mobilenet_v2": {"params": 3_504_872, "image": 224, "classes": 1000, "ctor": "mobilenet_v2"},
}
NVLINK_PEAK_GBS = 770.0  # measured peer copy per direction, /opt/skills/guides/B200_PROFILING.md
HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)  # 20 ms of sync path at N=1: robust to host hiccups
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--model", choices=sorted(MODELS), default="resnet50")
    ap.add_argument("--sync-period", type=int, default=1)
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--algo", choices=["auto", "oneshot", "twoshot", "push"], default="auto",
                    help="all-reduce / fused-round algorithm (push: K8, fused pipeline only)")
    ap.add_argument("--nblocks", type=int, default=128)
    ap.add_argument("--pipeline", choices=["overlap", "fused"], default="fused",
                    help="overlap: K5 | K4 | K2/K3 on a side stream; fused: one K7 pass per round boundary")
    ap.add_argument("--fused-nblocks", type=int, default=0, help="CTAs of the fused kernel (0 = 2 per SM)")
    ap.add_argument("--train-block", type=int, default=2, help="training steps per timed block")
    ap.add_argument("--train-reps", type=int, default=24, help="interleaved repetitions of every training leg")
    ap.add_argument("--train-warmup", type=int, default=4)
    ap.add_argument("--flat-align", type=int, default=256, help="byte alignment of every tensor in the flat buffer")
    ap.add_argument("--bucket-mb", type=int, default=25, help="gradient bucket size of the bucketed SGD-AR / DDP legs")
    ap.add_argument("--bucket-ctas", type=int, default=0, help="CTAs of each bucketed SGD-AR launch (0: 2 per SM)")
    ap.add_argument("--legs", default="", help="comma list: run only these training legs (and their baselines)")
    ap.add_argument("--step-graph", action="store_true",
                    help="N=1 training legs: capture forward + backward + the sync step in one graph per leg "
                         "(each leg then replays its own forward/backward graph, whose memory placement alone "
                         "moves the step time by up to ~0.4 ms; by default every leg replays the same "
                         "forward/backward graph and issues its sync step after it)")
    ap.add_argument("--nvls-leg", action="store_true",
                    help="N>1: add a training leg on the NVLS (in-switch, tolerance-mode) side-stream mean")
    ap.add_argument("--side-priority", type=int, default=0,
                    help="training legs: CUDA priority of the communicator's side stream (0 low, -1 high)")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="training leg: eager fwd/bwd instead of CUDA-graph replay")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernels-only", action="store_true", help="short run for ncu: sync path only")
    ap.add_argument("--no-virtual", action="store_true", help="skip the virtual-rank (P=2/4/8 on one GPU) kernels")
    ap.add_argument("--no-sync-graph", action="store_true",
                    help="N=1: issue the timed steps one by one instead of replaying them as one CUDA graph")
    ap.add_argument("--sync-graph", action="store_true",
                    help="N>1: replay the timed steps as one CUDA graph (fused pipeline; ~2.5%% slower per round "
                         "than eager launches behind the hold kernel, DESIGN.md §12)")
    return ap.parse_args()


def config_dict(args, world, fused_algo=None):
    return {
        "workload": f"{args.model}-lasgd-sync",
        "params": MODELS[args.model]["params"],
        "batch_per_gpu": args.batch,
        "sync_period": args.sync_period,
        "alpha": args.alpha,
        "local_step": "sgd momentum=0.9 nesterov weight_decay=1e-4 lr=0.1",
        "allreduce": args.algo,
        "fused_round_algo": fused_algo,
        "pipeline": args.pipeline,
        "sm_budget_ctas": args.nblocks,
        "parallelism": f"dp{world}",
        "l2": "no flush: every kernel streams 3-5 buffers of 102 MB (> 126 MB L2); gradients alternate between 2 buffers",
    }


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", str(gpu), "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
            return
        # nvidia-smi's NVML start-up contends with kernel launches in this process: wait
        # for its first sample so that start-up stays outside the timed region.
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 10.0 and self.p.poll() is None and os.path.getsize(self.f.name) == 0:
            time.sleep(0.01)

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        if not sm:
            return None
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}
        if pw:
            out["power_w_median"] = statistics.median(pw)
            out["sm_mhz_min"] = min(sm)
        return out


# ---------------------------------------------------------------------------- helpers
class Hold:
    """lasgd_hold: a one-thread kernel that holds a stream until released, so a whole
    timed region is enqueued before the device starts it (bounded: 5 s; under ncu, which serialises launches, it always waits the 5 s)."""

    def __init__(self, N):
        import ctypes

        self._N, self._c = N, ctypes
        self._h = ctypes.c_void_p()
        N.check(N.lib().lasgd_hold_create(ctypes.byref(self._h)), "lasgd_hold_create")

    def enqueue(self, stream):
        self._N.check(self._N.lib().lasgd_hold_enqueue(self._h, self._c.c_void_p(stream.cuda_stream), 5.0))

    def release(self):
        self._N.check(self._N.lib().lasgd_hold_release(self._h))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def ncu_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def kernel_bytes(name, n, world, comm, algo_code, sgd_momentum=True):
    """Algorithmic bytes per launch.  B = 4n.  Returns (bytes, bound)
    where bound is the resource whose roofline time is longest."""
    B = 4 * n
    if name == "fused_round":
        hbm = (7 if world > 1 else 6) * B  # read x,g,m(,own snap); write x,m,next snap
        nvl = (world - 1) * B  # one-shot: every peer's whole snapshot over NVLink
        fa = comm.resolve_fused_algo(algo_code) if world > 1 else 1
        if fa == 3:  # push: 2(P-1)/P*B out as stores; staged reads + landing writes in HBM
            nvl = comm.bytes_per_node(2)
            hbm += 2 * nvl
        elif fa == 2:  # two-shot: RS in + AG in, own chunk mean via HBM
            nvl = comm.bytes_per_node(2)
            hbm += 2 * B // world
        if nvl / NVLINK_PEAK_GBS > hbm / peaks()[0]:
            return nvl, "nvlink"
        return hbm, "hbm"
    if name == "sgd_step":
        return 5 * B if sgd_momentum else 3 * B, "hbm"
    if name == "pull":
        return 5 * B, "hbm"
    if name == "sgd_pull":  # x, g, m, snap, xbar in; x, m, next snapshot out
        return (8 if sgd_momentum else 7) * B, "hbm"
    if name == "finalize":
        return 4 * B, "hbm"
    if name == "snapshot":
        return 2 * B, "hbm"
    if name == "allreduce":
        return comm.bytes_per_node(algo_code), "nvlink"
    return 0, "hbm"


def virtual_rank_kernels(n, dev, stream, hbm_peak, traffic, reps=10):
    """The multi-rank kernels in their virtual-rank form (P ranks' buffers on this one
    GPU, the same device code minus the flag barriers, which stream order replaces):
    K8 mirror push (P=2), K8 staged push (P=4, 8), K3 two-shot mean (P=2, 4, 8), K2
    one-shot mean (P=2).  Every byte a rank would move over NVLink moves through this
    GPU's HBM instead, so the roofline is HBM.  Algorithmic bytes per round (all ranks;
    B = 4n): push P*(7B + 4(P-1)/P*B) (local step + pull + next snapshot, staged
    contributions read, mean pushed, peers' means read, next-snapshot chunks pushed);
    two-shot P*(3B - B/P); one-shot P*(P+1)*B (every rank reads all P sources and
    writes its mean)."""
    import torch

    from paper_2203_13085_b200 import _native as N
    from paper_2203_13085_b200 import kernels as K

    B = 4 * n
    out = {}

    def timeit(fn):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def entry(name, ms, byt, launches):
        ach = byt / (ms * 1e-3) / 1e9
        out[name] = {"avg_ms": ms, "bytes_per_round": byt, "bound": "hbm", "achieved_gbs": ach, "peak_gbs": hbm_peak,
                     "frac": ach / hbm_peak, "launches_per_round": launches, "traffic": traffic.get(name)}

    gen = torch.Generator(device=dev)
    with torch.cuda.stream(stream):
        for P in (2, 4, 8):
            gen.manual_seed(77 + P)
            xs = [torch.randn(n, device=dev, generator=gen) * 0.02 for _ in range(P)]
            gs = [torch.randn(n, device=dev, generator=gen) * 1e-2 for _ in range(P)]
            ms_ = [torch.zeros(n, device=dev) for _ in range(P)]
            snaps = [[x.clone() for x in xs], [torch.empty(n, device=dev) for _ in range(P)]]
            xbars = [torch.empty(n, device=dev) for _ in range(P)]
            # K8 push round (mirror at P=2, staged at P>=3); the staging launch runs once
            se = K.push_stage_elems(n, P)
            stages = [torch.zeros(2 * P * se, device=dev) for _ in range(P)]
            state = {"cur": 0, "init": True}
            fk = dict(ms=ms_, momentum=0.9, weight_decay=1e-4, nesterov=True, alpha=1.0, stream=stream)

            def push():
                c = state["cur"]
                K.fused_push_virtual(xs, gs, snaps[c], snaps[1 - c], xbars, stages, c, state["init"], 0.1,
                                     first_step=state["init"], **fk)
                state["cur"], state["init"] = 1 - c, False

            push()
            name = "push_mirror_virtual_p2" if P == 2 else f"push_staged_virtual_p{P}"
            entry(name, timeit(push), P * (7 * B + 4 * (P - 1) * B // P), 2)
            entry(f"twoshot_virtual_p{P}",
                  timeit(lambda: K.mean_virtual(xbars, snaps[0], algo=N.ALGO_TWOSHOT, stream=stream)),
                  P * (3 * B - B // P), 2)
            if P == 2:
                entry("oneshot_virtual_p2",
                      timeit(lambda: K.mean_virtual(xbars, snaps[0], algo=N.ALGO_ONESHOT, stream=stream)),
                      P * (P + 1) * B, 1)
            del xs, gs, ms_, snaps, xbars, stages
            torch.cuda.empty_cache()
    return out


def fused_algo_name(P, n):
    """The fused-round algorithm our arm runs at world size P for n fp32 parameters
    (lasgd_comm_resolve_fused_algo, csrc/lasgd_comm.cu), so both arms record one config."""
    if P <= 1:
        return "oneshot"
    b = 4 * n
    if P == 2:
        return "push" if b >= (32 << 20) else "oneshot"
    cutoff = (8 << 20) if P <= 4 else (1 << 20)
    return "oneshot" if b <= cutoff else "push"


def cpu_reference_run(n_full, P, k, steps, warmup, threads, target_step_s=1.0, rule="matched", alpha=1.0):
    """The LASGD sync path on the host through the C restatement in oracle/ (f64 like the
    reference, pinned to its outputs by tests/test_c_oracle.py), P workers in-process like
    LoopbackTransport, on a bounded sample of the parameter vector.

    rule "matched": the GPU arm's per-step work — every worker's local step with Nesterov
      momentum 0.9 and weight decay 1e-4 (oracle_sgd_momentum); every k steps the ring
      mean of the P snapshots (collective.py:154-203), the elastic pull writing the next
      snapshot (P > 1) or the snapshot copy (P = 1, optimizer.py:168-169).
    rule "reference": the reference's own rule — sgd_local_step on x and delta
      (optimizer.py:145-146), every k steps the ring mean and new = z + delta (:171).
    Returns (seconds per step, sample n)."""
    import numpy as np

    from oracle import c_oracle as C

    C.set_threads(threads)
    # bounded sample: estimate the per-element cost, keep one step near target_step_s
    probe_n = min(n_full, 1 << 22)
    xa, xb, da, db, g = (np.random.default_rng(i).standard_normal(probe_n) for i in range(5))
    t0 = time.perf_counter()
    for _ in range(3):
        if rule == "matched":
            C.sgd_momentum(xa, g, da, 0.1, 0.9, 0.0, 1e-4, True, False)
        else:
            C.sgd_delta(xb, db, xa, da, g, 0.1)
    per_elem = (time.perf_counter() - t0) / 3 / probe_n
    per_step_elem = per_elem * P * (1.0 + 1.5 / k)  # local step + amortised mean / pull
    n = int(min(n_full, max(1 << 16, target_step_s / per_step_elem)))
    mem = _mem_available()
    if mem:
        n = int(min(n, mem * 0.5 / (8 * (6 * P + 2))))
    rng = np.random.default_rng(0)
    g = rng.standard_normal(n) * 1e-2
    z = np.empty(n)
    if rule == "matched":
        xs = [rng.standard_normal(n) * 0.1 for _ in range(P)]
        ms = [np.zeros(n) for _ in range(P)]
        snaps = [[x.copy() for x in xs], [np.empty(n) for _ in range(P)]]
        st = {"cur": 0, "first": True}

        def one_step(t):
            for r in range(P):
                C.sgd_momentum(xs[r], g, ms[r], 0.1, 0.9, 0.0, 1e-4, True, st["first"])
            st["first"] = False
            if (t + 1) % k == 0:
                c = st["cur"]
                if P > 1:
                    C.ring_mean([z], snaps[c])
                    for r in range(P):
                        C.pull(xs[r], snaps[1 - c][r], snaps[c][r], z, alpha)
                else:
                    C.copy(snaps[1 - c][0], xs[0])
                st["cur"] = 1 - c
    else:
        xs = [[rng.standard_normal(n) * 0.1, np.empty(n)] for _ in range(P)]
        ds = [[np.zeros(n), np.empty(n)] for _ in range(P)]
        snaps = [x[0].copy() for x in xs]
        cur = [0] * P
        reset = [True] * P

        def one_step(t):
            for r in range(P):
                c = cur[r]
                C.sgd_delta(xs[r][1 - c], ds[r][1 - c], xs[r][c], ds[r][c], g, 0.1, delta_reset=reset[r])
                cur[r] = 1 - c
                reset[r] = False
            if (t + 1) % k == 0:
                if P > 1:
                    C.ring_mean([z], snaps)
                    for r in range(P):
                        C.finalize(xs[r][cur[r]], z, ds[r][cur[r]])
                        snaps[r] = xs[r][cur[r]]  # x_local = x_snapshot = new (aliased, optimizer.py:172-173)
                for r in range(P):
                    reset[r] = True

    for t in range(warmup):
        one_step(t)
    t0 = time.perf_counter()
    for t in range(steps):
        one_step(warmup + t)
    dt = (time.perf_counter() - t0) / steps
    return dt, n


def stock_reference_run(n_full, target_s=10.0):
    """The UNMODIFIED reference package (pip-installed into baseline/_ref, single-threaded
    numpy like the reference) timing its own sgd_local_step + lasgd_finalize_round
    (optimizer.py:136-178) for one worker at P = 1 on a bounded sample.  Returns
    (seconds per step at the full size, sample n) or None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "lasgd")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import numpy as np
    from lasgd.optimizer import NodeState, lasgd_finalize_round, sgd_local_step
    from lasgd.params import ParamVector

    n = min(n_full, 1 << 22)
    rng = np.random.default_rng(0)
    st = NodeState.fresh(0, ParamVector(rng.standard_normal(n) * 0.1))
    g = ParamVector(rng.standard_normal(n) * 1e-2)
    sgd_local_step(st, g, 0.1, tau_max=1)  # warm-up
    lasgd_finalize_round(st, None, 1)
    t0 = time.perf_counter()
    reps = 0
    while True:
        sgd_local_step(st, g, 0.1, tau_max=1)
        lasgd_finalize_round(st, None, 1)
        reps += 1
        if time.perf_counter() - t0 > target_s / 4 or reps >= 50:
            break
    dt = (time.perf_counter() - t0) / reps
    return dt * n_full / n, n


def _mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except Exception:
        return None
    return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference's algorithm on the host cores, on our arm's workload and config: the
    work-matched rule (value) and the reference's own plain-SGD + delta rule (extra)."""
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    P = world
    full = MODELS[args.model]["params"]
    dt, n = cpu_reference_run(full, P, args.sync_period, max(1, args.steps), max(1, args.warmup), threads,
                              rule="matched", alpha=args.alpha)
    scale = n / full  # elementwise work is linear in n: full-size step time = dt / scale
    value = P * args.batch / (dt / scale)
    dt_r, n_r = cpu_reference_run(full, P, args.sync_period, max(1, args.steps // 4), 1, threads, rule="reference",
                                  target_step_s=0.5)
    sample = (f"oracle/ C port (f64, pinned to the reference by tests/test_c_oracle.py), {P} workers in-process, "
              f"{threads} threads: per step every worker's Nesterov/weight-decay local step, every "
              f"{args.sync_period} steps the ring-order mean + elastic pull + next snapshot (the GPU arm's work); "
              f"{n} of {full} parameters per step, scaled linearly; {args.steps} timed steps after {args.warmup} "
              f"warm-up; host {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / scale * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, world, fused_algo_name(world, full)),
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "port", "sample": sample},
        "reference_rule": {"value": P * args.batch / (dt_r * full / n_r), "unit": "images/s", "cores": threads,
                           "sample": f"the reference's own rule (plain sgd_local_step + delta, finalize z + delta), "
                                     f"{n_r} of {full} parameters, scaled"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    stock = stock_reference_run(full)
    if stock is not None:
        line["stock_reference"] = {
            "value": args.batch / stock[0], "unit": "images/s", "cores": 1,
            "sample": f"unmodified reference package (baseline/_ref) sgd_local_step + lasgd_finalize_round, one "
                      f"worker, numpy single-threaded, {stock[1]} of {full} parameters, scaled"}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from paper_2203_13085_b200 import _native as N

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t.item())

    algo_code = {"auto": N.ALGO_AUTO, "oneshot": N.ALGO_ONESHOT, "twoshot": N.ALGO_TWOSHOT,
                 "push": N.ALGO_PUSH}[args.algo]
    n = MODELS[args.model]["params"]
    sgd = L.SgdConfig(0.9, 0.0, 1e-4, True)
    lr = 0.1
    comm = L.P2PCommunicator(n, nblocks=args.nblocks, timeout_s=60.0) if world > 1 else None
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    x = torch.randn(n, device=dev, generator=gen) * 0.02  # identical x0 on every rank
    grads = []
    for i in range(2):
        gen.manual_seed(1000 + 10 * rank + i)
        grads.append(torch.randn(n, device=dev, generator=gen) * 1e-2)
    compute = torch.cuda.Stream(device=dev, priority=-1)

    def make_worker(timed, sync=True, g=None):
        return L.LASGDWorker(x, g if g is not None else grads[0], comm=comm, sync_period=args.sync_period,
                             alpha=args.alpha, mode="pull", sgd=sgd, lr=lr, algo=algo_code, compute_stream=compute,
                             timed=timed, sync=sync, pipeline=args.pipeline, fused_nblocks=args.fused_nblocks)

    def run_sync_path(worker, steps, gsrc):
        for t in range(steps):
            worker.g = gsrc(t)
            worker.step()

    hold = Hold(N)

    # ---------------- value: HBM-resident gradients, device-timed.  At N=1 the K steps
    # replay as ONE CUDA graph (LASGDWorker.capture: the deterministic loop reads its
    # per-round scalars — rate, first step, snapshot slot, launch sequence — from the
    # device round descriptor; --sync-graph does the same at N>1).  The timed region is
    # enqueued behind a hold kernel and released at once, so host jitter cannot open gaps.
    with torch.cuda.stream(compute):
        w = make_worker(False)
        run_sync_path(w, args.warmup, lambda t: grads[t % 2])
        w.drain()
        graph = None
        use_graph = (world == 1 and not args.no_sync_graph) or (args.sync_graph and args.pipeline == "fused")
        if use_graph and args.steps % args.sync_period == 0:
            graph = w.capture([grads[t % 2] for t in range(args.steps)])
            graph.replay()  # graph upload; one more untimed pass
            w.drain()
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if rank == 0 else None
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w.reset_records()
    with torch.cuda.stream(compute):
        hold.enqueue(compute)
        if comm is not None:
            # the holds are released at slightly different host times on each rank; a
            # one-warp device barrier behind them lines the ranks' clocks up, so the max
            # over ranks does not count one rank's release skew as step time
            comm.device_barrier(compute)
        e0.record(compute)
        h0 = time.perf_counter()
        if graph is not None:
            graph.replay()
        else:
            run_sync_path(w, args.steps, lambda t: grads[t % 2])
        host_issue_ms = (time.perf_counter() - h0) * 1e3
        w.drain()
        e1.record(compute)
        hold.release()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1))
    host_issue_ms = max_over_ranks(host_issue_ms)
    value_kinds = dict(w.launches)  # kernel kind -> launches in the timed region
    launches = sum(value_kinds.values())
    barrier()

    # ---------------- per-kernel timing (same loop, events around every launch)
    with torch.cuda.stream(compute):
        wt = make_worker(True)
        run_sync_path(wt, args.warmup, lambda t: grads[t % 2])
        wt.drain()
    torch.cuda.synchronize()
    barrier()
    wt.reset_records()
    with torch.cuda.stream(compute):
        run_sync_path(wt, args.steps, lambda t: grads[t % 2])
        wt.drain()
    torch.cuda.synchronize()
    ktimes = wt.kernel_times()
    barrier()

    # ---------------- e2e: gradients from pinned host memory every step (H2D on a copy
    # stream, double-buffered) + D2H of the step's status word, through the public API
    host_g = [grads[i].cpu().pin_memory() for i in range(2)]
    dev_g = [torch.empty(n, device=dev) for _ in range(2)]
    status_h = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    # two copy streams, half the gradient each: two DMA engines keep the PCIe link fuller
    # (tools/h2d_probe.py: 102 MB in 1.88 ms vs 2.01 ms on one stream)
    copy_streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    halves = [(0, n // 2), (n // 2, n)]
    ready = [[torch.cuda.Event() for _ in range(2)] for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for ev in free:
        ev.record(compute)

    def e2e_loop(worker, steps):
        def issue(t):
            b = t % 2
            for cs, (lo, hi), ev in zip(copy_streams, halves, ready[b]):
                cs.wait_event(free[b])
                with torch.cuda.stream(cs):
                    dev_g[b][lo:hi].copy_(host_g[b][lo:hi], non_blocking=True)
                ev.record(cs)

        issue(0)
        for t in range(steps):
            b = t % 2
            if t + 1 < steps:
                issue(t + 1)
            for ev in ready[b]:
                compute.wait_event(ev)
            worker.g = dev_g[b]
            worker.step()
            free[b].record(compute)
            status_h.copy_(worker.state.nonfinite_counter, non_blocking=True)
        worker.drain()

    with torch.cuda.stream(compute):
        we = make_worker(False, g=dev_g[0])
        e2e_loop(we, args.warmup)
    torch.cuda.synchronize()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(compute):
        # no hold kernel here: end to end includes the host issuing every step
        f0.record(compute)
        for cs in copy_streams:
            cs.wait_event(f0)  # the first H2D starts inside the timed region
        e2e_loop(we, args.steps)
        f1.record(compute)
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks(f0.elapsed_time(f1))
    barrier()
    clk = clocks.stop() if clocks else None

    # ---------------- isolated kernel timings (each kernel alone, for the roofline detail)
    iso = {}
    ar_iso = {}
    with torch.cuda.stream(compute):
        m = torch.zeros_like(x)
        s0, s1, xb = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)

        def timeit(fn, reps=20):
            for _ in range(3):
                fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(compute)
            for _ in range(reps):
                fn()
            b.record(compute)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        from paper_2203_13085_b200 import kernels as K

        iso["sgd_step"] = timeit(lambda: K.sgd_step(x, grads[0], lr, m=m, momentum=0.9, weight_decay=1e-4,
                                                    nesterov=True, stream=compute))
        iso["pull"] = timeit(lambda: K.elastic_pull(x, s0, xb, 1.0, snap_next=s1, stream=compute))
        iso["snapshot"] = timeit(lambda: K.snapshot(s1, x, stream=compute))
        if comm is not None:
            barrier()

            def ar():
                seq = comm.allreduce(0, algo_code if algo_code != N.ALGO_PUSH else N.ALGO_AUTO, stream=compute)
                return seq

            iso["allreduce"] = timeit(ar, reps=10)
            # every transport of the exchange on the same snapshot, beside NCCL's all-reduce
            # of the same buffer (max over ranks; BASELINE configs[4]'s comparison at this size)
            for nm, code in (("oneshot", N.ALGO_ONESHOT), ("twoshot", N.ALGO_TWOSHOT), ("push", N.ALGO_PUSH),
                             ("ce", N.ALGO_CE)):
                barrier()
                ar_iso[nm] = max_over_ranks(timeit(lambda c=code: comm.allreduce(0, c, stream=compute), reps=10))
            nbuf = comm.snapshots[0].clone()
            barrier()
            ar_iso["nccl_allreduce_sum"] = max_over_ranks(timeit(lambda: dist.all_reduce(nbuf), reps=10))
            del nbuf
        fk = dict(m=m, momentum=0.9, weight_decay=1e-4, nesterov=True, alpha=args.alpha,
                  nblocks=args.fused_nblocks, stream=compute)
        if comm is not None:
            barrier()
            slot = [0]

            def fused():
                comm.fused_round(slot[0], x, grads[0], lr, algo=algo_code, **fk)
                slot[0] ^= 1

            iso["fused_round"] = timeit(fused, reps=10)
        else:
            iso["fused_round"] = timeit(lambda: K.fused_round_virtual(
                [x], [grads[0]], [s0], [s1], lr, ms=[m], **{k: v for k, v in fk.items() if k != "m"}))
    barrier()

    # ---------------- multi-rank kernels in virtual-rank form (one GPU: the N=1 record)
    vkernels = None
    if world == 1 and not args.no_virtual:
        vkernels = virtual_rank_kernels(n, dev, compute, peaks()[0], ncu_traffic())

    # ---------------- real training: ResNet-50 fwd/bwd + LASGD vs no-sync ceiling
    training = None
    if not args.no_train and not args.kernels_only:
        tclk = ClockSampler(local) if rank == 0 else None
        training = run_training(args, dev, comm, world, rank, sgd, lr, algo_code, compute, barrier, max_over_ranks)
        if tclk is not None:
            # clocks and power over the training legs: ResNet-50 bf16 at batch 256 runs at the
            # 1 kW cap, so SM clocks move with each leg's power draw
            training["clocks"] = tclk.stop()

    # ---------------- report
    imgs = world * args.batch * args.steps
    value = imgs / (ms / 1e3)
    e2e_val = imgs / (ms_e2e / 1e3)
    hbm_peak, peak_kind = peaks()
    traffic = ncu_traffic()
    kernels = {}
    for name, ts in ktimes.items():
        byt, bound = kernel_bytes(name, n, world, comm, algo_code)
        avg = sum(ts) / len(ts)
        pk = hbm_peak if bound == "hbm" else NVLINK_PEAK_GBS
        ach = byt / (avg * 1e-3) / 1e9 if avg > 0 else 0.0
        entry = {"launches": len(ts), "avg_ms": avg, "bytes_per_launch": byt, "bound": bound,
                 "achieved_gbs": ach, "peak_gbs": pk, "frac": ach / pk, "share_of_step": sum(ts) / ms}
        if name in iso:
            ia = byt / (iso[name] * 1e-3) / 1e9
            entry["isolated_ms"] = iso[name]
            entry["isolated_gbs"] = ia
            entry["isolated_frac"] = ia / pk
        kernels[name] = entry
    dom = max(kernels, key=lambda k: sum(ktimes[k]))
    d = kernels[dom]
    # ncu profiles one GPU only: the N=1 kernel is measured directly; a multi-rank round is
    # measured in its virtual-rank form (all ranks on one GPU, same device code, per rank)
    tr = traffic.get(dom) if world == 1 else traffic.get(f"{dom}_p{world}")
    # Launch duration: when the timed region is exactly one launch of the dominant kernel per
    # step, the region's device time / launches (max over ranks, inter-launch gaps included,
    # so conservative) is its average duration without per-launch event overhead; otherwise
    # the per-launch event pairs of the timing pass.
    if set(value_kinds) == {dom} and value_kinds[dom] == args.steps:
        avg_ms, method = ms / args.steps, "timed region device time / launches (one launch per step, gaps included)"
    else:
        avg_ms, method = d["avg_ms"], "CUDA events around every launch (timing pass)"
    achieved = d["bytes_per_launch"] / (avg_ms * 1e-3) / 1e9
    roofline = {"kernel": dom, "bound": "hbm" if d["bound"] == "hbm" else "nvlink", "achieved": achieved,
                "peak": d["peak_gbs"], "unit": "GB/s", "frac": achieved / d["peak_gbs"], "traffic": tr,
                "avg_launch_ms": avg_ms, "achieved_method": method,
                "achieved_per_launch_events": d["achieved_gbs"],
                "traffic_source": ("not measured: ncu runs on one GPU and this round has no virtual-rank capture"
                                   if tr is None else "ncu --set full, profiles/ncu_traffic.json" if world == 1
                                   else "ncu --set full of the virtual-rank form, per rank, profiles/ncu_traffic.json"),
                "algorithmic_bytes": d["bytes_per_launch"],
                "peak_source": (f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})" if d["bound"] == "hbm"
                                else "B200_PROFILING.md measured peer copy 770 GB/s/direction")}
    gpu_launches = int(sum_over_ranks(launches))

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        dt, ns = cpu_reference_run(n, 1, args.sync_period, 10, 2, threads, target_step_s=0.5, alpha=args.alpha)
        scale = ns / n
        cpu_base = {"value": args.batch / (dt / scale), "unit": "images/s", "cores": threads, "kind": "port",
                    "sample": f"oracle/ C port (f64, pinned by tests/test_c_oracle.py), 1 worker, the GPU arm's "
                              f"work (Nesterov/wd local step + next snapshot) on {ns} of {n} parameters, 10 steps, "
                              f"scaled linearly; host {cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "host_issue_ms_per_step": host_issue_ms / args.steps,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, world, {1: "oneshot", 2: "twoshot", 3: "push"}.get(
                comm.resolve_fused_algo(algo_code) if comm is not None else 1)),
            "timed_region": ("one CUDA-graph replay of the K steps (LASGDWorker.capture), behind a hold kernel"
                             if graph is not None else "K worker steps issued one by one, behind a hold kernel"),
            "roofline": roofline,
            "cpu_baseline": cpu_base,
            "e2e": {"value": e2e_val, "unit": "images/s", "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 8,
                    "ms_per_step": ms_e2e / args.steps,
                    "path": "public API (LASGDWorker) with gradients from pinned host memory each step"},
            "gpu_launches": gpu_launches,
            "clocks": clk,
            "sync_kernels": kernels,
            "allreduce_isolated_ms": ar_iso or None,
            "virtual_rank_kernels": vkernels,
            "training": training,
            # the BASELINE metric's ResNet-50 training throughput (images through forward,
            # backward and the LASGD step per second, all ranks) beside the sync-path value
            "training_summary": None if not training or "images_per_s_lasgd" not in training else {
                "images_per_s": training["images_per_s_lasgd"], "nosync_images_per_s": training["images_per_s_nosync"],
                "frac_of_nosync": training["images_per_s_lasgd"] / training["images_per_s_nosync"],
                "exposed_sync_ms_per_step": training["exposed_sync_ms_per_step"], "pipeline": args.pipeline},
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        barrier()
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _exposed_stats(leg, base, resamples=4000):
    """Exposed sync = median over repetitions of the paired difference (leg block - no-sync
    block of the same repetition), with a 95% bootstrap percentile interval of that
    median (repetitions resampled with replacement, fixed seed).  Pairing cancels the
    slow drifts of the step time (the GPU's step time switches between two levels ~0.4 ms
    apart for stretches of several blocks), the median ignores the rare repetition in
    which a switch falls between the two blocks."""
    import random
    import statistics as st

    diffs = [a - b for a, b in zip(leg, base)]
    rng = random.Random(12345)
    boots = sorted(st.median(rng.choices(diffs, k=len(diffs))) for _ in range(resamples))
    lo, hi = boots[int(0.025 * resamples)], boots[int(0.975 * resamples) - 1]
    return {"median": st.median(diffs), "ci95": [lo, hi], "ci95_halfwidth": (hi - lo) / 2, "blocks": len(diffs)}


def run_training(args, dev, comm, world, rank, sgd, lr, algo_code, compute, barrier, max_over_ranks):
    """Real training step (forward/backward in PyTorch, bf16 autocast, channels_last) with
    the sync path under each schedule, and with sync disabled (the no-sync ceiling).

    The legs run interleaved in blocks (every leg once per repetition, in the same order)
    and each leg's exposed sync time is the median over repetitions of its block time
    minus the no-sync baseline's block time in the same repetition, with a bootstrap 95%
    interval.
    Graphed legs (forward/backward replayed as a CUDA graph; at N=1 the local step and
    round boundary are captured into the same graph) compare with the graphed no-sync
    leg; eager legs (the bucketed SGD-AR, whose buckets launch from autograd hooks, and
    NCCL DDP) with the eager no-sync leg."""
    import torch
    import torchvision

    import paper_2203_13085_b200 as L
    from paper_2203_13085_b200 import _native as N

    spec = MODELS[args.model]
    torch.backends.cudnn.benchmark = True
    model = getattr(torchvision.models, spec["ctor"])(num_classes=spec["classes"]).to(dev)
    model = model.to(memory_format=torch.channels_last)
    flat = L.FlatParams(model, channels_last=True, align_bytes=args.flat_align)
    assert flat.n_params == spec["params"], (flat.n_params, spec["params"])
    tcomm = comm
    if comm is not None:
        import torch.distributed as dist

        # identical x0 on every rank (Algorithm 1 line 1)
        dist.broadcast(flat.x, 0)
        if comm.n != flat.numel:  # 256-B aligned tensors: the flat vector carries padding
            tcomm = L.P2PCommunicator(flat.numel, nblocks=args.nblocks, timeout_s=60.0,
                                      stream_priority=args.side_priority)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    hw = spec["image"]
    images = torch.randn(args.batch, 3, hw, hw, device=dev, generator=gen).to(memory_format=torch.channels_last)
    labels = torch.randint(0, spec["classes"], (args.batch,), device=dev, generator=gen)
    lossf = torch.nn.CrossEntropyLoss()

    def fwd_bwd_eager():
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            loss = lossf(model(images), labels)
        loss.backward()

    def fwd_bwd_zero():
        flat.zero_grad()
        fwd_bwd_eager()

    graphed = not args.no_graphs
    fwd_bwd = L.GraphedStep(flat, fwd_bwd_eager) if graphed else fwd_bwd_zero
    own_g = flat.g

    # ---- legs: make() -> (one_step, finish, close); one_step runs one training step on `compute`
    cached = {}  # N=1 graphed LASGD legs and DDP live across blocks (graphs captured once)

    def lasgd_leg(leg_comm=None, **wkw):
        key = repr(sorted(wkw.items())) + ("nvls" if leg_comm is not None else "")

        def make():
            flat.bind_grads(own_g)
            one_graph = None
            if key in cached:
                w, one_graph = cached[key]
            else:
                kw = dict(wkw)
                leg_algo = kw.pop("algo", algo_code)
                w = L.LASGDWorker(flat.x, flat.g, comm=leg_comm if leg_comm is not None else tcomm,
                                  sync_period=args.sync_period, alpha=args.alpha,
                                  mode="pull", sgd=sgd, lr=lr, algo=leg_algo, compute_stream=compute,
                                  fused_nblocks=args.fused_nblocks, **kw)
                if graphed and world == 1 and not wkw.get("adaptive") and args.step_graph:
                    # one CUDA graph: zero_grad + forward + backward + local step (+ round boundary)
                    fwd_bwd()  # the fwd/bwd graph exists: cuDNN autotuned, the shared pool warm
                    k = args.sync_period if wkw.get("sync", True) else 1
                    one_graph = w.capture_with(lambda t: (flat.zero_grad(), fwd_bwd_eager()), steps=k,
                                               pool=fwd_bwd.pool)
                    cached[key] = (w, one_graph)
            state = {"t": 0}

            def one():
                if one_graph is not None:
                    if state["t"] % one_graph.steps == 0:
                        one_graph.replay()
                    state["t"] += 1
                    return
                fwd_bwd()
                w.step()

            def finish():
                w.drain()
                return w

            return one, finish, (lambda: None) if key in cached else w.close
        return make

    def sgd_ar_leg(kind):
        import torch.distributed as dist

        from paper_2203_13085_b200 import kernels as K

        def make():
            if kind == "nccl":
                flat.bind_grads(own_g)
                m = torch.empty_like(flat.x)
                clock = [0]

                def one():
                    fwd_bwd()
                    dist.all_reduce(flat.g, op=dist.ReduceOp.AVG)
                    K.sgd_step(flat.x, flat.g, lr, m=m, momentum=sgd.momentum, weight_decay=sgd.weight_decay,
                               nesterov=sgd.nesterov, first_step=clock[0] == 0, stream=compute)
                    clock[0] += 1
                return one, lambda: None, lambda: None
            if kind == "p2p":
                w = L.SGDARWorker(flat.x, comm=tcomm, sgd=sgd, lr=lr, compute_stream=compute, flat=flat)

                def one():
                    fwd_bwd()
                    w.step()
                return one, lambda: None, lambda: flat.bind_grads(own_g)
            if kind == "bucketed":
                w = L.BucketedSGDARWorker(flat, tcomm, sgd=sgd, lr=lr, bucket_bytes=args.bucket_mb << 20,
                                          compute_stream=compute, nblocks=args.bucket_ctas)

                def one():
                    fwd_bwd_zero()
                    w.step()
                return one, lambda: None, lambda: (w.close(), flat.bind_grads(own_g))
            # torch DDP over NCCL (bucketed, overlapped with backward), our K5 after it
            from torch.nn.parallel import DistributedDataParallel as DDP

            flat.bind_grads(own_g)
            if "ddp" not in cached:
                cached["ddp"] = DDP(model, device_ids=[dev.index], bucket_cap_mb=args.bucket_mb,
                                    broadcast_buffers=False, gradient_as_bucket_view=False)
            ddp = cached["ddp"]
            m = torch.empty_like(flat.x)
            clock = [0]

            def one():
                flat.zero_grad()
                with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
                    loss = lossf(ddp(images), labels)
                loss.backward()
                K.sgd_step(flat.x, flat.g, lr, m=m, momentum=sgd.momentum, weight_decay=sgd.weight_decay,
                           nesterov=sgd.nesterov, first_step=clock[0] == 0, stream=compute)
                clock[0] += 1
            return one, lambda: None, lambda: None
        return make

    def nosync_eager_leg():
        from paper_2203_13085_b200 import kernels as K

        def make():
            flat.bind_grads(own_g)
            m = torch.empty_like(flat.x)
            clock = [0]

            def one():
                fwd_bwd_zero()
                K.sgd_step(flat.x, flat.g, lr, m=m, momentum=sgd.momentum, weight_decay=sgd.weight_decay,
                           nesterov=sgd.nesterov, first_step=clock[0] == 0, stream=compute)
                clock[0] += 1
            return one, lambda: None, lambda: None
        return make

    legs = {"nosync": (lasgd_leg(sync=False), "nosync"),
            "fused": (lasgd_leg(pipeline="fused"), "nosync"),
            "overlap": (lasgd_leg(pipeline="overlap"), "nosync"),
            "overlap_adaptive": (lasgd_leg(pipeline="overlap", adaptive=True, tau_max=5), "nosync")}
    ncomm = None
    if tcomm is not None and args.nvls_leg:
        # the overlap pipeline on the in-switch (NVLS, tolerance-mode) side-stream mean
        try:
            ncomm = L.P2PCommunicator(flat.numel, nblocks=args.nblocks, timeout_s=60.0, nvls=True)
        except ValueError:
            ncomm = None
        if ncomm is not None:
            legs["overlap_nvls"] = (lasgd_leg(leg_comm=ncomm, pipeline="overlap"), "nosync")
    if tcomm is not None:
        # the overlap pipeline with the side-stream mean's NVLink traffic on the copy engines
        # (the overlap leg's AUTO picks it at P >= 3; overlap_sm keeps the SM mean there)
        legs["overlap_ce"] = (lasgd_leg(pipeline="overlap", algo=N.ALGO_CE), "nosync")
        if world >= 3:
            legs["overlap_sm"] = (lasgd_leg(pipeline="overlap", algo=tcomm.resolve_algo(N.ALGO_AUTO)
                                            if tcomm.resolve_algo(N.ALGO_AUTO) != N.ALGO_CE else N.ALGO_TWOSHOT),
                                  "nosync")
        legs.update({"sgd_ar": (sgd_ar_leg("p2p"), "nosync"), "sgd_ar_nccl": (sgd_ar_leg("nccl"), "nosync"),
                     "nosync_eager": (nosync_eager_leg(), "nosync_eager"),
                     "sgd_ar_bucketed": (sgd_ar_leg("bucketed"), "nosync_eager"),
                     "ddp_nccl": (sgd_ar_leg("ddp"), "nosync_eager")})
    if args.legs:
        keep = set(args.legs.split(","))
        keep |= {legs[k][1] for k in keep if k in legs}
        legs = {k: v for k, v in legs.items() if k in keep}
    times = {k: [] for k in legs}
    hists = {}
    B, R = args.train_block, args.train_reps
    with torch.cuda.stream(compute):
        for name, (make, _) in legs.items():  # one untimed pass per leg: graphs, cuDNN, NCCL buckets
            one, finish, close = make()
            for _ in range(args.train_warmup):
                one()
            finish()
            close()
    torch.cuda.synchronize()
    for rep in range(R):
        for name, (make, _) in legs.items():
            with torch.cuda.stream(compute):
                one, finish, close = make()
                for _ in range(2):
                    one()
                w = finish()
            torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(compute):
                if w is not None and hasattr(w, "reset_records"):
                    w.reset_records()
                a.record(compute)
                for _ in range(B):
                    one()
                finish()
                b.record(compute)
            torch.cuda.synchronize()
            times[name].append(max_over_ranks(a.elapsed_time(b)) / B)
            if w is not None and hasattr(w, "tau_hist"):
                for t, c in w.tau_hist.items():
                    hists.setdefault(name, {}).setdefault(str(t), 0)
                    hists[name][str(t)] += c
            close()
            barrier()
    for key, v in list(cached.items()):
        if key != "ddp":
            v[0].close()
    cached.clear()
    if tcomm is not None and tcomm is not comm:
        tcomm.close()
    if ncomm is not None:
        ncomm.close()
    flat.bind_grads(own_g)

    import statistics as st

    out = {"model": f"{spec['ctor']} (torchvision, random init, {hw}x{hw}, {spec['classes']} classes)",
           "batch_per_gpu": args.batch, "precision": "bf16 autocast fwd/bwd, fp32 params",
           "flat_align_bytes": args.flat_align, "blocks": f"{R} repetitions x {B} steps per leg, legs interleaved",
           "fwd_bwd": (("cuda_graph (zero_grad+fwd+bwd+local step+round in one graph per leg)" if args.step_graph
                        and world == 1 else "cuda_graph (one zero_grad+fwd+bwd graph shared by the legs, sync "
                        "launches after it)") if graphed else "eager")}
    for name, (_, base) in legs.items():
        med = st.median(times[name])
        e = {"images_per_s": world * args.batch / (med / 1e3), "ms_per_step": med, "ms_per_step_blocks": times[name]}
        if name != base:
            d = _exposed_stats(times[name], times[base])
            e.update({"exposed_sync_ms_per_step": d["median"], "exposed_sync_ci95_ms": d["ci95"],
                      "exposed_sync_ci95_halfwidth_ms": d["ci95_halfwidth"],
                      "exposed_sync_frac": d["median"] / med, "baseline_leg": base})
        if name in hists:
            e["tau_histogram"] = hists[name]
        out[name] = e
    if args.pipeline in out and "nosync" in out:
        main = out[args.pipeline]
        out["images_per_s_lasgd"] = main["images_per_s"]
        out["images_per_s_nosync"] = out["nosync"]["images_per_s"]
        out["exposed_sync_ms_per_step"] = main["exposed_sync_ms_per_step"]
        out["exposed_sync_frac"] = main["exposed_sync_frac"]
    return out


if __name__ == "__main__":
    sys.exit(main())

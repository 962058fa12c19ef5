#!/usr/bin/env python
"""Single-GPU driver for the round-2 ncu captures, at ResNet-50 size (n = 25,557,032
fp32, B = 102.23 MB), every kernel in the order bench.py times it:

1. the N=1 bench kernel: the deterministic loop replayed from a CUDA graph
   (k_sgd_dyn: local step with Nesterov momentum + weight decay + next snapshot,
   scalars from the device round descriptor) — 2 replays of a 2-step graph;
2. the multi-rank rounds in virtual-rank form (P ranks on this GPU): K8 mirror push
   (P=2), K8 staged push (P=4, 8), K3 two-shot mean (P=2, 4, 8) — 2 rounds each
   (push: staging launch once, then phase A + phase B launches per round; two-shot:
   reduce-scatter + all-gather launches).

    python tools/profile_r02.py && ncu --set full --clock-control none --import-source on \\
        -k regex:'k_sgd_dyn|k_push|k_twoshot|k_oneshot' -o gpurun_out/prof_r02 python tools/profile_r02.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200 as L  # noqa: E402
from paper_2203_13085_b200 import _native as N  # noqa: E402
from paper_2203_13085_b200 import kernels as K  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = 25_557_032
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, device="cuda", generator=gen) * 0.02
    grads = [torch.randn(n, device="cuda", generator=gen) * 1e-2 for _ in range(2)]
    compute = torch.cuda.Stream()
    with torch.cuda.stream(compute):
        w = L.LASGDWorker(x, grads[0], sync_period=1, lr=0.1, sgd=L.SgdConfig(0.9, 0.0, 1e-4, True),
                          pipeline="fused", compute_stream=compute)
        w.step()
        graph = w.capture(grads)
        for _ in range(2):
            graph.replay()
    torch.cuda.synchronize()
    w.close()
    del x, grads
    for P in (2, 4, 8):
        xs = [torch.randn(n, device="cuda", generator=gen) * 0.02 for _ in range(P)]
        gs = [torch.randn(n, device="cuda", generator=gen) * 1e-2 for _ in range(P)]
        ms = [torch.zeros(n, device="cuda") for _ in range(P)]
        snaps = [[v.clone() for v in xs], [torch.empty(n, device="cuda") for _ in range(P)]]
        xbars = [torch.empty(n, device="cuda") for _ in range(P)]
        se = K.push_stage_elems(n, P)
        stages = [torch.zeros(2 * P * se, device="cuda") for _ in range(P)]
        for t in range(2):
            c = t % 2
            K.fused_push_virtual(xs, gs, snaps[c], snaps[1 - c], xbars, stages, c, t == 0, 0.1, ms=ms, momentum=0.9,
                                 weight_decay=1e-4, nesterov=True, first_step=t == 0, alpha=1.0)
        for _ in range(2):
            K.mean_virtual(xbars, snaps[0], algo=N.ALGO_TWOSHOT)
        if P == 2:
            for _ in range(2):
                K.mean_virtual(xbars, snaps[0], algo=N.ALGO_ONESHOT)
        torch.cuda.synchronize()
        del xs, gs, ms, snaps, xbars, stages
        torch.cuda.empty_cache()
    print("profile_r02 ok")


if __name__ == "__main__":
    main()

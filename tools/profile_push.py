#!/usr/bin/env python
"""Single-GPU driver for ncu (round 1, second part): the kernels the bench runs now, at
ResNet-50 size (n = 25,557,032 fp32), in a fixed launch order so a capture can be
attributed per launch:

  0  fused round at P = 1 (the N = 1 bench step: K5 + next snapshot, k_stream<SgdOp>)
  1  K8 mirror push, 2 virtual ranks: init launch (stages each snapshot at the peer)
  2  K8 mirror push round (phase 1)
  3  K8 mirror push, phase-2 launch (a no-op for the mirror form)
  4  K8 staged push, 4 virtual ranks: init launch
  5  K8 staged push phase A (own chunks: staged reduce, update, mean pushed)
  6  K8 staged push phase B (other chunks: update, next-snapshot chunks pushed)

Virtual ranks keep every rank's buffers on one GPU, so "remote" stores are local writes
and the traffic counts all P ranks' data; ncu must not wrap a multi-rank job.
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2203_13085_b200 import kernels as K  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = 25_557_032
    fk = dict(momentum=0.9, weight_decay=1e-4, nesterov=True)

    def vecs(k):
        return [torch.randn(n, device="cuda") * 0.01 for _ in range(k)]

    x, g, m, s0, s1 = vecs(5)
    K.fused_round_virtual([x], [g], [s0], [s1], 0.1, ms=[m], **fk)
    for P in (2, 4):
        xs, gs, ms, snaps, nexts, xbars = vecs(P), vecs(P), vecs(P), vecs(P), vecs(P), vecs(P)
        se = K.push_stage_elems(n, P)
        stages = [torch.zeros(2 * P * se, device="cuda") for _ in range(P)]
        K.fused_push_virtual(xs, gs, snaps, nexts, xbars, stages, 0, True, 0.1, ms=ms, alpha=1.0, **fk)
        del xs, gs, ms, snaps, nexts, xbars, stages
        torch.cuda.empty_cache()
    torch.cuda.synchronize()
    print("profile_push done")


if __name__ == "__main__":
    main()

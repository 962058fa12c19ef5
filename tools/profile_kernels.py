#!/usr/bin/env python
"""Single-GPU driver for ncu: launches every sync-path kernel a few times at
ResNet-50 size (n = 25,557,032 fp32) in a fixed order so an ncu capture can
attribute DRAM traffic per kernel.  The all-reduce kernels run in their
virtual-rank form (P contributions on one device, the same device code path
minus the flags), since ncu must not wrap a multi-rank job.

Order per repetition: sgd_step (momentum+nesterov+wd) -> elastic_pull(+snapshot)
-> snapshot -> finalize -> mean P=2 one-shot -> mean P=8 one-shot -> mean P=8 two-shot (RS, AG)
-> fused round P=1 -> fused round one-shot over 2 virtual ranks.
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2203_13085_b200 import _native as N  # noqa: E402
from paper_2203_13085_b200 import kernels as K  # noqa: E402


def main(reps: int = 3):
    torch.cuda.set_device(0)
    n = 25_557_032
    x, g, m, s0, s1, z, d = (torch.randn(n, device="cuda") for _ in range(7))
    srcs8 = [torch.randn(n, device="cuda") for _ in range(8)]
    outs8 = [torch.empty(n, device="cuda") for _ in range(8)]
    fk = dict(momentum=0.9, weight_decay=1e-4, nesterov=True)
    for _ in range(reps):
        K.sgd_step(x, g, 0.1, m=m, **fk)
        K.elastic_pull(x, s0, z, 1.0, snap_next=s1)
        K.snapshot(s1, x)
        K.finalize(x, z, d, snap_next=s1)
        K.mean_virtual([outs8[0]], srcs8[:2], algo=N.ALGO_ONESHOT, nblocks=128)
        K.mean_virtual([outs8[0]], srcs8, algo=N.ALGO_ONESHOT, nblocks=128)
        K.mean_virtual(outs8, srcs8, algo=N.ALGO_TWOSHOT, nblocks=128)
        # K7 at P = 1 (the N = 1 bench step: local step + next snapshot, one pass)
        K.fused_round_virtual([x], [g], [s0], [s1], 0.1, ms=[m], **fk)
        # K7 one-shot over 2 virtual ranks (x/g/m per rank = srcs8[0..5], snapshots = outs8)
        K.fused_round_virtual(srcs8[0:2], srcs8[2:4], outs8[0:2], outs8[2:4], 0.1, ms=srcs8[4:6], **fk)
    torch.cuda.synchronize()
    print("profile_kernels done")


if __name__ == "__main__":
    main()

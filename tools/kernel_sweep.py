#!/usr/bin/env python
"""Single-GPU sweep of the rank-local streaming kernels (K1/K4/K5) over the
streaming-grid occupancy (CTAs of 256 threads per SM) at ResNet-50 size and 1 GB.
Prints one JSON line per (kernel, size, ctas_per_sm) with achieved HBM GB/s."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200  # noqa: E402,F401
from paper_2203_13085_b200 import _native as N  # noqa: E402
from paper_2203_13085_b200 import kernels as K  # noqa: E402


def main():
    torch.cuda.set_device(0)
    peak = 6445.3
    for n in (25_557_032, 268_435_456):
        x, g, m, s0, s1, z = (torch.randn(n, device="cuda") for _ in range(6))
        B = 4 * n
        cases = {
            "sgd_momentum": (5 * B, lambda: K.sgd_step(x, g, 0.1, m=m, momentum=0.9, weight_decay=1e-4, nesterov=True)),
            "sgd_plain": (3 * B, lambda: K.sgd_step(x, g, 0.1)),
            "pull_snapshot": (5 * B, lambda: K.elastic_pull(x, s0, z, 1.0, snap_next=s1)),
            "snapshot": (2 * B, lambda: K.snapshot(s1, x)),
            "torch_copy": (2 * B, lambda: s1.copy_(x)),
        }
        for cps in (1, 2, 3, 4, 8):
            N.check(N.lib().lasgd_set_stream_ctas_per_sm(cps))
            for name, (byt, fn) in cases.items():
                for _ in range(3):
                    fn()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 20
                gbs = byt / (ms * 1e-3) / 1e9
                print(json.dumps({"kernel": name, "n": n, "ctas_per_sm": cps, "ms": ms, "gbs": gbs,
                                  "frac_of_measured": gbs / peak}), flush=True)
        del x, g, m, s0, s1, z
        torch.cuda.empty_cache()
    N.check(N.lib().lasgd_set_stream_ctas_per_sm(2))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""N=1 sync path replayed from a CUDA graph (k_sgd_dyn) against the streaming kernels'
CTAs per SM (lasgd_set_stream_ctas_per_sm): ms per step over 200 steps, best of 3."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200 as L  # noqa: E402
from paper_2203_13085_b200 import _native as N  # noqa: E402


def main():
    n = 25_557_032
    gen = torch.Generator(device="cuda").manual_seed(0)
    grads = [torch.randn(n, device="cuda", generator=gen) * 1e-2 for _ in range(2)]
    s = torch.cuda.Stream()
    for per_sm in (2, 3, 4, 6):
        N.check(N.lib().lasgd_set_stream_ctas_per_sm(per_sm))
        x = torch.randn(n, device="cuda", generator=gen) * 0.02
        with torch.cuda.stream(s):
            w = L.LASGDWorker(x, grads[0], sync_period=1, lr=0.1, sgd=L.SgdConfig(0.9, 0.0, 1e-4, True),
                              pipeline="fused", compute_stream=s)
            w.step()
            g = w.capture([grads[t % 2] for t in range(200)])
            g.replay()
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 200)
        print(json.dumps({"ctas_per_sm": per_sm, "ms_per_step": best, "hbm_frac": 6 * 4 * n / (best * 1e-3) / 1e9 / 6536.7}),
              flush=True)
        w.close()
    N.check(N.lib().lasgd_set_stream_ctas_per_sm(2))


if __name__ == "__main__":
    main()

"""Property-based parity of the fused round kernels on the GPU (hypothesis): random rank
counts, sizes (ragged, tiny, chunk-straddling), algorithms and modes, every result bit
for bit against the oracle.  Virtual ranks on cuda:0."""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import lasgd_oracle as O

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=120, deadline=None, suppress_health_check=[HealthCheck.too_slow])


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _bits(t):
    return t.cpu().numpy().view(np.uint32)


@SETTINGS
@given(P=st.integers(2, 8), n=st.integers(1, 40_000), algo=st.sampled_from([1, 2]),
       mode=st.sampled_from([0, 2]), momentum=st.booleans(), seed=st.integers(0, 2**31 - 1))
def test_k7_random(P, n, algo, mode, momentum, seed):
    from paper_2203_13085_b200 import kernels as K

    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = rng.standard_normal((2, P, n)).astype(np.float32)
    fk = dict(momentum=0.9, weight_decay=1e-4, nesterov=True) if momentum else {}
    cfg = O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True) if momentum else None
    xs = [_dev(x0) for _ in range(P)]
    ms = [torch.zeros(n, device="cuda") for _ in range(P)] if momentum else None
    xbars = [torch.zeros(n, device="cuda") for _ in range(P)]
    if mode == 0:  # LASGD pull rounds, sync period 1
        snaps = [[_dev(x0) for _ in range(P)], [torch.zeros(n, device="cuda") for _ in range(P)]]
        for t in range(2):
            K.fused_round_virtual(xs, [_dev(grads[t, r]) for r in range(P)], snaps[t % 2], snaps[1 - t % 2], 0.05,
                                  ms=ms, xbars=xbars, alpha=0.5, algo=algo, first_step=(t == 0), nblocks=5, **fk)
        torch.cuda.synchronize()
        ref, _, _, _ = O.run_lasgd_pull(x0, grads, [0.05, 0.05], P, 1, 0.5, sgd=cfg)
        for r in range(P):
            assert np.array_equal(_bits(xs[r]), ref[r].view(np.uint32)), (P, n, algo, r)
    else:  # SGD-AR rounds
        nexts = [torch.zeros(n, device="cuda") for _ in range(P)]
        for t in range(2):
            K.fused_round_virtual(xs, xs, [_dev(grads[t, r]) for r in range(P)], nexts, 0.05, ms=ms, xbars=xbars,
                                  algo=algo, mode=2, first_step=(t == 0), nblocks=5, **fk)
        torch.cuda.synchronize()
        ref, _ = O.run_sgd_ar(x0, grads, [0.05, 0.05], P, sgd=cfg)
        for r in range(P):
            assert np.array_equal(_bits(xs[r]), ref.view(np.uint32)), (P, n, algo, r)


@SETTINGS
@given(P=st.integers(2, 8), n=st.integers(1, 40_000), momentum=st.booleans(), seed=st.integers(0, 2**31 - 1))
def test_k8_push_random(P, n, momentum, seed):
    """K8 over virtual ranks: the mirror form at P=2, the staged form at P>=3."""
    from paper_2203_13085_b200 import kernels as K

    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = rng.standard_normal((3, P, n)).astype(np.float32)
    fk = dict(momentum=0.9, weight_decay=1e-4, nesterov=True) if momentum else {}
    cfg = O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True) if momentum else None
    xs = [_dev(x0) for _ in range(P)]
    ms = [torch.zeros(n, device="cuda") for _ in range(P)] if momentum else None
    snaps = [[_dev(x0) for _ in range(P)], [torch.zeros(n, device="cuda") for _ in range(P)]]
    xbars = [torch.zeros(n, device="cuda") for _ in range(P)]
    se = K.push_stage_elems(n, P)
    stages = [torch.zeros(2 * P * se, device="cuda") for _ in range(P)]
    for t in range(3):
        K.fused_push_virtual(xs, [_dev(grads[t, r]) for r in range(P)], snaps[t % 2], snaps[1 - t % 2], xbars, stages,
                             t % 2, t == 0, 0.05, ms=ms, alpha=0.5, first_step=(t == 0), nblocks=5, **fk)
    torch.cuda.synchronize()
    ref, _, _, _ = O.run_lasgd_pull(x0, grads, [0.05] * 3, P, 1, 0.5, sgd=cfg)
    for r in range(P):
        assert np.array_equal(_bits(xs[r]), ref[r].view(np.uint32)), (P, n, r)

"""K7 fused round (local step + ring-order mean + pull/finalize + next snapshot in one
pass) — bit-exact against the oracle's composition of the separate operations, which
is what the overlapped schedule computes."""

import numpy as np
import pytest
import torch

import paper_2203_13085_b200 as L
from oracle import lasgd_oracle as O
from paper_2203_13085_b200 import kernels as K

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    iv = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return a.shape == b.shape and np.array_equal(a.view(iv), b.view(iv))


CFGS = [O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True), O.SgdConfig(0.05, 0.0, 0.0, 0.0, False),
        O.SgdConfig(0.07, 0.8, 0.1, 5e-4, False)]


@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("n", [1, 7, 4099, 1_000_003])
@pytest.mark.parametrize("ci", [0, 1, 2])
@pytest.mark.parametrize("first", [True, False])
def test_fused_pull_bit_exact(algo, P, n, ci, first):
    cfg = CFGS[ci]
    rng = np.random.default_rng(P * 100 + n % 97 + ci)
    xs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    gs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    ms = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    snaps = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    alpha = 0.5 if ci == 1 else 1.0
    xt, gt, st = [dev(v) for v in xs], [dev(v) for v in gs], [dev(v) for v in snaps]
    mt = [dev(v) for v in ms] if cfg.momentum else None
    nt = [torch.full_like(x, float("nan")) for x in xt]
    xb = [torch.full_like(x, float("nan")) for x in xt] if algo == 2 else None
    K.fused_round_virtual(xt, gt, st, nt, cfg.lr, ms=mt, momentum=cfg.momentum, dampening=cfg.dampening,
                          weight_decay=cfg.weight_decay, nesterov=cfg.nesterov, first_step=first, alpha=alpha,
                          algo=algo, xbars=xb, nblocks=(7 if n > 1000 else 0))
    torch.cuda.synchronize()
    zbar = O.ring_mean(snaps) if P > 1 else None
    for r in range(P):
        x1, m1, _ = O.sgd_step_momentum(xs[r], gs[r], ms[r], cfg, first_step=first)
        ref = O.elastic_pull(x1, snaps[r], zbar, alpha) if P > 1 else x1
        assert same_bits(xt[r].cpu().numpy(), ref), (P, n, r)
        assert same_bits(nt[r].cpu().numpy(), ref), (P, n, r)
        if cfg.momentum:
            assert same_bits(mt[r].cpu().numpy(), m1)


@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_fused_finalize_matches_reference_bookkeeping(algo, P):
    n = 10_007
    rng = np.random.default_rng(P)
    xs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    gs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    ds = [rng.standard_normal(n).astype(np.float32) * 1e-2 for _ in range(P)]
    snaps = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    xt, gt, st, dt_ = [dev(v) for v in xs], [dev(v) for v in gs], [dev(v) for v in snaps], [dev(v) for v in ds]
    nt = [torch.empty_like(x) for x in xt]
    xb = [torch.empty_like(x) for x in xt] if algo == 2 else None
    K.fused_round_virtual(xt, gt, st, nt, 0.03, deltas=dt_, mode=1, algo=algo, xbars=xb)
    torch.cuda.synchronize()
    z = O.ring_mean(snaps)
    for r in range(P):
        _, d1 = O.sgd_step_delta(xs[r], ds[r], gs[r], 0.03)
        ref = O.finalize_delta(z, d1, None, P)
        assert same_bits(xt[r].cpu().numpy(), ref)
        assert same_bits(nt[r].cpu().numpy(), ref)


@pytest.mark.parametrize("mode", ["pull", "delta"])
@pytest.mark.parametrize("k", [1, 3])
def test_worker_fused_equals_overlap_single_gpu(mode, k):
    n, steps = 100_003, 7
    rng = np.random.default_rng(5)
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = [dev(rng.standard_normal(n).astype(np.float32)) for _ in range(steps)]
    sgd = L.SgdConfig(0.9, 0.0, 1e-4, True) if mode == "pull" else None
    out = {}
    for pipe in ("overlap", "fused"):
        x = dev(x0.copy())
        w = L.LASGDWorker(x, grads[0], sync_period=k, lr=0.05, mode=mode, sgd=sgd, pipeline=pipe)
        for t in range(steps):
            w.g = grads[t]
            w.step()
        torch.cuda.synchronize()
        out[pipe] = (x.cpu().numpy(), w.state.x_snapshot.cpu().numpy())
    assert same_bits(out["overlap"][0], out["fused"][0])
    assert same_bits(out["overlap"][1], out["fused"][1])
    # and both equal plain sequential SGD (P = 1)
    ref = x0.copy()
    m = np.zeros_like(ref)
    for t in range(steps):
        g = grads[t].cpu().numpy()
        if sgd is None:
            ref = O.sgd_step_plain(ref, g, 0.05)
        else:
            ref, m, _ = O.sgd_step_momentum(ref, g, m, O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True), t == 0)
    assert same_bits(out["fused"][0], ref)


def test_fused_rejects_bad_arguments():
    x = torch.zeros(16, device="cuda")
    with pytest.raises(ValueError):
        K.fused_round_virtual([x], [x], [x], [x], 0.1, alpha=0.0)
    with pytest.raises(ValueError):
        K.fused_round_virtual([x], [x], [x], [x], 0.1, mode=1)  # finalize needs delta
    with pytest.raises(ValueError):
        K.fused_round_virtual([x], [x], [x], [x], 0.1, momentum=0.9)  # momentum needs m


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [7, 4099, 100_003])
@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_push_round_multi_round_bit_exact(P, n, momentum):
    """K8 over virtual ranks, 3 rounds (sync period 1): staging, parity flips and the
    pushed means/contributions reproduce the oracle's deterministic loop bit for bit."""
    rng = np.random.default_rng(P * 31 + n % 101)
    steps = 3
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = rng.standard_normal((steps, P, n)).astype(np.float32)
    xs = [dev(x0.copy()) for _ in range(P)]
    ms = [torch.zeros(n, device="cuda") for _ in range(P)] if momentum else None
    snaps = [[dev(x0.copy()) for _ in range(P)], [torch.zeros(n, device="cuda") for _ in range(P)]]
    xbars = [torch.zeros(n, device="cuda") for _ in range(P)]
    se = K.push_stage_elems(n, P)
    stages = [torch.full((2 * P * se,), float("nan"), device="cuda") for _ in range(P)]
    cur = 0
    for t in range(steps):
        K.fused_push_virtual(xs, [dev(grads[t, r]) for r in range(P)], snaps[cur], snaps[1 - cur], xbars, stages, cur,
                             t == 0, 0.05, ms=ms, momentum=momentum, weight_decay=1e-4 if momentum else 0.0,
                             nesterov=bool(momentum), first_step=(t == 0), alpha=0.5, nblocks=5)
        cur = 1 - cur
    torch.cuda.synchronize()
    cfg = O.SgdConfig(0.05, momentum, 0.0, 1e-4, True) if momentum else None
    ref, _, _, _ = O.run_lasgd_pull(x0, grads, [0.05] * steps, P, 1, 0.5, sgd=cfg)
    for r in range(P):
        assert same_bits(xs[r].cpu().numpy(), ref[r]), (P, n, r)
        assert same_bits(snaps[cur][r].cpu().numpy(), ref[r]), (P, n, r)


def test_push_round_finalize_mode():
    P, n = 3, 10_007
    rng = np.random.default_rng(8)
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = rng.standard_normal((2, P, n)).astype(np.float32)
    xs = [dev(x0.copy()) for _ in range(P)]
    ds = [torch.zeros(n, device="cuda") for _ in range(P)]
    snaps = [[dev(x0.copy()) for _ in range(P)], [torch.zeros(n, device="cuda") for _ in range(P)]]
    xbars = [torch.zeros(n, device="cuda") for _ in range(P)]
    se = K.push_stage_elems(n, P)
    stages = [torch.zeros(2 * P * se, device="cuda") for _ in range(P)]
    for t in range(2):
        K.fused_push_virtual(xs, [dev(grads[t, r]) for r in range(P)], snaps[t % 2], snaps[1 - t % 2], xbars, stages,
                             t % 2, t == 0, 0.03, deltas=ds, delta_reset=(t > 0), mode=1)
    torch.cuda.synchronize()
    ref, _, _, _ = O.run_lasgd_delta(x0, grads, [0.03, 0.03], P, 1)
    for r in range(P):
        assert same_bits(xs[r].cpu().numpy(), ref[r])


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("n", [7, 4099, 100_003])
def test_sgd_ar_round_bit_exact(P, algo, n):
    """K7 mode 2 (SGD-AR, optimizer.py:214-242): one pass = ring-order mean of every
    rank's gradient slot + the momentum/Nesterov/wd step with it, bit-exact against the
    oracle's SGD-AR loop; the next-snapshot buffers are not written."""
    rng = np.random.default_rng(P * 7 + n % 13 + algo)
    steps = 3
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = rng.standard_normal((steps, P, n)).astype(np.float32)
    xs = [dev(x0.copy()) for _ in range(P)]
    ms = [torch.zeros(n, device="cuda") for _ in range(P)]
    xbars = [torch.zeros(n, device="cuda") for _ in range(P)]
    untouched = [torch.full((n,), 7.0, device="cuda") for _ in range(P)]
    etas = [0.1, 0.05, 0.2]
    for t in range(steps):
        slots = [dev(grads[t, r]) for r in range(P)]
        K.fused_round_virtual(xs, xs, slots, untouched, etas[t], ms=ms, xbars=xbars, momentum=0.9, weight_decay=1e-4,
                              nesterov=True, first_step=(t == 0), mode=2, algo=algo, nblocks=7)
    torch.cuda.synchronize()
    ref, _ = O.run_sgd_ar(x0, grads, etas, P, sgd=O.SgdConfig(1.0, 0.9, 0.0, 1e-4, True))
    for r in range(P):
        assert same_bits(xs[r].cpu().numpy(), ref), (P, algo, n, r)
        assert bool((untouched[r] == 7.0).all())


def test_sgd_ar_round_rejects_bad_arguments():
    x = torch.zeros(64, device="cuda")
    with pytest.raises(ValueError):  # needs peers
        K.fused_round_virtual([x], [x], [x], [x], 0.1, mode=2)
    with pytest.raises(ValueError):  # no delta bookkeeping in SGD-AR
        K.fused_round_virtual([x, x.clone()], [x, x], [x, x], [x, x], 0.1, deltas=[x, x], mode=2)
    st = [torch.zeros(2 * 2 * K.push_stage_elems(64, 2), device="cuda") for _ in range(2)]
    with pytest.raises(ValueError):  # no push form of the SGD-AR round
        K.fused_push_virtual([x, x.clone()], [x, x], [x, x], [x, x], [x, x], st, 0, True, 0.1, mode=2)


@pytest.mark.parametrize("P", [2, 8])
def test_push_round_1gib_exact_mean(P):
    """BASELINE configs[4]'s largest buffer (2^28 + 5 fp32 per rank) through K8 over
    virtual ranks (mirror form at P=2, staged form at P=8), checked by a size-independent
    property: small-integer contributions make every summation order exact, so with zero
    gradients and α = 1 every rank holds exactly sum/P (collective.py:200) after the
    first round, and the second round leaves it unchanged."""
    n = (1 << 28) + 5
    idx = torch.arange(n, device="cuda", dtype=torch.int64)
    xs = [((idx * 7 + 13 * r + (idx >> 11)) % 4096).to(torch.float32) for r in range(P)]
    del idx
    want = torch.zeros(n, device="cuda")
    for x in xs:
        want += x
    want /= P
    zero = torch.zeros(n, device="cuda")
    snaps = [[x.clone() for x in xs], [torch.empty(n, device="cuda") for _ in range(P)]]
    xbars = [torch.empty(n, device="cuda") for _ in range(P)]
    se = K.push_stage_elems(n, P)
    stages = [torch.empty(2 * P * se, device="cuda") for _ in range(P)]
    cur = 0
    for t in range(2):
        K.fused_push_virtual(xs, [zero] * P, snaps[cur], snaps[1 - cur], xbars, stages, cur, t == 0, 0.1,
                             alpha=1.0)
        cur = 1 - cur
        torch.cuda.synchronize()
        for r in range(P):
            assert torch.equal(xs[r].view(torch.int32), want.view(torch.int32)), (P, t, r)
            assert torch.equal(snaps[cur][r].view(torch.int32), want.view(torch.int32)), (P, t, r)
    del xs, snaps, xbars, stages
    torch.cuda.empty_cache()

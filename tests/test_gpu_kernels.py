"""Bit-exact parity of the rank-local kernels (K0 blend, K1 snapshot, K4 pull /
finalize, K5 local step) with the CPU oracle (fp32) and with the reference's own
golden outputs (f64).  Runs on the GPU box: ``pytest -m gpu``."""

import numpy as np
import pytest
import torch

from oracle import lasgd_oracle as O
from paper_2203_13085_b200 import kernels as K

pytestmark = pytest.mark.gpu

SIZES = [1, 3, 4, 5, 17, 1023, 4096, 100_609, 1_000_003]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    iv = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return np.array_equal(a.view(iv), b.view(iv))


def rnd(n, seed, dtype=np.float32, scale=1.0):
    return (np.random.default_rng(seed).standard_normal(n) * scale).astype(dtype)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("ab", [(1.0, -0.037), (0.5, 0.5), (0.3, 0.7), (1.0, -1.0)])
def test_blend_f32_bit_exact(n, ab):
    u, v = rnd(n, 1), rnd(n, 2)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    K.blend(out, ab[0], dev(u), ab[1], dev(v))
    assert same_bits(host(out), O.blend(ab[0], u, ab[1], v))


def test_blend_f64_matches_reference(golden_prims, golden_meta):
    u, v = golden_prims["blend_u"], golden_prims["blend_v"]
    for name in ("b1", "b2", "b3", "b4"):
        a, b = golden_meta[f"blend_{name}"]
        out = torch.empty(u.size, dtype=torch.float64, device="cuda")
        K.blend(out, a, dev(u), b, dev(v))
        assert same_bits(host(out), golden_prims[f"blend_{name}"])


def test_unaligned_views_use_scalar_path():
    base_u, base_v = rnd(10_001, 3), rnd(10_001, 4)
    u, v = dev(base_u)[1:], dev(base_v)[1:]
    out = torch.empty(10_001, dtype=torch.float32, device="cuda")[1:]
    K.blend(out, 1.0, u, -0.25, v)
    assert same_bits(host(out), O.blend(1.0, base_u[1:], -0.25, base_v[1:]))


@pytest.mark.parametrize("n", SIZES)
def test_snapshot_copy(n):
    x = rnd(n, 5)
    s = torch.empty(n, dtype=torch.float32, device="cuda")
    K.snapshot(s, dev(x))
    assert same_bits(host(s), x)


@pytest.mark.parametrize("n", SIZES)
def test_sgd_plain_and_delta_bit_exact(n):
    x, g, d = rnd(n, 6), rnd(n, 7), rnd(n, 8, scale=1e-3)
    eta = 0.0371
    xt, dt_ = dev(x), dev(d)
    K.sgd_step(xt, dev(g), eta, delta=dt_)
    rx, rd = O.sgd_step_delta(x, d, g, eta)
    assert same_bits(host(xt), rx) and same_bits(host(dt_), rd)
    # fresh accumulator (optimizer.py:174) without materialising zeros
    K.sgd_step(xt, dev(g), eta, delta=dt_, delta_reset=True)
    rx2, rd2 = O.sgd_step_delta(rx, None, g, eta, delta_reset=True)
    assert same_bits(host(xt), rx2) and same_bits(host(dt_), rd2)
    # plain step (no accumulator)
    xt = dev(x)
    K.sgd_step(xt, dev(g), eta)
    assert same_bits(host(xt), O.sgd_step_plain(x, g, eta))


@pytest.mark.parametrize("cfg", [
    O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True),
    O.SgdConfig(0.05, 0.9, 0.0, 0.0, False),
    O.SgdConfig(0.05, 0.8, 0.1, 5e-4, False),
    O.SgdConfig(0.2, 0.0, 0.0, 1e-2, False),
])
@pytest.mark.parametrize("n", [5, 4099, 1_000_003])
def test_sgd_momentum_bit_exact(cfg, n):
    x = rnd(n, 9)
    m = np.zeros_like(x)
    xt = dev(x)
    mt = torch.empty_like(xt) if cfg.momentum else None
    for t in range(4):
        g = rnd(n, 100 + t)
        K.sgd_step(xt, dev(g), cfg.lr, m=mt, momentum=cfg.momentum, dampening=cfg.dampening,
                   weight_decay=cfg.weight_decay, nesterov=cfg.nesterov, first_step=(t == 0))
        x, m, _ = O.sgd_step_momentum(x, g, m, cfg, first_step=(t == 0))
        assert same_bits(host(xt), x), t
        if cfg.momentum:
            assert same_bits(host(mt), m), t


def test_sgd_momentum_close_to_torch_optim():
    n = 1 << 16
    x = rnd(n, 11)
    p = torch.nn.Parameter(dev(x).clone())
    opt = torch.optim.SGD([p], lr=0.1, momentum=0.9, weight_decay=1e-4, nesterov=True)
    xt, mt = dev(x), torch.empty(n, device="cuda")
    for t in range(5):
        g = dev(rnd(n, 200 + t))
        p.grad = g.clone()
        opt.step()
        K.sgd_step(xt, g, 0.1, m=mt, momentum=0.9, weight_decay=1e-4, nesterov=True, first_step=(t == 0))
    torch.testing.assert_close(xt, p.detach(), rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("alpha", [1.0, 0.5, 0.25])
def test_elastic_pull_bit_exact(n, alpha):
    x, s, z = rnd(n, 12), rnd(n, 13), rnd(n, 14)
    xt, nxt = dev(x), torch.empty(n, dtype=torch.float32, device="cuda")
    K.elastic_pull(xt, dev(s), dev(z), alpha, snap_next=nxt)
    ref = O.elastic_pull(x, s, z, alpha)
    assert same_bits(host(xt), ref)
    assert same_bits(host(nxt), ref)


@pytest.mark.parametrize("n", SIZES)
def test_finalize_bit_exact(n):
    z, d, x = rnd(n, 15), rnd(n, 16), rnd(n, 17)
    xt, nxt = dev(x), torch.empty(n, dtype=torch.float32, device="cuda")
    K.finalize(xt, dev(z), dev(d), snap_next=nxt)
    ref = O.finalize_delta(z, d, x, 4)
    assert same_bits(host(xt), ref) and same_bits(host(nxt), ref)


def test_finalize_f64_matches_reference_kat():
    # z=[1,1], x=[3,0], snap=[2,1] (delta=[1,-1]) -> [2,0]
    xt = dev(np.array([3.0, 0.0]))
    K.finalize(xt, dev(np.array([1.0, 1.0])), dev(np.array([1.0, -1.0])))
    assert host(xt).tolist() == [2.0, 0.0]


def test_resnet50_size_bit_exact():
    n = 25_557_032
    x, g, s, z = rnd(n, 21), rnd(n, 22), rnd(n, 23), rnd(n, 24)
    cfg = O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True)
    xt, mt = dev(x), torch.empty(n, device="cuda")
    K.sgd_step(xt, dev(g), cfg.lr, m=mt, momentum=0.9, weight_decay=1e-4, nesterov=True, first_step=True)
    x1, m1, _ = O.sgd_step_momentum(x, g, np.zeros_like(x), cfg, True)
    assert same_bits(host(xt), x1) and same_bits(host(mt), m1)
    nxt = torch.empty_like(xt)
    K.elastic_pull(xt, dev(s), dev(z), 1.0, snap_next=nxt)
    ref = O.elastic_pull(x1, s, z, 1.0)
    assert same_bits(host(xt), ref) and same_bits(host(nxt), ref)


def test_nonfinite_counter():
    n = 100_003
    x, g = rnd(n, 30), rnd(n, 31)
    g[[0, 5000, n - 1]] = [np.inf, np.nan, -np.inf]
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    K.sgd_step(dev(x), dev(g), 0.1, nonfinite=nf)
    assert int(nf.item()) == 3
    nf.zero_()
    K.sgd_step(dev(x), dev(rnd(n, 32)), 0.1, nonfinite=nf)
    assert int(nf.item()) == 0


def test_dimension_and_dtype_errors():
    from paper_2203_13085_b200 import DimensionMismatchError

    a = torch.zeros(10, device="cuda")
    with pytest.raises(DimensionMismatchError):
        K.blend(a, 1.0, a, 1.0, torch.zeros(11, device="cuda"))
    with pytest.raises(TypeError):
        K.snapshot(a, torch.zeros(10, device="cuda", dtype=torch.float16))
    with pytest.raises(ValueError):
        K.elastic_pull(a, a, a, 1.5)


@pytest.mark.parametrize("n", [1, 7, 4099, 1_000_003])
@pytest.mark.parametrize("alpha", [1.0, 0.5])
@pytest.mark.parametrize("first", [True, False])
def test_sgd_pull_one_pass_equals_step_then_pull(n, alpha, first):
    """lasgd_sgd_pull (the deterministic overlap pipeline's round boundary) == K5 then K4,
    bit for bit, against the oracle; and the finalize form against step-then-finalize."""
    cfg = O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True)
    x, g, m, s, z, d = (rnd(n, 40 + i) for i in range(6))
    xt, gt, mt, st, zt = dev(x), dev(g), dev(m), dev(s), dev(z)
    nt = torch.full_like(xt, float("nan"))
    K.sgd_pull(xt, gt, nt, st, zt, cfg.lr, m=mt, momentum=0.9, weight_decay=1e-4, nesterov=True, first_step=first,
               alpha=alpha)
    x1, m1, _ = O.sgd_step_momentum(x, g, m, cfg, first_step=first)
    ref = O.elastic_pull(x1, s, z, alpha)
    assert same_bits(host(xt), ref) and same_bits(host(nt), ref) and same_bits(host(mt), m1)
    # finalize form (reference bookkeeping, plain SGD): x = z + (delta + (-lr) g)
    xt, dt, nt = dev(x), dev(d), torch.empty_like(dev(x))
    K.sgd_pull(xt, dev(g), nt, dev(s), dev(z), 0.05, delta=dt, mode=1)
    _, d1 = O.sgd_step_delta(x, d, g, 0.05)
    ref = O.finalize_delta(z, d1, x, 2)
    assert same_bits(host(xt), ref) and same_bits(host(nt), ref)

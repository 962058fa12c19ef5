"""Pin the C restatement of the oracle (oracle/lasgd_oracle.c, the timed CPU baseline and
the `--impl reference` arm of bench.py) to the reference's own outputs
(tests/golden/*.npz, made by tests/golden/make_golden.py from /root/reference) in f64,
and to the pinned Python oracle bit for bit in f32, at 1 and 16 OpenMP threads.  CPU only."""

import os
import subprocess

import numpy as np
import pytest

from lasgd_testutil import loop_cases
from oracle import lasgd_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def C():
    from oracle import c_oracle

    if not os.path.exists(c_oracle.LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    c_oracle.lib()
    yield c_oracle
    c_oracle.set_threads(os.cpu_count() or 1)


@pytest.fixture(params=[1, 16])
def threads(request, C):
    C.set_threads(request.param)
    return request.param


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    iv = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return a.shape == b.shape and np.array_equal(a.view(iv), b.view(iv))


def test_blend_f64_vs_reference(C, threads, golden_prims, golden_meta):
    u, v = golden_prims["blend_u"], golden_prims["blend_v"]
    for name in ("b1", "b2", "b3", "b4"):
        a, b = golden_meta[f"blend_{name}"]
        out = np.empty_like(u)
        C.blend(out, a, u, b, v)
        assert same_bits(out, golden_prims[f"blend_{name}"]), name


def test_ring_mean_f64_vs_reference(C, threads, golden_prims):
    for P in range(1, 9):
        for d in (1, 5, 7, 1000, 1001, 4099):
            vecs = [np.ascontiguousarray(v) for v in golden_prims[f"mean_in_{P}_{d}"]]
            outs = [np.empty(d) for _ in range(min(P, 3))]
            C.ring_mean(outs, vecs)
            for o in outs:
                assert same_bits(o, golden_prims[f"mean_out_{P}_{d}"]), (P, d)


def _c_delta_loop(C, x0, grads, etas, P, k):
    """The reference node loop (optimizer.py:181-207, collective_complete = (tau_i == k))
    driven through the C primitives: sgd_local_step -> oracle_sgd_delta, the ring mean
    -> oracle_ring_mean, lasgd_finalize_round -> oracle_finalize."""
    xs = [x0.copy() for _ in range(P)]
    ds = [np.zeros_like(x0) for _ in range(P)]
    snaps = [x0.copy() for _ in range(P)]
    z = np.empty_like(x0)
    C.ring_mean([z], snaps)
    hist, tau = [], 0
    for t, eta in enumerate(etas):
        for r in range(P):
            xn, dn = np.empty_like(x0), np.empty_like(x0)
            C.sgd_delta(xn, dn, xs[r], ds[r], np.ascontiguousarray(grads[t][r]), float(eta), delta_reset=False)
            xs[r], ds[r] = xn, dn
        tau += 1
        if tau == k:
            for r in range(P):
                if P > 1:
                    out = np.empty_like(x0)
                    C.finalize(out, z, ds[r])
                    xs[r] = out
                snaps[r] = xs[r].copy()
                ds[r] = np.zeros_like(x0)
            z = np.empty_like(x0)
            C.ring_mean([z], snaps)
            tau = 0
        hist.append(np.stack(xs))
    return hist, snaps, ds


def test_node_loop_delta_f64_vs_reference(C, threads, golden_loops):
    for tag, c in loop_cases(golden_loops, "abcde"):
        P, k = int(c["P"]), int(c["k"])
        hist, snaps, ds = _c_delta_loop(C, c["x0"], c["grads"], c["etas"], P, k)
        for t in range(len(hist)):
            assert same_bits(hist[t], c["xs_hist"][t]), (tag, t)
        assert same_bits(np.stack(snaps), c["final_snap"]), tag
        assert same_bits(np.stack(ds), c["final_delta"]), tag


def test_pull_loop_f64_vs_reference(C, threads, golden_pulls):
    """pull x -= alpha*(snap - xbar) (blend order of optimizer.py:256-257) + plain SGD."""
    for tag, c in loop_cases(golden_pulls, "abc"):
        P, k, alpha = int(c["P"]), int(c["k"]), float(c["alpha"])
        x0 = c["x0"]
        xs = [x0.copy() for _ in range(P)]
        snaps = [x0.copy() for _ in range(P)]
        z = np.empty_like(x0)
        C.ring_mean([z], snaps)
        tau = 0
        for t, eta in enumerate(c["etas"]):
            for r in range(P):
                xn, dn = np.empty_like(x0), np.empty_like(x0)
                C.sgd_delta(xn, dn, xs[r], np.zeros_like(x0), np.ascontiguousarray(c["grads"][t][r]), float(eta),
                            delta_reset=True)
                xs[r] = xn
            tau += 1
            if tau == k:
                for r in range(P):
                    if P > 1:
                        nxt = np.empty_like(x0)
                        C.pull(xs[r], nxt, snaps[r], z, alpha)
                        snaps[r] = nxt
                    else:
                        snaps[r] = xs[r].copy()
                z = np.empty_like(x0)
                C.ring_mean([z], snaps)
                tau = 0
            assert same_bits(np.stack(xs), c["xs_hist"][t]), (tag, t)


def test_f32_ops_bit_exact_vs_python_oracle(C, threads):
    rng = np.random.default_rng(11)
    n = 100_003
    x, g, m, d, s, z = (rng.standard_normal(n).astype(np.float32) for _ in range(6))
    # blend
    out = np.empty_like(x)
    C.blend(out, 0.3, x, -0.7, g)
    assert same_bits(out, O.blend(0.3, x, -0.7, g))
    # sgd_local_step with the delta accumulator, fresh and live
    for reset in (False, True):
        xn, dn = np.empty_like(x), np.empty_like(x)
        C.sgd_delta(xn, dn, x, d, g, 0.05, delta_reset=reset)
        ex, ed = O.sgd_step_delta(x, d, g, 0.05, delta_reset=reset)
        assert same_bits(xn, ex) and same_bits(dn, ed)
    # momentum / Nesterov / weight decay step (the GPU arm's local step)
    for first in (True, False):
        for nest in (True, False):
            xc, mc = x.copy(), m.copy()
            C.sgd_momentum(xc, g, mc, 0.1, 0.9, 0.0, 1e-4, nest, first)
            ex, em, _ = O.sgd_step_momentum(x, g, m, O.SgdConfig(0.1, 0.9, 0.0, 1e-4, nest), first_step=first)
            assert same_bits(xc, ex) and same_bits(mc, em), (first, nest)
    # finalize and pull
    out = np.empty_like(x)
    C.finalize(out, z, d)
    assert same_bits(out, O.finalize_delta(z, d, x, 2))
    for alpha in (1.0, 0.5):
        xc, nxt = x.copy(), np.empty_like(x)
        C.pull(xc, nxt, s, z, alpha)
        assert same_bits(xc, O.elastic_pull(x, s, z, alpha)) and same_bits(nxt, xc)
    # ring mean, ragged sizes
    for P in (2, 3, 5, 8):
        for nn in (7, 1001, 100_003):
            vs = [rng.standard_normal(nn).astype(np.float32) for _ in range(P)]
            o = np.empty(nn, np.float32)
            C.ring_mean([o], vs)
            assert same_bits(o, O.ring_mean(vs)), (P, nn)


def test_f64_momentum_step_vs_python_oracle(C, threads):
    rng = np.random.default_rng(12)
    n = 50_001
    x, g, m = (rng.standard_normal(n) for _ in range(3))
    xc, mc = x.copy(), m.copy()
    C.sgd_momentum(xc, g, mc, 0.1, 0.9, 0.0, 1e-4, True, False)
    ex, em, _ = O.sgd_step_momentum(x, g, m, O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True), first_step=False)
    assert same_bits(xc, ex) and same_bits(mc, em)

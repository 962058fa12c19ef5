"""Out-of-bounds guard: every buffer a kernel touches is carved out of a larger
allocation whose head and tail guard bands hold a sentinel bit pattern, and after the
launch the guards must be bit-for-bit intact while the payload matches the oracle.
This is the repo's memory-safety net in place of compute-sanitizer (closed on this
GPU pool: runs under it left GPUs needing a reset).  It covers every streaming kernel
(scalar tail, unaligned scalar path), the virtual-rank mean / fused / push rounds at
P = 2..8 (ragged chunks, empty chunks when n < P) and the graph-replayed worker loop."""

import numpy as np
import pytest
import torch

import paper_2203_13085_b200 as L
from oracle import lasgd_oracle as O
from paper_2203_13085_b200 import _native as N
from paper_2203_13085_b200 import kernels as K

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side (16 KiB for fp32): a full pack-loop stride of slack
SENTINEL = 0x7FC0DEAD  # a quiet-NaN payload no kernel produces from finite inputs
SIZES = [1, 3, 4, 5, 17, 1000, 1001, 65_539]


class Guarded:
    """A device vector of n elements with guard bands; ``shift`` misaligns its start."""

    def __init__(self, n, values=None, shift=0):
        self.n, self.shift = n, shift
        self.buf = torch.empty(2 * GUARD + n + shift, dtype=torch.float32, device="cuda")
        self.buf.view(torch.int32).fill_(SENTINEL)
        self.t = self.buf[GUARD + shift:GUARD + shift + n]
        if values is not None:
            self.t.copy_(torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)))

    def intact(self):
        b = self.buf.view(torch.int32)
        head, tail = b[:GUARD + self.shift], b[GUARD + self.shift + self.n:]
        return bool((head == SENTINEL).all()) and bool((tail == SENTINEL).all())

    def np(self):
        return self.t.cpu().numpy()


def same_bits(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


def rnd(n, seed):
    return np.random.default_rng(seed).standard_normal(n).astype(np.float32)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("shift", [0, 1])
def test_streaming_kernels_stay_in_bounds(n, shift):
    x, g, m, d, s, z = (rnd(n, i) for i in range(6))
    bufs = {k: Guarded(n, v, shift) for k, v in dict(x=x, g=g, m=m, d=d, s=s, z=z).items()}
    out = Guarded(n, shift=shift)
    K.blend(out.t, 0.5, bufs["x"].t, -0.25, bufs["g"].t)
    torch.cuda.synchronize()
    assert same_bits(out.np(), O.blend(0.5, x, -0.25, g))
    snap = Guarded(n, shift=shift)
    K.snapshot(snap.t, bufs["x"].t)
    K.sgd_step(bufs["x"].t, bufs["g"].t, 0.1, m=bufs["m"].t, delta=bufs["d"].t, momentum=0.9, weight_decay=1e-4,
               nesterov=True)
    K.elastic_pull(bufs["x"].t, bufs["s"].t, bufs["z"].t, 0.5, snap_next=snap.t)
    K.finalize(out.t, bufs["z"].t, bufs["d"].t, snap_next=snap.t)
    torch.cuda.synchronize()
    for b in list(bufs.values()) + [out, snap]:
        assert b.intact(), (n, shift)


@pytest.mark.parametrize("P", [2, 3, 5, 8])
@pytest.mark.parametrize("n", [3, 5, 1001, 65_539])
@pytest.mark.parametrize("algo", [N.ALGO_ONESHOT, N.ALGO_TWOSHOT])
def test_virtual_mean_stays_in_bounds(P, n, algo):
    vs = [rnd(n, 10 + r) for r in range(P)]
    srcs = [Guarded(n, v) for v in vs]
    outs = [Guarded(n) for _ in range(P)]
    K.mean_virtual([o.t for o in outs], [s.t for s in srcs], algo=algo, nblocks=5)
    torch.cuda.synchronize()
    want = O.ring_mean(vs)
    for o in outs:
        assert o.intact() and same_bits(o.np(), want), (P, n)
    assert all(s.intact() for s in srcs)


@pytest.mark.parametrize("P", [1, 2, 4, 7])
@pytest.mark.parametrize("n", [3, 1001, 65_539])
@pytest.mark.parametrize("algo", [N.ALGO_ONESHOT, N.ALGO_TWOSHOT])
def test_virtual_fused_round_stays_in_bounds(P, n, algo):
    cfg = O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True)
    xs, gs, ms, ss = ([rnd(n, 100 * k + r) for r in range(P)] for k in range(4))
    X, G, M, S = ([Guarded(n, v) for v in arr] for arr in (xs, gs, ms, ss))
    NX = [Guarded(n) for _ in range(P)]
    XB = [Guarded(n) for _ in range(P)]
    K.fused_round_virtual([b.t for b in X], [b.t for b in G], [b.t for b in S], [b.t for b in NX], cfg.lr,
                          ms=[b.t for b in M], momentum=0.9, weight_decay=1e-4, nesterov=True, alpha=0.5,
                          algo=algo, xbars=[b.t for b in XB] if algo == N.ALGO_TWOSHOT else None, nblocks=3)
    torch.cuda.synchronize()
    zbar = O.ring_mean(ss) if P > 1 else None
    for r in range(P):
        x1, _, _ = O.sgd_step_momentum(xs[r], gs[r], ms[r], cfg, first_step=False)
        ref = O.elastic_pull(x1, ss[r], zbar, 0.5) if P > 1 else x1
        assert same_bits(X[r].np(), ref) and same_bits(NX[r].np(), ref), (P, n, r)
    for b in X + G + M + S + NX + (XB if algo == N.ALGO_TWOSHOT else []):
        assert b.intact(), (P, n)


@pytest.mark.parametrize("P", [2, 3, 6, 8])
@pytest.mark.parametrize("n", [5, 1001, 65_539])
def test_virtual_push_round_stays_in_bounds(P, n):
    cfg = O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True)
    xs, gs, ss = ([rnd(n, 300 * k + r) for r in range(P)] for k in range(3))
    X, G, S0 = ([Guarded(n, v) for v in arr] for arr in (xs, gs, ss))
    M = [Guarded(n, np.zeros(n, np.float32)) for _ in range(P)]
    S1 = [Guarded(n) for _ in range(P)]
    XB = [Guarded(n) for _ in range(P)]
    se = K.push_stage_elems(n, P)
    ST = [Guarded(2 * P * se) for _ in range(P)]
    snaps = [[b.t for b in S0], [b.t for b in S1]]
    xr = [x.copy() for x in xs]
    mr = [np.zeros(n, np.float32) for _ in range(P)]
    sr = [s.copy() for s in ss]
    for t in range(2):
        c = t % 2
        K.fused_push_virtual([b.t for b in X], [b.t for b in G], snaps[c], snaps[1 - c], [b.t for b in XB],
                             [b.t for b in ST], c, t == 0, 0.1, ms=[b.t for b in M], momentum=0.9,
                             weight_decay=1e-4, nesterov=True, first_step=t == 0, alpha=1.0)
        zbar = O.ring_mean(sr)
        for r in range(P):
            x1, mr[r], _ = O.sgd_step_momentum(xr[r], gs[r], mr[r], cfg, first_step=t == 0)
            xr[r] = O.elastic_pull(x1, sr[r], zbar, 1.0)
        sr = [x.copy() for x in xr]
    torch.cuda.synchronize()
    for r in range(P):
        assert same_bits(X[r].np(), xr[r]), (P, n, r)
    for b in X + G + M + S0 + S1 + XB + ST:
        assert b.intact(), (P, n)


@pytest.mark.parametrize("n", [5, 1001, 65_539])
def test_graph_replayed_worker_stays_in_bounds(n):
    x0, g0, g1 = rnd(n, 1), rnd(n, 2), rnd(n, 3)
    X, G0, G1 = Guarded(n, x0), Guarded(n, g0), Guarded(n, g1)
    w = L.LASGDWorker(X.t, G0.t, sync_period=2, lr=0.05, sgd=L.SgdConfig(0.9, 0.0, 1e-4, True), pipeline="fused")
    graph = w.capture([G0.t, G1.t])
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert X.intact() and G0.intact() and G1.intact()
    assert w.state.momentum_buf is not None
    w.close()

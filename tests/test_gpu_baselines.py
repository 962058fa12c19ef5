"""SGD-AR baseline (optimizer.py:214-242) and adaptive completion on one GPU."""

import os

import numpy as np
import pytest
import torch

import paper_2203_13085_b200 as L
from oracle import lasgd_oracle as O

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    iv = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return a.shape == b.shape and np.array_equal(a.view(iv), b.view(iv))


def test_sgd_ar_f64_bit_exact_vs_reference():
    g = dict(np.load(os.path.join(GOLDEN, "sgd_ar.npz")))
    P = g["grads"].shape[1]
    tr = L.CudaLoopbackTransport(P, dtype=torch.float64)
    states = [L.NodeState.fresh(r, g["x0"], dtype=torch.float64) for r in range(P)]
    for t in range(len(g["etas"])):
        grads = [torch.from_numpy(g["grads"][t, r]).cuda() for r in range(P)]
        mg = L.sync_allreduce_sgd_round(states, grads, float(g["etas"][t]), transport=tr, round_id=t)
        torch.cuda.synchronize()
        assert same_bits(mg.cpu().numpy(), g["mean_hist"][t])
        for st in states:
            assert same_bits(st.x_local.cpu().numpy(), g["x_hist"][t])
            assert same_bits(st.x_snapshot.cpu().numpy(), g["x_hist"][t])


def test_sgd_ar_f32_matches_oracle_and_detects_divergence():
    rng = np.random.default_rng(2)
    P, n = 4, 10_007
    x0 = rng.standard_normal(n).astype(np.float32)
    states = [L.NodeState.fresh(r, x0) for r in range(P)]
    ref = x0.copy()
    for t in range(3):
        grads = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
        L.sync_allreduce_sgd_round(states, [torch.from_numpy(v).cuda() for v in grads], 0.1, round_id=t)
        ref = O.sgd_step_plain(ref, O.ring_mean(grads), 0.1)
    torch.cuda.synchronize()
    for st in states:
        assert same_bits(st.x_local.cpu().numpy(), ref)
    states[2].x_local[5] += 1.0
    with pytest.raises(L.ModelDivergenceError):
        L.sync_allreduce_sgd_round(states, [torch.zeros(n, device="cuda")] * P, 0.1, round_id=9)


def test_adaptive_single_rank_closes_every_step():
    rng = np.random.default_rng(4)
    n, steps = 50_003, 9
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = [torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda() for _ in range(steps)]
    x = torch.from_numpy(x0.copy()).cuda()
    w = L.LASGDWorker(x, grads[0], lr=0.05, adaptive=True, tau_max=4, sync_period=4)
    for t in range(steps):
        w.g = grads[t]
        assert w.step()  # with one rank the mean is always "landed": every step closes a round
    torch.cuda.synchronize()
    assert dict(w.tau_hist) == {1: steps}
    ref = x0.copy()
    for t in range(steps):
        ref = O.sgd_step_plain(ref, grads[t].cpu().numpy(), 0.05)
    assert same_bits(x.cpu().numpy(), ref)
    assert same_bits(w.state.x_snapshot.cpu().numpy(), ref)


def test_worker_rejects_fused_adaptive_and_bad_config():
    x = torch.zeros(64, device="cuda")
    with pytest.raises(ValueError):
        L.LASGDWorker(x, x, lr=0.1, adaptive=True, pipeline="fused")
    with pytest.raises(ValueError):
        L.LASGDWorker(x, x, lr=0.1, alpha=0.0)
    with pytest.raises(ValueError):
        L.LASGDWorker(x, x, lr=0.1, sync_period=0)


def test_integration_doc_loop_runs():
    """The reference-style loop of INTEGRATION.md §2 (poll-driven ticks, loopback)."""
    P, n, tau_max = 3, 4099, 2
    rng = np.random.default_rng(6)
    x0 = rng.standard_normal(n).astype(np.float32)
    tr = L.CudaLoopbackTransport(P)
    states = [L.NodeState.fresh(r, x0, mode="delta") for r in range(P)]
    for r, st in enumerate(states):
        st.pending = tr.submit(0, r, st.x_snapshot)
    grad_fn = [lambda x, r=r: torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda() for r in range(P)]
    schedule = L.LrSchedule(0.01, 1, 0)
    finalized = 0
    for _ in range(20):
        for r, st in enumerate(states):
            done = L.poll(st.pending) is L.Status.COMPLETE
            act = L.lasgd_node_tick(st, grad_fn[r], schedule, done, st.pending if done else None, tau_max, P,
                                    submit=lambda v, r=r, st=st: tr.submit(st.global_clock, r, v))
            finalized += act is L.TickAction.FINALIZED
            assert st.tau_i <= tau_max
    torch.cuda.synchronize()
    assert finalized > 0
    for st in states:
        st.check_finite()

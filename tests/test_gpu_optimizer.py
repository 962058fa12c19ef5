"""End-to-end parity of the reference-facing API (NodeState / sgd_local_step /
lasgd_finalize_round / lasgd_node_tick + CudaLoopbackTransport) on one GPU:

* f64: the reference's own node loop (tests/golden/node_loops.npz) reproduced
  bit for bit at every step;
* fp32: bit-exact against the fp32 oracle restatement;
* config 1 (BASELINE configs[0]): MLP [784,128,1], 4 workers, tau=4,
  alpha in {1, 0.5}: loss trajectory within 1e-4 of the reference over 100 steps.
"""

import numpy as np
import pytest
import torch

import paper_2203_13085_b200 as L
from lasgd_testutil import loop_cases
from oracle import lasgd_oracle as O
from oracle import problems_oracle as PO

pytestmark = pytest.mark.gpu


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    iv = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return a.shape == b.shape and np.array_equal(a.view(iv), b.view(iv))


class ConstSchedule(L.LrSchedule):
    pass


def run_api_loop(x0, grads, etas, P, k, dtype, mode, alpha=None, sgd=None):
    """Drive the reference-facing API exactly like tests/golden/make_golden.py drives the reference."""
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    tr = L.CudaLoopbackTransport(P, dtype=tdt)
    states = [L.NodeState.fresh(r, x0.astype(dtype), mode=mode, dtype=tdt, sgd=sgd) for r in range(P)]
    for r, st in enumerate(states):
        st.pending = tr.submit(0, r, st.x_snapshot)
    hist = []
    for t in range(len(etas)):
        for r, st in enumerate(states):
            g = torch.from_numpy(grads[t, r].astype(dtype)).cuda()
            sch = L.LrSchedule(float(etas[t]), 1, 0)  # lr_at -> peak/10**0 = eta exactly
            act = L.lasgd_node_tick(st, lambda _x, g=g: g, sch, False, None, k, P)
            assert act is L.TickAction.COMPUTED_STEP
        if states[0].tau_i == k:
            z = states[0].pending.result_async()
            rid = states[0].global_clock + 1
            for r, st in enumerate(states):
                act = L.lasgd_node_tick(st, None, None, True, z, k, P,
                                        submit=lambda v, r=r, rid=rid: tr.submit(rid, r, v), alpha=alpha)
                assert act is L.TickAction.FINALIZED
        torch.cuda.synchronize()
        hist.append(np.stack([st.x_local.cpu().numpy() for st in states]))
    return hist, states


def test_node_loop_f64_bit_exact_vs_reference(golden_loops):
    for tag, c in loop_cases(golden_loops, "abcde"):
        P, k = int(c["P"]), int(c["k"])
        hist, states = run_api_loop(c["x0"], c["grads"], c["etas"], P, k, np.float64, "delta")
        for t in range(len(hist)):
            assert same_bits(hist[t], c["xs_hist"][t]), (tag, t)
        snaps = np.stack([st.x_snapshot.cpu().numpy() for st in states])
        assert same_bits(snaps, c["final_snap"]), tag


def test_node_loop_f32_bit_exact_vs_oracle(golden_loops):
    for tag, c in loop_cases(golden_loops, "abcde"):
        P, k = int(c["P"]), int(c["k"])
        x0, grads = c["x0"].astype(np.float32), c["grads"].astype(np.float32)
        hist, _ = run_api_loop(x0, grads, c["etas"], P, k, np.float32, "delta")
        _, _, _, ref = O.run_lasgd_delta(x0, grads, c["etas"], P, k)
        for t in range(len(hist)):
            assert same_bits(hist[t], np.stack(ref[t])), (tag, t)


def test_pull_loop_f64_bit_exact_vs_reference(golden_pulls):
    for tag, c in loop_cases(golden_pulls, "abc"):
        P, k, alpha = int(c["P"]), int(c["k"]), float(c["alpha"])
        hist, _ = run_api_loop(c["x0"], c["grads"], c["etas"], P, k, np.float64, "pull", alpha=alpha)
        for t in range(len(hist)):
            assert same_bits(hist[t], c["xs_hist"][t]), (tag, t)


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_momentum_pull_loop_f32_bit_exact_vs_oracle(alpha):
    rng = np.random.default_rng(77)
    P, k, steps, n = 4, 2, 8, 10_007
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = rng.standard_normal((steps, P, n)).astype(np.float32)
    etas = np.full(steps, 0.05)
    cfg = O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True)
    sgd = L.SgdConfig(0.9, 0.0, 1e-4, True)
    hist, _ = run_api_loop(x0, grads, etas, P, k, np.float32, "pull", alpha=alpha, sgd=sgd)
    _, _, _, ref = O.run_lasgd_pull(x0, grads, etas, P, k, alpha, sgd=cfg)
    for t in range(steps):
        assert same_bits(hist[t], np.stack(ref[t])), t


def test_budget_and_missing_center_errors():
    st = L.NodeState.fresh(0, np.zeros(8, np.float32))
    g = torch.ones(8, device="cuda")
    L.sgd_local_step(st, g, 0.1, tau_max=1)
    with pytest.raises(RuntimeError):
        L.sgd_local_step(st, g, 0.1, tau_max=1)  # optimizer.py:141-144
    with pytest.raises(ValueError):
        L.lasgd_node_tick(st, None, None, True, None, 1, 2)
    assert L.lasgd_node_tick(st, None, L.LrSchedule(0.1, 1, 0), False, None, 1, 2) is L.TickAction.WAITING_ON_COLLECTIVE


def test_single_node_bit_identical_to_sequential_sgd():
    """AC2: P = 1 LASGD == sequential SGD, bit for bit, 500 steps."""
    rng = np.random.default_rng(1)
    n = 4099
    x0 = rng.standard_normal(n).astype(np.float32)
    st = L.NodeState.fresh(0, x0, mode="delta")
    ref = x0.copy()
    sch = L.LrSchedule(0.01, 1, 0)
    for t in range(500):
        g = rng.standard_normal(n).astype(np.float32)
        L.sgd_local_step(st, torch.from_numpy(g).cuda(), L.lr_at(sch, t), tau_max=3)
        ref = O.sgd_step_plain(ref, g, L.lr_at(sch, t))
        if st.tau_i == 3:
            L.lasgd_finalize_round(st, None, 1)
    assert same_bits(st.x_local.cpu().numpy(), ref)


def test_lazy_nonfinite_detection():
    st = L.NodeState.fresh(0, np.zeros(1024, np.float32), mode="pull")
    g = torch.ones(1024, device="cuda")
    g[3] = float("nan")
    L.sgd_local_step(st, g, 0.1, tau_max=10)
    with pytest.raises(L.NonFiniteError):
        st.check_finite()
    st2 = L.NodeState.fresh(0, np.zeros(16, np.float32), check_finite="eager")
    with pytest.raises(L.NonFiniteError):
        L.sgd_local_step(st2, torch.full((16,), float("inf"), device="cuda"), 0.1, tau_max=10)


# ------------------------------------------------------------------ config 1
class Mlp(torch.nn.Module):
    def __init__(self, dims):
        super().__init__()
        self.layers = torch.nn.ModuleList(torch.nn.Linear(i, o) for i, o in zip(dims[:-1], dims[1:]))

    def forward(self, X):
        h = X
        for i, layer in enumerate(self.layers):
            h = layer(h)
            if i < len(self.layers) - 1:
                h = torch.tanh(h)
        return h[:, 0]


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_config1_loss_trajectory_within_1e4(golden_config1, alpha):
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    P, k, steps, dims = 4, 4, 100, [784, 128, 1]
    X, y = PO.make_synthetic(0, 4096, 784, 0.1, "regression")
    Xd = torch.from_numpy(X.astype(np.float32)).cuda()
    yd = torch.from_numpy(y.astype(np.float32)).cuda()
    n = PO.mlp_dim(dims)
    x0 = (np.random.default_rng(0).standard_normal(n) * 0.05).astype(np.float32)
    mode = "delta" if alpha == 1.0 else "pull"
    models, flats, states = [], [], []
    tr = L.CudaLoopbackTransport(P)
    for r in range(P):
        m = Mlp(dims).cuda()
        f = L.FlatParams(m)
        f.x.copy_(torch.from_numpy(x0))
        st = L.NodeState.fresh(r, f.x, mode=mode, copy=False)
        st.pending = tr.submit(0, r, st.x_snapshot)
        models.append(m)
        flats.append(f)
        states.append(st)
    samplers = [PO.ShardSampler(4096, r, P, 32, seed=0) for r in range(P)]
    sch = L.LrSchedule(0.01, 1, 0)
    losses = np.zeros((steps, P))
    for t in range(steps):
        for r in range(P):
            def grad_fn(_x, r=r, t=t):
                b = torch.from_numpy(samplers[r].next_batch()).cuda()
                flats[r].zero_grad()
                resid = models[r](Xd[b]) - yd[b]
                loss = (resid @ resid) / (2.0 * b.numel())
                loss.backward()
                losses[t, r] = float(loss)
                return flats[r].g

            assert L.lasgd_node_tick(states[r], grad_fn, sch, False, None, k, P) is L.TickAction.COMPUTED_STEP
        if states[0].tau_i == k:
            z = states[0].pending.result_async()
            rid = states[0].global_clock + 1
            for r in range(P):
                L.lasgd_node_tick(states[r], None, sch, True, z, k, P,
                                  submit=lambda v, r=r, rid=rid: tr.submit(rid, r, v), alpha=alpha)
    ref = golden_config1[f"a{int(alpha * 100)}_losses"]
    rel = np.abs(losses - ref) / np.abs(ref)
    assert rel.max() < 1e-4, rel.max()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_finalize_twice_without_a_step_uses_zero_delta(dtype):
    """optimizer.py:171-174: finalize resets delta to zero, so a second finalize with no
    local step in between computes new = z + 0 (the poll-driven lasgd_node_tick loop hits
    this when a round is already complete at the next tick), and delta reads back as 0."""
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    rng = np.random.default_rng(5)
    n = 4099
    x0 = rng.standard_normal(n).astype(dtype)
    g = rng.standard_normal(n).astype(dtype)
    z1 = rng.standard_normal(n).astype(dtype)
    z2 = rng.standard_normal(n).astype(dtype)
    st = L.NodeState.fresh(0, x0, mode="delta", dtype=tdt)
    L.sgd_local_step(st, torch.from_numpy(g).cuda(), 0.1, tau_max=4)
    L.lasgd_finalize_round(st, torch.from_numpy(z1).cuda(), 2)
    L.lasgd_finalize_round(st, torch.from_numpy(z2).cuda(), 2)  # no step in between
    torch.cuda.synchronize()
    want = z2 + np.zeros(n, dtype)  # blend(1, z, 1, zeros) == z + 0
    assert same_bits(st.x_local.cpu().numpy(), want)
    assert same_bits(st.x_snapshot.cpu().numpy(), want)
    assert not st.delta.cpu().numpy().any()
    # the accumulator is live again after the next step: delta = 0 + (-eta)*g
    L.sgd_local_step(st, torch.from_numpy(g).cuda(), 0.1, tau_max=4)
    torch.cuda.synchronize()
    assert same_bits(st.delta.cpu().numpy(), np.zeros(n, dtype) + dtype(-0.1) * g)


def test_worker_rejects_communicator_of_another_shape():
    comm = L.P2PCommunicator(1000)
    x = torch.zeros(999, device="cuda")
    with pytest.raises(ValueError, match="communicator"):
        L.LASGDWorker(x, torch.zeros_like(x), comm=comm, lr=0.1)
    xd = torch.zeros(1000, device="cuda", dtype=torch.float64)
    with pytest.raises(ValueError, match="communicator"):
        L.LASGDWorker(xd, torch.zeros_like(xd), comm=comm, lr=0.1)
    comm.close()

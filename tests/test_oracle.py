"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/, made by
tests/golden/make_golden.py from /root/reference).  CPU only."""

import numpy as np
import pytest

from oracle import lasgd_oracle as O
from oracle import problems_oracle as PO
from lasgd_testutil import loop_cases


def test_partition_matches_reference(golden_meta):
    for key, bounds in golden_meta["partition"].items():
        d, P = map(int, key.split(","))
        assert [list(b) for b in O.partition_chunks(d, P)] == bounds
        # closed-form chunk id agrees with the bounds (used by the CUDA kernels)
        if d < 10**6:
            j = np.arange(d)
            cid = O.chunk_of(j, d, P)
            for c, (s, e) in enumerate(bounds):
                assert np.all(cid[s:e] == c)


def test_bytes_per_node_matches_reference(golden_meta):
    for key, vals in golden_meta["bytes_per_node"].items():
        d, P, b = map(int, key.split(","))
        assert O.bytes_per_node(d, P, b) == vals[0]
        for r in range(P):
            assert O.bytes_per_node(d, P, b, rank=r) == vals[1 + r]
    assert O.bytes_per_node(100, 4, 8) == 1200


def test_blend_bit_exact_f64(golden_prims, golden_meta):
    u, v = golden_prims["blend_u"], golden_prims["blend_v"]
    for name in ("b1", "b2", "b3", "b4"):
        a, b = golden_meta[f"blend_{name}"]
        assert np.array_equal(O.blend(a, u, b, v), golden_prims[f"blend_{name}"])
    # SPEC.md:53-56 KATs
    assert np.array_equal(O.blend(1, np.array([1.0, 2]), 1, np.array([3.0, 4])), [4, 6])
    assert np.array_equal(O.blend(0.5, np.array([2.0, 2]), 0.5, np.array([0.0, 4])), [1, 3])


def test_ring_mean_bit_exact_f64(golden_prims):
    for P in range(1, 9):
        for d in (1, 5, 7, 1000, 1001, 4099):
            vecs = list(golden_prims[f"mean_in_{P}_{d}"])
            assert np.array_equal(O.ring_mean(vecs), golden_prims[f"mean_out_{P}_{d}"]), (P, d)


def test_ring_mean_order_is_not_naive_order(golden_prims):
    # documents why the order matters: ascending-order mean differs somewhere
    diffs = 0
    for P in (3, 5, 7, 8):
        vecs = list(golden_prims[f"mean_in_{P}_4099"])
        diffs += int(np.count_nonzero(O.ring_mean(vecs) != O.naive_mean(vecs)))
    assert diffs > 0


def test_mean_kat():
    out = O.ring_mean([np.array([1.0, 2, 3]), np.array([4.0, 5, 6]), np.array([7.0, 8, 9])])
    assert np.array_equal(out, [4, 5, 6])


def test_lr_at_matches_reference(golden_meta):
    b, s, w, dec, f, spe = golden_meta["lr_sched"]
    sch = O.LrSchedule(b, s, w, tuple(dec), f, spe)
    for step, val in golden_meta["lr_vals"]:
        assert O.lr_at(sch, step) == val
    sch2 = O.LrSchedule(0.01, 1, 0)
    for step, val in golden_meta["lr_vals_flat"]:
        assert O.lr_at(sch2, step) == val


def test_node_loop_delta_bit_exact_f64(golden_loops):
    for tag, c in loop_cases(golden_loops, "abcde"):
        P, k = int(c["P"]), int(c["k"])
        xs, snaps, _, hist = O.run_lasgd_delta(c["x0"], c["grads"], c["etas"], P, k)
        for t in range(len(hist)):
            assert np.array_equal(np.stack(hist[t]), c["xs_hist"][t]), (tag, t)
        assert np.array_equal(np.stack(snaps), c["final_snap"]), tag


def test_pull_loop_bit_exact_f64(golden_pulls):
    for tag, c in loop_cases(golden_pulls, "abc"):
        P, k, alpha = int(c["P"]), int(c["k"]), float(c["alpha"])
        _, _, _, hist = O.run_lasgd_pull(c["x0"], c["grads"], c["etas"], P, k, alpha)
        for t in range(len(hist)):
            assert np.array_equal(np.stack(hist[t]), c["xs_hist"][t]), (tag, t)


def test_sgd_ar_loop_bit_exact_f64():
    """run_sgd_ar vs the reference's sync_allreduce_sgd_round (tests/golden/sgd_ar.npz)."""
    import os

    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "sgd_ar.npz")))
    P = g["grads"].shape[1]
    for t in range(1, len(g["etas"]) + 1):
        x, means = O.run_sgd_ar(g["x0"], g["grads"][:t], g["etas"][:t], P)
        assert np.array_equal(x, g["x_hist"][t - 1]), t
        assert np.array_equal(means[-1], g["mean_hist"][t - 1]), t


def test_alpha1_pull_close_to_reference_finalize(golden_loops):
    """x - (snap - z) vs z + delta: equal up to rounding."""
    for tag, c in loop_cases(golden_loops, "abe"):
        P, k = int(c["P"]), int(c["k"])
        _, _, _, hist = O.run_lasgd_pull(c["x0"], c["grads"], c["etas"], P, k, 1.0)
        ref = c["xs_hist"][-1]
        got = np.stack(hist[-1])
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_f32_restatement_close_to_f64_reference(golden_loops):
    for tag, c in loop_cases(golden_loops, "ab"):
        P, k = int(c["P"]), int(c["k"])
        _, _, _, hist = O.run_lasgd_delta(c["x0"].astype(np.float32), c["grads"].astype(np.float32), c["etas"], P, k)
        assert np.allclose(np.stack(hist[-1]), c["xs_hist"][-1], rtol=1e-5, atol=1e-5)


def test_momentum_step_matches_torch_sgd_to_tolerance():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    x = rng.standard_normal(10007).astype(np.float32)
    p = torch.nn.Parameter(torch.from_numpy(x.copy()))
    opt = torch.optim.SGD([p], lr=0.1, momentum=0.9, weight_decay=1e-4, nesterov=True, dampening=0.0)
    m = np.zeros_like(x)
    cfg = O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True)
    for t in range(5):
        g = rng.standard_normal(x.size).astype(np.float32)
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        x, m, _ = O.sgd_step_momentum(x, g, m, cfg, first_step=(t == 0))
    np.testing.assert_allclose(x, p.detach().numpy(), rtol=1e-5, atol=1e-6)


def test_config1_data_and_sampler_match_reference(golden_config1):
    g = golden_config1
    X, y = PO.make_synthetic(0, 4096, 784, 0.1, "regression")
    assert np.array_equal(np.array([X.sum(), y.sum(), X[17, 300], y[4095]]), g["a100_ds_checksum"])
    samplers = [PO.ShardSampler(4096, r, 4, 32, seed=0) for r in range(4)]
    for t in range(100):
        for r in range(4):
            assert np.array_equal(samplers[r].next_batch(), g["a100_batches"][t, r])
    x0 = np.random.default_rng(0).standard_normal(PO.mlp_dim([784, 128, 1])) * 0.05
    assert np.array_equal(x0[:64], g["a100_x0_head"])


def _config1_oracle(dtype, alpha, steps=100, P=4, k=4):
    X, y = PO.make_synthetic(0, 4096, 784, 0.1, "regression")
    dims = [784, 128, 1]
    n = PO.mlp_dim(dims)
    x0 = (np.random.default_rng(0).standard_normal(n) * 0.05).astype(dtype)
    Xd, yd = X.astype(dtype), y.astype(dtype)
    samplers = [PO.ShardSampler(4096, r, P, 32, seed=0) for r in range(P)]
    sch = O.LrSchedule(0.01, 1, 0)
    xs = [x0.copy() for _ in range(P)]
    snaps = [x0.copy() for _ in range(P)]
    deltas = [np.zeros_like(x0) for _ in range(P)]
    z = O.ring_mean(snaps)
    losses = np.zeros((steps, P))
    tau = 0
    for t in range(steps):
        eta = O.lr_at(sch, t)
        for r in range(P):
            b = samplers[r].next_batch()
            loss, g = PO.mlp_loss_and_grad(xs[r], dims, Xd[b], yd[b])
            losses[t, r] = loss
            if alpha == 1.0:
                xs[r], deltas[r] = O.sgd_step_delta(xs[r], deltas[r], g.astype(dtype), eta)
            else:
                xs[r] = O.sgd_step_plain(xs[r], g.astype(dtype), eta)
        tau += 1
        if tau == k:
            for r in range(P):
                if alpha == 1.0:
                    xs[r] = O.finalize_delta(z, deltas[r], xs[r], P)
                    deltas[r] = np.zeros_like(x0)
                else:
                    xs[r] = O.elastic_pull(xs[r], snaps[r], z, alpha)
                snaps[r] = xs[r].copy()
            z = O.ring_mean(snaps)
            tau = 0
    return losses, np.stack(xs)


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_config1_trajectory_f64_matches_reference(golden_config1, alpha):
    tag = f"a{int(alpha * 100)}_"
    losses, xs = _config1_oracle(np.float64, alpha)
    np.testing.assert_allclose(losses, golden_config1[tag + "losses"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(xs[:, golden_config1[tag + "final_sample_idx"]], golden_config1[tag + "final_sample"],
                               rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_config1_trajectory_f32_within_1e4(golden_config1, alpha):
    tag = f"a{int(alpha * 100)}_"
    losses, _ = _config1_oracle(np.float32, alpha)
    rel = np.abs(losses - golden_config1[tag + "losses"]) / np.abs(golden_config1[tag + "losses"])
    assert rel.max() < 1e-4, rel.max()


def test_easgd_templates_bit_exact_f64():
    """elastic_local_step / elastic_center_step / easgd_round_robin_exchange /
    mean_of_vectors restated in the oracle vs the reference (tests/golden/easgd.npz)."""
    import os

    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "easgd.npz")))
    x, z, gr, xs = g["x"], g["z"], g["g"], g["xs"]
    for i in range(4):
        eta, alpha = g[f"els_{i}_args"]
        assert np.array_equal(O.elastic_local_step(x, z, gr, float(eta), float(alpha)), g[f"els_{i}"]), i
    for i in range(4):
        beta, k = g[f"ecs_{i}_args"]
        assert np.array_equal(O.elastic_center_step(z, list(xs[: int(k)]), float(beta)), g[f"ecs_{i}"]), i
    for i in range(3):
        nx, nz = O.easgd_round_robin_exchange(x, z, float(g[f"rr_{i}_args"][0]))
        assert np.array_equal(nx, g[f"rr_{i}_x"]) and np.array_equal(nz, g[f"rr_{i}_z"]), i
    for k in (1, 2, 3, 5):
        assert np.array_equal(O.naive_mean(list(xs[:k])), g[f"mean_{k}"]), k

"""The reference's α≠1 templates on the device (optimizer.py:113-133, 245-259;
params.py:150-158), built from the K0 blend kernel: bit-exact against the reference
in f64 (tests/golden/easgd.npz) and against the oracle's fp32 restatement."""

import os

import numpy as np
import pytest
import torch

from oracle import lasgd_oracle as O

pytestmark = pytest.mark.gpu

G = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "easgd.npz")))


def _d(a, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


def test_f64_bit_exact_vs_reference():
    import paper_2203_13085_b200 as L

    x, z, g, xs = _d(G["x"]), _d(G["z"]), _d(G["g"]), [_d(v) for v in G["xs"]]
    for i in range(4):
        eta, alpha = (float(v) for v in G[f"els_{i}_args"])
        assert np.array_equal(L.elastic_local_step(x, z, g, eta, alpha).cpu().numpy(), G[f"els_{i}"]), i
    for i in range(4):
        beta, k = G[f"ecs_{i}_args"]
        got = L.elastic_center_step(z, xs[: int(k)], float(beta)).cpu().numpy()
        assert np.array_equal(got, G[f"ecs_{i}"]), i
    for i in range(3):
        nx, nz = L.easgd_round_robin_exchange(x, z, float(G[f"rr_{i}_args"][0]))
        assert np.array_equal(nx.cpu().numpy(), G[f"rr_{i}_x"]) and np.array_equal(nz.cpu().numpy(), G[f"rr_{i}_z"])
    for k in (1, 2, 3, 5):
        assert np.array_equal(L.mean_of_vectors(xs[:k]).cpu().numpy(), G[f"mean_{k}"]), k


def test_f32_bit_exact_vs_oracle_and_errors():
    import paper_2203_13085_b200 as L

    rng = np.random.default_rng(5)
    x, z, g = (rng.standard_normal(10_007).astype(np.float32) for _ in range(3))
    xs = [rng.standard_normal(10_007).astype(np.float32) for _ in range(7)]
    dx, dz, dg = _d(x, torch.float32), _d(z, torch.float32), _d(g, torch.float32)
    dxs = [_d(v, torch.float32) for v in xs]
    got = L.elastic_local_step(dx, dz, dg, 0.05, 0.3).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), O.elastic_local_step(x, z, g, 0.05, 0.3).view(np.uint32))
    got = L.elastic_center_step(dz, dxs, 0.4).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), O.elastic_center_step(z, xs, 0.4).view(np.uint32))
    nx, nz = L.easgd_round_robin_exchange(dx, dz, 0.35)
    ox, oz = O.easgd_round_robin_exchange(x, z, 0.35)
    assert np.array_equal(nx.cpu().numpy().view(np.uint32), ox.view(np.uint32))
    assert np.array_equal(nz.cpu().numpy().view(np.uint32), oz.view(np.uint32))
    for k in (3, 7):  # non-power-of-two counts: true division, not a reciprocal multiply
        got = L.mean_of_vectors(dxs[:k]).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), O.naive_mean(xs[:k]).view(np.uint32)), k
    with pytest.raises(L.HyperParamError):
        L.elastic_local_step(dx, dz, dg, 0.05, 1.5)
    with pytest.raises(L.HyperParamError):
        L.elastic_local_step(dx, dz, dg, 0.0, 0.5)
    with pytest.raises(L.HyperParamError):
        L.easgd_round_robin_exchange(dx, dz, 1.0)
    with pytest.raises(L.HyperParamError):
        L.elastic_center_step(dz, dxs, -0.1)
    with pytest.raises(ValueError):
        L.elastic_center_step(dz, [], 0.5)
    with pytest.raises(L.DimensionMismatchError):
        L.easgd_round_robin_exchange(dx, dz[:100], 0.5)


def test_execute_allreduce_matches_reference(golden_prims):
    """collective.py:154-203 on the device: per-rank means bit-exact (f64) against the
    reference's outputs, exact byte accounting, on_step abort, default plan only."""
    import paper_2203_13085_b200 as L

    for P in range(1, 9):
        for d in (1, 5, 7, 1000, 1001, 4099):
            vecs = list(golden_prims[f"mean_in_{P}_{d}"])
            out = L.execute_allreduce(vecs)
            ref = golden_prims[f"mean_out_{P}_{d}"]
            assert len(out.per_rank) == P
            for r in range(P):
                assert np.array_equal(out.per_rank[r].cpu().numpy(), ref if P > 1 else vecs[0]), (P, d, r)
            assert out.bytes_sent == ([O.bytes_per_node(d, P, 8, r) for r in range(P)] if P > 1 else [0])
            sizes = [e - s for s, e in O.partition_chunks(d, P)]
            assert out.peak_step_bytes == (8 * max(sizes) if P > 1 else 0)
    vecs = list(golden_prims["mean_in_4_1001"])
    seen = []

    def on_step(i, step_bytes):
        seen.append((i, list(step_bytes)))
        if i == 2:
            raise L.TransportFault("injected at step 2")

    with pytest.raises(L.TransportFault):
        L.execute_allreduce(vecs, on_step=on_step)
    assert [i for i, _ in seen] == [0, 1, 2] and all(len(b) == 4 for _, b in seen)
    custom = L.ChunkSpec(4, ((0, 500), (500, 600), (600, 700), (700, 1001)))
    with pytest.raises(NotImplementedError):
        L.execute_allreduce(vecs, chunks=custom)
    with pytest.raises(L.DimensionMismatchError):
        L.execute_allreduce([vecs[0], vecs[1][:10]])

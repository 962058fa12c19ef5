"""Mean all-reduce parity on one GPU (P virtual ranks, the GPU analogue of the
reference's LoopbackTransport): one-shot and two-shot kernels against the
reference's execute_allreduce outputs (f64, bit-exact) and the fp32 ring-order
oracle (bit-exact), plus the transport / handle contract."""

import numpy as np
import pytest
import torch

import paper_2203_13085_b200 as L
from oracle import lasgd_oracle as O
from paper_2203_13085_b200 import _native as N
from paper_2203_13085_b200 import kernels as K

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    iv = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return a.shape == b.shape and np.array_equal(a.view(iv), b.view(iv))


def gpu_mean(vecs, algo, nblocks=0, dtype=torch.float32):
    srcs = [dev(v) for v in vecs]
    P = len(vecs)
    outs = [torch.full_like(srcs[0], float("nan")) for _ in range(P if algo == N.ALGO_TWOSHOT else 1)]
    K.mean_virtual(outs, srcs, algo=algo, nblocks=nblocks)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("algo", [N.ALGO_ONESHOT, N.ALGO_TWOSHOT])
def test_mean_f64_bit_exact_vs_reference(golden_prims, algo):
    for P in range(1, 9):
        for d in (1, 5, 7, 1000, 1001, 4099):
            vecs = list(golden_prims[f"mean_in_{P}_{d}"])
            for out in gpu_mean(vecs, algo):
                assert same_bits(out, golden_prims[f"mean_out_{P}_{d}"]), (P, d, algo)


@pytest.mark.parametrize("algo", [N.ALGO_ONESHOT, N.ALGO_TWOSHOT])
@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("n", [1, 2, 9, 31, 4097, 65_539, 1_000_001])
def test_mean_f32_bit_exact_vs_oracle(algo, P, n):
    rng = np.random.default_rng(P * 1000 + n)
    vecs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    ref = O.ring_mean(vecs)
    outs = gpu_mean(vecs, algo)
    for out in outs:
        assert same_bits(out, ref), (algo, P, n)


@pytest.mark.parametrize("nblocks", [1, 3, 32, 128, 1000])
def test_twoshot_slicing_any_cta_count(nblocks):
    rng = np.random.default_rng(nblocks)
    for P, n in [(3, 10_007), (8, 123_457), (5, 3)]:
        vecs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
        ref = O.ring_mean(vecs)
        for out in gpu_mean(vecs, N.ALGO_TWOSHOT, nblocks=nblocks):
            assert same_bits(out, ref)
        for out in gpu_mean(vecs, N.ALGO_ONESHOT, nblocks=nblocks):
            assert same_bits(out, ref)


def test_mean_resnet50_size_p8():
    n, P = 25_557_032, 8
    rng = np.random.default_rng(5)
    vecs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    ref = O.ring_mean(vecs)
    for algo in (N.ALGO_ONESHOT, N.ALGO_TWOSHOT):
        outs = gpu_mean(vecs, algo, nblocks=32)
        assert all(same_bits(o, ref) for o in outs)


def test_mean_differs_from_naive_order_but_within_1e6():
    rng = np.random.default_rng(9)
    vecs = [rng.standard_normal(100_000).astype(np.float32) for _ in range(7)]
    out = gpu_mean(vecs, N.ALGO_ONESHOT)[0]
    naive = np.mean(np.stack(vecs).astype(np.float64), axis=0)
    np.testing.assert_allclose(out, naive, rtol=1e-6, atol=1e-6)


def test_allreduce_average_kat():
    h = L.all_reduce_average([np.array([1.0, 2, 3]), np.array([4.0, 5, 6]), np.array([7.0, 8, 9])])
    assert h.wait(10.0)
    assert L.poll(h) is L.Status.COMPLETE
    assert h.result.cpu().tolist() == [4.0, 5.0, 6.0]


def test_loopback_transport_contract(golden_meta):
    tr = L.CudaLoopbackTransport(3, dtype=torch.float64)
    v = [np.random.default_rng(i).standard_normal(1001) for i in range(3)]
    h = tr.submit(0, 0, v[0])
    assert L.poll(h) is L.Status.IN_FLIGHT
    with pytest.raises(RuntimeError):
        h.result  # collective.py:115-116
    with pytest.raises(RuntimeError):
        tr.submit(0, 0, v[0])  # double contribution, collective.py:255-256
    tr.submit(0, 1, v[1])
    h2 = tr.submit(0, 2, v[2])
    assert h2 is h
    assert h.wait(10.0) and h.status is L.Status.COMPLETE
    assert same_bits(h.result.cpu().numpy(), O.ring_mean(v))
    # byte accounting equals the reference's counters (collective.py:280-286)
    assert tr.bytes_sent == golden_meta["mean_bytes_3_1001"]
    assert h.bytes_sent_per_node == max(golden_meta["mean_bytes_3_1001"])
    with pytest.raises(KeyError):
        tr.submit(0, 0, v[0])  # late contribution to a completed round


def test_loopback_fault_injection_matches_reference(golden_meta):
    tr = L.CudaLoopbackTransport(3, fault_at=(0, 1))
    h = tr.all_reduce([np.ones(10), np.ones(10), np.ones(10)], round_id=0)
    assert h.status.value == golden_meta["fault_status"]
    assert h.diagnostic == golden_meta["fault_diag"]
    with pytest.raises(L.CollectiveFailure):
        h.result


def test_dimension_mismatch():
    tr = L.CudaLoopbackTransport(2)
    tr.submit(0, 0, np.ones(5))
    with pytest.raises(L.DimensionMismatchError):
        tr.submit(0, 1, np.ones(6))


def test_nonfinite_in_mean_counted():
    vecs = [np.ones(1000, np.float32), np.ones(1000, np.float32)]
    vecs[1][10] = np.inf
    srcs = [dev(v) for v in vecs]
    out = torch.empty_like(srcs[0])
    nf = torch.zeros(1, dtype=torch.int64, device="cuda")
    K.mean_virtual([out], srcs, nonfinite=nf)
    assert int(nf.item()) == 1

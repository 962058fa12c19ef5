"""CPU-only checks of the C-ABI library: it loads, exports every symbol the header
declares, and its host utilities agree with the reference's golden values."""

import ctypes
import os
import re

import pytest

import paper_2203_13085_b200 as L
from paper_2203_13085_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lasgd_sync.h")).read()
    return sorted(set(re.findall(r"\b(lasgd_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_all_exported():
    lib = ctypes.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_binding_covers_header():
    assert set(header_symbols()) == set(N.SIGNATURES)


def test_abi_version_and_errors():
    assert N.lib().lasgd_abi_version() == 1
    assert N.lib().lasgd_strerror(N.ERR_COLLECTIVE) == b"collective failed"
    with pytest.raises(L.CollectiveFailure):
        N.check(N.ERR_COLLECTIVE)
    with pytest.raises(L.DimensionMismatchError):
        N.check(N.ERR_DIMENSION)
    with pytest.raises(L.NonFiniteError):
        N.check(N.ERR_NONFINITE)
    with pytest.raises(ValueError):
        N.check(N.ERR_INVALID_ARGUMENT)


def test_partition_chunks_matches_reference(golden_meta):
    for key, bounds in golden_meta["partition"].items():
        d, P = map(int, key.split(","))
        assert [list(b) for b in L.partition_chunks(d, P).bounds] == bounds
    with pytest.raises(ValueError):
        L.partition_chunks(0, 3)
    with pytest.raises(ValueError):
        L.partition_chunks(3, 0)


def test_bytes_per_node_matches_reference(golden_meta):
    for key, vals in golden_meta["bytes_per_node"].items():
        d, P, b = map(int, key.split(","))
        assert L.bytes_per_node(d, P, b) == vals[0]
        for r in range(P):
            assert L.bytes_per_node(d, P, b, rank=r) == vals[1 + r]


def test_ring_schedule_matches_reference(golden_meta):
    for P, steps in golden_meta["ring_steps"].items():
        assert L.ring_schedule(int(P)).num_steps == steps
    got = [[[e.send_chunk, e.recv_chunk, e.send_to, e.recv_from, e.phase] for e in step]
           for step in L.ring_schedule(3).steps]
    assert got == golden_meta["ring_schedule_3"]


def test_lr_at_matches_reference(golden_meta):
    b, s, w, dec, f, spe = golden_meta["lr_sched"]
    sch = L.LrSchedule(b, s, w, tuple(dec), f, spe)
    for step, val in golden_meta["lr_vals"]:
        assert L.lr_at(sch, step) == val
    with pytest.raises(ValueError):
        L.lr_at(sch, -1)
    with pytest.raises(ValueError):
        L.LrSchedule(0.0, 1, 0)


def test_hyperparams_validation():
    sch = L.LrSchedule(0.01, 1, 0)
    L.HyperParams(sch, 4, 4).validate("lasgd")
    with pytest.raises(L.HyperParamError):
        L.HyperParams(sch, 4, 4, alpha=0.5).validate("lasgd")  # optimizer.py:71-72
    L.HyperParams(sch, 4, 4, alpha=0.5).validate("lasgd_pull")
    with pytest.raises(L.HyperParamError):
        L.HyperParams(sch, 0, 0).validate()
    with pytest.raises(L.HyperParamError):
        L.HyperParams(sch, 4, 1, alpha=0.5, rho=1.0).validate("lasgd_pull")


def test_sgd_config_validation():
    L.SgdConfig(0.9, 0.0, 1e-4, True).validate()
    with pytest.raises(L.HyperParamError):
        L.SgdConfig(0.0, 0.0, 0.0, True).validate()


def test_entry_points_reject_bad_arguments_without_gpu():
    # argument validation happens on the host before any CUDA call
    lib = N.lib()
    assert lib.lasgd_blend(None, 1.0, None, 1.0, None, 10, N.F32, None, None) == N.ERR_INVALID_ARGUMENT
    assert lib.lasgd_sgd_step(None, None, None, None, 0, N.F32, None, None, None) == N.ERR_INVALID_ARGUMENT
    assert lib.lasgd_elastic_pull(ctypes.c_void_p(16), None, ctypes.c_void_p(16), ctypes.c_void_p(16), 4, N.F32, 2.0,
                                  None, None) == N.ERR_INVALID_ARGUMENT
    assert lib.lasgd_mean_virtual(None, 1, None, 9, 10, N.F32, 1, 0, None, None) == N.ERR_UNSUPPORTED
    h = ctypes.c_void_p()
    assert lib.lasgd_comm_create(0, 9, 0, 10, N.F32, None, ctypes.byref(h)) == N.ERR_UNSUPPORTED
    assert lib.lasgd_comm_create(2, 2, 0, 10, N.F32, None, ctypes.byref(h)) == N.ERR_INVALID_ARGUMENT
    assert b"rank" in lib.lasgd_last_error()


def test_allreduce_auto_choices():
    """The standalone all-reduce's AUTO (lasgd_comm_allreduce without NVLS): one-shot at
    P=2; at the measured P = 3-4 the push mean where the two-shot would run (and at P=4
    from 4 MB), the copy-engine mean from 512 MB; P >= 5 keeps one-shot / two-shot."""
    from paper_2203_13085_b200 import _native as N

    MB = 1 << 20
    f = N.lib().lasgd_resolve_allreduce_algo_for
    one, two, push, ce = N.ALGO_ONESHOT, N.ALGO_TWOSHOT, N.ALGO_PUSH, N.ALGO_CE
    cases = [(2, 4 * MB, one), (2, 1024 * MB, one),
             (3, 4 * MB, one), (3, 16 * MB, push), (3, 102 * MB, push), (3, 1024 * MB, ce),
             (4, 1 * MB, one), (4, 4 * MB, push), (4, 102 * MB, push), (4, 256 * MB, push), (4, 512 * MB, ce),
             (8, 1 * MB, one), (8, 16 * MB, two), (8, 1024 * MB, two)]
    for world, nbytes, want in cases:
        assert f(world, nbytes) == want, (world, nbytes)

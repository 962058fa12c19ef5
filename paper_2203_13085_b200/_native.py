"""ctypes binding of the C-ABI CUDA library (include/lasgd_sync.h).

The library is built in-tree (``make -C paper_2203_13085_b200/csrc`` or
``__graft_entry__.build()``) to ``paper_2203_13085_b200/_lib/liblasgd_sync.so``.
There is no fallback: if the library is missing, importing the product path
raises ``ImportError``.  Error codes map to the reference's exception types
(params.py:15-20, collective.py:22-27, optimizer.py:24-25).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "liblasgd_sync.so")

OK = 0
ERR_INVALID_ARGUMENT = -1
ERR_DIMENSION = -2
ERR_NONFINITE = -3
ERR_CUDA = -4
ERR_COLLECTIVE = -5
ERR_TIMEOUT = -6
ERR_STATE = -7
ERR_UNSUPPORTED = -8

F32 = 0
F64 = 1
ALGO_AUTO = 0
ALGO_ONESHOT = 1
ALGO_TWOSHOT = 2
ALGO_PUSH = 3
ALGO_NVLS = 4
ALGO_CE = 5  # side-stream all-reduce with the NVLink traffic on the copy engines
MAX_RANKS = 8
MAX_BLOCKS = 512
IPC_HANDLE_BYTES = 64


class DimensionMismatchError(ValueError):
    """params.py:15-16."""


class NonFiniteError(FloatingPointError):
    """params.py:19-20."""


class TransportFault(RuntimeError):
    """collective.py:22-23."""


class CollectiveFailure(RuntimeError):
    """collective.py:26-27."""


class SgdParams(ctypes.Structure):
    _fields_ = [
        ("lr", ctypes.c_double),
        ("momentum", ctypes.c_double),
        ("dampening", ctypes.c_double),
        ("weight_decay", ctypes.c_double),
        ("nesterov", ctypes.c_int),
        ("first_step", ctypes.c_int),
        ("delta_reset", ctypes.c_int),
    ]


class CommConfig(ctypes.Structure):
    _fields_ = [
        ("nblocks", ctypes.c_int),
        ("threads", ctypes.c_int),
        ("timeout_s", ctypes.c_double),
        ("fault_seq", ctypes.c_longlong),
        ("fault_phase", ctypes.c_int),
    ]


TAU_HIST = 64
KERNEL_KINDS = ("sgd_step", "snapshot", "pull", "finalize", "allreduce", "fused_round", "sgd_pull")


class WorkerConfig(ctypes.Structure):
    _fields_ = [
        ("sync_period", ctypes.c_int),
        ("alpha", ctypes.c_double),
        ("mode", ctypes.c_int),
        ("pipeline", ctypes.c_int),
        ("algo", ctypes.c_int),
        ("fused_nblocks", ctypes.c_int),
        ("momentum", ctypes.c_double),
        ("dampening", ctypes.c_double),
        ("weight_decay", ctypes.c_double),
        ("nesterov", ctypes.c_int),
        ("sync", ctypes.c_int),
        ("adaptive", ctypes.c_int),
        ("tau_max", ctypes.c_int),
        ("max_host_lead", ctypes.c_int),
        ("max_host_wait_us", ctypes.c_int),
    ]


class WorkerState(ctypes.Structure):
    _fields_ = [
        ("tau_i", ctypes.c_int),
        ("snap_idx", ctypes.c_int),
        ("local_clock", ctypes.c_longlong),
        ("global_clock", ctypes.c_longlong),
        ("seq", ctypes.c_ulonglong),
        ("momentum_started", ctypes.c_int),
        ("delta_fresh", ctypes.c_int),
        ("launches", ctypes.c_longlong * len(KERNEL_KINDS)),
        ("tau_hist", ctypes.c_longlong * TAU_HIST),
    ]


_P = ctypes.c_void_p
_SZ = ctypes.c_size_t
_I = ctypes.c_int
_D = ctypes.c_double
_ULLP = ctypes.POINTER(ctypes.c_ulonglong)

# every symbol include/lasgd_sync.h declares: (name, restype, argtypes)
SIGNATURES = {
    "lasgd_abi_version": (_I, []),
    "lasgd_strerror": (ctypes.c_char_p, [_I]),
    "lasgd_last_error": (ctypes.c_char_p, []),
    "lasgd_set_stream_ctas_per_sm": (_I, [_I]),
    "lasgd_blend": (_I, [_P, _D, _P, _D, _P, _SZ, _I, _P, _P]),
    "lasgd_snapshot": (_I, [_P, _P, _SZ, _I, _P]),
    "lasgd_sgd_step": (_I, [_P, _P, _P, _P, _SZ, _I, ctypes.POINTER(SgdParams), _P, _P]),
    "lasgd_elastic_pull": (_I, [_P, _P, _P, _P, _SZ, _I, _D, _P, _P]),
    "lasgd_finalize": (_I, [_P, _P, _P, _P, _SZ, _I, _P, _P]),
    "lasgd_sgd_pull": (_I, [_P, _P, _P, _P, _P, _P, _P, _SZ, _I, ctypes.POINTER(SgdParams), _D, _I, _P, _P]),
    "lasgd_mean_virtual": (_I, [_P, _I, _P, _I, _SZ, _I, _I, _I, _P, _P]),
    "lasgd_comm_create": (_I, [_I, _I, _I, _SZ, _I, ctypes.POINTER(CommConfig), ctypes.POINTER(_P)]),
    "lasgd_comm_ipc_handle": (_I, [_P, _P]),
    "lasgd_comm_open": (_I, [_P, _P]),
    "lasgd_comm_buffer": (_I, [_P, _I, ctypes.POINTER(_P)]),
    "lasgd_comm_allreduce": (_I, [_P, _I, _I, _P, _ULLP]),
    "lasgd_comm_fused_round": (_I, [_P, _I, _I, _P, _P, _P, _P, ctypes.POINTER(SgdParams), _D, _I, _I, _P, _P,
                                    _ULLP]),
    "lasgd_fused_round_virtual": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _SZ, _I, ctypes.POINTER(SgdParams), _D,
                                       _I, _I, _P, _P]),
    "lasgd_comm_sgd_ar_range": (_I, [_P, _I, _SZ, _SZ, _I, _P, _P, ctypes.POINTER(SgdParams), _I, _P, _P, _ULLP]),
    "lasgd_comm_query": (_I, [_P, ctypes.c_ulonglong]),
    "lasgd_comm_stream_wait": (_I, [_P, ctypes.c_ulonglong, _P]),
    "lasgd_comm_wait": (_I, [_P, ctypes.c_ulonglong, _D]),
    "lasgd_comm_diagnostic": (_I, [_P, ctypes.c_char_p, _SZ]),
    "lasgd_comm_bytes_per_node": (ctypes.c_ulonglong, [_P, _I]),
    "lasgd_comm_resolve_algo": (_I, [_P, _I]),
    "lasgd_comm_resolve_fused_algo": (_I, [_P, _I]),
    "lasgd_resolve_fused_algo_for": (_I, [_I, _SZ]),
    "lasgd_resolve_allreduce_algo_for": (_I, [_I, _SZ]),
    "lasgd_comm_peers_ahead": (_I, [_P, ctypes.c_ulonglong]),
    "lasgd_comm_set_gate": (_I, [_P, _I]),
    "lasgd_comm_barrier": (_I, [_P, _P]),
    "lasgd_comm_set_nblocks": (_I, [_P, _I]),
    "lasgd_comm_set_trace": (_I, [_P, _I]),
    "lasgd_comm_read_trace": (_I, [_P, _P, _I]),
    "lasgd_comm_destroy": (_I, [_P]),
    "lasgd_comm_info": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_P)]),
    "lasgd_comm_shape": (_I, [_P, ctypes.POINTER(_SZ), ctypes.POINTER(_I)]),
    "lasgd_comm_nvls_supported": (_I, [_P]),
    "lasgd_comm_nvls_create": (_I, [_P, ctypes.POINTER(_I)]),
    "lasgd_comm_nvls_import": (_I, [_P, _I]),
    "lasgd_comm_nvls_add_device": (_I, [_P]),
    "lasgd_comm_nvls_bind": (_I, [_P]),
    "lasgd_comm_peer_max_seq": (_I, [_P, _ULLP]),
    "lasgd_comm_launches": (_I, [_P, _ULLP]),
    "lasgd_comm_invalidate_staging": (_I, [_P]),
    "lasgd_fused_push_virtual": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _SZ, _I, ctypes.POINTER(SgdParams),
                                      _D, _I, _I, _P, _P]),
    "lasgd_push_stage_elems": (_SZ, [_SZ, _I, _I]),
    "lasgd_worker_create": (_I, [_P, _P, _P, _P, _P, _P, _SZ, _I, ctypes.POINTER(WorkerConfig), _P, _P, _P,
                                 ctypes.POINTER(_P)]),
    "lasgd_worker_step": (_I, [_P, _P, _D]),
    "lasgd_worker_drain": (_I, [_P]),
    "lasgd_worker_get_state": (_I, [_P, ctypes.POINTER(WorkerState)]),
    "lasgd_worker_set_timing": (_I, [_P, _I]),
    "lasgd_worker_timings": (_I, [_P, _I, ctypes.POINTER(ctypes.c_float), _I]),
    "lasgd_worker_reset_stats": (_I, [_P]),
    "lasgd_worker_destroy": (_I, [_P]),
    "lasgd_worker_set_lr_table": (_I, [_P, ctypes.POINTER(ctypes.c_double), _SZ]),
    "lasgd_worker_graph_capture": (_I, [_P, _I, _P, ctypes.POINTER(_P)]),
    "lasgd_worker_capture_begin": (_I, [_P, ctypes.POINTER(_P)]),
    "lasgd_worker_capture_end": (_I, [_P]),
    "lasgd_graph_launch": (_I, [_P]),
    "lasgd_graph_destroy": (_I, [_P]),
    "lasgd_stamp": (_I, [_P, _P]),
    "lasgd_hold_create": (_I, [ctypes.POINTER(_P)]),
    "lasgd_hold_enqueue": (_I, [_P, _P, _D]),
    "lasgd_hold_release": (_I, [_P]),
    "lasgd_hold_destroy": (_I, [_P]),
    "lasgd_partition_chunks": (_I, [_SZ, _I, ctypes.POINTER(_SZ)]),
    "lasgd_bytes_per_node": (ctypes.c_ulonglong, [_SZ, _I, _I, _I]),
}

_lib = None


def lib():
    """Load the library (once).  Raises ImportError when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"LASGD CUDA library not built: {LIB_PATH} is missing "
                "(run `make -C paper_2203_13085_b200/csrc` or __graft_entry__.build()); "
                "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.lasgd_abi_version() != 1:
            raise ImportError("liblasgd_sync ABI version mismatch; rebuild the library")
        _lib = L
    return _lib


def last_error() -> str:
    return lib().lasgd_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> int:
    """Map a negative C-ABI return code to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc in (ERR_INVALID_ARGUMENT, ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == ERR_DIMENSION:
        raise DimensionMismatchError(msg)
    if rc == ERR_NONFINITE:
        raise NonFiniteError(msg)
    if rc == ERR_COLLECTIVE:
        raise CollectiveFailure(msg)
    if rc == ERR_TIMEOUT:
        raise TimeoutError(msg)
    raise RuntimeError(msg)

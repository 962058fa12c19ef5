"""Tensor-level wrappers of the C-ABI kernels (one launch each, on the current
CUDA stream unless ``stream`` is given).  Inputs must be contiguous CUDA
tensors of one element type (float32 = product path, float64 = reference
precision); nothing here ever falls back to a CPU or torch implementation.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import _native as N

_DTYPES = {torch.float32: N.F32, torch.float64: N.F64}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported element type {t.dtype}; use float32 or float64") from None


def _check(*ts: Optional[torch.Tensor]) -> tuple[int, int]:
    ref = next(t for t in ts if t is not None)
    code = dtype_code(ref)
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("LASGD kernels need CUDA tensors (there is no CPU path)")
        if not t.is_contiguous():
            raise ValueError("LASGD kernels need contiguous (flat) tensors")
        if t.dtype != ref.dtype:
            raise TypeError(f"mixed element types {t.dtype} vs {ref.dtype}")
        if t.numel() != ref.numel():
            raise N.DimensionMismatchError(f"dimension mismatch: {t.numel()} vs {ref.numel()}")
        if t.device != ref.device:
            raise ValueError("tensors on different devices")
    return code, ref.numel()


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def blend(out, a: float, u, b: float, v, nonfinite=None, stream=None) -> torch.Tensor:
    """K0: ``out = a*u + b*v`` (params.py:80-89)."""
    code, n = _check(out, u, v)
    N.check(N.lib().lasgd_blend(_ptr(out), float(a), _ptr(u), float(b), _ptr(v), n, code, _ptr(nonfinite),
                                _stream(stream)), "blend")
    return out


def snapshot(snap, x, stream=None) -> torch.Tensor:
    """K1: ``snap = x``."""
    code, n = _check(snap, x)
    N.check(N.lib().lasgd_snapshot(_ptr(snap), _ptr(x), n, code, _stream(stream)), "snapshot")
    return snap


def sgd_step(x, g, lr: float, *, m=None, delta=None, momentum=0.0, dampening=0.0, weight_decay=0.0,
             nesterov=False, first_step=False, delta_reset=False, nonfinite=None, stream=None) -> torch.Tensor:
    """K5: fused local step (see include/lasgd_sync.h).  At momentum = wd = 0 this is
    optimizer.py:145-146 exactly (x and, if given, the delta accumulator)."""
    code, n = _check(x, g, m, delta)
    p = N.SgdParams(float(lr), float(momentum), float(dampening), float(weight_decay), int(bool(nesterov)),
                    int(bool(first_step)), int(bool(delta_reset)))
    N.check(N.lib().lasgd_sgd_step(_ptr(x), _ptr(g), _ptr(m), _ptr(delta), n, code, ctypes.byref(p),
                                   _ptr(nonfinite), _stream(stream)), "sgd_step")
    return x


def elastic_pull(x, snap, xbar, alpha: float, snap_next=None, nonfinite=None, stream=None) -> torch.Tensor:
    """K4a: ``x -= alpha*(snap - xbar)`` in blend order, optional fused ``snap_next = x``."""
    code, n = _check(x, snap, xbar, snap_next)
    N.check(N.lib().lasgd_elastic_pull(_ptr(x), _ptr(snap_next), _ptr(snap), _ptr(xbar), n, code, float(alpha),
                                       _ptr(nonfinite), _stream(stream)), "elastic_pull")
    return x


def finalize(x, z, delta, snap_next=None, nonfinite=None, stream=None) -> torch.Tensor:
    """K4b: ``x = z + delta`` (optimizer.py:171), optional fused ``snap_next = x``;
    ``delta=None`` is a zero accumulator (x = z + 0)."""
    code, n = _check(x, z, delta, snap_next)
    N.check(N.lib().lasgd_finalize(_ptr(x), _ptr(snap_next), _ptr(z), _ptr(delta), n, code, _ptr(nonfinite),
                                   _stream(stream)), "finalize")
    return x


def sgd_pull(x, g, snap_next, snap, xbar, lr: float, *, m=None, delta=None, momentum=0.0, dampening=0.0,
             weight_decay=0.0, nesterov=False, first_step=False, delta_reset=False, alpha: float = 1.0, mode: int = 0,
             nonfinite=None, stream=None) -> torch.Tensor:
    """K5 + K4 in one pass: the local step, then the pull towards ``xbar`` (mode 0) or the
    reference finalize ``x = xbar + delta'`` (mode 1); ``snap_next = x``."""
    code, n = _check(x, g, snap_next, xbar, snap, m, delta)
    p = sgd_params(lr, momentum, dampening, weight_decay, nesterov, first_step, delta_reset)
    N.check(N.lib().lasgd_sgd_pull(_ptr(x), _ptr(g), _ptr(m), _ptr(delta), _ptr(snap_next), _ptr(snap), _ptr(xbar), n,
                                   code, ctypes.byref(p), float(alpha), int(mode), _ptr(nonfinite), _stream(stream)),
            "sgd_pull")
    return x


def sgd_params(lr: float, momentum=0.0, dampening=0.0, weight_decay=0.0, nesterov=False, first_step=False,
               delta_reset=False) -> N.SgdParams:
    return N.SgdParams(float(lr), float(momentum), float(dampening), float(weight_decay), int(bool(nesterov)),
                       int(bool(first_step)), int(bool(delta_reset)))


def fused_round_virtual(xs, gs, snaps, snap_nexts, lr: float, *, ms=None, deltas=None, momentum=0.0,
                        dampening=0.0, weight_decay=0.0, nesterov=False, first_step=False, delta_reset=False,
                        alpha: float = 1.0, mode: int = 0, algo: int = N.ALGO_ONESHOT, xbars=None, nblocks: int = 0,
                        nonfinite=None, stream=None) -> None:
    """K7 for P ranks on one device: local step + ring-order mean of ``snaps`` + pull
    (mode 0) or finalize (mode 1) + next snapshot, one pass (two launches for the
    two-shot form, which needs per-rank ``xbars`` scratch).  Mode 2 (SGD-AR): ``snaps``
    hold the gradients, x = local step with their mean; ``gs`` unused, nothing else
    written."""
    P = len(xs)
    flat = list(xs) + list(gs) + list(snaps) + list(snap_nexts) + list(ms or []) + list(deltas or []) + list(xbars or [])
    code, n = _check(*flat)

    def arr(ts):
        return None if ts is None else (ctypes.c_void_p * P)(*[t.data_ptr() for t in ts])

    p = sgd_params(lr, momentum, dampening, weight_decay, nesterov, first_step, delta_reset)
    N.check(N.lib().lasgd_fused_round_virtual(P, int(algo), arr(xs), arr(gs), arr(ms), arr(deltas), arr(snaps),
                                              arr(xbars), arr(snap_nexts), n, code, ctypes.byref(p), float(alpha),
                                              int(mode), int(nblocks), _ptr(nonfinite), _stream(stream)),
            "fused_round_virtual")


def push_stage_elems(n: int, P: int, dtype: torch.dtype = torch.float32) -> int:
    return int(N.lib().lasgd_push_stage_elems(n, P, _DTYPES[dtype]))


def fused_push_virtual(xs, gs, snaps, snap_nexts, xbars, stages, cur: int, init: bool, lr: float, *, ms=None,
                       deltas=None, momentum=0.0, dampening=0.0, weight_decay=0.0, nesterov=False, first_step=False,
                       delta_reset=False, alpha: float = 1.0, mode: int = 0, nblocks: int = 0, nonfinite=None,
                       stream=None) -> None:
    """K8 (push round) for P ranks on one device; ``stages[r]`` holds
    2 * P * push_stage_elems(n, P) elements."""
    P = len(xs)
    code, n = _check(*(list(xs) + list(gs) + list(snaps) + list(snap_nexts) + list(xbars) + list(ms or []) +
                       list(deltas or [])))

    def arr(ts):
        return None if ts is None else (ctypes.c_void_p * P)(*[t.data_ptr() for t in ts])

    p = sgd_params(lr, momentum, dampening, weight_decay, nesterov, first_step, delta_reset)
    N.check(N.lib().lasgd_fused_push_virtual(P, arr(xs), arr(gs), arr(ms), arr(deltas), arr(snaps), arr(snap_nexts),
                                             arr(xbars), arr(stages), int(cur), int(bool(init)), n, code,
                                             ctypes.byref(p), float(alpha), int(mode), int(nblocks), _ptr(nonfinite),
                                             _stream(stream)), "fused_push_virtual")


def mean_virtual(outs: Sequence[torch.Tensor], srcs: Sequence[torch.Tensor], algo: int = N.ALGO_ONESHOT,
                 nblocks: int = 0, nonfinite=None, stream=None) -> None:
    """Ring-order mean of P same-device contributions (collective.py:154-203)."""
    code, n = _check(*srcs, *outs)
    src_arr = (ctypes.c_void_p * len(srcs))(*[s.data_ptr() for s in srcs])
    out_arr = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    N.check(N.lib().lasgd_mean_virtual(out_arr, len(outs), src_arr, len(srcs), n, code, int(algo), int(nblocks),
                                       _ptr(nonfinite), _stream(stream)), "mean_virtual")

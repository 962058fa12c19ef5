"""ctypes wrapper for oracle/build/liblasgd_oracle.so — TEST INFRASTRUCTURE / CPU BASELINE ONLY.

Build with ``make -C oracle`` (``__graft_entry__.build()`` does this).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "build", "liblasgd_oracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"C oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = ctypes.CDLL(LIB_PATH)
        for sfx in ("f32", "f64"):
            getattr(L, f"oracle_blend_{sfx}").argtypes = [_P, _D, _P, _D, _P, _I64]
            getattr(L, f"oracle_sgd_delta_{sfx}").argtypes = [_P, _P, _P, _P, _P, _I64, _D, _INT]
            getattr(L, f"oracle_sgd_momentum_{sfx}").argtypes = [_P, _P, _P, _I64, _D, _D, _D, _D, _INT, _INT]
            getattr(L, f"oracle_finalize_{sfx}").argtypes = [_P, _P, _P, _I64]
            getattr(L, f"oracle_pull_{sfx}").argtypes = [_P, _P, _P, _P, _I64, _D]
            getattr(L, f"oracle_ring_mean_{sfx}").argtypes = [_P, _INT, _P, _INT, _I64]
            getattr(L, f"oracle_copy_{sfx}").argtypes = [_P, _P, _I64]
            for name in ("blend", "sgd_delta", "sgd_momentum", "finalize", "pull", "ring_mean"):
                getattr(L, f"oracle_{name}_{sfx}").restype = _I64
        L.oracle_get_threads.restype = _INT
        _lib = L
    return _lib


def _sfx(a: np.ndarray) -> str:
    return {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}[a.dtype]


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return lib().oracle_get_threads()


def blend(out, a, u, b, v):
    return getattr(lib(), f"oracle_blend_{_sfx(u)}")(_p(out), a, _p(u), b, _p(v), u.size)


def sgd_delta(x_out, d_out, x, d, g, eta, delta_reset=False):
    return getattr(lib(), f"oracle_sgd_delta_{_sfx(x)}")(_p(x_out), _p(d_out), _p(x), _p(d), _p(g), x.size, eta,
                                                         int(delta_reset))


def sgd_momentum(x, g, m, lr, mu, damp, wd, nesterov, first):
    return getattr(lib(), f"oracle_sgd_momentum_{_sfx(x)}")(_p(x), _p(g), _p(m), x.size, lr, mu, damp, wd,
                                                            int(nesterov), int(first))


def finalize(out, z, d):
    return getattr(lib(), f"oracle_finalize_{_sfx(z)}")(_p(out), _p(z), _p(d), z.size)


def pull(x, snap_next, snap, xbar, alpha):
    return getattr(lib(), f"oracle_pull_{_sfx(x)}")(_p(x), _p(snap_next), _p(snap), _p(xbar), x.size, alpha)


def ring_mean(outs, srcs):
    P = len(srcs)
    src_arr = (ctypes.c_void_p * P)(*[s.ctypes.data for s in srcs])
    out_arr = (ctypes.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
    return getattr(lib(), f"oracle_ring_mean_{_sfx(srcs[0])}")(out_arr, len(outs), src_arr, P, srcs[0].size)


def copy(dst, src):
    getattr(lib(), f"oracle_copy_{_sfx(src)}")(_p(dst), _p(src), src.size)

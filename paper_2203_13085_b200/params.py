"""Flat parameter vectors on the device (mirror of /root/reference/pkg/src/lasgd/params.py).

The reference keeps immutable f64 host vectors (``ParamVector``, params.py:29-72)
and allocates on every operation.  Here a rank's parameters live in ONE
contiguous fp32 (or f64) CUDA buffer that the kernels update in place; the
functions below keep the reference's names, argument order and exceptions.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from ._native import DimensionMismatchError, NonFiniteError  # noqa: F401  (re-exported, params.py:15-20)


def as_device_vector(v, dtype: torch.dtype = torch.float32, device=None) -> torch.Tensor:
    """Accept a torch tensor, a numpy array or a reference-style ``ParamVector``
    (anything with a ``.data`` ndarray) and return a contiguous 1-D CUDA tensor.
    Host inputs are copied (one H2D transfer); CUDA inputs of the right type are
    returned as-is (flattened view)."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    if isinstance(v, torch.Tensor):
        t = v
    else:
        arr = getattr(v, "data", v)
        if isinstance(arr, memoryview):
            arr = np.asarray(v)
        arr = np.asarray(arr)
        if arr.ndim == 0:  # np.ascontiguousarray would promote a scalar to shape (1,)
            raise ValueError(f"parameter vector must be 1-D, got shape {arr.shape}")
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dim() != 1:
        if t.dim() == 0:
            raise ValueError(f"parameter vector must be 1-D, got shape {tuple(t.shape)}")
        t = t.reshape(-1)
    if t.numel() == 0:
        raise ValueError("parameter vector must have positive dimension")
    if t.dtype != dtype or t.device != torch.device(device) or not t.is_contiguous():
        t = t.to(device=device, dtype=dtype, non_blocking=False).contiguous()
    return t


def vector_dtype(v) -> torch.dtype:
    """The element type a vector argument computes in: f64 for f64 inputs (e.g. the
    reference's ParamVector, bit-exact with it), f32 otherwise."""
    if isinstance(v, torch.Tensor):
        return torch.float64 if v.dtype == torch.float64 else torch.float32
    return torch.float64 if np.asarray(getattr(v, "data", v)).dtype == np.float64 else torch.float32


def require_same_dim(u: torch.Tensor, v: torch.Tensor) -> None:
    """params.py:75-77."""
    if u.numel() != v.numel():
        raise DimensionMismatchError(f"dimension mismatch: {u.numel()} vs {v.numel()}")


def blend(a: float, u: torch.Tensor, b: float, v: torch.Tensor, *, out: Optional[torch.Tensor] = None,
          check_finite: bool = True) -> torch.Tensor:
    """params.py:80-89: ``a*u + b*v`` as a new (or the given) device vector.

    ``check_finite`` reproduces the reference's eager NonFiniteError (it costs one
    device sync); the fused counter itself is free."""
    require_same_dim(u, v)
    if out is None:
        out = torch.empty_like(u)
    nf = torch.zeros(1, dtype=torch.int64, device=u.device) if check_finite else None
    K.blend(out, a, u, b, v, nonfinite=nf)
    if check_finite:
        bad = int(nf.item())
        if bad:
            raise NonFiniteError(f"blend: {bad} non-finite entries out of {u.numel()}")
    return out


@dataclass(frozen=True)
class ChunkSpec:
    """params.py:92-127: balanced partition of [0, d) into contiguous ranges."""

    num_chunks: int
    bounds: tuple

    def __post_init__(self) -> None:
        if self.num_chunks != len(self.bounds):
            raise ValueError("bounds must have one range per chunk")
        cursor = 0
        for start, end in self.bounds:
            if start != cursor or end < start:
                raise ValueError(f"chunk ranges must be contiguous and ordered, got {self.bounds}")
            cursor = end

    @property
    def dim(self) -> int:
        return self.bounds[-1][1] if self.bounds else 0

    def size(self, index: int) -> int:
        s, e = self.bounds[index]
        return e - s

    def slice(self, index: int) -> slice:
        s, e = self.bounds[index]
        return slice(s, e)

    @property
    def max_size(self) -> int:
        return max(e - s for s, e in self.bounds)


def partition_chunks(d: int, num_chunks: int) -> ChunkSpec:
    """params.py:130-147 via the C ABI (the same closed form the kernels use)."""
    import ctypes

    if d < 1:
        raise ValueError("d must be positive")
    if num_chunks < 1:
        raise ValueError("num_chunks must be positive")
    arr = (ctypes.c_size_t * (num_chunks + 1))()
    N.check(N.lib().lasgd_partition_chunks(d, num_chunks, arr), "partition_chunks")
    return ChunkSpec(num_chunks=num_chunks, bounds=tuple((int(arr[i]), int(arr[i + 1])) for i in range(num_chunks)))


def mean_of_vectors(vectors) -> torch.Tensor:
    """params.py:150-158: the mean in fixed ascending-index order (``acc += v`` then
    ``acc / len``) — NOT the ring order of the all-reduce.  Sums with the K0 blend
    (``1*acc + 1*v`` is exact in the rounding contract); the division is a true
    division by a device scalar tensor (a Python-scalar divisor would be turned into a
    reciprocal multiply)."""
    vectors = list(vectors)
    if not vectors:
        raise ValueError("need at least one vector")
    dt = vector_dtype(vectors[0])
    vs = [as_device_vector(v, dtype=dt) for v in vectors]
    acc = vs[0].clone()
    for v in vs[1:]:
        require_same_dim(vs[0], v)
        blend(1.0, acc, 1.0, v, out=acc)
    return acc / torch.tensor(float(len(vs)), dtype=acc.dtype, device=acc.device)


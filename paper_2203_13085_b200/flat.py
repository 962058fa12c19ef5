"""Flat parameter / gradient buffers behind a torch module.

Every trainable parameter becomes a view into ONE contiguous fp32 buffer ``x``
and its ``.grad`` a view into ONE contiguous buffer ``g``, so cuDNN's backward
accumulates gradients straight into the buffer the sync kernels stream over.
The layout is the module's parameter order, each tensor row-major — for an MLP
this is exactly the reference MlpOracle's flat vector (problems.py:202-205:
W_l row-major then b_l).  4-D weights can be exposed as channels_last-strided
views over the same contiguous storage.  BatchNorm running statistics are
buffers, not parameters: they stay rank-local (not averaged).

``align_bytes`` (e.g. 256) starts every tensor at an aligned offset so cuDNN sees
aligned weights and gradients; the gaps are zero in ``x`` and ``g`` and stay zero
under every sync kernel (zero gradient, zero weight decay term, zero mean).  The
default 0 packs the tensors back to back (the reference's flat layout).
"""

from __future__ import annotations

import torch


class FlatParams:
    def __init__(self, module: torch.nn.Module, dtype: torch.dtype = torch.float32, device=None,
                 channels_last: bool = False, align_bytes: int = 0):
        params = [p for p in module.parameters() if p.requires_grad]
        if not params:
            raise ValueError("module has no trainable parameters")
        device = device or params[0].device
        esize = torch.empty(0, dtype=dtype).element_size()
        if align_bytes < 0 or (align_bytes and align_bytes % esize):
            raise ValueError(f"align_bytes must be a non-negative multiple of {esize}")
        step = max(1, align_bytes // esize)
        self.offsets = []
        off = 0
        for p in params:
            off = (off + step - 1) // step * step
            self.offsets.append(off)
            off += p.numel()
        self.n_params = sum(p.numel() for p in params)
        self.numel = off
        self.x = torch.zeros(self.numel, dtype=dtype, device=device)
        self.g = torch.zeros(self.numel, dtype=dtype, device=device)
        self.params = params
        self.channels_last = channels_last
        self._grad_views = {}
        with torch.no_grad():
            for p, o in zip(params, self.offsets):
                v = self._view(self.x, o, p.shape, channels_last)
                v.copy_(p.detach())
                p.data = v
                p.grad = self._view(self.g, o, p.shape, channels_last)

    @staticmethod
    def _view(buf: torch.Tensor, off: int, shape, channels_last: bool) -> torch.Tensor:
        n = 1
        for s in shape:
            n *= s
        flat = buf[off:off + n]
        if channels_last and len(shape) == 4:
            o, i, h, w = shape
            return flat.view(o, h, w, i).permute(0, 3, 1, 2)  # NHWC storage, NCHW shape
        return flat.view(shape)

    def bind_grads(self, buf: torch.Tensor) -> None:
        """Point every ``.grad`` into ``buf`` (e.g. a communicator's registered slot, so
        backward writes the all-reduce input in place)."""
        if buf.dtype != self.x.dtype or buf.numel() != self.numel or not buf.is_contiguous():
            raise ValueError("gradient buffer must be a contiguous vector like x")
        key = (buf.data_ptr(), buf.device)
        views = self._grad_views.get(key)
        if views is None:  # views are built once per buffer: rebinding every step stays cheap
            views = [self._view(buf, off, p.shape, self.channels_last) for p, off in zip(self.params, self.offsets)]
            self._grad_views[key] = views
        for p, v in zip(self.params, views):
            p.grad = v
        self.g = buf

    def zero_grad(self) -> None:
        """One memset over the flat gradient buffer (grads stay attached as views)."""
        self.g.zero_()

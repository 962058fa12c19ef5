"""CUDA-graph capture of the step on the compute side of the sync path.

A minibatch step of fixed shape (zero the flat gradient, forward, backward) is
captured once into a CUDA graph and replayed every step, so a launch-bound model
(ResNet-18 on 32x32 inputs issues ~500 kernels per step) costs one graph launch of
host time instead of ~4 ms of PyTorch dispatch.  The sync path stays outside the
graph: its launches carry per-round arguments (sequence number, snapshot slot, rate)
and are issued natively by the worker right after the replay on the same stream.

Gradients land in whatever buffer ``FlatParams`` has bound at capture time; callers
that alternate gradient buffers (``SGDARWorker``) get one graph per buffer.
"""

from __future__ import annotations

from typing import Callable, Optional

import torch


class GraphedStep:
    def __init__(self, flat, fn: Callable[[], object], warmup: int = 3, pool=None):
        """``fn()`` runs forward + backward on static input tensors (it is traced once
        per gradient buffer and must not synchronise with the host)."""
        self.flat = flat
        self.fn = fn
        self.warmup = warmup
        self.pool = pool if pool is not None else torch.cuda.graph_pool_handle()
        self.graphs: dict = {}

    def _capture(self) -> torch.cuda.CUDAGraph:
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream(device=cur.device)
        side.wait_stream(cur)
        with torch.cuda.stream(side):  # warm-up off the capture stream (cuDNN autotuning, allocator)
            for _ in range(self.warmup):
                self.flat.zero_grad()
                self.fn()
        cur.wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, pool=self.pool):
            self.flat.zero_grad()
            self.fn()
        return g

    def __call__(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Replay on ``stream`` (default: the current stream)."""
        key = self.flat.g.data_ptr()
        g = self.graphs.get(key)
        if g is None:
            g = self.graphs[key] = self._capture()
        if stream is None:
            g.replay()
        else:
            with torch.cuda.stream(stream):
                g.replay()

"""``torch.optim``-style front end of the LASGD worker, for training scripts written
against PyTorch optimizers: ``opt = LASGD(model, lr=0.1, momentum=0.9, ...)``, then the
usual ``opt.zero_grad(); loss.backward(); opt.step()``.

The module's parameters become views of one flat fp32 buffer (``FlatParams``) and their
gradients views of another, so ``step()`` is the native worker's step
(``LASGDWorker.step``): the fused local step every minibatch and, every
``sync_period`` minibatches, the round boundary of Algorithm 1 (PAPER.md:158-193,
optimizer.py:181-207) — the ring-order mean of every rank's snapshot over NVLink, the
elastic pull and the next snapshot.  With ``comm=None`` and more than one process under
``torch.distributed``, a ``P2PCommunicator`` is created (collective: every rank must
construct the optimizer).  The local step is ``torch.optim.SGD``'s update (momentum,
dampening, weight decay, Nesterov) with every operation rounded separately.
"""

from __future__ import annotations

from typing import Optional

import torch

from . import _native as N
from .collective import P2PCommunicator
from .engine import LASGDWorker
from .flat import FlatParams
from .optimizer import SgdConfig
from .problems import LrSchedule


class LASGD(torch.optim.Optimizer):
    def __init__(self, module: torch.nn.Module, lr: Optional[float] = None, *, momentum: float = 0.0,
                 dampening: float = 0.0, weight_decay: float = 0.0, nesterov: bool = False,
                 schedule: Optional[LrSchedule] = None, sync_period: int = 1, alpha: float = 1.0,
                 pipeline: str = "fused", adaptive: bool = False, tau_max: Optional[int] = None, comm="auto",
                 algo: int = N.ALGO_AUTO, nvls: bool = False, channels_last: bool = False, align_bytes: int = 256,
                 compute_stream: Optional[torch.cuda.Stream] = None):
        if (lr is None) == (schedule is None):
            raise ValueError("give exactly one of lr / schedule")
        self.flat = FlatParams(module, channels_last=channels_last, align_bytes=align_bytes)
        defaults = dict(lr=lr, momentum=momentum, dampening=dampening, weight_decay=weight_decay, nesterov=nesterov)
        super().__init__(self.flat.params, defaults)
        self._own_comm = False
        if comm == "auto":
            import torch.distributed as dist

            world = dist.get_world_size() if dist.is_initialized() else 1
            comm = None
            if world > 1:
                dist.broadcast(self.flat.x, 0)  # identical x0 on every rank (Algorithm 1 line 1)
                comm = P2PCommunicator(self.flat.numel, nvls=nvls)
                self._own_comm = True
        self.comm = comm
        self.worker = LASGDWorker(self.flat.x, self.flat.g, comm=comm, sync_period=sync_period, alpha=alpha,
                                  mode="pull", sgd=SgdConfig(momentum, dampening, weight_decay, nesterov),
                                  schedule=schedule, lr=lr, adaptive=adaptive, tau_max=tau_max, algo=algo,
                                  compute_stream=compute_stream, pipeline=pipeline)

    def zero_grad(self, set_to_none: bool = False) -> None:
        """One memset over the flat gradient buffer (the views stay attached)."""
        self.flat.zero_grad()

    @torch.no_grad()
    def step(self, closure=None):
        """One local step from the gradients backward left in the flat buffer; returns the
        closure's loss (if given) like ``torch.optim.SGD``.  The per-group ``lr`` is honoured
        when no schedule was given."""
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        if self.worker.schedule is None:
            self.worker.lr = float(self.param_groups[0]["lr"])
        self.worker.step()
        return loss

    def state_dict(self):
        """Not provided: the optimizer state lives in the native worker (momentum, snapshot
        slots, round counters, the communicator's sequence numbers), and the reference
        has no checkpointing either.  Refusing beats silently returning a
        state without the momentum."""
        raise NotImplementedError("LASGD state lives in the native worker; checkpoint the model and re-create the optimizer")

    def load_state_dict(self, state_dict) -> None:
        raise NotImplementedError("LASGD state lives in the native worker; checkpoint the model and re-create the optimizer")

    def add_param_group(self, param_group) -> None:
        # the flat buffers are laid out once, at construction (torch.optim.Optimizer's own
        # __init__ calls this for the module's parameters, before the worker exists)
        if hasattr(self, "worker"):
            raise NotImplementedError("the flat parameter buffer is fixed at construction: no new parameter groups")
        super().add_param_group(param_group)

    def drain(self) -> None:
        """Order the compute stream after any in-flight mean (end of training)."""
        self.worker.drain()

    @property
    def state_view(self):
        """NodeState-shaped view of the worker (tau_i, clocks, snapshot)."""
        return self.worker.state

    def close(self) -> None:
        self.worker.close()
        if self._own_comm:
            self.comm.close()

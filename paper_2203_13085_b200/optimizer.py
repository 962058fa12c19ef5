"""LASGD node state machine on device buffers (mirror of
/root/reference/pkg/src/lasgd/optimizer.py).

Same names, argument order and error behaviour as the reference:
``HyperParams``, ``NodeState.fresh``, ``sgd_local_step``,
``lasgd_finalize_round``, ``lasgd_node_tick``, ``TickAction``.  The state holds
CUDA tensors that the fused kernels update in place (stream-ordered, no host
sync), instead of immutable f64 host vectors.

Two bookkeeping modes:

* ``mode="delta"`` — the reference's exact algorithm: the local step also
  accumulates ``delta`` (optimizer.py:145-146) and finalize is
  ``new = z + delta`` (optimizer.py:171).  Bit-exact against the reference in
  f64 and against its fp32 restatement in fp32.
* ``mode="pull"`` — the north-star elastic pull ``x -= alpha*(snap - xbar)``
  (Algorithm 1 line 9a for alpha = 1; blend order of
  optimizer.py:256-257), which needs no delta buffer (one fewer HBM stream in
  every local step) and supports alpha in (0, 1].

Optional torch-style momentum / weight decay / Nesterov (SPEC.md:176
"optional ... default off") is fused into the same local-step kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import Callable, Optional

import torch

from . import kernels as K
from ._native import NonFiniteError
from .collective import CollectiveHandle
from .params import as_device_vector, blend, mean_of_vectors, require_same_dim, vector_dtype
from .problems import LrSchedule, lr_at


class HyperParamError(ValueError):
    """optimizer.py:24-25."""


@dataclass
class SgdConfig:
    """Local-step modifiers (all off = the reference's plain SGD step)."""

    momentum: float = 0.0
    dampening: float = 0.0
    weight_decay: float = 0.0
    nesterov: bool = False

    def validate(self) -> None:
        if self.momentum < 0 or self.weight_decay < 0 or not 0 <= self.dampening <= 1:
            raise HyperParamError("momentum/weight_decay must be >= 0 and dampening in [0, 1]")
        if self.nesterov and (self.momentum <= 0 or self.dampening != 0):
            raise HyperParamError("Nesterov momentum requires a momentum and zero dampening")


@dataclass
class HyperParams:
    """optimizer.py:28-76.  ``mode="lasgd"`` keeps the reference rule alpha = beta = 1;
    ``mode="lasgd_pull"`` admits the north-star elastic pull with 0 < alpha <= 1."""

    eta: LrSchedule
    num_nodes: int
    tau_max: int
    alpha: float = 1.0
    beta: float = 1.0
    rho: Optional[float] = None
    gamma: Optional[float] = None

    def validate(self, mode: str = "lasgd") -> None:
        errors = []
        if self.num_nodes < 1:
            errors.append("num_nodes must be >= 1")
        if self.tau_max < 1:
            errors.append("tau_max must be >= 1")
        if not 0.0 <= self.alpha <= 1.0:
            errors.append(f"alpha must be in [0, 1], got {self.alpha}")
        if not 0.0 <= self.beta <= 1.0:
            errors.append(f"beta must be in [0, 1], got {self.beta}")
        if self.rho is not None:
            if self.rho < 0:
                errors.append("rho must be >= 0")
            else:
                implied = self.eta.peak_lr * self.rho
                if not math.isclose(self.alpha, implied, rel_tol=1e-9, abs_tol=1e-12):
                    errors.append(f"alpha={self.alpha} inconsistent with peak_lr*rho={implied}")
        if self.gamma is not None:
            if self.gamma < 0:
                errors.append("gamma must be >= 0")
            else:
                implied = self.num_nodes * self.gamma
                if not math.isclose(self.beta, implied, rel_tol=1e-9, abs_tol=1e-12):
                    errors.append(f"beta={self.beta} inconsistent with num_nodes*gamma={implied}")
        if mode == "lasgd" and (self.alpha != 1.0 or self.beta != 1.0):
            errors.append("asynchronous mode requires alpha = beta = 1")
        if mode == "lasgd_pull" and (not 0.0 < self.alpha <= 1.0 or self.beta != 1.0):
            errors.append("elastic-pull mode requires 0 < alpha <= 1 and beta = 1")
        if mode == "easgd" and not 0.0 < self.alpha < 1.0:
            errors.append("round-robin elastic averaging requires 0 < alpha < 1")
        if errors:
            raise HyperParamError("; ".join(errors))


class _FiniteMonitor:
    """Fused non-finite counter (device) read back lazily: each ``poll`` copies the
    counter to pinned host memory asynchronously and inspects the PREVIOUS copy
    if it has landed — detection lags by at most one poll and never blocks.
    ``check`` is the eager, synchronising variant (params.py:23-26 semantics)."""

    def __init__(self, device):
        self.counter = torch.zeros(1, dtype=torch.int64, device=device)
        self._host = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        self._event: Optional[torch.cuda.Event] = None

    def _raise_if(self, bad: int, n: int) -> None:
        if bad:
            raise NonFiniteError(f"blend: {bad} non-finite entries out of {n}")

    def poll(self, n: int) -> None:
        if self._event is not None:
            if not self._event.query():
                return
            self._raise_if(int(self._host.item()), n)
        self._host.copy_(self.counter, non_blocking=True)
        self._event = torch.cuda.Event()
        self._event.record()

    def check(self, n: int) -> None:
        self._raise_if(int(self.counter.item()), n)


class NodeState:
    """optimizer.py:79-104 on device buffers.

    ``x_snapshot`` is one of two snapshot slots (double-buffered by round parity
    so a finalize never overwrites a snapshot a peer may still be reading); with
    ``snapshot_buffers`` from a P2P communicator the slots ARE the IPC-exported
    contribution buffers, so submitting costs no copy."""

    def __init__(self, rank: int, x_local: torch.Tensor, snapshots, delta: Optional[torch.Tensor],
                 sgd: Optional[SgdConfig] = None, check_finite: str = "lazy"):
        self.rank = rank
        self.x_local = x_local
        self.snapshots = list(snapshots)
        self.snap_idx = 0
        self._delta_buf = delta
        self.tau_i = 0
        self.local_clock = 0
        self.global_clock = 0
        self.pending: Optional[CollectiveHandle] = None
        self.sgd = sgd or SgdConfig()
        self.sgd.validate()
        self.momentum_buf = torch.empty_like(x_local) if self.sgd.momentum != 0 else None
        self._momentum_started = False
        self._delta_fresh = False
        if check_finite not in ("lazy", "eager", "off"):
            raise ValueError("check_finite must be 'lazy', 'eager' or 'off'")
        self.check_mode = check_finite
        self._finite = _FiniteMonitor(x_local.device)

    @property
    def x_snapshot(self) -> torch.Tensor:
        return self.snapshots[self.snap_idx]

    @property
    def delta(self) -> Optional[torch.Tensor]:
        """The delta accumulator (optimizer.py:84).  A finalize resets it to zero
        (optimizer.py:174) lazily: the next local step overwrites instead of adding, so
        the reset costs no pass of its own.  Reading it here materialises the zeros."""
        if self._delta_buf is not None and self._delta_fresh:
            self._delta_buf.zero_()
            self._delta_fresh = False
        return self._delta_buf

    @property
    def nonfinite_counter(self) -> Optional[torch.Tensor]:
        return None if self.check_mode == "off" else self._finite.counter

    def check_finite(self) -> None:
        """Synchronising NaN/Inf check of everything computed so far."""
        self._finite.check(self.x_local.numel())

    def _after_op(self, boundary: bool = False) -> None:
        if self.check_mode == "eager":
            self._finite.check(self.x_local.numel())
        elif self.check_mode == "lazy" and boundary:
            self._finite.poll(self.x_local.numel())

    @classmethod
    def fresh(cls, rank: int, x0, *, mode: str = "delta", sgd: Optional[SgdConfig] = None, snapshot_buffers=None,
              dtype: torch.dtype = torch.float32, device=None, copy: bool = True,
              check_finite: str = "lazy") -> "NodeState":
        """optimizer.py:97-104: x_local = x_snapshot = x0, delta = 0."""
        if mode not in ("delta", "pull"):
            raise ValueError("mode must be 'delta' or 'pull'")
        x = as_device_vector(x0, dtype, device)
        if copy and (isinstance(x0, torch.Tensor) and x.data_ptr() == x0.data_ptr()):
            x = x.clone()
        if snapshot_buffers is None:
            snapshot_buffers = [torch.empty_like(x), torch.empty_like(x)]
        for s in snapshot_buffers:
            if s.numel() != x.numel() or s.dtype != x.dtype:
                raise ValueError("snapshot buffers must match the parameter vector")
        K.snapshot(snapshot_buffers[0], x)
        delta = torch.zeros_like(x) if mode == "delta" else None
        return cls(rank, x, snapshot_buffers, delta, sgd=sgd, check_finite=check_finite)


class TickAction(Enum):
    COMPUTED_STEP = "computed_step"
    FINALIZED = "finalized"
    WAITING_ON_COLLECTIVE = "waiting_on_collective"


def sgd_local_step(state: NodeState, g, eta: float, tau_max: int) -> NodeState:
    """optimizer.py:136-149 as one fused kernel: x (and delta) += (-eta)*direction."""
    if state.tau_i >= tau_max:
        raise RuntimeError(
            f"node {state.rank} has exhausted its local budget (tau_i={state.tau_i}, tau_max={tau_max})")
    g = g if isinstance(g, torch.Tensor) and g.is_cuda else as_device_vector(g, state.x_local.dtype,
                                                                             state.x_local.device)
    c = state.sgd
    K.sgd_step(state.x_local, g.reshape(-1), eta, m=state.momentum_buf, delta=state._delta_buf, momentum=c.momentum,
               dampening=c.dampening, weight_decay=c.weight_decay, nesterov=c.nesterov,
               first_step=not state._momentum_started, delta_reset=state._delta_fresh,
               nonfinite=state.nonfinite_counter)
    state._momentum_started = state.momentum_buf is not None
    state._delta_fresh = False
    state.tau_i += 1
    state.local_clock += 1
    state._after_op()
    return state


def lasgd_finalize_round(state: NodeState, z, num_nodes: int,
                         submit: Optional[Callable[[torch.Tensor], CollectiveHandle]] = None, *,
                         alpha: Optional[float] = None) -> NodeState:
    """optimizer.py:152-178.

    P == 1 short-circuits to the live model (new snapshot = x_local).  Otherwise,
    in delta mode with alpha in (None, 1) the reference rule new = z + delta;
    in pull mode (or alpha != 1) x -= alpha*(snap - z).  Either way the new model
    is written to the other snapshot slot in the same pass, the budget resets and
    the snapshot is submitted when ``submit`` is given.  ``z`` may be a tensor or
    a handle (then ordered with ``result_async``, without a host sync)."""
    nxt = 1 - state.snap_idx
    x = state.x_local
    if num_nodes == 1:
        K.snapshot(state.snapshots[nxt], x)
    else:
        if isinstance(z, CollectiveHandle):
            z = z.result_async()
        if z is None:
            raise ValueError("collective reported complete but no center vector supplied")
        z = z if isinstance(z, torch.Tensor) and z.is_cuda else as_device_vector(z, x.dtype, x.device)
        if state._delta_buf is not None and (alpha is None or alpha == 1.0):
            # no local step since the last finalize: delta is logically zero (optimizer.py:174),
            # so new = z + 0 — the kernel reads no delta at all
            d = None if state._delta_fresh else state._delta_buf
            K.finalize(x, z, d, snap_next=state.snapshots[nxt], nonfinite=state.nonfinite_counter)
        else:
            a = 1.0 if alpha is None else float(alpha)
            if not 0.0 < a <= 1.0:
                raise HyperParamError(f"alpha must be in (0, 1], got {a}")
            K.elastic_pull(x, state.x_snapshot, z, a, snap_next=state.snapshots[nxt],
                           nonfinite=state.nonfinite_counter)
    state.snap_idx = nxt
    state._delta_fresh = state._delta_buf is not None
    state.tau_i = 0
    state.global_clock += 1
    state._after_op(boundary=True)
    state.pending = submit(state.x_snapshot) if submit is not None else None
    return state


class ModelDivergenceError(RuntimeError):
    """optimizer.py:210-211: synchronous replicas stopped being bit-identical."""


def elastic_local_step(x, z, g, eta: float, alpha: float) -> torch.Tensor:
    """optimizer.py:113-122: ``alpha*z + (1-alpha)*x - eta*g`` as two K0 blends, in the
    reference's order (new device vector)."""
    if not 0.0 <= alpha <= 1.0:
        raise HyperParamError(f"alpha must be in [0, 1], got {alpha}")
    if eta <= 0:
        raise HyperParamError(f"eta must be positive, got {eta}")
    dt = vector_dtype(x)
    x, z, g = (as_device_vector(v, dtype=dt) for v in (x, z, g))
    pulled = blend(alpha, z, 1.0 - alpha, x)
    return blend(1.0, pulled, -eta, g, out=pulled)


def elastic_center_step(z, xs, beta: float) -> torch.Tensor:
    """optimizer.py:125-133: ``(1-beta)*z + beta*mean(xs)`` (ascending-order mean)."""
    xs = list(xs)
    if not xs:
        raise ValueError("need at least one local model")
    if not 0.0 <= beta <= 1.0:
        raise HyperParamError(f"beta must be in [0, 1], got {beta}")
    dt = vector_dtype(z)
    z = as_device_vector(z, dtype=dt)
    xs = [as_device_vector(v, dtype=dt) for v in xs]
    for v in xs:
        require_same_dim(z, v)
    return blend(1.0 - beta, z, beta, mean_of_vectors(xs))


def easgd_round_robin_exchange(x, z, alpha: float):
    """optimizer.py:245-259: symmetric elastic pull between one node and the center,
    ``x' = x - alpha*(x - z)``, ``z' = z + alpha*(x - z)`` (three K0 blends)."""
    if not 0.0 < alpha < 1.0:
        raise HyperParamError(f"round-robin exchange needs 0 < alpha < 1, got {alpha}")
    dt = vector_dtype(x)
    x, z = as_device_vector(x, dtype=dt), as_device_vector(z, dtype=dt)
    require_same_dim(x, z)
    diff = blend(1.0, x, -1.0, z)
    return blend(1.0, x, -alpha, diff), blend(1.0, z, alpha, diff)


def sync_allreduce_sgd_round(states, grads, eta: float, transport=None, round_id: int = 0) -> torch.Tensor:
    """optimizer.py:214-242 (SGD-AR baseline): average the gradients with the same
    ring-order mean all-reduce, apply x = x + (-eta)*mean_g on every replica and move
    its snapshot.  Replicas on one device (loopback) are checked bit for bit first;
    with a per-process P2P transport each process passes its own single state."""
    from .collective import all_reduce_average

    if len(states) != len(grads):
        raise ValueError("need one gradient per node")
    ref = states[0].x_local
    for st in states[1:]:
        if not torch.equal(st.x_local.view(torch.int32 if ref.dtype == torch.float32 else torch.int64),
                           ref.view(torch.int32 if ref.dtype == torch.float32 else torch.int64)):
            raise ModelDivergenceError(f"node {st.rank} model differs from node {states[0].rank}")
    handle = all_reduce_average(grads, transport=transport, round_id=round_id)
    mean_g = handle.result_async()
    for st in states:
        K.sgd_step(st.x_local, mean_g, eta, nonfinite=st.nonfinite_counter)
        nxt = 1 - st.snap_idx
        K.snapshot(st.snapshots[nxt], st.x_local)
        st.snap_idx = nxt
        st.local_clock += 1
        st.global_clock += 1
        st._after_op(boundary=True)
    return mean_g


def lasgd_node_tick(state: NodeState, grad_fn: Callable, schedule: LrSchedule, collective_complete: bool,
                    z, tau_max: int, num_nodes: int,
                    submit: Optional[Callable[[torch.Tensor], CollectiveHandle]] = None, *,
                    alpha: Optional[float] = None) -> TickAction:
    """optimizer.py:181-207: finalize if the collective is done, else step while budget remains, else wait."""
    if collective_complete:
        if z is None:
            raise ValueError("collective reported complete but no center vector supplied")
        lasgd_finalize_round(state, z, num_nodes, submit=submit, alpha=alpha)
        return TickAction.FINALIZED
    if state.tau_i < tau_max:
        g = grad_fn(state.x_local)
        eta = lr_at(schedule, state.local_clock)
        sgd_local_step(state, g, eta, tau_max)
        return TickAction.COMPUTED_STEP
    return TickAction.WAITING_ON_COLLECTIVE

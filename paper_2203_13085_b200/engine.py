"""Per-rank LASGD worker: the round protocol on CUDA streams and events.

This is Algorithm 1 (optimizer.py:181-207) driven by real
asynchrony instead of the reference's caller-supplied ``collective_complete``
flag:

* compute stream (high priority): forward/backward (PyTorch), then K5 — the
  fused local step on the flat buffer — every minibatch;
* at a round boundary: the compute stream waits for the previous round's mean
  (event), applies the fused pull / finalize that also writes the next
  snapshot slot (K4+K1), and hands the snapshot to the side stream;
* side stream (low priority, bounded CTA budget): the NVLink P2P mean
  all-reduce (K2/K3 with K6 flags) overlaps the next minibatches.

Round boundaries are either deterministic (exactly ``sync_period`` local steps
per round — the parity schedule) or adaptive (finalize as soon as the
host-mapped completion flag says the mean landed, or block the compute stream
when ``tau_max`` steps have been taken — the paper's dynamic rate, Table 3).

``pipeline="fused"`` (deterministic only) replaces the boundary step's
K5 -> (mean lands) -> K4 -> K2/K3 chain by ONE kernel (K7) that applies the local
step, reads every peer's snapshot over NVLink, forms the ring-order mean, pulls and
writes the next snapshot in the same pass — bit-identical results, HBM and NVLink
streamed concurrently.  ``pipeline="overlap"`` (default) keeps the mean on the side
stream so it overlaps the next minibatches' forward/backward.
"""

from __future__ import annotations

import collections
from typing import Optional

import torch

from . import _native as N
from . import kernels as K
from .optimizer import NodeState, SgdConfig
from .problems import LrSchedule, lr_at


class LASGDWorker:
    def __init__(self, x: torch.Tensor, g: torch.Tensor, *, comm=None, sync_period: int = 1, alpha: float = 1.0,
                 mode: str = "pull", sgd: Optional[SgdConfig] = None, schedule: Optional[LrSchedule] = None,
                 lr: Optional[float] = None, adaptive: bool = False, tau_max: Optional[int] = None,
                 algo: int = N.ALGO_AUTO, compute_stream: Optional[torch.cuda.Stream] = None, sync: bool = True,
                 timed: bool = False, check_finite: str = "lazy", max_host_lead: int = 2,
                 pipeline: str = "overlap", fused_nblocks: int = 0):
        if (schedule is None) == (lr is None):
            raise ValueError("give exactly one of schedule / lr")
        if sync_period < 1:
            raise ValueError("sync_period must be >= 1")
        if not 0.0 < alpha <= 1.0:
            raise ValueError("alpha must be in (0, 1]")
        if mode not in ("pull", "delta"):
            raise ValueError("mode must be 'pull' or 'delta'")
        if pipeline not in ("overlap", "fused"):
            raise ValueError("pipeline must be 'overlap' or 'fused'")
        if pipeline == "fused" and adaptive:
            raise ValueError("the fused pipeline implements the deterministic schedule only")
        self.pipeline = pipeline
        self.fused_nblocks = fused_nblocks
        self.comm = comm
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.k = sync_period
        self.alpha = alpha
        self.mode = mode
        self.schedule, self.lr = schedule, lr
        self.adaptive = adaptive
        self.tau_max = tau_max if tau_max is not None else sync_period
        self.algo = algo
        self.sync = sync
        self.timed = timed
        self.g = g
        self.compute = compute_stream if compute_stream is not None else torch.cuda.current_stream(x.device)
        snaps = comm.snapshots if comm is not None else [torch.empty_like(x), torch.empty_like(x)]
        delta = torch.zeros_like(x) if mode == "delta" else None
        self.state = NodeState(self.rank, x, snaps, delta, sgd=sgd, check_finite=check_finite)
        self.xbar = comm.xbar if comm is not None else None
        self.seq = 0
        self.launches = collections.Counter()
        self.records = []  # (name, start_event, end_event)
        self.tau_hist = collections.Counter()
        self._lead = collections.deque()
        self._max_lead = max_host_lead
        with torch.cuda.stream(self.compute):
            self._launch("snapshot", self.compute, lambda: K.snapshot(self.state.snapshots[0], x))
            if self.sync and self.world > 1 and pipeline == "overlap":
                self._submit(0)

    # ------------------------------------------------------------------ helpers
    def _launch(self, name: str, stream, fn) -> None:
        if self.timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            self.records.append((name, e0, e1))
        else:
            fn()
        self.launches[name] += 1

    def _submit(self, slot: int) -> None:
        self.comm.stream.wait_stream(self.compute)
        box = {}
        self._launch("allreduce", self.comm.stream, lambda: box.setdefault("s", self.comm.allreduce(slot, self.algo)))
        self.seq = box["s"]

    def current_lr(self) -> float:
        return self.lr if self.schedule is None else lr_at(self.schedule, self.state.local_clock)

    # ------------------------------------------------------------------ protocol
    def step(self) -> bool:
        """One local step from the gradient already in ``g`` (call on the compute
        stream after backward).  Returns True if this step closed a round."""
        st = self.state
        c = st.sgd
        lr = self.current_lr()
        if self.pipeline == "fused" and self.sync and st.tau_i + 1 == self.k:
            self._fused_round(lr)
            return True
        self._launch("sgd_step", self.compute, lambda: K.sgd_step(
            st.x_local, self.g, lr, m=st.momentum_buf, delta=st.delta, momentum=c.momentum, dampening=c.dampening,
            weight_decay=c.weight_decay, nesterov=c.nesterov, first_step=not st._momentum_started,
            delta_reset=st._delta_fresh, nonfinite=st.nonfinite_counter, stream=self.compute))
        st._momentum_started = st.momentum_buf is not None
        st._delta_fresh = False
        st.tau_i += 1
        st.local_clock += 1
        if not self.sync:
            return False
        if self.adaptive:
            self._throttle()
            done = self.world == 1 or self.comm.query(self.seq) == 1
            if done or st.tau_i >= self.tau_max:
                self._round()
                return True
            return False
        if st.tau_i == self.k:
            self._round()
            return True
        return False

    def _fused_round(self, lr: float) -> None:
        st = self.state
        c = st.sgd
        cur, nxt = st.snap_idx, 1 - st.snap_idx
        mode = 1 if (self.mode == "delta" and self.alpha == 1.0) else 0
        kw = dict(momentum=c.momentum, dampening=c.dampening, weight_decay=c.weight_decay, nesterov=c.nesterov,
                  first_step=not st._momentum_started, delta_reset=st._delta_fresh, alpha=self.alpha, mode=mode,
                  nonfinite=st.nonfinite_counter)
        self.tau_hist[st.tau_i + 1] += 1
        if self.world == 1:
            # P == 1 (optimizer.py:168-169): local step + snapshot in one pass, no mean
            self._launch("fused_round", self.compute, lambda: K.fused_round_virtual(
                [st.x_local], [self.g], [st.snapshots[cur]], [st.snapshots[nxt]], lr,
                ms=None if st.momentum_buf is None else [st.momentum_buf],
                deltas=None if st.delta is None else [st.delta], nblocks=self.fused_nblocks, stream=self.compute,
                **kw))
        else:
            box = {}
            self._launch("fused_round", self.compute, lambda: box.setdefault("s", self.comm.fused_round(
                cur, st.x_local, self.g, lr, m=st.momentum_buf, delta=st.delta, algo=self.algo,
                nblocks=self.fused_nblocks,
                stream=self.compute, **kw)))
            self.seq = box["s"]
        st._momentum_started = st.momentum_buf is not None
        st._delta_fresh = st.delta is not None
        st.snap_idx = nxt
        st.tau_i = 0
        st.local_clock += 1
        st.global_clock += 1
        if st.check_mode == "lazy":
            with torch.cuda.stream(self.compute):
                st._finite.poll(st.x_local.numel())

    def _throttle(self) -> None:
        ev = torch.cuda.Event()
        ev.record(self.compute)
        self._lead.append(ev)
        while len(self._lead) > self._max_lead:
            self._lead.popleft().synchronize()

    def _round(self) -> None:
        st = self.state
        nxt = 1 - st.snap_idx
        x = st.x_local
        self.tau_hist[st.tau_i] += 1
        if self.world == 1:
            # optimizer.py:168-169: P == 1 keeps the live model; only the snapshot moves
            self._launch("snapshot", self.compute, lambda: K.snapshot(st.snapshots[nxt], x, stream=self.compute))
        else:
            self.comm.stream_wait(self.seq, self.compute)
            if self.mode == "delta" and self.alpha == 1.0:
                self._launch("finalize", self.compute, lambda: K.finalize(
                    x, self.xbar, st.delta, snap_next=st.snapshots[nxt], nonfinite=st.nonfinite_counter,
                    stream=self.compute))
            else:
                cur = st.snapshots[st.snap_idx]
                self._launch("pull", self.compute, lambda: K.elastic_pull(
                    x, cur, self.xbar, self.alpha, snap_next=st.snapshots[nxt], nonfinite=st.nonfinite_counter,
                    stream=self.compute))
        st.snap_idx = nxt
        st._delta_fresh = st.delta is not None
        st.tau_i = 0
        st.global_clock += 1
        if st.check_mode == "lazy":
            with torch.cuda.stream(self.compute):
                st._finite.poll(x.numel())
        if self.world > 1:
            self._submit(nxt)

    def drain(self) -> None:
        """Order the compute stream after the in-flight all-reduce."""
        if self.world > 1 and self.seq and self.pipeline == "overlap":
            self.comm.stream_wait(self.seq, self.compute)

    # ------------------------------------------------------------------ measurement
    def kernel_times(self) -> dict:
        """Per-kernel list of durations (ms) of the timed launches (after a sync)."""
        out = collections.defaultdict(list)
        for name, e0, e1 in self.records:
            out[name].append(e0.elapsed_time(e1))
        return dict(out)

    def reset_records(self) -> None:
        self.records.clear()
        self.launches.clear()

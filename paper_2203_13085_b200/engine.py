"""Per-rank LASGD worker: the round protocol on CUDA streams and events.

This is Algorithm 1 (optimizer.py:181-207) driven by real
asynchrony instead of the reference's caller-supplied ``collective_complete``
flag.  The protocol itself runs natively (``lasgd_worker_*`` in
csrc/lasgd_worker.cu): one ctypes call per local step issues every launch of
that step, so the host keeps well ahead of the GPU.

* compute stream (high priority): forward/backward (PyTorch), then K5 — the
  fused local step on the flat buffer — every minibatch;
* ``pipeline="overlap"``: at a round boundary the compute stream waits for the
  previous round's mean (event), applies the fused pull / finalize that also
  writes the next snapshot slot (K4+K1) and hands the snapshot to the side
  stream (low priority, bounded CTA budget), where the NVLink P2P mean
  all-reduce (K2/K3 with K6 flags) overlaps the next minibatches;
* ``pipeline="fused"`` (deterministic only): the boundary step is ONE kernel
  that applies the local step, forms the ring-order mean of every rank's snapshot,
  pulls and writes the next snapshot — K7 (peers' snapshots read over NVLink) or the
  K8 push round (data moved by remote stores: the peer's snapshot mirrored at P=2,
  staged chunks at P>=3); bit-identical results, HBM and NVLink streamed concurrently.

Round boundaries are deterministic (exactly ``sync_period`` local steps per
round — the parity schedule) or adaptive (finalize as soon as the host-mapped
completion flag says the mean landed or the peers are already ahead, or make the
compute stream wait when ``tau_max`` steps have been taken — the paper's dynamic
rate, Table 3).
"""

from __future__ import annotations

import collections
import ctypes
from typing import Optional

import torch

from . import _native as N
from . import kernels as K
from .optimizer import SgdConfig, _FiniteMonitor
from .problems import LrSchedule, lr_at


class WorkerState:
    """NodeState-shaped view (optimizer.py:79-104) of the native worker."""

    def __init__(self, worker: "LASGDWorker", x, snapshots, delta, momentum_buf, finite):
        self._w = worker
        self.rank = worker.rank
        self.x_local = x
        self.snapshots = snapshots
        self.delta = delta
        self.momentum_buf = momentum_buf
        self._finite = finite

    def _s(self):
        return self._w._native_state()

    @property
    def tau_i(self) -> int:
        return self._s().tau_i

    @property
    def snap_idx(self) -> int:
        return self._s().snap_idx

    @property
    def local_clock(self) -> int:
        return self._s().local_clock

    @property
    def global_clock(self) -> int:
        return self._s().global_clock

    @property
    def x_snapshot(self) -> torch.Tensor:
        return self.snapshots[self.snap_idx]

    @property
    def nonfinite_counter(self):
        return self._finite.counter

    def check_finite(self) -> None:
        self._finite.check(self.x_local.numel())


class LASGDWorker:
    def __init__(self, x: torch.Tensor, g: torch.Tensor, *, comm=None, sync_period: int = 1, alpha: float = 1.0,
                 mode: str = "pull", sgd: Optional[SgdConfig] = None, schedule: Optional[LrSchedule] = None,
                 lr: Optional[float] = None, adaptive: bool = False, tau_max: Optional[int] = None,
                 algo: int = N.ALGO_AUTO, compute_stream: Optional[torch.cuda.Stream] = None, sync: bool = True,
                 timed: bool = False, check_finite: str = "lazy", max_host_lead: int = 2,
                 pipeline: str = "overlap", fused_nblocks: int = 0, check_every: int = 16,
                 max_host_wait_us: int = 250_000):
        if (schedule is None) == (lr is None):
            raise ValueError("give exactly one of schedule / lr")
        if mode not in ("pull", "delta"):
            raise ValueError("mode must be 'pull' or 'delta'")
        if pipeline not in ("overlap", "fused"):
            raise ValueError("pipeline must be 'overlap' or 'fused'")
        if check_finite not in ("lazy", "eager", "off"):
            raise ValueError("check_finite must be 'lazy', 'eager' or 'off'")
        sgd = sgd or SgdConfig()
        sgd.validate()
        K._check(x, g)
        if comm is not None and (comm.n != x.numel() or comm.dtype != x.dtype):
            raise ValueError("communicator buffers do not match x")
        if algo == N.ALGO_CE and pipeline == "fused" and comm is not None and comm.world > 1 and sync:
            raise ValueError("the copy-engine mean is a side-stream all-reduce: use pipeline='overlap'")
        self.comm = comm
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.k = sync_period
        self.schedule, self.lr = schedule, lr
        self.pipeline = pipeline
        self.adaptive = adaptive
        self.algo = algo
        self.timed = timed
        self.sync = bool(sync)
        self._graphs: list = []  # SyncGraphs point into the native worker: closed with it
        self.g = g
        self.compute = compute_stream if compute_stream is not None else torch.cuda.current_stream(x.device)
        self._local_clock = 0
        self._rounds = 0
        self._check_mode = check_finite
        self._check_every = max(1, check_every)
        snaps = comm.snapshots if comm is not None else [torch.empty_like(x), torch.empty_like(x)]
        delta = torch.zeros_like(x) if mode == "delta" else None
        mbuf = torch.empty_like(x) if sgd.momentum != 0 else None
        finite = _FiniteMonitor(x.device)
        self.state = WorkerState(self, x, snaps, delta, mbuf, finite)
        self.xbar = comm.xbar if comm is not None else None
        cfg = N.WorkerConfig(sync_period, float(alpha), 1 if mode == "delta" else 0, 1 if pipeline == "fused" else 0,
                             int(algo), int(fused_nblocks), float(sgd.momentum), float(sgd.dampening),
                             float(sgd.weight_decay), int(sgd.nesterov), int(bool(sync)), int(bool(adaptive)),
                             int(tau_max or 0), int(max_host_lead), int(max_host_wait_us))
        side = comm.stream if comm is not None else None
        h = ctypes.c_void_p()
        ptr = K._ptr
        N.check(N.lib().lasgd_worker_create(
            comm._h if comm is not None else None, ptr(x), ptr(mbuf), ptr(delta),
            None if comm is not None else ptr(snaps[0]), None if comm is not None else ptr(snaps[1]),
            x.numel(), K.dtype_code(x), ctypes.byref(cfg), ctypes.c_void_p(self.compute.cuda_stream),
            ctypes.c_void_p(side.cuda_stream) if side is not None else None,
            None if check_finite == "off" else ptr(finite.counter), ctypes.byref(h)), "lasgd_worker_create")
        self._h = h
        self._keep = (x, g, snaps, delta, mbuf, finite)  # buffers the native worker points into
        if timed:
            N.check(N.lib().lasgd_worker_set_timing(self._h, 1))

    # ------------------------------------------------------------------ protocol
    def current_lr(self) -> float:
        return self.lr if self.schedule is None else lr_at(self.schedule, self._local_clock)

    def step(self) -> bool:
        """One local step from the gradient in ``self.g`` (call on the compute stream
        after backward).  Returns True if this step closed a round."""
        rc = N.lib().lasgd_worker_step(self._h, self.g.data_ptr(), self.current_lr())
        if rc < 0:
            N.check(rc, "lasgd_worker_step")
        self._local_clock += 1
        if self._check_mode == "eager":
            self.state.check_finite()
        if getattr(self, "_capturing", False):
            return rc == 1  # inside a stream capture: the replay does the bookkeeping
        if rc == 1:
            self._rounds += 1
            if self._check_mode == "lazy" and self._rounds % self._check_every == 0:
                with torch.cuda.stream(self.compute):
                    self.state._finite.poll(self.state.x_local.numel())
            return True
        return False

    # ------------------------------------------------------------------ graph replay
    def _ensure_lr_table(self, clock_end: int) -> None:
        """Device learning-rate table covering local clocks [0, clock_end)."""
        if self.schedule is None:
            # a constant rate may have been changed since the last capture (an LR
            # scheduler writing worker.lr): re-upload whenever it differs
            if getattr(self, "_lr_len", 0) != 1 or getattr(self, "_lr_const", None) != float(self.lr):
                table = (ctypes.c_double * 1)(float(self.lr))
                N.check(N.lib().lasgd_worker_set_lr_table(self._h, table, 1), "lasgd_worker_set_lr_table")
                self._lr_len, self._lr_const = 1, float(self.lr)
            return
        if getattr(self, "_lr_len", 0) >= clock_end:
            return
        n = max(clock_end, 2 * getattr(self, "_lr_len", 0), 1024)
        table = (ctypes.c_double * n)(*[lr_at(self.schedule, t) for t in range(n)])
        N.check(N.lib().lasgd_worker_set_lr_table(self._h, table, n), "lasgd_worker_set_lr_table")
        self._lr_len = n

    def capture(self, grads, steps: Optional[int] = None) -> "SyncGraph":
        """Capture ``steps`` local steps (default ``len(grads)``; a whole number of rounds),
        step t reading gradient ``grads[t % len(grads)]``, as one CUDA graph.  Nothing runs
        until ``replay()``; each replay advances the worker exactly as ``steps`` calls of
        ``step()`` would, with bit-identical results (deterministic schedule; one rank, or
        the fused pipeline over a communicator after one eager round)."""
        grads = list(grads)
        steps = len(grads) if steps is None else int(steps)
        for t in grads:
            K._check(self.state.x_local, t)
        self._ensure_lr_table(self._local_clock + steps)
        arr = (ctypes.c_void_p * steps)(*[grads[t % len(grads)].data_ptr() for t in range(steps)])
        h = ctypes.c_void_p()
        N.check(N.lib().lasgd_worker_graph_capture(self._h, steps, arr, ctypes.byref(h)), "lasgd_worker_graph_capture")
        gr = SyncGraph(self, h, steps, grads)
        self._graphs.append(gr)
        return gr

    def capture_with(self, fn, steps: int = 1, pool=None) -> "SyncGraph":
        """Capture ``steps`` iterations of ``fn(t)`` (forward + backward writing the
        gradient into ``self.g``) followed by ``step()`` into ONE CUDA graph on the compute
        stream: the whole training step — minibatch compute, local step and round
        boundary — replays as a single launch.  ``fn`` must have run eagerly before
        (cuDNN autotuning, allocator warm-up) and must not synchronise with the host."""
        self._ensure_lr_table(self._local_clock + steps)
        graph = torch.cuda.CUDAGraph()
        h = ctypes.c_void_p()
        self._capturing = True
        clock0 = self._local_clock
        try:
            with torch.cuda.graph(graph, stream=self.compute, pool=pool):
                N.check(N.lib().lasgd_worker_capture_begin(self._h, ctypes.byref(h)), "lasgd_worker_capture_begin")
                try:
                    for t in range(steps):
                        fn(t)
                        self.step()
                finally:
                    rc_end = N.lib().lasgd_worker_capture_end(h)
            N.check(rc_end, "lasgd_worker_capture_end")
        except BaseException:
            if h:
                N.lib().lasgd_graph_destroy(h)
            raise
        finally:
            self._capturing = False
            self._local_clock = clock0  # step() advanced the Python clock during capture
        gr = SyncGraph(self, h, steps, [self.g], external=graph)
        self._graphs.append(gr)
        return gr

    def drain(self, group=None) -> None:
        """Order the compute stream after the in-flight all-reduce.

        Adaptive mode: ranks close rounds on their own clock, so at the end of a run
        one rank may have launched more all-reduces than another, and its last launch
        would wait for a peer launch that never comes.  The launch counts are
        exchanged over torch.distributed and lagging ranks contribute their current
        snapshot to the missing rounds (exactly what a node that keeps running would
        submit), so every launched collective completes."""
        N.check(N.lib().lasgd_worker_drain(self._h), "lasgd_worker_drain")
        if not (self.adaptive and self.world > 1):
            return
        import time

        import torch.distributed as dist

        comm = self.comm
        slot = self._native_state().snap_idx

        def pad_to(target: int) -> None:
            extra = target - comm.launches()
            if extra <= 0:
                return
            comm.stream.wait_stream(self.compute)  # the padding reads the current snapshot slot
            for _ in range(extra):
                comm.allreduce(slot, self.algo)

        # A peer that launched more rounds may be stalled (device waiting on our missing
        # launch, host possibly blocked behind it), so never block on a host collective
        # here: pad to what the peers' entry flags show while an asynchronous MAX of the
        # launch counts completes, then pad to the agreed maximum.
        side = torch.cuda.Stream(device=self.state.x_local.device)
        backend = dist.get_backend(group)
        with torch.cuda.stream(side):
            t = torch.tensor([comm.launches()], dtype=torch.int64,
                             device=self.state.x_local.device if backend == "nccl" else "cpu")
            work = dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group, async_op=True)
            while not work.is_completed():
                pad_to(comm.peer_max_seq())
                time.sleep(1e-3)
            work.wait()
        pad_to(int(t.item()))
        last = comm.launches()
        if last:
            comm.stream_wait(last, self.compute)

    # ------------------------------------------------------------------ state / measurement
    def _native_state(self) -> N.WorkerState:
        s = N.WorkerState()
        N.check(N.lib().lasgd_worker_get_state(self._h, ctypes.byref(s)))
        return s

    @property
    def seq(self) -> int:
        return self._native_state().seq

    @property
    def launches(self) -> collections.Counter:
        s = self._native_state()
        return collections.Counter({k: s.launches[i] for i, k in enumerate(N.KERNEL_KINDS) if s.launches[i]})

    @property
    def tau_hist(self) -> collections.Counter:
        s = self._native_state()
        return collections.Counter({t: s.tau_hist[t] for t in range(N.TAU_HIST) if s.tau_hist[t]})

    def kernel_times(self) -> dict:
        """Per-kernel durations (ms) of the timed launches (call after a sync)."""
        out = {}
        for i, name in enumerate(N.KERNEL_KINDS):
            buf = (ctypes.c_float * 65536)()
            k = N.check(N.lib().lasgd_worker_timings(self._h, i, buf, 65536))
            if k:
                out[name] = list(buf[:k])
        return out

    def reset_records(self) -> None:
        N.check(N.lib().lasgd_worker_reset_stats(self._h))

    def close(self) -> None:
        for gr in getattr(self, "_graphs", ()):
            gr.close()
        if getattr(self, "_h", None):
            N.lib().lasgd_worker_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SyncGraph:
    """A captured run of worker steps (``LASGDWorker.capture``): ``replay()`` is one graph
    launch on the worker's compute stream."""

    def __init__(self, worker: LASGDWorker, handle, steps: int, grads, external=None):
        self.worker = worker
        self._h = handle
        self.steps = steps
        self.rounds = steps // worker.k if worker.sync else 0
        self._keep = grads  # the captured gradient buffers
        self.external = external  # capture_with: the torch graph holding fwd/bwd + the steps

    def replay(self) -> None:
        w = self.worker
        w._ensure_lr_table(w._local_clock + self.steps)
        N.check(N.lib().lasgd_graph_launch(self._h), "lasgd_graph_launch")
        if self.external is not None:
            with torch.cuda.stream(w.compute):
                self.external.replay()
        w._local_clock += self.steps
        before = w._rounds
        w._rounds += self.rounds
        if w._check_mode == "eager":
            w.state.check_finite()
        elif w._check_mode == "lazy" and w._rounds // w._check_every != before // w._check_every:
            with torch.cuda.stream(w.compute):
                w.state._finite.poll(w.state.x_local.numel())

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().lasgd_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SGDARWorker:
    """SGD-AR baseline (optimizer.py:214-242, ``sync_allreduce_sgd_round``) per process.

    Backward writes the gradient straight into one of the communicator's registered
    snapshot slots (``grad_buffer``); ``step()`` then runs ONE fused kernel on the compute
    stream (K7 mode 2): the ring-order mean of every rank's gradient slot over NVLink
    (one-shot or two-shot; the reference ring's per-chunk order, so the mean and therefore
    every replica's model stay bit-identical) and K5 with the mean gradient — the
    synchronous data-parallel step LASGD is compared against (Table 4).

    The slots alternate per step: peers may still be reading this step's slot while
    this rank runs the next backward; the slot is rewritten two steps later, after the
    next all-reduce's entry barrier has proved every peer finished this one.  Pass
    ``flat`` (FlatParams) to have ``.grad`` rebound to the current slot automatically."""

    def __init__(self, x: torch.Tensor, *, comm=None, sgd: Optional[SgdConfig] = None,
                 schedule: Optional[LrSchedule] = None, lr: Optional[float] = None, algo: int = N.ALGO_AUTO,
                 compute_stream: Optional[torch.cuda.Stream] = None, flat=None):
        if (schedule is None) == (lr is None):
            raise ValueError("give exactly one of schedule / lr")
        if algo in (N.ALGO_PUSH, N.ALGO_CE):
            raise ValueError("the SGD-AR round is one kernel: one-shot or two-shot (push / copy-engine are LASGD forms)")
        self.sgd = sgd or SgdConfig()
        self.sgd.validate()
        K._check(x)
        self.x, self.comm, self.algo = x, comm, algo
        self.schedule, self.lr = schedule, lr
        self.compute = compute_stream if compute_stream is not None else torch.cuda.current_stream(x.device)
        if comm is not None and (comm.n != x.numel() or comm.dtype != x.dtype):
            raise ValueError("communicator buffers do not match x")
        self._bufs = comm.snapshots if comm is not None else [torch.zeros_like(x)]
        self._slot = 0
        self.flat = flat
        self.m = torch.empty_like(x) if self.sgd.momentum != 0 else None
        self._finite = _FiniteMonitor(x.device)
        self.local_clock = 0
        self.launches = collections.Counter()
        if flat is not None:
            flat.bind_grads(self.grad_buffer)

    @property
    def grad_buffer(self) -> torch.Tensor:
        """Where the next backward must write its gradient."""
        return self._bufs[self._slot]

    def current_lr(self) -> float:
        return self.lr if self.schedule is None else lr_at(self.schedule, self.local_clock)

    def step(self) -> None:
        """Mean of every rank's ``grad_buffer`` then ``x = K5(x, mean)`` (call on the
        compute stream after backward; every rank must call it the same number of times)."""
        s = self.sgd
        if self.comm is not None:
            # one fused pass (K7 mode 2): ring-order mean of every rank's gradient slot
            # (over NVLink) and the local step with it
            self.comm.fused_round(self._slot, self.x, self.x, self.current_lr(), m=self.m, momentum=s.momentum,
                                  dampening=s.dampening, weight_decay=s.weight_decay, nesterov=s.nesterov,
                                  first_step=self.local_clock == 0, mode=2, algo=self.algo,
                                  nonfinite=self._finite.counter, stream=self.compute)
            self.launches["fused_round"] += 1
            self._slot ^= 1
        else:
            K.sgd_step(self.x, self.grad_buffer, self.current_lr(), m=self.m, momentum=s.momentum,
                       dampening=s.dampening, weight_decay=s.weight_decay, nesterov=s.nesterov,
                       first_step=self.local_clock == 0, nonfinite=self._finite.counter, stream=self.compute)
            self.launches["sgd_step"] += 1
        self.local_clock += 1
        if self.flat is not None and self.comm is not None:
            self.flat.bind_grads(self.grad_buffer)

    def check_finite(self) -> None:
        self._finite.check(self.x.numel())


def plan_buckets(n: int, tensors, bucket_bytes: int, esize: int):
    """Gradient buckets of ``BucketedSGDARWorker``: contiguous ranges covering [0, n) from
    the END of the flat vector (backward produces the last layers' gradients first), at
    most ``bucket_bytes`` each, every boundary a 16-byte multiple (the kernels' pack
    alignment).  ``tensors`` = (offset, numel) of every parameter.  Returns (buckets as
    (lo, hi) in launch order, the buckets each tensor overlaps, the number of tensors each
    bucket waits for)."""
    wpack = max(1, 16 // esize)
    cap = max(wpack, bucket_bytes // esize // wpack * wpack)
    buckets = []
    hi = n
    while hi > 0:
        lo = max(0, hi - cap) // wpack * wpack
        buckets.append((lo, hi))
        hi = lo
    member, need = [], [0] * len(buckets)
    for off, cnt in tensors:
        end = off + cnt
        bs = [b for b, (lo, hi) in enumerate(buckets) if lo < end and off < hi]
        member.append(bs)
        for b in bs:
            need[b] += 1
    return buckets, member, need


class BucketedSGDARWorker:
    """SGD-AR (optimizer.py:214-242, ``sync_allreduce_sgd_round``) as a data-parallel
    trainer runs it: the gradient all-reduce is split into buckets in reverse parameter
    order and each bucket is reduced over NVLink — with the local step of its slice of x
    fused in — on a side stream as soon as backward has accumulated every gradient in it,
    so the exchange overlaps the rest of backward.  Only the last bucket's round is
    exposed.  The per-element summation order is the whole-vector ring order whatever the
    bucketing (lasgd_comm_sgd_ar_range), so x stays bit-identical to ``SGDARWorker`` and to
    the reference's round.

    Backward must write the gradients into the communicator's slots: the worker binds
    ``flat``'s ``.grad`` views to slot ``grad_buffer`` and rebinds them every step.  Use:
    ``flat.zero_grad(); loss.backward(); worker.step()`` on the compute stream, eagerly
    (the buckets launch from autograd hooks), one backward per ``step()``.  A parameter
    must receive exactly one gradient accumulation per backward (no weight sharing)."""

    def __init__(self, flat, comm, *, sgd: Optional[SgdConfig] = None, schedule: Optional[LrSchedule] = None,
                 lr: Optional[float] = None, bucket_bytes: int = 25 << 20,
                 compute_stream: Optional[torch.cuda.Stream] = None, side_stream: Optional[torch.cuda.Stream] = None,
                 nblocks: int = 0, algo: int = N.ALGO_AUTO):
        if (schedule is None) == (lr is None):
            raise ValueError("give exactly one of schedule / lr")
        if comm is None or comm.world < 2:
            raise ValueError("the bucketed SGD-AR worker needs a communicator with P >= 2")
        if comm.n != flat.numel or comm.dtype != flat.x.dtype:
            raise ValueError("communicator buffers do not match the flat parameters")
        if bucket_bytes <= 0:
            raise ValueError("bucket_bytes must be positive")
        if algo in (N.ALGO_PUSH, N.ALGO_CE):
            raise ValueError("bucketed SGD-AR rounds are one-shot or two-shot")
        self.sgd = sgd or SgdConfig()
        self.sgd.validate()
        self.flat, self.comm = flat, comm
        self.x = flat.x
        self.schedule, self.lr = schedule, lr
        self.compute = compute_stream if compute_stream is not None else torch.cuda.current_stream(flat.x.device)
        self.side = side_stream if side_stream is not None else comm.stream
        self.nblocks = nblocks
        self.algo = algo
        self.m = torch.empty_like(flat.x) if self.sgd.momentum != 0 else None
        self._finite = _FiniteMonitor(flat.x.device)
        self.local_clock = 0
        self.launches = collections.Counter()
        self._slot = 0
        self.buckets, self._param_buckets, self._need = plan_buckets(
            flat.numel, [(off, p.numel()) for p, off in zip(flat.params, flat.offsets)], bucket_bytes,
            flat.x.element_size())
        self._hooks = [p.register_post_accumulate_grad_hook(self._make_hook(i)) for i, p in enumerate(flat.params)]
        self._reset_step()
        flat.bind_grads(self.grad_buffer)

    @property
    def grad_buffer(self) -> torch.Tensor:
        """Where the next backward must write its gradient."""
        return self.comm.snapshots[self._slot]

    def current_lr(self) -> float:
        return self.lr if self.schedule is None else lr_at(self.schedule, self.local_clock)

    def _reset_step(self) -> None:
        self._pending = list(self._need)
        self._ready = set(b for b, k in enumerate(self._pending) if k == 0)
        self._next = 0
        self._step_lr = None

    def _make_hook(self, i):
        def hook(_p):
            for b in self._param_buckets[i]:
                self._pending[b] -= 1
                if self._pending[b] == 0:
                    self._ready.add(b)
            self._launch_ready()
        return hook

    def _launch(self, b: int) -> None:
        if self._step_lr is None:
            self._step_lr = self.current_lr()
        lo, hi = self.buckets[b]
        ev = torch.cuda.Event()
        ev.record(self.compute)  # every gradient of the bucket has been accumulated on it
        self.side.wait_event(ev)
        s = self.sgd
        self.comm.sgd_ar_range(self._slot, lo, hi - lo, self.x, self._step_lr, m=self.m, momentum=s.momentum,
                               dampening=s.dampening, weight_decay=s.weight_decay, nesterov=s.nesterov,
                               first_step=self.local_clock == 0, algo=self.algo, nblocks=self.nblocks,
                               nonfinite=self._finite.counter, stream=self.side)
        self.launches["sgd_ar_bucket"] += 1

    def _launch_ready(self) -> None:
        # strictly in bucket order: every rank issues the same launch sequence
        while self._next < len(self.buckets) and self._next in self._ready:
            self._launch(self._next)
            self._next += 1

    def step(self) -> None:
        """Close the step (call on the compute stream after backward): launch whatever
        bucket backward did not complete, order the compute stream after every bucket's
        round (x is updated there) and move the gradients to the other slot."""
        self._ready.update(range(len(self.buckets)))
        self._launch_ready()
        self.compute.wait_stream(self.side)
        self.local_clock += 1
        self._slot ^= 1
        self._reset_step()
        self.flat.bind_grads(self.grad_buffer)

    def check_finite(self) -> None:
        self._finite.check(self.x.numel())

    def close(self) -> None:
        for h in getattr(self, "_hooks", ()):
            h.remove()
        self._hooks = []

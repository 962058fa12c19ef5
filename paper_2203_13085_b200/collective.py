"""Mean all-reduce transports with non-blocking handles (mirror of
/root/reference/pkg/src/lasgd/collective.py).

Two transports keep the reference's duck type (``submit(round_id, rank,
contribution) -> CollectiveHandle`` and ``all_reduce(contributions, round_id)``,
collective.py:248-268):

* ``CudaLoopbackTransport`` — all P ranks' contributions on ONE device (the
  GPU analogue of ``LoopbackTransport``, collective.py:229-287): the round's
  mean kernel launches when the last contribution arrives.
* ``CudaP2PTransport`` — one process per GPU; the contribution is this rank's
  snapshot in IPC-mapped memory and the mean is computed by the NVLink P2P
  kernel (one-shot / two-shot) on a low-priority side stream.

Handles are backed by CUDA completion state (an event for the loopback, a
host-mapped flag written by the kernel for P2P), so ``poll`` never blocks.
Results are bit-identical to ``execute_allreduce`` (ring order, /P after the
sum) — see tests/test_gpu_collective.py.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass
from enum import Enum
from typing import Optional

import torch

from . import _native as N
from . import kernels as K
from ._native import CollectiveFailure, DimensionMismatchError, TransportFault  # noqa: F401 (collective.py:22-27)
from .params import ChunkSpec, as_device_vector, partition_chunks


# ---------------------------------------------------------------- ring plan (host replica)
@dataclass(frozen=True)
class RingStep:
    send_chunk: int
    recv_chunk: int
    send_to: int
    recv_from: int
    phase: str


@dataclass(frozen=True)
class RingSchedule:
    num_ranks: int
    steps: tuple

    @property
    def num_steps(self) -> int:
        return len(self.steps)


def ring_schedule(num_ranks: int) -> RingSchedule:
    """collective.py:51-83.  Kept for byte accounting and for the fault-injection
    step numbering; the device kernels do not execute a ring (one NVSwitch hop
    reaches every peer) but reproduce its per-chunk summation order."""
    if num_ranks < 1:
        raise ValueError("num_ranks must be positive")
    P = num_ranks
    steps = []
    for s in range(P - 1):
        steps.append(tuple(RingStep((r - s) % P, (r - s - 1) % P, (r + 1) % P, (r - 1) % P, "reduce") for r in range(P)))
    for k in range(P - 1):
        steps.append(tuple(RingStep((r + 1 - k) % P, (r - k) % P, (r + 1) % P, (r - 1) % P, "gather") for r in range(P)))
    return RingSchedule(num_ranks=P, steps=tuple(steps))


def bytes_per_node(d: int, num_ranks: int, bytes_per_element: int, rank: Optional[int] = None) -> int:
    """collective.py:206-226 (C ABI replay of the schedule)."""
    if bytes_per_element < 1:
        raise ValueError("bytes_per_element must be positive")
    return int(N.lib().lasgd_bytes_per_node(d, num_ranks, bytes_per_element, -1 if rank is None else rank))


# ---------------------------------------------------------------- handles
class Status(Enum):
    IN_FLIGHT = "in_flight"
    COMPLETE = "complete"
    FAILED = "failed"


class CollectiveHandle:
    """collective.py:92-139: IN_FLIGHT -> COMPLETE | FAILED, exactly once.

    ``status`` polls the device completion state without blocking.  ``result``
    keeps the reference contract (raises while in flight / on failure);
    ``result_async(stream)`` is the overlap-friendly accessor: it orders
    ``stream`` after the collective and returns the mean without a host sync.
    """

    def __init__(self, round_id: int):
        self.round_id = round_id
        self._status = Status.IN_FLIGHT
        self._result: Optional[torch.Tensor] = None
        self._diagnostic: Optional[str] = None
        self.bytes_sent_per_node = 0

    # backend hooks
    def _probe(self) -> Status:
        return self._status

    def _order(self, stream) -> None:
        pass

    @property
    def status(self) -> Status:
        if self._status is Status.IN_FLIGHT:
            self._probe()
        return self._status

    @property
    def result(self) -> torch.Tensor:
        st = self.status
        if st is Status.FAILED:
            raise CollectiveFailure(self._diagnostic or "collective failed")
        if st is not Status.COMPLETE:
            raise RuntimeError(f"round {self.round_id} still in flight")
        return self._result

    def result_async(self, stream=None) -> torch.Tensor:
        if self._status is Status.FAILED or (self._status is Status.IN_FLIGHT and self._probe() is Status.FAILED):
            raise CollectiveFailure(self._diagnostic or "collective failed")
        self._order(stream if stream is not None else torch.cuda.current_stream())
        return self._result

    @property
    def diagnostic(self) -> Optional[str]:
        self.status
        return self._diagnostic

    def _complete(self, bytes_sent_per_node: Optional[int] = None) -> None:
        if self._status is not Status.IN_FLIGHT:
            raise RuntimeError("handle already resolved")
        if bytes_sent_per_node is not None:
            self.bytes_sent_per_node = bytes_sent_per_node
        self._status = Status.COMPLETE

    def _fail(self, diagnostic: str) -> None:
        if self._status is not Status.IN_FLIGHT:
            raise RuntimeError("handle already resolved")
        self._diagnostic = diagnostic
        self._status = Status.FAILED

    def wait(self, timeout: Optional[float] = None) -> bool:
        """collective.py:138-139: True once resolved (complete or failed)."""
        t0 = time.monotonic()
        while self.status is Status.IN_FLIGHT:
            if timeout is not None and time.monotonic() - t0 > timeout:
                return False
            time.sleep(20e-6)
        return True


def poll(handle: CollectiveHandle) -> Status:
    """collective.py:142-144: non-destructive status read."""
    return handle.status


class _EventHandle(CollectiveHandle):
    def __init__(self, round_id: int):
        super().__init__(round_id)
        self._event: Optional[torch.cuda.Event] = None
        self._nf_host: Optional[torch.Tensor] = None  # pinned copy of the mean's non-finite count

    @property
    def result(self) -> torch.Tensor:
        out = super().result
        # collective.py:201-202 checks the mean; the fused counter landed with the event
        bad = int(self._nf_host.item()) if self._nf_host is not None else 0
        if bad:
            raise N.NonFiniteError(f"all-reduce result: {bad} non-finite entries out of {out.numel()}")
        return out

    def _probe(self) -> Status:
        if self._status is Status.IN_FLIGHT and self._event is not None and self._event.query():
            self._complete()
        return self._status

    def _order(self, stream) -> None:
        if self._event is not None:
            stream.wait_event(self._event)


# ---------------------------------------------------------------- single-device transport
class CudaLoopbackTransport:
    """collective.py:229-287 on one GPU: contributions accumulate per round and the
    mean kernel launches on the last submit (stream-ordered after every
    contribution).  ``fault_at=(round, step)`` reproduces the reference's injected
    ``TransportFault`` (the handle fails with the same diagnostic)."""

    def __init__(self, num_ranks: int, fault_at: Optional[tuple] = None, algo: int = N.ALGO_AUTO,
                 dtype: torch.dtype = torch.float32, device=None):
        if num_ranks < 1:
            raise ValueError("num_ranks must be positive")
        if num_ranks > N.MAX_RANKS:
            raise ValueError(f"num_ranks {num_ranks} > {N.MAX_RANKS}")
        self.num_ranks = num_ranks
        self.fault_at = fault_at
        self.algo = algo
        self.dtype = dtype
        self.device = device
        self.bytes_sent = [0] * num_ranks
        self.peak_step_bytes = 0
        self._pending: dict = {}
        self._handles: dict = {}
        self._done: set = set()  # completed rounds (the reference retains their handles forever)

    def submit(self, round_id: int, rank: int, contribution) -> CollectiveHandle:
        if round_id in self._done:
            raise KeyError(round_id)  # late contribution to a completed round, collective.py:254
        handle = self._handles.get(round_id)
        if handle is None:
            handle = _EventHandle(round_id)
            self._handles[round_id] = handle
            self._pending[round_id] = [None] * self.num_ranks
        slot = self._pending[round_id]  # KeyError after completion, like collective.py:254
        if slot[rank] is not None:
            raise RuntimeError(f"rank {rank} already contributed to round {round_id}")
        slot[rank] = as_device_vector(contribution, self.dtype, self.device)
        if all(v is not None for v in slot):
            self._run_round(round_id, slot, handle)
        return handle

    def all_reduce(self, contributions, round_id: int = 0) -> CollectiveHandle:
        if len(contributions) != self.num_ranks:
            raise ValueError(f"expected {self.num_ranks} contributions, got {len(contributions)}")
        handle = None
        for rank, vec in enumerate(contributions):
            handle = self.submit(round_id, rank, vec)
        return handle

    def _run_round(self, round_id: int, vectors: list, handle: _EventHandle) -> None:
        P = self.num_ranks
        d = vectors[0].numel()
        for v in vectors:
            if v.numel() != d:
                raise DimensionMismatchError(f"contribution dims differ: {v.numel()} vs {d}")
        if self.fault_at is not None and self.fault_at[0] == round_id and 0 <= self.fault_at[1] < 2 * (P - 1):
            handle._fail(f"injected fault in round {round_id} at ring step {self.fault_at[1]}")
            return
        if P == 1:
            handle._result = vectors[0]  # collective.py:174-175: input unchanged
        else:
            out = torch.empty_like(vectors[0])
            nf = torch.zeros(1, dtype=torch.int64, device=out.device)
            K.mean_virtual([out], vectors, algo=N.ALGO_ONESHOT if self.algo == N.ALGO_AUTO else self.algo,
                           nonfinite=nf)
            handle._result = out
            handle._nf_host = torch.empty(1, dtype=torch.int64, pin_memory=True)
            handle._nf_host.copy_(nf, non_blocking=True)
        handle._event = torch.cuda.Event()
        handle._event.record()
        bpe = vectors[0].element_size()
        for r in range(P):
            self.bytes_sent[r] += bytes_per_node(d, P, bpe, rank=r) if P > 1 else 0
        if P > 1:
            self.peak_step_bytes = max(self.peak_step_bytes, partition_chunks(d, P).max_size * bpe)
        handle.bytes_sent_per_node = bytes_per_node(d, P, bpe) if P > 1 else 0
        del self._pending[round_id]
        del self._handles[round_id]
        self._done.add(round_id)


@dataclass
class AllReduceOutcome:
    """collective.py:147-151."""

    per_rank: list  # mean vector per rank (device tensors), bit-identical
    bytes_sent: list  # exact bytes each rank's ring schedule transmits
    peak_step_bytes: int  # largest single-step payload any rank sends


def execute_allreduce(vectors, chunks: Optional[ChunkSpec] = None, schedule: Optional[RingSchedule] = None,
                      on_step=None) -> AllReduceOutcome:
    """collective.py:154-203 on the device: the ring-order mean of P contributions held
    on one GPU, computed by the one-shot mean kernel (K2 over virtual ranks), which
    writes the P bit-identical per-rank results in one launch.

    Byte accounting is the exact replay of the ring schedule (``bytes_sent``,
    ``peak_step_bytes``).  ``on_step(step_index, step_bytes)`` is called for every step
    with the reference's payload sizes, in step order, BEFORE the kernel runs: a
    ``TransportFault`` raised there aborts the collective with no result, as in the
    reference.  f64 inputs compute in f64 (bit-exact with the reference), others in
    f32.  Only the default partition and schedule are supported (the kernels implement
    exactly that order); anything else raises ``NotImplementedError``."""
    from .params import vector_dtype

    vectors = list(vectors)
    P = len(vectors)
    if P == 0:
        raise ValueError("need at least one contribution")
    dt = vector_dtype(vectors[0])
    vs = [as_device_vector(v, dtype=dt) for v in vectors]
    d = vs[0].numel()
    for v in vs:
        if v.numel() != d:
            raise DimensionMismatchError(f"contribution dims differ: {v.numel()} vs {d}")
    if P == 1:
        return AllReduceOutcome(per_rank=[vs[0]], bytes_sent=[0], peak_step_bytes=0)
    default_chunks = partition_chunks(d, P)
    if chunks is not None and tuple(map(tuple, chunks.bounds)) != tuple(map(tuple, default_chunks.bounds)):
        raise NotImplementedError("the device ring mean implements the default partition_chunks(d, P) only")
    if schedule is not None and schedule != ring_schedule(P):
        raise NotImplementedError("the device ring mean implements the default ring_schedule(P) only")
    bpe = vs[0].element_size()
    sizes = [default_chunks.size(c) * bpe for c in range(P)]
    peak = 0
    for step_index, step in enumerate(ring_schedule(P).steps):
        step_bytes = [0] * P
        for entry in step:  # rank entry.recv_from sends chunk entry.recv_chunk
            step_bytes[entry.recv_from] = sizes[entry.recv_chunk]
        peak = max(peak, max(step_bytes))
        if on_step is not None:
            on_step(step_index, step_bytes)
    outs = [torch.empty_like(vs[0]) for _ in range(P)]
    nf = torch.zeros(1, dtype=torch.int64, device=vs[0].device)
    K.mean_virtual(outs, vs, algo=N.ALGO_ONESHOT, nonfinite=nf)
    bad = int(nf.item())
    if bad:
        raise N.NonFiniteError(f"all-reduce result: {bad} non-finite entries out of {d * P}")
    return AllReduceOutcome(per_rank=outs, bytes_sent=[bytes_per_node(d, P, bpe, r) for r in range(P)],
                            peak_step_bytes=peak)


def all_reduce_average(contributions, transport=None, round_id: int = 0) -> CollectiveHandle:
    """collective.py:290-294."""
    if transport is None:
        transport = CudaLoopbackTransport(len(contributions))
    return transport.all_reduce(contributions, round_id=round_id)


# ---------------------------------------------------------------- multi-GPU (NVLink P2P)
class _CudaBuf:
    """Minimal __cuda_array_interface__ exporter so comm-owned memory becomes a torch view."""

    def __init__(self, ptr: int, n: int, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 2,
                                         "strides": None}
        self._owner = owner


def exchange_handles(mine: bytes, world: int, group=None) -> bytes:
    """All-gather every rank's fixed-size IPC handle, concatenated in rank order
    (the layout lasgd_comm_open expects).  Works over any torch.distributed backend."""
    import torch.distributed as dist

    if len(mine) != N.IPC_HANDLE_BYTES:
        raise ValueError(f"IPC handle must be {N.IPC_HANDLE_BYTES} bytes, got {len(mine)}")
    if world == 1:
        return mine
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    for r, h in enumerate(gathered):
        if not isinstance(h, bytes) or len(h) != N.IPC_HANDLE_BYTES:
            raise RuntimeError(f"rank {r} sent a malformed IPC handle")
    return b"".join(gathered)


def share_fd(fd: Optional[int], rank: int, world: int, group=None) -> int:
    """Pass a file descriptor from rank 0 to every other rank of this node (SCM_RIGHTS
    over an abstract-namespace UNIX socket whose name rank 0 broadcasts).  Returns the
    descriptor valid in this process."""
    import secrets
    import socket
    import time

    import torch.distributed as dist

    import os
    import struct

    name = [f"\0lasgd-nvls-{secrets.token_hex(8)}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0, group=group)
    pids = [None] * world
    dist.all_gather_object(pids, os.getpid(), group=group)
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name[0])
        srv.listen(world)
        dist.barrier(group=group)
        try:
            served = 0
            while served < world - 1:
                conn, _ = srv.accept()
                with conn:
                    # hand the descriptor only to this job's ranks (the socket name is
                    # visible to every process on the node)
                    pid, _, _ = struct.unpack("3i", conn.getsockopt(socket.SOL_SOCKET, socket.SO_PEERCRED,
                                                                    struct.calcsize("3i")))
                    if pid not in pids[1:]:
                        continue
                    socket.send_fds(conn, [b"f"], [fd])
                    served += 1
        finally:
            srv.close()
        return fd
    dist.barrier(group=group)
    deadline = time.monotonic() + 60.0
    while True:
        cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        try:
            cli.connect(name[0])
            break
        except OSError:
            cli.close()
            if time.monotonic() > deadline:
                raise
            time.sleep(0.01)
    with cli:
        _, fds, _, _ = socket.recv_fds(cli, 16, 1)
    if not fds:
        raise RuntimeError("no file descriptor received from rank 0")
    return fds[0]


class P2PCommunicator:
    """One rank's endpoint of the NVLink P2P mean all-reduce (K2/K3/K6).

    Owns an IPC-exportable region (signal pads, two snapshot slots, the mean
    buffer) and maps every peer's region.  Handles are exchanged once at
    construction through ``torch.distributed`` (any backend; gloo works).
    All ranks must issue the same sequence of ``allreduce`` calls.

    ``nvls=True`` (fp32, P >= 2): the snapshot slots and the mean buffer move into a
    multicast-bound allocation and ``allreduce`` reduces inside the NVSwitch
    (``ALGO_NVLS``, tolerance mode: within rounding of the ring-order mean, identical
    bits on every rank); fused rounds are then unavailable (use the overlap pipeline).
    """

    def __init__(self, n: int, *, dtype: torch.dtype = torch.float32, rank: Optional[int] = None,
                 world: Optional[int] = None, device=None, group=None, nblocks: int = 96, threads: int = 256,
                 timeout_s: float = 30.0, fault_seq: int = -1, fault_phase: int = 0, stream_priority: int = 0,
                 nvls: bool = False):
        import torch.distributed as dist

        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.rank, self.world, self.n, self.dtype = rank, world, n, dtype
        self._code = K.dtype_code(torch.empty(0, dtype=dtype))
        cfg = N.CommConfig(nblocks, threads, timeout_s, fault_seq, fault_phase)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib().lasgd_comm_create(rank, world, self.device.index, n, self._code, ctypes.byref(cfg),
                                              ctypes.byref(h)), "lasgd_comm_create")
        self._h = h
        buf = ctypes.create_string_buffer(N.IPC_HANDLE_BYTES)
        N.check(N.lib().lasgd_comm_ipc_handle(self._h, buf), "lasgd_comm_ipc_handle")
        mine = bytes(buf.raw)
        if world > 1:
            allh = exchange_handles(mine, world, group)
            N.check(N.lib().lasgd_comm_open(self._h, allh), "lasgd_comm_open")
        self.nvls = bool(nvls)
        if self.nvls:
            self._setup_nvls(group)
        typestr = "<f4" if dtype == torch.float32 else "<f8"
        self.snapshots = []
        for which in (0, 1):
            p = ctypes.c_void_p()
            N.check(N.lib().lasgd_comm_buffer(self._h, which, ctypes.byref(p)))
            self.snapshots.append(torch.as_tensor(_CudaBuf(p.value, n, typestr, self), device=self.device))
        p = ctypes.c_void_p()
        N.check(N.lib().lasgd_comm_buffer(self._h, 2, ctypes.byref(p)))
        self.xbar = torch.as_tensor(_CudaBuf(p.value, n, typestr, self), device=self.device)
        self.stream = torch.cuda.Stream(device=self.device, priority=stream_priority)
        if world > 1 and dist.is_initialized():
            dist.barrier(group=group)

    def _setup_nvls(self, group) -> None:
        import torch.distributed as dist

        if self.world < 2 or not dist.is_initialized():
            raise ValueError("NVLS needs P >= 2 ranks under torch.distributed")
        ok = [bool(N.lib().lasgd_comm_nvls_supported(self._h))]
        oks = [None] * self.world
        dist.all_gather_object(oks, ok[0], group=group)
        if not all(oks):
            raise ValueError("NVLink SHARP multicast is not supported on every rank's device")
        with torch.cuda.device(self.device):
            fd = ctypes.c_int(-1)
            if self.rank == 0:
                N.check(N.lib().lasgd_comm_nvls_create(self._h, ctypes.byref(fd)), "lasgd_comm_nvls_create")
            got = share_fd(fd.value if self.rank == 0 else None, self.rank, self.world, group)
            if self.rank != 0:
                N.check(N.lib().lasgd_comm_nvls_import(self._h, got), "lasgd_comm_nvls_import")
            N.check(N.lib().lasgd_comm_nvls_add_device(self._h), "lasgd_comm_nvls_add_device")
            dist.barrier(group=group)  # every device added before anyone binds
            N.check(N.lib().lasgd_comm_nvls_bind(self._h), "lasgd_comm_nvls_bind")
            if self.rank == 0:
                import os

                os.close(fd.value)
        dist.barrier(group=group)

    def slot_of(self, t: torch.Tensor) -> Optional[int]:
        for i, s in enumerate(self.snapshots):
            if t.data_ptr() == s.data_ptr() and t.numel() == s.numel():
                return i
        return None

    def allreduce(self, slot: int, algo: int = N.ALGO_AUTO, stream=None) -> int:
        """Launch the mean of snapshot slot ``slot`` over all ranks into ``self.xbar``
        on ``stream`` (default: the communicator's low-priority side stream).  ``algo``:
        ``ALGO_ONESHOT`` / ``ALGO_TWOSHOT`` (SM loads), ``ALGO_PUSH`` (NVLink stores),
        ``ALGO_CE`` (copy engines) — all the ring order of collective.py:154-203, bit for
        bit — or ``ALGO_NVLS`` on an NVLS communicator; ``ALGO_AUTO`` picks by world size
        and buffer size (``resolve_algo``).  Returns the launch's sequence number."""
        s = stream if stream is not None else self.stream
        seq = ctypes.c_ulonglong()
        N.check(N.lib().lasgd_comm_allreduce(self._h, slot, algo, ctypes.c_void_p(s.cuda_stream), ctypes.byref(seq)),
                "lasgd_comm_allreduce")
        return seq.value

    def fused_round(self, slot: int, x: torch.Tensor, g: torch.Tensor, lr: float, *, m=None, delta=None,
                    momentum=0.0, dampening=0.0, weight_decay=0.0, nesterov=False, first_step=False,
                    delta_reset=False, alpha: float = 1.0, mode: int = 0, algo: int = N.ALGO_AUTO, nblocks: int = 0,
                    nonfinite=None, stream=None) -> int:
        """One fused round on ``stream`` (default: the current stream): local step + mean of
        snapshot slot ``slot`` over all ranks (NVLink) + pull (mode 0) / finalize (mode 1)
        + write snapshot slot ``1 - slot`` — K7, or the K8 push round for ``ALGO_PUSH``
        (what AUTO picks for large buffers).  Mode 2 = one SGD-AR round: the slots hold
        gradients and x takes the local step with their mean (K7 one-/two-shot only)."""
        K._check(x, g, m, delta, self.snapshots[0])
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        p = K.sgd_params(lr, momentum, dampening, weight_decay, nesterov, first_step, delta_reset)
        seq = ctypes.c_ulonglong()
        N.check(N.lib().lasgd_comm_fused_round(self._h, slot, int(algo), K._ptr(x), K._ptr(g), K._ptr(m), K._ptr(delta),
                                               ctypes.byref(p), float(alpha), int(mode), int(nblocks),
                                               K._ptr(nonfinite), ctypes.c_void_p(s.cuda_stream), ctypes.byref(seq)),
                "lasgd_comm_fused_round")
        return seq.value

    def sgd_ar_range(self, slot: int, off: int, length: int, x: torch.Tensor, lr: float, *, m=None, momentum=0.0,
                     dampening=0.0, weight_decay=0.0, nesterov=False, first_step=False, algo: int = N.ALGO_AUTO,
                     nblocks: int = 0, nonfinite=None, stream=None) -> int:
        """One bucket of a bucketed SGD-AR step (optimizer.py:214-242): the ring-order
        mean over all ranks of gradient slot ``slot`` on elements [off, off + length), and
        the local step of ``x`` (and ``m``) there — bit-identical to the whole-vector round
        for any bucketing."""
        K._check(x, m, self.snapshots[0])
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        p = K.sgd_params(lr, momentum, dampening, weight_decay, nesterov, first_step)
        seq = ctypes.c_ulonglong()
        N.check(N.lib().lasgd_comm_sgd_ar_range(self._h, slot, int(off), int(length), int(algo), K._ptr(x), K._ptr(m),
                                                ctypes.byref(p), int(nblocks), K._ptr(nonfinite),
                                                ctypes.c_void_p(s.cuda_stream), ctypes.byref(seq)),
                "lasgd_comm_sgd_ar_range")
        return seq.value

    def launches(self) -> int:
        """Sequence number of this rank's latest launch."""
        v = ctypes.c_ulonglong()
        N.check(N.lib().lasgd_comm_launches(self._h, ctypes.byref(v)))
        return v.value

    def peer_max_seq(self) -> int:
        """Highest launch any peer has started (from its entry flags in our pad)."""
        v = ctypes.c_ulonglong()
        N.check(N.lib().lasgd_comm_peer_max_seq(self._h, ctypes.byref(v)), "peer_max_seq")
        return v.value

    def query(self, seq: int) -> int:
        return N.check(N.lib().lasgd_comm_query(self._h, seq), "all-reduce")

    def stream_wait(self, seq: int, stream) -> None:
        N.check(N.lib().lasgd_comm_stream_wait(self._h, seq, ctypes.c_void_p(stream.cuda_stream)))

    def wait(self, seq: int, timeout_s: float = -1.0) -> int:
        return N.check(N.lib().lasgd_comm_wait(self._h, seq, timeout_s), "all-reduce")

    def diagnostic(self) -> str:
        buf = ctypes.create_string_buffer(256)
        N.lib().lasgd_comm_diagnostic(self._h, buf, 256)
        return buf.value.decode()

    def resolve_algo(self, algo: int = N.ALGO_AUTO) -> int:
        return N.lib().lasgd_comm_resolve_algo(self._h, algo)

    def resolve_fused_algo(self, algo: int = N.ALGO_AUTO) -> int:
        """Algorithm fused_round runs for `algo` (AUTO -> one-shot or push)."""
        return N.lib().lasgd_comm_resolve_fused_algo(self._h, algo)

    def set_nblocks(self, nblocks: int) -> None:
        """SM budget of later launches (collective: every rank must call it identically)."""
        N.check(N.lib().lasgd_comm_set_nblocks(self._h, int(nblocks)), "set_nblocks")

    def set_trace(self, on: bool) -> None:
        N.check(N.lib().lasgd_comm_set_trace(self._h, int(bool(on))))

    def invalidate_staging(self) -> None:
        """Call after writing a snapshot slot outside the fused rounds (e.g. loading a
        checkpoint into it): the next round re-stages / re-enters through the per-CTA
        barrier instead of trusting the previous round's end-of-round signals."""
        N.check(N.lib().lasgd_comm_invalidate_staging(self._h))

    def set_gate(self, on: bool) -> None:
        """Gate every all-reduce behind a one-warp wait for all peers (collective setting)."""
        N.check(N.lib().lasgd_comm_set_gate(self._h, int(bool(on))))

    def device_barrier(self, stream=None) -> None:
        """Stream-ordered barrier across the ranks (one warp; no launch sequence number, so
        the round chain and push staging are untouched).  Collective."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        N.check(N.lib().lasgd_comm_barrier(self._h, ctypes.c_void_p(s.cuda_stream)), "lasgd_comm_barrier")

    def peers_ahead(self, seq: int) -> bool:
        """True if some peer already entered a launch later than ``seq``."""
        return bool(N.check(N.lib().lasgd_comm_peers_ahead(self._h, seq)))

    def read_trace(self):
        """Per-CTA globaltimer stamps (ns) of the last traced launch: list of
        (start, entry_passed, mid_passed, end); synchronises the device."""
        buf = (ctypes.c_ulonglong * (N.MAX_BLOCKS * 4))()
        nb = N.check(N.lib().lasgd_comm_read_trace(self._h, buf, N.MAX_BLOCKS), "read_trace")
        return [tuple(buf[4 * b + k] for k in range(4)) for b in range(nb)]

    def bytes_per_node(self, algo: int = N.ALGO_AUTO) -> int:
        return int(N.lib().lasgd_comm_bytes_per_node(self._h, algo))

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().lasgd_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _P2PHandle(CollectiveHandle):
    def __init__(self, round_id: int, comm: P2PCommunicator, seq: int):
        super().__init__(round_id)
        self._comm, self._seq = comm, seq
        self._result = comm.xbar
        self.bytes_sent_per_node = comm.bytes_per_node()

    def _probe(self) -> Status:
        if self._status is Status.IN_FLIGHT:
            try:
                if self._comm.query(self._seq) == 1:
                    self._complete()
            except CollectiveFailure as e:
                self._fail(str(e))
        return self._status

    def _order(self, stream) -> None:
        self._comm.stream_wait(self._seq, stream)


class CudaP2PTransport:
    """Per-process transport over a ``P2PCommunicator`` (same duck type as
    LoopbackTransport).  ``submit`` accepts this rank's contribution only; if it
    is not already one of the communicator's snapshot slots it is copied (K1)
    into the next slot.  The launch is ordered after the submitting stream and
    runs on the communicator's side stream.  One outstanding collective per node
    (SPEC collective "Single outstanding collective"): a handle's result is the
    shared mean buffer, valid until the next launch."""

    def __init__(self, comm: P2PCommunicator, algo: int = N.ALGO_AUTO):
        self.comm = comm
        self.num_ranks = comm.world
        self.algo = algo
        self._next_slot = 0
        self.bytes_sent = [0] * comm.world
        self.launches = 0

    def submit(self, round_id: int, rank: int, contribution) -> CollectiveHandle:
        if rank != self.comm.rank:
            raise ValueError(f"this process is rank {self.comm.rank}; cannot submit for rank {rank}")
        cur = torch.cuda.current_stream(self.comm.device)
        t = contribution if isinstance(contribution, torch.Tensor) else as_device_vector(contribution, self.comm.dtype,
                                                                                         self.comm.device)
        if t.numel() != self.comm.n:
            raise DimensionMismatchError(f"contribution dims differ: {t.numel()} vs {self.comm.n}")
        slot = self.comm.slot_of(t)
        if slot is None:
            slot = self._next_slot
            K.snapshot(self.comm.snapshots[slot], t.reshape(-1), stream=cur)
        self._next_slot = 1 - slot
        self.comm.stream.wait_stream(cur)
        seq = self.comm.allreduce(slot, self.algo)
        self.launches += 1
        h = _P2PHandle(round_id, self.comm, seq)
        self.bytes_sent[rank] += h.bytes_sent_per_node
        return h

    def all_reduce(self, contributions, round_id: int = 0) -> CollectiveHandle:
        if len(contributions) == self.num_ranks:
            contributions = [contributions[self.comm.rank]]
        if len(contributions) != 1:
            raise ValueError("a per-process transport takes this rank's contribution (or all ranks' list)")
        return self.submit(round_id, self.comm.rank, contributions[0])

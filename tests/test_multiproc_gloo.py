"""N > 1 host-side logic on CPU (world_size 2, gloo): the IPC-handle exchange the P2P
communicator performs at start-up, and the per-rank decomposition of the round
protocol (each rank steps locally, one exchange per round) reproducing the
reference's in-process loop bit for bit."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    return dist


def _w_exchange(rank, world, port):
    dist = _init(rank, world, port)
    from paper_2203_13085_b200.collective import exchange_handles

    mine = bytes([rank + 1]) * 64
    allh = exchange_handles(mine, world)
    assert allh == b"".join(bytes([r + 1]) * 64 for r in range(world))
    try:
        exchange_handles(b"short", world)
        raise AssertionError("expected ValueError")
    except ValueError:
        pass
    dist.destroy_process_group()


def _w_protocol(rank, world, port, out_dir):
    dist = _init(rank, world, port)
    import torch

    from oracle import lasgd_oracle as O

    n, steps, k, alpha = 1001, 7, 2, 0.5
    rng = np.random.default_rng(3)
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = rng.standard_normal((steps, world, n)).astype(np.float32)
    x = x0.copy()
    snap = x0.copy()

    def mean_of_snapshots(s):
        parts = [torch.zeros(n) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(s))
        return O.ring_mean([p.numpy() for p in parts])

    z = mean_of_snapshots(snap)
    tau = 0
    for t in range(steps):
        x = O.sgd_step_plain(x, grads[t, rank], 0.05)
        tau += 1
        if tau == k:
            x = O.elastic_pull(x, snap, z, alpha)
            snap = x.copy()
            z = mean_of_snapshots(snap)
            tau = 0
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    dist.destroy_process_group()


def test_ipc_handle_exchange_gloo():
    mp.spawn(_w_exchange, args=(2, _port()), nprocs=2, join=True)


def test_per_rank_protocol_matches_in_process_reference(tmp_path):
    from oracle import lasgd_oracle as O

    mp.spawn(_w_protocol, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    rng = np.random.default_rng(3)
    x0 = rng.standard_normal(1001).astype(np.float32)
    grads = rng.standard_normal((7, 2, 1001)).astype(np.float32)
    xs, _, _, _ = O.run_lasgd_pull(x0, grads, [0.05] * 7, 2, 2, 0.5)
    for r in range(2):
        got = np.load(tmp_path / f"x{r}.npy")
        assert np.array_equal(got.view(np.uint32), xs[r].view(np.uint32))


def _w_share_fd(rank, world, port):
    """The NVLS set-up's descriptor hand-off: rank 0's file descriptor reaches every other
    rank (SCM_RIGHTS over the abstract UNIX socket, peers checked by SO_PEERCRED)."""
    import tempfile

    dist = _init(rank, world, port)
    from paper_2203_13085_b200.collective import share_fd

    fd = None
    if rank == 0:
        f = tempfile.TemporaryFile()
        f.write(b"multicast handle stand-in")
        f.flush()
        fd = os.dup(f.fileno())
    got = share_fd(fd, rank, world)
    # the descriptors share one open file description (one offset): read positionally
    assert os.pread(got, 64, 0) == b"multicast handle stand-in"
    if rank != 0:
        assert got != fd
    os.close(got)
    dist.destroy_process_group()


def test_share_fd_reaches_every_rank():
    mp.spawn(_w_share_fd, args=(3, _port()), nprocs=3, join=True)

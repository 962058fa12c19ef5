"""Multi-GPU parity of the NVLink P2P path (one process per GPU, IPC-mapped peers):
K2 one-shot / K3 two-shot bit-exact against the ring-order oracle on every rank,
the LASGDWorker round protocol (double-buffered snapshots, side stream) bit-exact
against the oracle's deterministic-k loop, and the watchdog turning a missing
peer flag into CollectiveFailure on every rank.  Skipped with < 2 GPUs."""

import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import torch.distributed as dist

    import os

    # LASGD_TEST_GPUS=k: rank r on GPU r % k, several ranks (processes, contexts) per GPU
    # (test_gpu_p2p_one_gpu.py: k = 1)
    torch.cuda.set_device(rank % int(os.environ.get("LASGD_TEST_GPUS", 1 << 30)))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


def _same_bits(a, b):
    iv = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return a.shape == b.shape and np.array_equal(a.view(iv), b.view(iv))


def _vec(seed, n, dtype=np.float32):
    return np.random.default_rng(seed).standard_normal(n).astype(dtype)


def _w_allreduce(rank, world, port):
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O
    from paper_2203_13085_b200 import _native as N

    _init(rank, world, port)
    for dtype in (torch.float32, torch.float64):
        npdt = np.float32 if dtype == torch.float32 else np.float64
        for n in (3, 1001, 65_537, 4_000_037):
            comm = L.P2PCommunicator(n, dtype=dtype, nblocks=24, timeout_s=20.0)
            ar = comm.resolve_algo(N.ALGO_AUTO)
            big = world == 2 and n * dtype.itemsize >= (32 << 20)
            assert comm.resolve_fused_algo(N.ALGO_AUTO) == (N.ALGO_PUSH if ar == N.ALGO_TWOSHOT or big else ar)
            assert comm.resolve_fused_algo(N.ALGO_TWOSHOT) == N.ALGO_TWOSHOT
            if world >= 3 and n * dtype.itemsize > (8 << 20):
                # the push mean where the two-shot would run, at the measured P = 3-4
                assert ar == (N.ALGO_PUSH if world <= 4 else N.ALGO_TWOSHOT)
            for rnd in range(4):
                for algo in (N.ALGO_ONESHOT, N.ALGO_TWOSHOT, N.ALGO_PUSH):
                    slot = rnd % 2
                    vecs = [_vec(1000 * rnd + 10 * r + algo + n, n, npdt) for r in range(world)]
                    comm.snapshots[slot].copy_(torch.from_numpy(vecs[rank]))
                    torch.cuda.synchronize()
                    seq = comm.allreduce(slot, algo)
                    assert comm.wait(seq, 30.0) == 1
                    torch.cuda.synchronize()
                    got = comm.xbar.cpu().numpy()
                    assert _same_bits(got, O.ring_mean(vecs)), (n, rnd, algo, rank)
            # gated launches (side-stream use): same results; peers_ahead sees later launches
            comm.set_gate(True)
            for rnd in range(2):
                vecs = [_vec(77 + 10 * r + rnd, n, npdt) for r in range(world)]
                comm.snapshots[rnd].copy_(torch.from_numpy(vecs[rank]))
                torch.cuda.synchronize()
                seq = comm.allreduce(rnd)
                assert comm.wait(seq, 30.0) == 1
                assert _same_bits(comm.xbar.cpu().numpy(), O.ring_mean(vecs)), (n, "gated", rank)
                dist.barrier()
            assert comm.peers_ahead(seq - 1) and not comm.peers_ahead(seq)
            comm.set_gate(False)
            dist.barrier()
            comm.close()
    dist.destroy_process_group()


def _w_worker_loop(rank, world, port):
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O

    _init(rank, world, port)
    n, steps = 100_003, 9
    x0 = _vec(7, n)
    grads = np.stack([np.stack([_vec(100 * t + r, n) for r in range(world)]) for t in range(steps)])
    mom = L.SgdConfig(0.9, 0.0, 1e-4, True)
    cases = [(2, 1.0, None, "overlap", 1), (1, 0.5, mom, "overlap", 2), (3, 0.25, None, "overlap", 1),
             (1, 1.0, mom, "fused", 1), (2, 0.5, None, "fused", 1), (1, 0.5, mom, "fused", 2), (3, 1.0, None, "fused", 2),
             (1, 0.5, mom, "fused", 3), (2, 1.0, None, "fused", 3)]
    for k, alpha, sgd, pipe, algo in cases:
        comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
        x = torch.from_numpy(x0.copy()).cuda()
        g = torch.empty_like(x)
        compute = torch.cuda.Stream(priority=-1)
        with torch.cuda.stream(compute):
            w = L.LASGDWorker(x, g, comm=comm, sync_period=k, alpha=alpha, sgd=sgd, lr=0.05, mode="pull",
                              compute_stream=compute, pipeline=pipe, algo=algo)
            for t in range(steps):
                g.copy_(torch.from_numpy(grads[t, rank]), non_blocking=False)
                w.step()
            w.drain()
        torch.cuda.synchronize()
        cfg = None if sgd is None else O.SgdConfig(0.05, sgd.momentum, sgd.dampening, sgd.weight_decay, sgd.nesterov)
        xs, _, _, _ = O.run_lasgd_pull(x0, grads, np.full(steps, 0.05), world, k, alpha, sgd=cfg)
        assert _same_bits(x.cpu().numpy(), xs[rank]), (k, alpha, pipe, algo, rank)
        dist.barrier()
        comm.close()
    # reference bookkeeping (delta mode) through the worker
    comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
    x = torch.from_numpy(x0.copy()).cuda()
    g = torch.empty_like(x)
    xs, _, _, _ = O.run_lasgd_delta(x0, grads, np.full(steps, 0.05), world, 2)
    for pipe, algo in (("overlap", 2), ("fused", 1), ("fused", 2), ("fused", 3)):
        x = torch.from_numpy(x0.copy()).cuda()
        w = L.LASGDWorker(x, g, comm=comm, sync_period=2, lr=0.05, mode="delta", pipeline=pipe, algo=algo)
        for t in range(steps):
            g.copy_(torch.from_numpy(grads[t, rank]))
            w.step()
        w.drain()
        torch.cuda.synchronize()
        assert _same_bits(x.cpu().numpy(), xs[rank]), pipe
        dist.barrier()
    # adaptive completion: ranks close rounds on their own clock (rank 1 is slowed down);
    # drain() must equalise the launch counts so every collective completes
    for tau_max in (1, 3):
        x = torch.from_numpy(x0.copy()).cuda()
        w = L.LASGDWorker(x, g, comm=comm, sync_period=tau_max, lr=0.05, mode="pull", adaptive=True,
                          tau_max=tau_max)
        for t in range(12):
            if rank == 1:
                torch.cuda._sleep(2_000_000)
            g.copy_(torch.from_numpy(grads[t % steps, rank]))
            w.step()
        w.drain()
        torch.cuda.synchronize()
        hist = dict(w.tau_hist)
        assert all(1 <= k <= tau_max for k in hist), hist
        assert np.isfinite(x.cpu().numpy()).all()
        dist.barrier()
    comm.close()
    dist.destroy_process_group()


def _w_sgd_ar(rank, world, port):
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O

    _init(rank, world, port)
    n, steps = 65_541, 7
    x0 = _vec(3, n)
    grads = np.stack([np.stack([_vec(500 * t + r, n) for r in range(world)]) for t in range(steps)])
    etas = np.array([0.1, 0.05, 0.2, 0.01, 0.07, 0.03, 0.11])
    for sgd in (None, L.SgdConfig(0.9, 0.0, 1e-4, True)):
        for algo in (1, 2):
            comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
            x = torch.from_numpy(x0.copy()).cuda()
            compute = torch.cuda.Stream()
            with torch.cuda.stream(compute):
                w = L.SGDARWorker(x, comm=comm, sgd=sgd, lr=1.0, algo=algo, compute_stream=compute)
                for t in range(steps):
                    w.lr = float(etas[t])
                    w.grad_buffer.copy_(torch.from_numpy(grads[t, rank]))
                    w.step()
            torch.cuda.synchronize()
            cfg = None if sgd is None else O.SgdConfig(1.0, sgd.momentum, sgd.dampening, sgd.weight_decay,
                                                       sgd.nesterov)
            ref, _ = O.run_sgd_ar(x0, grads, etas, world, sgd=cfg)
            assert _same_bits(x.cpu().numpy(), ref), (sgd, algo, rank)
            dist.barrier()
            comm.close()
    # gradients written by backward straight into the registered slots (FlatParams rebinding)
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(32, 16), torch.nn.Tanh(), torch.nn.Linear(16, 1)).cuda()
    flat = L.FlatParams(model)
    comm = L.P2PCommunicator(flat.numel, nblocks=8, timeout_s=20.0)
    w = L.SGDARWorker(flat.x, comm=comm, lr=0.05, flat=flat)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(10 + rank)
    for _ in range(5):
        flat.zero_grad()
        model(torch.randn(8, 32, device="cuda", generator=gen)).square().mean().backward()
        w.step()
    torch.cuda.synchronize()
    xs = [torch.empty_like(flat.x) for _ in range(world)]
    dist.all_gather_object(xs, flat.x.cpu())
    assert all(torch.equal(xs[0], v) for v in xs), "SGD-AR replicas diverged"
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


def _w_sgd_ar_bucketed(rank, world, port):
    """Bucketed SGD-AR (rounds over sub-ranges launched from autograd hooks): bit-exact
    against the oracle's SGD-AR loop (optimizer.py:214-242) for ragged buckets, and
    bit-identical to the one-launch SGDARWorker when backward drives the buckets."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O

    _init(rank, world, port)

    class _Flat:  # a flat vector with no module: gradients are written by hand
        def __init__(self, n):
            self.numel, self.n_params = n, n
            self.x = torch.empty(n, device="cuda")
            self.params, self.offsets = [], []

        def bind_grads(self, buf):
            self.g = buf

    n, steps = 65_541, 6
    x0 = _vec(3, n)
    grads = np.stack([np.stack([_vec(700 * t + r, n) for r in range(world)]) for t in range(steps)])
    etas = np.array([0.1, 0.05, 0.2, 0.01, 0.07, 0.03])
    from paper_2203_13085_b200 import _native as N

    for sgd, algo in ((None, N.ALGO_ONESHOT), (L.SgdConfig(0.9, 0.0, 1e-4, True), N.ALGO_ONESHOT),
                      (L.SgdConfig(0.9, 0.0, 1e-4, True), N.ALGO_TWOSHOT)):
        for bucket_bytes in (16_000, 65_536 * 4, 1 << 30):
            comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
            flat = _Flat(n)
            flat.x.copy_(torch.from_numpy(x0))
            compute = torch.cuda.Stream()
            with torch.cuda.stream(compute):
                w = L.BucketedSGDARWorker(flat, comm, sgd=sgd, lr=1.0, bucket_bytes=bucket_bytes,
                                          compute_stream=compute, algo=algo)
                for t in range(steps):
                    w.lr = float(etas[t])
                    w.grad_buffer.copy_(torch.from_numpy(grads[t, rank]))
                    w.step()
            torch.cuda.synchronize()
            cfg = None if sgd is None else O.SgdConfig(1.0, sgd.momentum, sgd.dampening, sgd.weight_decay,
                                                       sgd.nesterov)
            ref, _ = O.run_sgd_ar(x0, grads, etas, world, sgd=cfg)
            assert _same_bits(flat.x.cpu().numpy(), ref), (sgd, algo, bucket_bytes, rank)
            assert w.launches["sgd_ar_bucket"] == steps * len(w.buckets)
            w.close()
            dist.barrier()
            comm.close()

    # backward drives the buckets: same bits as the one-launch SGD-AR round
    def train(bucketed):
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.Tanh(), torch.nn.Linear(256, 256),
                                    torch.nn.Tanh(), torch.nn.Linear(256, 1)).cuda()
        flat = L.FlatParams(model, align_bytes=256)
        comm = L.P2PCommunicator(flat.numel, nblocks=8, timeout_s=20.0)
        compute = torch.cuda.Stream()
        sgd = L.SgdConfig(0.9, 0.0, 1e-4, True)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(10 + rank)
        with torch.cuda.stream(compute):
            if bucketed:
                w = L.BucketedSGDARWorker(flat, comm, sgd=sgd, lr=0.05, bucket_bytes=64 * 1024,
                                          compute_stream=compute)
                assert len(w.buckets) >= 3
            else:
                w = L.SGDARWorker(flat.x, comm=comm, sgd=sgd, lr=0.05, compute_stream=compute, flat=flat)
            for _ in range(5):
                flat.zero_grad()
                model(torch.randn(32, 64, device="cuda", generator=gen)).square().mean().backward()
                w.step()
        torch.cuda.synchronize()
        out = flat.x.cpu()
        if bucketed:
            w.close()
        dist.barrier()
        comm.close()
        return out

    a, b = train(True), train(False)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32)), rank
    xs = [None] * world
    dist.all_gather_object(xs, a)
    assert all(torch.equal(xs[0], v) for v in xs), "bucketed SGD-AR replicas diverged"
    dist.destroy_process_group()


def _w_graph_replay(rank, world, port):
    """Multi-rank graph replay (device round descriptor carries the launch sequence and
    the snapshot slot): fused rounds replayed from a CUDA graph — K8 push (mirror at P=2,
    staged at P>=3) and K7 one-shot — are bit-identical to the same steps issued one by
    one and to the oracle's deterministic loop, on every rank."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O
    from paper_2203_13085_b200 import _native as N

    _init(rank, world, port)
    n = 65_541
    x0 = _vec(5, n)
    gsrc = [[_vec(900 + 10 * i + r, n) for r in range(world)] for i in range(2)]
    sgd = L.SgdConfig(0.9, 0.0, 1e-4, True)
    for algo in (N.ALGO_PUSH, N.ALGO_ONESHOT):
        for k, alpha in ((1, 1.0), (2, 0.5)):
            pre, S, R, post = k, 4 * k, 3, k
            total = pre + S * R + post
            grads = [torch.from_numpy(gsrc[i][rank]).cuda() for i in range(2)]

            def run(graphed):
                comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
                x = torch.from_numpy(x0.copy()).cuda()
                compute = torch.cuda.Stream()
                with torch.cuda.stream(compute):
                    w = L.LASGDWorker(x, grads[0], comm=comm, sync_period=k, alpha=alpha, mode="pull", sgd=sgd,
                                      lr=0.05, algo=algo, pipeline="fused", compute_stream=compute)
                    t = 0
                    for _ in range(pre if graphed else total):
                        w.g = grads[t % 2]
                        w.step()
                        t += 1
                    if graphed:
                        graph = w.capture([grads[(pre + i) % 2] for i in range(S)])
                        for _ in range(R):
                            graph.replay()
                        t += S * R
                        for _ in range(post):
                            w.g = grads[t % 2]
                            w.step()
                            t += 1
                    w.drain()
                torch.cuda.synchronize()
                out = (x.cpu().numpy(), w.state.x_snapshot.cpu().numpy(), w.state.local_clock, w.state.global_clock,
                       comm.launches())
                w.close()
                dist.barrier()
                comm.close()
                return out

            a, b = run(True), run(False)
            assert a[2:4] == b[2:4] == (total, total // k), (a[2:], b[2:])
            if algo == N.ALGO_PUSH and k == 1:
                # a replay is refused once another launch moved the communicator, and
                # accepted again after one eager round
                comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
                x = torch.from_numpy(x0.copy()).cuda()
                compute = torch.cuda.Stream()
                with torch.cuda.stream(compute):
                    w = L.LASGDWorker(x, grads[0], comm=comm, sync_period=1, sgd=sgd, lr=0.05, algo=algo,
                                      pipeline="fused", compute_stream=compute)
                    w.step()
                    graph = w.capture(grads)
                    graph.replay()
                    comm.stream.wait_stream(compute)
                    comm.wait(comm.allreduce(w.state.snap_idx), 20.0)
                    compute.wait_stream(comm.stream)
                    with pytest.raises(RuntimeError, match="eager round"):
                        graph.replay()
                    w.g = grads[0]
                    w.step()
                    graph.replay()
                torch.cuda.synchronize()
                w.close()
                dist.barrier()
                comm.close()
            assert _same_bits(a[0], b[0]) and _same_bits(a[1], b[1]), (algo, k, rank)
            gl = np.stack([np.stack(gsrc[t % 2]) for t in range(total)])
            ref, _, _, _ = O.run_lasgd_pull(x0, gl, [0.05] * total, world, k, alpha,
                                            sgd=O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True))
            assert _same_bits(a[0], ref[rank]), (algo, k, rank)
    # >= 32 MB: the staged push round's pipelined halves (P >= 3) in graph form == eager
    nb = 9_000_001
    xb0 = _vec(6, nb)
    gb = [torch.from_numpy(_vec(950 + 10 * i + rank, nb)).cuda() for i in range(2)]

    def run_big(graphed):
        comm = L.P2PCommunicator(nb, timeout_s=30.0)
        x = torch.from_numpy(xb0.copy()).cuda()
        compute = torch.cuda.Stream()
        with torch.cuda.stream(compute):
            w = L.LASGDWorker(x, gb[0], comm=comm, sync_period=1, mode="pull", sgd=sgd, lr=0.05,
                              algo=N.ALGO_PUSH, pipeline="fused", compute_stream=compute)
            w.step()
            if graphed:
                graph = w.capture(gb)
                for _ in range(3):
                    graph.replay()
            else:
                for t in range(6):
                    w.g = gb[t % 2]
                    w.step()
            w.drain()
        torch.cuda.synchronize()
        out = x.cpu().numpy()
        w.close()
        dist.barrier()
        comm.close()
        return out

    assert _same_bits(run_big(True), run_big(False)), rank
    # the whole training step (zero_grad + forward + backward + fused round over NVLink)
    # captured into one CUDA graph per minibatch: the same bits as eager steps
    def train(graphed):
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.Tanh(), torch.nn.Linear(256, 8)).cuda()
        flat = L.FlatParams(model, align_bytes=256)
        comm = L.P2PCommunicator(flat.numel, nblocks=16, timeout_s=20.0)
        gen = torch.Generator(device="cuda").manual_seed(5 + rank)
        inp = torch.randn(32, 64, device="cuda", generator=gen)
        tgt = torch.randn(32, 8, device="cuda", generator=gen)
        compute = torch.cuda.Stream()
        w = L.LASGDWorker(flat.x, flat.g, comm=comm, sync_period=2, alpha=0.5, mode="pull", sgd=sgd, lr=0.05,
                          algo=N.ALGO_PUSH, pipeline="fused", compute_stream=compute)

        def fwd_bwd(t=0):
            flat.zero_grad()
            torch.nn.functional.mse_loss(model(inp), tgt).backward()

        with torch.cuda.stream(compute):
            for _ in range(4):  # eager warm-up rounds (also the staging of the push round)
                fwd_bwd()
                w.step()
            if graphed:
                g = w.capture_with(fwd_bwd, steps=2)
                for _ in range(4):
                    g.replay()
            else:
                for _ in range(8):
                    fwd_bwd()
                    w.step()
        torch.cuda.synchronize()
        out = flat.x.cpu()
        w.close()
        dist.barrier()
        comm.close()
        return out

    a, b = train(True), train(False)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32)), rank
    dist.destroy_process_group()


def _w_nvls(rank, world, port):
    """NVLink SHARP mean (tolerance mode): within 1e-6 of the ring-order mean relative to
    the contributions' magnitude (the north star's reduction-order tolerance), the same bits
    on every rank, and the overlap pipeline on it within rounding of the oracle's loop."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O
    from paper_2203_13085_b200 import _native as N

    _init(rank, world, port)
    try:
        probe = L.P2PCommunicator(1024, nvls=True, timeout_s=20.0)
    except ValueError as e:  # no multicast on this box: nothing to check
        print(f"rank {rank}: NVLS unavailable ({e})")
        dist.destroy_process_group()
        return
    probe.close()
    for n in (3, 1001, 65_537, 4_000_037):
        comm = L.P2PCommunicator(n, nvls=True, nblocks=24, timeout_s=20.0)
        for rnd in range(3):
            slot = rnd % 2
            vecs = [_vec(300 * rnd + 7 * r + n % 13, n) for r in range(world)]
            comm.snapshots[slot].copy_(torch.from_numpy(vecs[rank]))
            torch.cuda.synchronize()
            seq = comm.allreduce(slot, N.ALGO_NVLS)
            assert comm.wait(seq, 30.0) == 1
            torch.cuda.synchronize()
            got = comm.xbar.cpu().numpy().astype(np.float64)
            ref = O.ring_mean(vecs).astype(np.float64)
            scale = np.sum(np.abs(np.stack(vecs).astype(np.float64)), axis=0) / world
            assert np.all(np.abs(got - ref) <= 1e-6 * scale + 1e-30), (n, rnd, rank)
            sums = [None] * world
            dist.all_gather_object(sums, comm.xbar.cpu().numpy().tobytes())
            assert all(x == sums[0] for x in sums), "ranks received different means"
        dist.barrier()
        comm.close()
    # the reference-facing transport on it: all_reduce_average through CudaP2PTransport
    n = 10_007
    comm = L.P2PCommunicator(n, nvls=True, nblocks=8, timeout_s=20.0)
    tr = L.CudaP2PTransport(comm)
    vecs = [_vec(55 + r, n) for r in range(world)]
    h = tr.submit(0, rank, torch.from_numpy(vecs[rank]).cuda())
    assert h.wait(30.0) and h.status is L.Status.COMPLETE
    got = h.result.cpu().numpy().astype(np.float64)
    scale = np.sum(np.abs(np.stack(vecs).astype(np.float64)), axis=0) / world
    assert np.all(np.abs(got - O.ring_mean(vecs).astype(np.float64)) <= 1e-6 * scale + 1e-30)
    dist.barrier()
    comm.close()
    # the overlap pipeline (side-stream mean + one-pass boundary) on the in-switch mean
    n, steps = 65_541, 6
    x0 = _vec(3, n)
    grads = np.stack([np.stack([_vec(40 * t + r, n) for r in range(world)]) for t in range(steps)])
    comm = L.P2PCommunicator(n, nvls=True, nblocks=16, timeout_s=20.0)
    x = torch.from_numpy(x0.copy()).cuda()
    compute = torch.cuda.Stream()
    sgd = L.SgdConfig(0.9, 0.0, 1e-4, True)
    with torch.cuda.stream(compute):
        w = L.LASGDWorker(x, torch.zeros_like(x), comm=comm, sync_period=2, alpha=0.5, mode="pull", sgd=sgd,
                          lr=0.05, pipeline="overlap", compute_stream=compute)
        for t in range(steps):
            w.g = torch.from_numpy(grads[t, rank]).cuda()
            w.step()
        w.drain()
    torch.cuda.synchronize()
    ref, _, _, _ = O.run_lasgd_pull(x0, grads, [0.05] * steps, world, 2, 0.5,
                                    sgd=O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True))
    np.testing.assert_allclose(x.cpu().numpy(), ref[rank], rtol=1e-5, atol=1e-6)
    w.close()
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


def _w_full_size(rank, world, port):
    """The bench's configuration at BASELINE size: ResNet-50's n, Nesterov momentum +
    weight decay, sync period 1, fused pipeline with the AUTO algorithm (mirror push at
    P=2, staged push at P>=3) — bit-exact against the oracle on every rank."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O

    _init(rank, world, port)
    n, steps = 25_557_032, 2
    rng = np.random.default_rng(2024)
    x0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    grads = np.stack([np.stack([(np.random.default_rng(10 * t + r).standard_normal(n) * 0.01).astype(np.float32)
                                for r in range(world)]) for t in range(steps)])
    comm = L.P2PCommunicator(n, timeout_s=60.0)
    x = torch.from_numpy(x0.copy()).cuda()
    g = torch.empty_like(x)
    sgd = L.SgdConfig(0.9, 0.0, 1e-4, True)
    w = L.LASGDWorker(x, g, comm=comm, sync_period=1, alpha=1.0, sgd=sgd, lr=0.1, mode="pull", pipeline="fused")
    for t in range(steps):
        g.copy_(torch.from_numpy(grads[t, rank]))
        w.step()
    w.drain()
    torch.cuda.synchronize()
    ref, _, _, _ = O.run_lasgd_pull(x0, grads, np.full(steps, 0.1), world, 1, 1.0,
                                    sgd=O.SgdConfig(0.1, 0.9, 0.0, 1e-4, True))
    assert _same_bits(x.cpu().numpy(), ref[rank]), (world, rank)
    dist.barrier()
    w.close()
    comm.close()
    dist.destroy_process_group()


def _w_max_size(rank, world, port):
    """BASELINE configs[4]'s largest buffer (1 GiB of fp32, ragged: 2^28 + 5 elements)
    through the fused AUTO round, checked by a size-independent property: contributions
    are small integers, so every summation order is exact; with zero gradients and
    α = 1 each rank must end on x + (-1)·(x + (-1)·sum/P) (K4a's rounding order,
    optimizer.py:113-133), which is sum/P itself when P is a power of two — then a
    second round must leave it unchanged."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L

    _init(rank, world, port)
    n = (1 << 28) + 5
    idx = torch.arange(n, device="cuda", dtype=torch.int64)

    def contrib(r):
        return ((idx * 7 + 13 * r + (idx >> 11)) % 4096).to(torch.float32)

    want = contrib(0)
    for r in range(1, world):
        want += contrib(r)
    want /= world
    x = contrib(rank)
    del idx
    want = x - (x - want)  # separately rounded ops, as the kernel (exact when P is a power of two)
    rounds = 2 if world & (world - 1) == 0 else 1
    g = torch.zeros_like(x)
    comm = L.P2PCommunicator(n, timeout_s=60.0)
    w = L.LASGDWorker(x, g, comm=comm, sync_period=1, alpha=1.0, sgd=L.SgdConfig(0.0, 0.0, 0.0, False), lr=0.1,
                      mode="pull", pipeline="fused")
    for _ in range(rounds):
        w.step()
    w.drain()
    torch.cuda.synchronize()
    assert torch.equal(x.view(torch.int32), want.view(torch.int32)), (world, rank, rounds)
    dist.barrier()
    w.close()
    comm.close()
    dist.destroy_process_group()


def _w_ragged(rank, world, port):
    """Fused rounds through the communicator at tiny / ragged n (empty chunks when n < P,
    packs straddling chunk bounds) for every fused algorithm, bit-exact vs the oracle."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O

    _init(rank, world, port)
    steps = 4
    mom = L.SgdConfig(0.9, 0.0, 1e-4, True)
    for n in (1, 3, 5, 7, 33, 4099):
        x0 = _vec(n + 1, n)
        grads = np.stack([np.stack([_vec(1000 * n + 10 * t + r, n) for r in range(world)]) for t in range(steps)])
        for algo in (1, 2, 3):
            comm = L.P2PCommunicator(n, nblocks=8, timeout_s=20.0)
            x = torch.from_numpy(x0.copy()).cuda()
            g = torch.empty_like(x)
            w = L.LASGDWorker(x, g, comm=comm, sync_period=1, alpha=0.5, sgd=mom, lr=0.05, mode="pull",
                              pipeline="fused", algo=algo)
            for t in range(steps):
                g.copy_(torch.from_numpy(grads[t, rank]))
                w.step()
            w.drain()
            torch.cuda.synchronize()
            xs, _, _, _ = O.run_lasgd_pull(x0, grads, np.full(steps, 0.05), world, 1, 0.5,
                                           sgd=O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True))
            assert _same_bits(x.cpu().numpy(), xs[rank]), (n, algo, rank)
            dist.barrier()
            w.close()
            comm.close()
    dist.destroy_process_group()


def _w_fault(rank, world, port):
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from paper_2203_13085_b200 import _native as N

    _init(rank, world, port)
    for algo, phase in ((N.ALGO_TWOSHOT, 1), (N.ALGO_ONESHOT, 0), (N.ALGO_PUSH, 1), (N.ALGO_PUSH, 2)):
        comm = L.P2PCommunicator(4096, nblocks=8, timeout_s=1.0, fault_seq=2 if rank == 1 else -1, fault_phase=phase)
        tr = L.CudaP2PTransport(comm, algo=algo)
        h1 = tr.submit(0, rank, comm.snapshots[0])
        assert h1.wait(30.0) and h1.status is L.Status.COMPLETE
        h2 = tr.submit(1, rank, comm.snapshots[1])
        assert h2.wait(30.0)
        assert h2.status is L.Status.FAILED, (rank, h2.status)
        assert ("timed out" in h2.diagnostic) or ("injected" in h2.diagnostic)
        with pytest.raises(L.CollectiveFailure):
            h2.result
        with pytest.raises(L.CollectiveFailure):
            tr.submit(2, rank, comm.snapshots[0])  # poisoned communicator
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
    dist.destroy_process_group()


def _w_adaptive_laggard(rank, world, port):
    """Adaptive schedule with the last rank much slower: the fast ranks take up to
    tau_max local steps per round while the laggard closes its rounds early (peers
    already ahead), i.e. the dynamic rate of the paper's Table 3.  Measured on B200:
    mean tau 3.25-3.8 on the fast ranks, 2.4 on the laggard (P=2 and P=4)."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L

    from paper_2203_13085_b200 import _native as N

    _init(rank, world, port)
    n = 100_003
    comm = L.P2PCommunicator(n, nblocks=16, timeout_s=30.0)
    # every side-stream transport: the laggard must see its peers' progress through the
    # flags each one writes (per-CTA entry flags, or the rank-level rows of the push and
    # copy-engine means)
    for algo in (N.ALGO_AUTO, N.ALGO_PUSH, N.ALGO_CE):
        x = torch.randn(n, device="cuda")
        g = torch.randn(n, device="cuda") * 1e-3
        w = L.LASGDWorker(x, g, comm=comm, sync_period=4, lr=0.01, mode="pull", adaptive=True, tau_max=4, algo=algo)
        for _ in range(40):
            if rank == world - 1:
                torch.cuda._sleep(3_000_000)  # ~1.5 ms per step on the laggard
            w.step()
        w.drain()
        torch.cuda.synchronize()
        hist = dict(w.tau_hist)
        mean_tau = sum(k * v for k, v in hist.items()) / max(1, sum(hist.values()))
        allm = [None] * world
        dist.all_gather_object(allm, mean_tau)
        assert np.isfinite(x.cpu().numpy()).all()
        if rank == 0:
            # fast ranks run ahead (several local steps per round); the laggard closes as soon
            # as it sees its peers ahead, which its host learns at most max_host_lead (2)
            # steps late, so its rounds last at most ~1 + 2 steps
            fast, lag = allm[:-1], allm[world - 1]
            assert all(m > lag for m in fast) and sum(fast) / len(fast) >= lag + 0.5, (algo, allm)
            assert lag <= 3.0, (algo, allm)
        dist.barrier()
        w.close()
    comm.close()
    dist.destroy_process_group()


def _w_fault_end_signal(rank, world, port):
    """A rank that never raises its end-of-round signal (fault phase 2) in a fused push /
    mirror round: the next round's entry wait trips the watchdog and every rank's worker
    raises CollectiveFailure instead of hanging."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L

    _init(rank, world, port)
    # small (one-pass round) and >= 32 MB at P >= 3 (pipelined halves: phase 1 drops the
    # first half's signal, phase 2 the end signal)
    cases = [(4099, 2), (9_000_001, 2)] + ([(9_000_001, 1)] if world >= 3 else [])  # P=2 mirror: no mid signal
    for n, phase in cases:
        comm = L.P2PCommunicator(n, nblocks=8, timeout_s=1.0, fault_seq=3 if rank == 1 else -1, fault_phase=phase)
        x = torch.randn(n, device="cuda")
        g = torch.randn(n, device="cuda")
        w = L.LASGDWorker(x, g, comm=comm, sync_period=1, lr=0.01, pipeline="fused", algo=3)
        with pytest.raises(L.CollectiveFailure):
            for _ in range(6):  # launch 1 stages the snapshot, 2.. are rounds; rank 1 skips a signal of 3
                w.step()
            torch.cuda.synchronize()  # in-flight rounds time out after 1 s
            w.step()
        torch.cuda.synchronize()
        diag = comm.diagnostic()
        assert "timed out" in diag or "injected" in diag, (n, phase, diag)
        if phase == 2:
            assert "end-of-round" in diag or "injected" in diag, diag
        dist.barrier()
        w.close()
        comm.close()
    dist.destroy_process_group()


def _w_torch_optim(rank, world, port):
    """The torch.optim front end across ranks (comm="auto": x0 broadcast from rank 0, a
    P2PCommunicator built inside): bit-identical to driving LASGDWorker over an explicit
    communicator (parameters and snapshot)."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L

    _init(rank, world, port)
    g = torch.Generator(device="cuda").manual_seed(100 + rank)  # rank-local data
    inp, tgt = torch.randn(32, 16, device="cuda", generator=g), torch.randn(32, 3, device="cuda", generator=g)

    def model():
        torch.manual_seed(rank)  # different init per rank: auto mode must broadcast rank 0's
        return torch.nn.Sequential(torch.nn.Linear(16, 40), torch.nn.ReLU(), torch.nn.Linear(40, 3)).cuda()

    def run(use_opt):
        m = model()
        if use_opt:
            opt = L.LASGD(m, lr=0.05, momentum=0.9, weight_decay=1e-4, sync_period=3)
            w, comm = opt.worker, None
        else:
            flat = L.FlatParams(m, align_bytes=256)
            dist.broadcast(flat.x, 0)
            comm = L.P2PCommunicator(flat.numel)
            w = L.LASGDWorker(flat.x, flat.g, comm=comm, sync_period=3, lr=0.05, pipeline="fused",
                              sgd=L.SgdConfig(0.9, 0.0, 1e-4, False))
        for _ in range(9):
            if use_opt:
                opt.zero_grad()
            else:
                flat.zero_grad()
            torch.nn.functional.mse_loss(m(inp), tgt).backward()
            (opt if use_opt else w).step()
        (opt if use_opt else w).drain()
        torch.cuda.synchronize()
        x = torch.cat([p.detach().reshape(-1) for p in m.parameters()]).cpu().numpy()
        snap = w.state.x_snapshot.cpu().numpy()
        dist.barrier()
        if use_opt:
            opt.close()
        else:
            w.close()
            comm.close()
        return x, snap

    (xa, sa), (xb, sb) = run(True), run(False)
    assert _same_bits(xa, xb) and _same_bits(sa, sb), rank
    dist.destroy_process_group()


def _w_ce(rank, world, port):
    """The copy-engine mean (ALGO_CE: contributions and means moved by cudaMemcpyAsync over
    the IPC-mapped regions, flags by one-warp kernels): bit-exact against the ring-order
    oracle at ragged sizes in f32 and f64, interleaved with SM all-reduces and push rounds
    on the same communicator (the CE mean clobbers the push staging), gated launches, the
    overlap worker loop on it against the oracle, and a dropped signal failing every rank."""
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from oracle import lasgd_oracle as O
    from paper_2203_13085_b200 import _native as N

    _init(rank, world, port)
    for dtype in (torch.float32, torch.float64):
        npdt = np.float32 if dtype == torch.float32 else np.float64
        for n in (1, 3, 1001, 65_537, 4_000_037):
            comm = L.P2PCommunicator(n, dtype=dtype, nblocks=24, timeout_s=20.0)
            assert comm.resolve_algo(N.ALGO_CE) == N.ALGO_CE
            for rnd, algo in enumerate((N.ALGO_CE, N.ALGO_CE, N.ALGO_TWOSHOT, N.ALGO_CE, N.ALGO_ONESHOT, N.ALGO_CE,
                                        N.ALGO_PUSH, N.ALGO_PUSH, N.ALGO_CE, N.ALGO_PUSH)):
                slot = rnd % 2
                vecs = [_vec(5000 * rnd + 10 * r + n, n, npdt) for r in range(world)]
                comm.snapshots[slot].copy_(torch.from_numpy(vecs[rank]))
                torch.cuda.synchronize()
                seq = comm.allreduce(slot, algo)
                assert comm.wait(seq, 30.0) == 1
                torch.cuda.synchronize()
                assert _same_bits(comm.xbar.cpu().numpy(), O.ring_mean(vecs)), (n, rnd, algo, rank)
            comm.set_gate(True)
            for rnd in range(2):
                vecs = [_vec(91 + 10 * r + rnd, n, npdt) for r in range(world)]
                comm.snapshots[rnd].copy_(torch.from_numpy(vecs[rank]))
                torch.cuda.synchronize()
                seq = comm.allreduce(rnd, N.ALGO_CE)
                assert comm.wait(seq, 30.0) == 1
                assert _same_bits(comm.xbar.cpu().numpy(), O.ring_mean(vecs)), (n, "gated", rank)
            comm.set_gate(False)
            # the device barrier takes no launch sequence number
            before = comm.launches()
            for _ in range(3):
                comm.device_barrier()
            torch.cuda.synchronize()
            assert comm.launches() == before
            dist.barrier()
            comm.close()
    # large buffers: the push mean's pipelined halves (>= 32 MB), beside the CE mean
    for dtype, n in ((torch.float32, 9_000_001), (torch.float64, 4_500_007)):
        npdt = np.float32 if dtype == torch.float32 else np.float64
        comm = L.P2PCommunicator(n, dtype=dtype, timeout_s=30.0)
        for rnd, algo in enumerate((N.ALGO_PUSH, N.ALGO_CE, N.ALGO_PUSH, N.ALGO_AUTO)):
            slot = rnd % 2
            vecs = [_vec(7000 * rnd + 10 * r + n, n, npdt) for r in range(world)]
            comm.snapshots[slot].copy_(torch.from_numpy(vecs[rank]))
            torch.cuda.synchronize()
            seq = comm.allreduce(slot, algo)
            assert comm.wait(seq, 30.0) == 1
            torch.cuda.synchronize()
            assert _same_bits(comm.xbar.cpu().numpy(), O.ring_mean(vecs)), (n, rnd, algo, rank)
        dist.barrier()
        comm.close()
    # the overlap pipeline on the CE mean, mixed with fused push rounds on one communicator
    n, steps = 100_003, 8
    x0 = _vec(11, n)
    grads = np.stack([np.stack([_vec(300 * t + r, n) for r in range(world)]) for t in range(steps)])
    mom = L.SgdConfig(0.9, 0.0, 1e-4, True)
    comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
    for k, pipe, algo in ((1, "overlap", N.ALGO_CE), (2, "fused", N.ALGO_PUSH), (1, "overlap", N.ALGO_CE),
                          (3, "overlap", N.ALGO_CE), (1, "fused", N.ALGO_PUSH), (2, "overlap", N.ALGO_PUSH)):
        x = torch.from_numpy(x0.copy()).cuda()
        g = torch.empty_like(x)
        compute = torch.cuda.Stream()
        with torch.cuda.stream(compute):
            w = L.LASGDWorker(x, g, comm=comm, sync_period=k, alpha=0.5, sgd=mom, lr=0.05, mode="pull",
                              compute_stream=compute, pipeline=pipe, algo=algo)
            for t in range(steps):
                g.copy_(torch.from_numpy(grads[t, rank]))
                w.step()
                if t % 3 == 1:  # device barriers between rounds leave the round chain intact
                    comm.device_barrier(compute)
            w.drain()
        torch.cuda.synchronize()
        xs, _, _, _ = O.run_lasgd_pull(x0, grads, np.full(steps, 0.05), world, k, 0.5,
                                       sgd=O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True))
        assert _same_bits(x.cpu().numpy(), xs[rank]), (k, pipe, algo, rank)
        w.close()
        dist.barrier()
    with pytest.raises(ValueError):
        L.LASGDWorker(x, g, comm=comm, pipeline="fused", algo=N.ALGO_CE, lr=0.1)
    comm.close()
    # ResNet-50 size, overlap pipeline with AUTO: the side-stream mean is the CE mean at
    # P >= 4 (the SM mean below), bit-exact either way
    n, steps = 25_557_032, 3
    x0 = _vec(12, n)
    grads = np.stack([np.stack([_vec(310 * t + r, n) for r in range(world)]) for t in range(steps)])
    comm = L.P2PCommunicator(n, timeout_s=30.0)
    x = torch.from_numpy(x0.copy()).cuda()
    g = torch.empty_like(x)
    w = L.LASGDWorker(x, g, comm=comm, sync_period=1, lr=0.05, mode="pull", pipeline="overlap")
    for t in range(steps):
        g.copy_(torch.from_numpy(grads[t, rank]))
        w.step()
    w.drain()
    torch.cuda.synchronize()
    xs, _, _, _ = O.run_lasgd_pull(x0, grads, np.full(steps, 0.05), world, 1, 1.0)
    assert _same_bits(x.cpu().numpy(), xs[rank]), ("full size overlap", rank)
    w.close()
    dist.barrier()
    comm.close()
    # watchdog: rank 1 drops its contributions signal (phase 1) or its means signal (phase 2)
    for phase in (1, 2):
        comm = L.P2PCommunicator(4096, nblocks=8, timeout_s=1.0, fault_seq=2 if rank == 1 else -1, fault_phase=phase)
        tr = L.CudaP2PTransport(comm, algo=N.ALGO_CE)
        h1 = tr.submit(0, rank, comm.snapshots[0])
        assert h1.wait(30.0) and h1.status is L.Status.COMPLETE
        h2 = tr.submit(1, rank, comm.snapshots[1])
        assert h2.wait(30.0)
        assert h2.status is L.Status.FAILED, (rank, h2.status)
        assert ("copy-engine" in h2.diagnostic) or ("injected" in h2.diagnostic), h2.diagnostic
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
    dist.destroy_process_group()


def _spawn(fn):
    import torch.multiprocessing as mp

    world = min(NGPU, 4)
    mp.spawn(fn, args=(world, _free_port()), nprocs=world, join=True)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_p2p_allreduce_bit_exact():
    _spawn(_w_allreduce)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_worker_round_protocol_bit_exact():
    _spawn(_w_worker_loop)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_sgd_ar_worker_bit_exact():
    _spawn(_w_sgd_ar)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_sgd_ar_bucketed_bit_exact():
    _spawn(_w_sgd_ar_bucketed)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_graph_replay_multi_rank_bit_exact():
    _spawn(_w_graph_replay)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_nvls_mean_within_tolerance():
    _spawn(_w_nvls)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_fused_auto_full_resnet50_size_bit_exact():
    _spawn(_w_full_size)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_fused_auto_1gib_exact_mean():
    _spawn(_w_max_size)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_fused_rounds_ragged_sizes_bit_exact():
    _spawn(_w_ragged)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_adaptive_fast_ranks_run_ahead_of_a_laggard():
    _spawn(_w_adaptive_laggard)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_watchdog_missing_end_signal_fails_every_rank():
    _spawn(_w_fault_end_signal)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_watchdog_fault_fails_every_rank():
    _spawn(_w_fault)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_torch_optim_front_end_multi_rank_bit_exact():
    _spawn(_w_torch_optim)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_copy_engine_mean_bit_exact():
    _spawn(_w_ce)

"""Graph replay of the deterministic schedule (lasgd_worker_graph_capture /
lasgd_worker_capture_begin, the device round descriptor): a captured run of worker
steps replayed as one CUDA graph launch leaves x, the momentum buffer, the delta
accumulator, the snapshot slots and the protocol counters bit-identical to the same
steps issued one by one (which tests/test_gpu_optimizer.py pins to the oracle), and
the P = 1 loop matches the oracle directly (optimizer.py:181-207, collective_complete
= (tau_i == k))."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N_ELEM = 70_001  # odd: exercises the scalar tail of the streaming kernels


def _grads(n, count=2, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn(n, device="cuda", generator=g) * 1e-2 for _ in range(count)]


def _worker(x, g, **kw):
    import paper_2203_13085_b200 as L

    kw.setdefault("sgd", L.SgdConfig(0.9, 0.0, 1e-4, True))
    kw.setdefault("lr", 0.05)
    return L.LASGDWorker(x, g, **kw)


def _state(w):
    st = w.state
    t = [st.x_local.clone(), st.x_snapshot.clone()]
    if st.momentum_buf is not None:
        t.append(st.momentum_buf.clone())
    if st.delta is not None:
        t.append(st.delta.clone())
    return t, (st.tau_i, st.snap_idx, st.local_clock, st.global_clock)


def _bits_equal(a, b):
    return torch.equal(a.view(torch.int32), b.view(torch.int32))


@pytest.mark.parametrize("pipeline", ["fused", "overlap"])
@pytest.mark.parametrize("k", [1, 3])
@pytest.mark.parametrize("mode", ["pull", "delta"])
@pytest.mark.parametrize("sched", [False, True])
def test_graph_replay_bit_identical_to_eager(pipeline, k, mode, sched):
    import paper_2203_13085_b200 as L

    torch.manual_seed(1)
    x0 = torch.randn(N_ELEM, device="cuda") * 0.1
    grads = _grads(N_ELEM)
    kw = dict(sync_period=k, mode=mode, pipeline=pipeline)
    if sched:
        kw["schedule"] = L.LrSchedule(0.02, 4, 0.5, (1.0, 2.0), 10.0, steps_per_epoch=12)
        kw.pop("lr", None)
        kw["lr"] = None
    pre, S, R, post = 2 * k, 6 * k, 3, k  # eager, captured x replays, eager again
    total = pre + S * R + post

    xe = x0.clone()
    we = _worker(xe, grads[0], **kw)
    for t in range(total):
        we.g = grads[t % 2]
        we.step()
    torch.cuda.synchronize()
    ref, ref_ctr = _state(we)

    xg = x0.clone()
    wg = _worker(xg, grads[0], **kw)
    for t in range(pre):
        wg.g = grads[t % 2]
        wg.step()
    graph = wg.capture([grads[(pre + i) % 2] for i in range(S)])
    for _ in range(R):
        graph.replay()
    for t in range(pre + S * R, total):
        wg.g = grads[t % 2]
        wg.step()
    torch.cuda.synchronize()
    got, got_ctr = _state(wg)
    assert got_ctr == ref_ctr
    for a, b in zip(got, ref):
        assert _bits_equal(a, b)
    assert wg.launches == we.launches or pipeline == "overlap"  # overlap: boundary K5+K1 fuse in the graph
    assert wg.tau_hist == we.tau_hist
    we.close()
    wg.close()


def test_graph_replay_matches_oracle_p1():
    """P = 1 fused loop with momentum/Nesterov/wd at sync period 1, replayed from a graph,
    against the oracle's deterministic driver."""
    from oracle import lasgd_oracle as O

    n, steps = 10_007, 8
    rng = np.random.default_rng(3)
    x0 = rng.standard_normal(n).astype(np.float32)
    g_np = rng.standard_normal((2, n)).astype(np.float32) * np.float32(0.01)
    grads = [torch.from_numpy(g_np[i]).cuda() for i in range(2)]
    x = torch.from_numpy(x0).cuda()
    w = _worker(x, grads[0], sync_period=1, pipeline="fused", lr=0.05)
    graph = w.capture(grads)
    for _ in range(steps // 2):
        graph.replay()
    torch.cuda.synchronize()
    gl = np.stack([g_np[t % 2][None, :] for t in range(steps)])
    ref, snaps, _, _ = O.run_lasgd_pull(x0, gl, [0.05] * steps, 1, 1, 1.0,
                                        sgd=O.SgdConfig(0.05, 0.9, 0.0, 1e-4, True))
    assert np.array_equal(x.cpu().numpy().view(np.uint32), ref[0].view(np.uint32))
    assert np.array_equal(w.state.x_snapshot.cpu().numpy().view(np.uint32), snaps[0].view(np.uint32))
    w.close()


def test_capture_with_training_step_matches_eager():
    """Forward + backward + local step + round boundary as ONE graph (capture_with)."""
    import paper_2203_13085_b200 as L

    def run(graphed):
        torch.manual_seed(7)
        model = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.Tanh(), torch.nn.Linear(128, 8)).cuda()
        flat = L.FlatParams(model)
        gen = torch.Generator("cuda").manual_seed(11)
        inp = torch.randn(32, 64, device="cuda", generator=gen)
        tgt = torch.randn(32, 8, device="cuda", generator=gen)
        compute = torch.cuda.Stream()
        w = L.LASGDWorker(flat.x, flat.g, sync_period=2, lr=0.05, pipeline="fused",
                          sgd=L.SgdConfig(0.9, 0.0, 1e-4, True), compute_stream=compute)

        def fwd_bwd(t=0):
            flat.zero_grad()
            torch.nn.functional.mse_loss(model(inp), tgt).backward()

        with torch.cuda.stream(compute):
            for _ in range(4):  # eager warm-up (also the autograd / allocator warm-up)
                fwd_bwd()
                w.step()
            if graphed:
                g = w.capture_with(fwd_bwd, steps=2)
                for _ in range(5):
                    g.replay()
            else:
                for _ in range(10):
                    fwd_bwd()
                    w.step()
        torch.cuda.synchronize()
        out = flat.x.clone(), w.state.local_clock, w.state.global_clock
        w.close()
        return out

    a, b = run(True), run(False)
    assert a[1:] == b[1:] == (14, 7)
    assert _bits_equal(a[0], b[0])


def test_graph_capture_rejections():
    grads = _grads(1024)
    x = torch.zeros(1024, device="cuda")
    w = _worker(x, grads[0], sync_period=2, pipeline="fused")
    with pytest.raises(ValueError, match="whole rounds"):
        w.capture(grads[:1] * 3)
    graph = w.capture(grads)
    w.g = grads[0]
    w.step()  # now mid-round: the graph was captured at a round start
    with pytest.raises(RuntimeError, match="round"):
        graph.replay()
    w.step()
    graph.replay()
    torch.cuda.synchronize()
    w.close()
    xa = torch.zeros(1024, device="cuda")
    wa = _worker(xa, grads[0], sync_period=2, adaptive=True, tau_max=3)
    with pytest.raises(ValueError, match="deterministic"):
        wa.capture(grads)
    wa.close()


def test_hold_releases_queued_work():
    """The measurement hold: work queued behind it starts only after the release."""
    import ctypes

    from paper_2203_13085_b200 import _native as N
    from paper_2203_13085_b200 import kernels as K

    h = ctypes.c_void_p()
    N.check(N.lib().lasgd_hold_create(ctypes.byref(h)))
    s = torch.cuda.Stream()
    x = torch.zeros(4096, device="cuda")
    y = torch.ones(4096, device="cuda")
    N.check(N.lib().lasgd_hold_enqueue(h, ctypes.c_void_p(s.cuda_stream), 10.0))
    K.snapshot(x, y, stream=s)
    ev = torch.cuda.Event()
    ev.record(s)
    import time

    time.sleep(0.05)
    assert not ev.query()  # still held
    N.check(N.lib().lasgd_hold_release(h))
    ev.synchronize()
    assert torch.equal(x, y)
    N.lib().lasgd_hold_destroy(h)

"""The torch.optim front end (LASGD): bit-identical to driving LASGDWorker directly, within
floating-point contraction of torch.optim.SGD at P = 1, and compatible with torch's LR
schedulers through param_groups."""

import pytest
import torch

import paper_2203_13085_b200 as L

pytestmark = pytest.mark.gpu


def _mlp(seed=0):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(32, 64), torch.nn.Tanh(), torch.nn.Linear(64, 4)).cuda()


def _data():
    g = torch.Generator(device="cuda").manual_seed(3)
    return torch.randn(64, 32, device="cuda", generator=g), torch.randn(64, 4, device="cuda", generator=g)


def test_optimizer_equals_worker():
    inp, tgt = _data()

    def run(use_opt):
        model = _mlp()
        if use_opt:
            opt = L.LASGD(model, lr=0.05, momentum=0.9, weight_decay=1e-4, nesterov=True, sync_period=2)
        else:
            flat = L.FlatParams(model, align_bytes=256)
            w = L.LASGDWorker(flat.x, flat.g, sync_period=2, lr=0.05, pipeline="fused",
                              sgd=L.SgdConfig(0.9, 0.0, 1e-4, True))
        for _ in range(9):
            if use_opt:
                opt.zero_grad()
            else:
                flat.zero_grad()
            torch.nn.functional.mse_loss(model(inp), tgt).backward()
            if use_opt:
                opt.step()
            else:
                w.step()
        torch.cuda.synchronize()
        return torch.cat([p.detach().reshape(-1) for p in model.parameters()])

    a, b = run(True), run(False)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_optimizer_close_to_torch_sgd_and_scheduler():
    inp, tgt = _data()
    m1, m2 = _mlp(1), _mlp(1)
    opt = L.LASGD(m1, lr=0.1, momentum=0.9, weight_decay=1e-4, nesterov=True)
    ref = torch.optim.SGD(m2.parameters(), lr=0.1, momentum=0.9, weight_decay=1e-4, nesterov=True)
    s1 = torch.optim.lr_scheduler.StepLR(opt, step_size=3, gamma=0.5)
    s2 = torch.optim.lr_scheduler.StepLR(ref, step_size=3, gamma=0.5)
    for _ in range(8):
        for m, o, s in ((m1, opt, s1), (m2, ref, s2)):
            o.zero_grad()
            loss = torch.nn.functional.mse_loss(m(inp), tgt)
            loss.backward()
            o.step()
            s.step()
    torch.cuda.synchronize()
    assert opt.param_groups[0]["lr"] == ref.param_groups[0]["lr"] == 0.1 * 0.5 ** 2
    for p1, p2 in zip(m1.parameters(), m2.parameters()):
        torch.testing.assert_close(p1, p2, rtol=1e-5, atol=1e-6)
    assert opt.state_view.local_clock == 8
    with pytest.raises(NotImplementedError):
        opt.state_dict()
    with pytest.raises(NotImplementedError):
        opt.add_param_group({"params": [torch.zeros(3, device="cuda", requires_grad=True)]})
    opt.close()


def test_graph_replay_follows_changed_constant_lr():
    """A constant rate changed between replays (what an LR scheduler does) reaches the
    replayed kernels: replay at lr a, then at lr b == eager steps at a, then at b."""
    n = 4099
    gen = torch.Generator(device="cuda").manual_seed(5)
    x0 = torch.randn(n, device="cuda", generator=gen)
    grads = [torch.randn(n, device="cuda", generator=gen) for _ in range(2)]

    def run(graph):
        x = x0.clone()
        w = L.LASGDWorker(x, grads[0], sync_period=2, lr=0.1, pipeline="fused", sgd=L.SgdConfig(0.9, 0.0, 0.0, False))
        w.step()
        w.g = grads[1]
        w.step()
        g = w.capture(grads) if graph else None
        for lr in (0.1, 0.025):
            w.lr = lr
            if graph:
                g.replay()
            else:
                for t in range(2):
                    w.g = grads[t]
                    w.step()
        torch.cuda.synchronize()
        out = x.clone()
        if g is not None:
            g.close()
        w.close()
        return out

    a, b = run(True), run(False)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))

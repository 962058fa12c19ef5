"""CUDA-graph capture of zero_grad + forward + backward (graphs.GraphedStep): the
replayed step writes the same gradients as the eager step into the bound flat
buffer, one graph per bound buffer, and composes with the native LASGD worker."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _mlp(seed=0):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.Tanh(), torch.nn.Linear(128, 8)).cuda()


def test_graphed_step_matches_eager_and_rebinds():
    import paper_2203_13085_b200 as L

    model = _mlp()
    flat = L.FlatParams(model)
    inp = torch.randn(32, 64, device="cuda")
    tgt = torch.randn(32, 8, device="cuda")

    def fn():
        torch.nn.functional.mse_loss(model(inp), tgt).backward()

    flat.zero_grad()
    fn()
    eager = flat.g.clone()
    step = L.GraphedStep(flat, fn)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    assert torch.equal(flat.g, eager)
    # new input values flow through the static input tensor
    inp.mul_(2.0)
    step()
    flat2 = flat.g.clone()
    flat.zero_grad()
    fn()
    assert torch.equal(flat.g, flat2)
    # a second gradient buffer gets its own graph; the first buffer is left untouched
    other = torch.full_like(flat.g, 7.0)
    before = flat.g.clone()
    first = flat.g
    flat.bind_grads(other)
    step()
    torch.cuda.synchronize()
    assert len(step.graphs) == 2
    assert torch.equal(other, flat2)
    assert torch.equal(first, before)


def test_graphed_step_with_worker_equals_eager_training():
    import paper_2203_13085_b200 as L

    def train(graphed):
        model = _mlp(1)
        flat = L.FlatParams(model)
        inp = torch.randn(32, 64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
        tgt = torch.randn(32, 8, device="cuda", generator=torch.Generator("cuda").manual_seed(6))

        def fn():
            torch.nn.functional.mse_loss(model(inp), tgt).backward()

        step = L.GraphedStep(flat, fn) if graphed else None
        w = L.LASGDWorker(flat.x, flat.g, sync_period=2, lr=0.05, sgd=L.SgdConfig(0.9, 0.0, 1e-4, True))
        for _ in range(12):
            if graphed:
                step()
            else:
                flat.zero_grad()
                fn()
            w.step()
        w.drain()
        torch.cuda.synchronize()
        return flat.x.clone()

    assert torch.equal(train(True), train(False))

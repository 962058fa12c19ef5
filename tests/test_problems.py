"""Config-1 problem plumbing of the package (problems.py) against the oracle's
restatement (itself pinned to the reference by tests/golden/config1.npz): same data,
same per-node batches, same flat parameter layout, loss and gradient (CPU, f64)."""

import numpy as np
import torch

from oracle import problems_oracle as PO
from oracle.lasgd_oracle import partition_chunks
from paper_2203_13085_b200 import FlatParams
from paper_2203_13085_b200 import problems as PR


def test_synthetic_data_and_sampler_identical():
    a = PR.make_synthetic(0, 4096, 784, 0.1)
    b = PO.make_synthetic(0, 4096, 784, 0.1, "regression")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for rank in range(4):
        s1, s2 = PR.ShardSampler(4096, rank, 4, 32, 7), PO.ShardSampler(4096, rank, 4, 32, 7)
        for _ in range(70):  # crosses an epoch boundary (32 batches per shard epoch)
            assert np.array_equal(s1.next_batch(), s2.next_batch())


def test_shards_follow_partition_chunks():
    for n, P in ((10, 3), (3, 5), (9, 3), (4096, 4), (7, 1)):
        for r, (s, e) in enumerate(partition_chunks(n, P)):
            assert np.array_equal(PR.shard_of(n, r, P), np.arange(s, e))


def test_mlp_flat_layout_loss_and_grad_match_oracle():
    dims = [20, 16, 8, 1]
    X, y = PR.make_synthetic(3, 64, 20, 0.1)
    model = PR.mlp(dims, dtype=torch.float64)
    flat = FlatParams(model, dtype=torch.float64)
    assert flat.numel == PO.mlp_dim(dims)
    x = np.random.default_rng(0).standard_normal(flat.numel) * 0.3
    flat.x.copy_(torch.from_numpy(x))
    flat.zero_grad()
    loss = PR.mlp_loss(model, torch.from_numpy(X), torch.from_numpy(y))
    loss.backward()
    ref_loss, ref_grad = PO.mlp_loss_and_grad(x, dims, X, y)
    assert abs(loss.item() - ref_loss) <= 1e-12 * abs(ref_loss)
    np.testing.assert_allclose(flat.g.numpy(), ref_grad, rtol=1e-10, atol=1e-13)

"""Config-1 data + gradient oracle — TEST INFRASTRUCTURE ONLY (see lasgd_oracle.py header).

Restates the reference's seeded synthetic problem so the GPU box (which has no
/root/reference) can rebuild config 1 bit-identically:

* ``make_synthetic``  — problems.py:67-88 (numpy Generator on
  SeedSequence(entropy=seed, spawn_key=(902,)));
* ``ShardSampler``    — problems.py:91-113 (per-rank SeedSequence(seed, (rank, 0)),
  without-replacement permutation of the contiguous shard, problems.py:45-53);
* ``mlp_loss_and_grad`` — problems.py:195-275 (tanh hidden layers, linear output,
  loss (1/2m)·Σ resid², flat layout W_l row-major then b_l).

Pinned against the reference by tests/golden/config1.npz (dataset checksum,
batch order, f64 loss trajectory).
"""

from __future__ import annotations

import numpy as np

from .lasgd_oracle import partition_chunks


def make_synthetic(seed: int, n: int, d: int, noise: float, kind: str):
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(902,)))
    features = rng.standard_normal((n, d))
    w_true = rng.standard_normal(d)
    eps = rng.standard_normal(n)
    logits = features @ w_true + noise * eps
    if kind == "regression":
        targets = logits
    else:
        targets = (logits > 0.0).astype(np.float64)
    return features, targets


class ShardSampler:
    def __init__(self, n: int, rank: int, num_nodes: int, batch_size: int, seed: int):
        s, e = partition_chunks(n, num_nodes)[rank]
        self.indices = np.arange(s, e)
        self.batch_size = min(batch_size, self.indices.size)
        self._rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(rank, 0)))
        self._order = np.empty(0, dtype=np.int64)
        self._pos = 0

    def next_batch(self) -> np.ndarray:
        if self._pos >= self._order.size:
            self._order = self._rng.permutation(self.indices)
            self._pos = 0
        batch = self._order[self._pos : self._pos + self.batch_size]
        self._pos += batch.size
        return batch


def mlp_dim(layer_dims) -> int:
    return sum(o * i + o for i, o in zip(layer_dims[:-1], layer_dims[1:]))


def mlp_loss_and_grad(x: np.ndarray, layer_dims, X: np.ndarray, y: np.ndarray):
    shapes = [(layer_dims[i + 1], layer_dims[i]) for i in range(len(layer_dims) - 1)]
    layers, off = [], 0
    for n_out, n_in in shapes:
        W = x[off : off + n_out * n_in].reshape(n_out, n_in)
        off += n_out * n_in
        b = x[off : off + n_out]
        off += n_out
        layers.append((W, b))
    m = X.shape[0]
    acts = [X]
    pre = None
    for idx, (W, b) in enumerate(layers):
        pre = acts[-1] @ W.T + b
        if idx < len(layers) - 1:
            acts.append(np.tanh(pre))
    resid = pre[:, 0] - y
    loss = float(resid @ resid) / (2.0 * m)
    parts = []
    delta = (resid / m)[:, None]
    for idx in range(len(layers) - 1, -1, -1):
        W, b = layers[idx]
        gW = delta.T @ acts[idx]
        parts.append(np.concatenate([gW.ravel(), delta.sum(axis=0)]))
        if idx > 0:
            delta = (delta @ W) * (1.0 - acts[idx] ** 2)
    return loss, np.concatenate(parts[::-1])

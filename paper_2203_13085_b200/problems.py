"""Learning-rate schedule (mirror of problems.py:322-365 of the reference) and the
config-1 problem the CLI runs on the GPU.

The rate is a host scalar; the K5 kernel rounds it to the element type
(``(float)(-lr)``), exactly as numpy's NEP 50 does for ``f32_array * -eta``.

Config 1 (BASELINE.json configs[0]): the reference's seeded synthetic regression
(``make_synthetic``, problems.py:67-88), per-node shards with without-replacement
minibatches (``ShardSampler``, problems.py:91-113) and the tanh MLP with squared loss
(``MlpOracle``, problems.py:195-275) as a torch module whose ``FlatParams`` layout is
the reference's flat vector (W_l row-major, then b_l).  The data generator and the
sampler use numpy's seeded generators like the reference, so batches are identical;
forward/backward is PyTorch.  (The oracle keeps its own restatement for the parity
tests, oracle/problems_oracle.py.)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class LrSchedule:
    """Linear warmup from base_lr to base_lr*scale_nodes, then step decays (problems.py:322-352)."""

    base_lr: float
    scale_nodes: int
    warmup_epochs: float
    decay_epochs: tuple = ()
    decay_factor: float = 10.0
    steps_per_epoch: int = 1

    def __post_init__(self) -> None:
        if self.base_lr <= 0:
            raise ValueError("base_lr must be positive")
        if self.scale_nodes < 1:
            raise ValueError("scale_nodes must be a positive integer")
        if self.warmup_epochs < 0:
            raise ValueError("warmup_epochs must be nonnegative")
        if self.decay_factor <= 0:
            raise ValueError("decay_factor must be positive")
        if self.steps_per_epoch < 1:
            raise ValueError("steps_per_epoch must be positive")
        object.__setattr__(self, "decay_epochs", tuple(float(e) for e in self.decay_epochs))

    @property
    def peak_lr(self) -> float:
        return self.base_lr * self.scale_nodes


def lr_at(schedule: LrSchedule, step: int) -> float:
    """problems.py:355-365: indexed by the node's LOCAL clock (optimizer.py:204)."""
    if step < 0:
        raise ValueError("step must be nonnegative")
    epoch = step / schedule.steps_per_epoch
    peak = schedule.peak_lr
    if schedule.warmup_epochs > 0 and epoch < schedule.warmup_epochs:
        frac = epoch / schedule.warmup_epochs
        return schedule.base_lr + (peak - schedule.base_lr) * frac
    decays = sum(1 for e in schedule.decay_epochs if epoch >= e)
    return peak / schedule.decay_factor**decays


# ---------------------------------------------------------------------------- config 1


def make_synthetic(seed: int, n: int, d: int, noise: float, kind: str = "regression"):
    """problems.py:67-88: (features [n, d], targets [n]) as float64 numpy arrays."""
    if n < 1 or d < 1:
        raise ValueError("n and d must be positive")
    if noise < 0:
        raise ValueError("noise must be nonnegative")
    if kind not in ("regression", "classification"):
        raise ValueError(f"unknown dataset kind {kind!r}")
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(902,)))
    features = rng.standard_normal((n, d))
    w_true = rng.standard_normal(d)
    eps = rng.standard_normal(n)
    logits = features @ w_true + noise * eps
    targets = logits if kind == "regression" else (logits > 0.0).astype(np.float64)
    return features, targets


def shard_of(n: int, rank: int, num_nodes: int) -> np.ndarray:
    """Dataset.shard_of (problems.py:45-53): contiguous partition_chunks shard."""
    base, extra = divmod(n, num_nodes)
    start = rank * base + min(rank, extra)
    return np.arange(start, start + base + (1 if rank < extra else 0))


class ShardSampler:
    """problems.py:91-113: reshuffle the node's shard every epoch with a generator
    seeded by (seed, rank); batch order is a pure function of the seed."""

    def __init__(self, n: int, rank: int, num_nodes: int, batch_size: int, seed: int):
        if batch_size < 1:
            raise ValueError("batch_size must be positive")
        self.indices = shard_of(n, rank, num_nodes)
        self.batch_size = min(batch_size, self.indices.size)
        self._rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(rank, 0)))
        self._order = np.empty(0, dtype=np.int64)
        self._pos = 0

    def next_batch(self) -> np.ndarray:
        if self._pos >= self._order.size:
            self._order = self._rng.permutation(self.indices)
            self._pos = 0
        batch = self._order[self._pos:self._pos + self.batch_size]
        self._pos += batch.size
        return batch


def mlp(layer_dims, dtype=None, device=None):
    """MlpOracle's network (problems.py:195-275) as a torch module: Linear layers with
    tanh between them, scalar linear output.  ``FlatParams`` over it yields the
    reference's flat layout."""
    import torch

    if len(layer_dims) < 2 or layer_dims[-1] != 1:
        raise ValueError("need at least input and output dims, output arity 1")
    layers = []
    for i, (a, b) in enumerate(zip(layer_dims[:-1], layer_dims[1:])):
        layers.append(torch.nn.Linear(a, b, dtype=dtype, device=device))
        if i < len(layer_dims) - 2:
            layers.append(torch.nn.Tanh())
    return torch.nn.Sequential(*layers)


def mlp_loss(model, X, y):
    """(1/2m) * sum of squared output errors (problems.py, MlpOracle loss)."""
    r = model(X)[:, 0] - y
    return 0.5 * (r * r).mean()

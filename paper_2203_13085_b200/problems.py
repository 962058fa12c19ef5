"""Learning-rate schedule (mirror of problems.py:322-365 of the reference).

The rate is a host scalar; the K5 kernel rounds it to the element type
(``(float)(-lr)``), exactly as numpy's NEP 50 does for ``f32_array * -eta``.
The reference's datasets and gradient oracles (problems.py:21-315) are not
part of the sync path — forward/backward stays in PyTorch; the config-1
restatement used by the parity tests lives in oracle/problems_oracle.py.
"""

from __future__ import annotations

from dataclasses import dataclass


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

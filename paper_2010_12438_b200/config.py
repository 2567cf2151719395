"""Configuration dataclasses mirroring the reference (embedding.py:17-21,
policy.py:18-41, simulator.py:24-28,80-83, training.py:28,47-67)."""
from __future__ import annotations

from dataclasses import dataclass

TASK_ORDER = ("placement", "schedule_priority", "fusion_priority")
TASKS = TASK_ORDER
NUM_PRIORITY_LEVELS = 8
INVALID_REWARD = -10.0


@dataclass(frozen=True)
class EmbedConfig:
    gs_layers: int = 4
    gs_dim: int = 128
    gs_knn: int = 5


@dataclass(frozen=True)
class PolicyConfig:
    trf_layers: int = 4
    d_model: int = 128
    n_head: int = 3
    d_head: int = 15
    d_inner: int = 512
    segment_len: int = 64
    iterations: int = 2

    @property
    def attn_width(self) -> int:
        return self.n_head * self.d_head


@dataclass
class FusionConfig:
    max_group: int = 8
    num_levels: int = NUM_PRIORITY_LEVELS


@dataclass
class PPOHyper:
    """training.py:47-67 (same defaults and validation)."""

    lr: float = 1e-3
    rollouts: int = 800
    minibatches: int = 40
    epochs: int = 20
    clip_epsilon: float = 0.2
    entropy_coef: float = 0.5
    value_coef: float = 1.0
    temperature: float = 1.0
    advantage_norm: bool = True

    def __post_init__(self):
        if min(self.lr, self.rollouts, self.minibatches, self.epochs) <= 0:
            raise ValueError("hyperparameters must be positive")
        if not (0.0 < self.clip_epsilon < 1.0):
            raise ValueError("clip epsilon must be in (0,1)")


def ordered_tasks(task_sizes: dict) -> list[tuple[str, int]]:
    """policy.py:36-41."""
    unknown = set(task_sizes) - set(TASK_ORDER)
    if unknown:
        raise ValueError(f"unknown tasks: {sorted(unknown)}")
    return [(t, task_sizes[t]) for t in TASK_ORDER if t in task_sizes]

"""DST mask-update API: schedules, budgets and the device TopK entry points.

Host-scalar parts (schedules, budget allocation, K rule) mirror the reference's
``selection.py`` / ``diagcore.py`` with the same names, argument meaning and
exceptions; the per-candidate work (soft TopK, its gradient, hard TopK) runs
on the GPU through ``ops`` (K4/K5 in ``csrc/topk_kernels.cu``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import EmptyLayerList, NonPositiveTemperature, ShapeMismatch, StepOutOfRange
from .ops import select_hard, soft_topk, soft_topk_grad, soft_topk_select  # noqa: F401

EPS_ACTIVE = 1e-3  # layers.py:41


def candidate_count(rows: int, cols: int) -> int:
    """diagcore.py:22-26."""
    if rows < 1 or cols < 1:
        raise ShapeMismatch(f"dimensions must be positive, got {rows}x{cols}")
    return max(rows, cols)


def required_diagonals(rows: int, cols: int, sparsity: float) -> int:
    """diagcore.py:29-48: K = floor((1-s) M N / min(M,N) + 0.5) clamped to [1, C]."""
    s = float(sparsity)
    if not 0.0 <= s < 1.0:
        raise ValueError(f"sparsity must be in [0, 1), got {sparsity}")
    k = math.floor((1.0 - s) * rows * cols / min(rows, cols) + 0.5)
    return max(1, min(candidate_count(rows, cols), k))


@dataclass(frozen=True)
class TemperatureSchedule:
    """selection.py:43-58."""

    kind: str = "cosine"
    t_init: float = 4.0
    t_final: float = 0.05
    total_steps: int = 1

    def __post_init__(self) -> None:
        if self.kind not in ("constant", "linear", "cosine"):
            raise ValueError(f"unknown schedule kind {self.kind!r}")
        if not self.t_init >= self.t_final > 0:
            raise NonPositiveTemperature(
                f"need t_init >= t_final > 0, got {self.t_init}, {self.t_final}")
        if self.total_steps < 1:
            raise ValueError("total_steps must be positive")


@dataclass(frozen=True)
class SparsitySchedule:
    """selection.py:61-76."""

    kind: str = "constant"
    s_init: float = 0.0
    s_final: float = 0.9
    total_steps: int = 1

    def __post_init__(self) -> None:
        if self.kind not in ("constant", "linear", "cosine"):
            raise ValueError(f"unknown schedule kind {self.kind!r}")
        if not (0 <= self.s_init < 1 and 0 <= self.s_final < 1):
            raise ValueError("sparsities must lie in [0, 1)")
        if self.s_init > self.s_final:
            raise ValueError("s_init must not exceed s_final")
        if self.total_steps < 1:
            raise ValueError("total_steps must be positive")


@dataclass(frozen=True)
class BudgetAllocation:
    """selection.py:79-88."""

    method: str = "uniform"
    global_sparsity: float = 0.9

    def __post_init__(self) -> None:
        if self.method not in ("uniform", "erk", "compute_fraction"):
            raise ValueError(f"unknown allocation method {self.method!r}")
        if not 0 <= self.global_sparsity < 1:
            raise ValueError("global_sparsity must be in [0, 1)")


def _interp(kind: str, a: float, b: float, step: int, total: int) -> float:
    frac = step / total
    if kind == "linear":
        return a + (b - a) * frac
    return b + 0.5 * (a - b) * (1.0 + float(np.cos(np.pi * frac)))


def temperature_at(step: int, sched: TemperatureSchedule) -> float:
    """selection.py:189-200."""
    if not 0 <= step <= sched.total_steps:
        raise StepOutOfRange(f"step {step} outside [0, {sched.total_steps}]")
    if sched.kind == "constant":
        return sched.t_init
    return _interp(sched.kind, sched.t_init, sched.t_final, step, sched.total_steps)


def sparsity_at(step: int, sched: SparsitySchedule) -> float:
    """selection.py:203-214."""
    if not 0 <= step <= sched.total_steps:
        raise StepOutOfRange(f"step {step} outside [0, {sched.total_steps}]")
    if sched.kind == "constant":
        return sched.s_final
    return _interp(sched.kind, sched.s_init, sched.s_final, step, sched.total_steps)


def allocate_budgets(layer_shapes, alloc: BudgetAllocation) -> list[float]:
    """selection.py:225-262: per-layer sparsities meeting the global nonzero budget."""
    shapes = [(int(m), int(n)) for m, n in layer_shapes]
    if not shapes:
        raise EmptyLayerList("need at least one layer shape")
    if alloc.method == "uniform":
        return [alloc.global_sparsity for _ in shapes]
    sizes = np.array([m * n for m, n in shapes], dtype=np.float64)
    if alloc.method == "erk":
        raw = np.array([(m + n) / (m * n) for m, n in shapes])
    else:
        raw = sizes / sizes.sum()
    budget = (1.0 - alloc.global_sparsity) * sizes.sum()
    dense = np.zeros(len(shapes), dtype=bool)
    densities = np.ones(len(shapes))
    for _ in range(len(shapes)):
        free = ~dense
        if not free.any():
            break
        scale = (budget - sizes[dense].sum()) / float((raw[free] * sizes[free]).sum())
        cand = scale * raw
        over = free & (cand >= 1.0)
        if not over.any():
            densities[free] = cand[free]
            break
        dense |= over
    return [float(1.0 - d) for d in densities]


def layer_diagonal_counts(layer_shapes, alloc: BudgetAllocation) -> list[int]:
    """selection.py:265-270."""
    rhos = allocate_budgets(layer_shapes, alloc)
    return [required_diagonals(m, n, r) for (m, n), r in zip(layer_shapes, rhos)]


def schedule_layer_budgets(layers, budget_method: str, step: int, s_sched: SparsitySchedule) -> float:
    """training.py:608-619: set every DiagLinear's k from the sparsity schedule."""
    s_t = sparsity_at(min(step, s_sched.total_steps), s_sched)
    if layers:
        shapes = [(lyr.out_features, lyr.in_features) for lyr in layers]
        for lyr, s_layer in zip(layers, allocate_budgets(shapes, BudgetAllocation(budget_method, s_t))):
            lyr.set_k(required_diagonals(lyr.out_features, lyr.in_features, s_layer))
    return s_t

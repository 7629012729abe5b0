"""Soft/hard TopK diagonal selection and schedules (float64) — TEST INFRASTRUCTURE ONLY.

Restates reference ``pkg/src/diagsparse/selection.py`` and the active-set rule
of ``layers.py:41,234``.
"""

from __future__ import annotations

import numpy as np

from .geometry import required_diagonals

EPS_ACTIVE = 1e-3  # layers.py:41


def _validate(alpha, k: int, temperature: float) -> np.ndarray:
    """selection.py:91-97."""
    a = np.asarray(alpha, dtype=np.float64)
    if temperature <= 0:
        raise ValueError(f"temperature must be positive, got {temperature}")
    if not (1 <= k <= a.size):
        raise ValueError(f"k={k} outside [1, {a.size}]")
    return a


def waterfill(z: np.ndarray, k: int):
    """selection.py:100-124 — capped budget redistribution over softmax(z).

    Returns (tilde, clamped, m, order): ``order`` is the stable descending sort
    of z (ties to the smaller index), ``m`` the number of clamped entries.
    suffix[i] = logsumexp(z_sorted[i:]) is accumulated from the tail with
    ``np.logaddexp`` exactly as the reference does (selection.py:112).
    """
    n = z.size
    order = np.argsort(-z, kind="stable")
    zs = z[order]
    tail = np.logaddexp.accumulate(zs[::-1])[::-1]
    lim = min(k, n)
    share = (k - np.arange(lim)) * np.exp(zs[:lim] - tail[:lim])
    ok = share >= 1.0
    m = lim if bool(ok.all()) else int(np.argmin(ok))
    tilde = np.empty(n)
    clamped = np.zeros(n, dtype=bool)
    head, rest = order[:m], order[m:]
    clamped[head] = True
    tilde[head] = 1.0
    if rest.size:
        tilde[rest] = (k - m) * np.exp(zs[m:] - tail[m])
    return tilde, clamped, m, order


def soft_topk(alpha, k: int, temperature: float) -> np.ndarray:
    """selection.py:127-142."""
    a = _validate(alpha, k, temperature)
    return waterfill(a / temperature, k)[0]


def soft_topk_grad(alpha, k: int, temperature: float, upstream) -> np.ndarray:
    """selection.py:145-173 — d<upstream, soft_topk>/d alpha; clamped entries get 0."""
    a = _validate(alpha, k, temperature)
    up = np.asarray(upstream, dtype=np.float64)
    if up.shape != a.shape:
        raise ValueError("upstream must match alpha's shape")
    _, clamped, _, _ = waterfill(a / temperature, k)
    g = np.zeros_like(a)
    free = ~clamped
    budget = k - int(clamped.sum())
    if not free.any() or budget <= 0:
        return g
    z = a[free] / temperature
    q = np.exp(z - z.max())
    q /= q.sum()
    w = up[free] * q
    g[free] = (budget / temperature) * (w - q * w.sum())
    return g


def select_hard(alpha, k: int) -> np.ndarray:
    """selection.py:176-186 — indices of the k largest, ties to the smaller index, ascending."""
    a = np.asarray(alpha, dtype=np.float64)
    if not (1 <= k <= a.size):
        raise ValueError(f"k={k} outside [1, {a.size}]")
    return np.sort(np.argsort(-a, kind="stable")[:k])


def active_offsets(alpha_soft: np.ndarray) -> np.ndarray:
    """layers.py:234 — candidates whose soft score reaches EPS_ACTIVE, ascending."""
    return np.flatnonzero(alpha_soft >= EPS_ACTIVE)


def _schedule(kind: str, start: float, end: float, step: int, total: int) -> float:
    """Shared body of selection.py:189-214."""
    if not (0 <= step <= total):
        raise ValueError(f"step {step} outside [0, {total}]")
    if kind == "constant":
        return None  # caller decides which endpoint a constant schedule holds
    frac = step / total
    if kind == "linear":
        return start + (end - start) * frac
    return end + 0.5 * (start - end) * (1.0 + np.cos(np.pi * frac))


def temperature_at(step: int, kind: str, t_init: float, t_final: float, total: int) -> float:
    """selection.py:189-200 (constant schedules hold t_init)."""
    v = _schedule(kind, t_init, t_final, step, total)
    return t_init if v is None else v


def sparsity_at(step: int, kind: str, s_init: float, s_final: float, total: int) -> float:
    """selection.py:203-214 (constant schedules hold s_final)."""
    v = _schedule(kind, s_init, s_final, step, total)
    return s_final if v is None else v


def l1_term(alpha, coeff: float):
    """selection.py:217-222 — (coeff * sum|alpha|, coeff * sign(alpha)), sign(0) = 0."""
    if coeff < 0:
        raise ValueError("l1 coefficient must be nonnegative")
    a = np.asarray(alpha, dtype=np.float64)
    return coeff * float(np.abs(a).sum()), coeff * np.sign(a)


def allocate_budgets(layer_shapes, method: str, global_sparsity: float) -> list[float]:
    """selection.py:225-262 — per-layer sparsities meeting a global nonzero budget."""
    shapes = [(int(m), int(n)) for m, n in layer_shapes]
    if not shapes:
        raise ValueError("need at least one layer shape")
    if method == "uniform":
        return [global_sparsity] * len(shapes)
    size = np.array([m * n for m, n in shapes], dtype=np.float64)
    if method == "erk":
        raw = np.array([(m + n) / (m * n) for m, n in shapes])
    elif method == "compute_fraction":
        raw = size / size.sum()
    else:
        raise ValueError(f"unknown allocation method {method!r}")
    budget = (1.0 - global_sparsity) * size.sum()
    dense = np.zeros(len(shapes), dtype=bool)
    dens = np.ones(len(shapes))
    for _ in range(len(shapes)):
        free = ~dense
        if not free.any():
            break
        scale = (budget - size[dense].sum()) / float((raw[free] * size[free]).sum())
        cand = scale * raw
        over = free & (cand >= 1.0)
        if not over.any():
            dens[free] = cand[free]
            break
        dense |= over
    return [float(1.0 - d) for d in dens]


def layer_diagonal_counts(layer_shapes, method: str, global_sparsity: float) -> list[int]:
    """selection.py:265-270."""
    rho = allocate_budgets(layer_shapes, method, global_sparsity)
    return [required_diagonals(m, n, r) for (m, n), r in zip(layer_shapes, rho)]

"""DynaDiag layer step, optimizer and DiagHeur update (float64) — TEST INFRASTRUCTURE ONLY.

Restates reference ``layers.py`` (``DynaDiagLayer``, ``_record_diag_matmul``,
``diagheur_update``) and ``training.py`` (``adamw_step``, ``clip_global_norm``,
``lr_at``) without the tape: forward returns what backward needs, backward
returns the gradients the tape would accumulate.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import ceil, sqrt

import numpy as np

from .geometry import candidate_count, csr_spmm, diag_spmm, entry_coords, required_diagonals, transpose_diagonals
from .topk import EPS_ACTIVE, l1_term, select_hard, soft_topk, soft_topk_grad, temperature_at


def _product(rows, cols, offsets, vals, X, use_csr):
    """layers.py:133-137 — blocked (scipy CSR) product while few diagonals are active,
    the diagonal-by-diagonal reference product otherwise."""
    if use_csr:
        return csr_spmm(rows, cols, offsets, vals, X)
    return diag_spmm(rows, cols, offsets, vals, X)


def diag_matmul_forward(x, weights, active, rows, cols, use_csr=False):
    """layers.py:126-137: y = x @ W^T for W built from the active diagonals' weights."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] != cols:
        raise ValueError(f"input has shape {x.shape}, expected (B, {cols})")
    return _product(rows, cols, list(int(a) for a in active), weights, x.T, use_csr).T


def diag_matmul_backward(up, x, values, weights, active, rows, cols, alpha=None,
                         alpha_soft=None, k=None, temperature=None, use_csr=False):
    """layers.py:143-167 — (gx, g_values[, g_alpha]) for upstream ``up`` (B, M)."""
    offs = [int(a) for a in active]
    offs_t, w_t = transpose_diagonals(rows, cols, offs, weights)
    gx = _product(cols, rows, offs_t, w_t, np.asarray(up).T, use_csr).T
    L = min(rows, cols)
    n_act = len(offs)
    r_idx, c_idx = entry_coords(rows, cols, offs)
    if 4 * n_act * L >= rows * cols:
        gw = (up.T @ x)[r_idx, c_idx]
    else:
        gw = np.empty((n_act, L))
        for j in range(n_act):
            gw[j] = (up[:, r_idx[j]] * x[:, c_idx[j]]).sum(axis=0)
    g_values = np.zeros_like(values)
    if alpha is None:
        g_values[offs] = gw
        return gx, g_values
    g_values[offs] = alpha_soft[offs, None] * gw
    g_soft = np.zeros(values.shape[0])
    g_soft[offs] = (gw * values[offs]).sum(axis=1)
    return gx, g_values, soft_topk_grad(alpha, k, temperature, g_soft)


@dataclass
class OracleDiagLayer:
    """State of ``DynaDiagLayer`` (layers.py:173-287) with the same init stream."""

    in_features: int
    out_features: int
    sparsity: float = 0.9
    t_kind: str = "cosine"
    t_init: float = 4.0
    t_final: float = 0.05
    t_total: int = 1
    l1_coeff: float = 1e-4
    bias: bool = True
    seed: int = 0
    values: np.ndarray = field(init=False)
    alpha: np.ndarray = field(init=False)
    b: np.ndarray | None = field(init=False)

    def __post_init__(self):
        M, N = self.out_features, self.in_features
        self.C = candidate_count(M, N)
        self.L = min(M, N)
        self.k = required_diagonals(M, N, self.sparsity)
        rng = np.random.default_rng(self.seed)          # layers.py:201-208, same draw order
        bound = sqrt(1.0 / N)
        self.values = rng.uniform(-bound, bound, (self.C, self.L))
        self.alpha = rng.normal(0.0, 0.01, self.C)
        self.b = np.zeros(M) if self.bias else None

    def temperature(self, step: int) -> float:
        """layers.py:217-219."""
        return temperature_at(min(step, self.t_total), self.t_kind, self.t_init, self.t_final, self.t_total)

    def select(self, step: int):
        T = self.temperature(step)
        a_soft = soft_topk(self.alpha, self.k, T)
        return T, a_soft, np.flatnonzero(a_soft >= EPS_ACTIVE)

    def forward(self, x, step: int):
        """layers.py:230-251 -> (y, cache for backward)."""
        T, a_soft, active = self.select(step)
        weights = a_soft[active, None] * self.values[active]
        use_csr = active.size <= 2 * self.k
        y = diag_matmul_forward(x, weights, active, self.out_features, self.in_features, use_csr)
        if self.b is not None:
            y = y + self.b
        return y, (np.asarray(x, dtype=np.float64), T, a_soft, active, weights, use_csr)

    def backward(self, up, cache):
        """Tape.backward of the layer op + add_bias (autodiff.py:72-81) -> dict of grads."""
        x, T, a_soft, active, weights, use_csr = cache
        gx, g_values, g_alpha = diag_matmul_backward(
            up, x, self.values, weights, active, self.out_features, self.in_features,
            alpha=self.alpha, alpha_soft=a_soft, k=self.k, temperature=T, use_csr=use_csr)
        grads = {"x": gx, "values": g_values, "alpha": g_alpha}
        if self.b is not None:
            grads["bias"] = up.sum(axis=0)
        return grads

    def penalty_grad(self):
        """layers.py:253-257 via l1_term."""
        return l1_term(self.alpha, self.l1_coeff)

    def params(self):
        """layers.py:259-266: (name, array, decay)."""
        out = [("values", self.values, True), ("alpha", self.alpha, False)]
        if self.b is not None:
            out.append(("bias", self.b, False))
        return out

    def freeze(self):
        """layers.py:277-287 -> (offsets, baked values)."""
        sel = select_hard(self.alpha, self.k)
        a_soft = soft_topk(self.alpha, self.k, self.t_final)
        return sel, a_soft[sel, None] * self.values[sel]


def adamw_update(param, grad, state: dict, *, lr, beta1, beta2, eps, weight_decay):
    """training.py:346-358 — returns the new param, mutates state (m, v, t)."""
    state["t"] += 1
    t = state["t"]
    state["m"] = beta1 * state["m"] + (1.0 - beta1) * grad
    state["v"] = beta2 * state["v"] + (1.0 - beta2) * grad * grad
    m_hat = state["m"] / (1.0 - beta1 ** t)
    v_hat = state["v"] / (1.0 - beta2 ** t)
    return param - lr * (m_hat / (np.sqrt(v_hat) + eps) + weight_decay * param)


def clip_by_global_norm(grads: list, max_norm: float):
    """training.py:406-417 — returns (scaled grads, norm)."""
    total = 0.0
    for g in grads:
        total += float((g ** 2).sum())
    norm = np.sqrt(total)
    if norm > max_norm and norm > 0:
        s = max_norm / norm
        grads = [g * s for g in grads]
    return grads, norm


def lr_at(step: int, total: int, warmup: float, lr_peak: float, lr_final: float = 0.0) -> float:
    """training.py:393-403."""
    if step > total:
        raise ValueError(f"step {step} beyond total {total}")
    if warmup > 0 and step < warmup:
        return lr_peak * step / warmup
    if total <= warmup:
        return lr_peak
    frac = (step - warmup) / (total - warmup)
    return lr_final + 0.5 * (lr_peak - lr_final) * (1.0 + np.cos(np.pi * frac))


def diagheur_swap(values, active, k, candidates, prune_fraction, rng, step=None, total_steps=None):
    """layers.py:381-413 — returns (new values, new active)."""
    frac = prune_fraction
    if step is not None and total_steps:
        frac = frac * 0.5 * (1.0 + np.cos(np.pi * min(step, total_steps) / total_steps))
    n = min(ceil(frac * k), candidates - k)
    if n <= 0:
        return values, active
    norms = np.linalg.norm(values[active], axis=1)
    order = np.lexsort((active, norms))
    survivors = np.setdiff1d(active, active[order[:n]])
    free = np.ones(candidates, dtype=bool)
    free[active] = False
    grown = rng.choice(np.flatnonzero(free), n, replace=False)
    values = values.copy()
    values[grown] = 0.0
    return values, np.sort(np.concatenate([survivors, grown]))


def layer_train_step(layer: OracleDiagLayer, x, up, step: int, opt_state: dict, *, lr=1e-3,
                     betas=(0.9, 0.99), eps=1e-8, weight_decay=5e-5, grad_clip=1.0):
    """One reference layer step as bench_train_step times it (bench.py:168-179):
    forward, backward (+l1 penalty), clip_global_norm, AdamW over all params."""
    y, cache = layer.forward(x, step)
    grads = layer.backward(up, cache)
    if layer.l1_coeff > 0:
        grads["alpha"] = grads["alpha"] + layer.penalty_grad()[1]
    names = [n for n, _, _ in layer.params()]
    scaled, _ = clip_by_global_norm([grads[n] for n in names], grad_clip)
    for (name, arr, decay), g in zip(layer.params(), scaled):
        st = opt_state.setdefault(name, {"m": np.zeros_like(arr), "v": np.zeros_like(arr), "t": 0})
        new = adamw_update(arr, g, st, lr=lr, beta1=betas[0], beta2=betas[1], eps=eps,
                           weight_decay=weight_decay if decay else 0.0)
        if name == "values":
            layer.values = new
        elif name == "alpha":
            layer.alpha = new
        else:
            layer.b = new
    return y, grads

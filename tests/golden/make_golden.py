"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  These fixtures pin the oracle (``oracle/``)
and are the ground truth the CUDA path is checked against at small sizes; the
GPU box never reads /root/reference.  Re-running reproduces them bit-for-bit
(all inputs come from fixed seeds).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("DIAGSPARSE_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

from diagsparse import autodiff, diagcore, layers, selection, training  # noqa: E402

OUT = Path(__file__).resolve().parent

# (M, N, K, B, seed): tall, wide, square, degenerate, dense-switch shapes
SPMM_CASES = [
    (8, 6, 3, 5, 0), (6, 8, 3, 5, 1), (7, 7, 4, 3, 2), (32, 24, 5, 7, 3), (24, 32, 5, 7, 4),
    (16, 16, 16, 2, 5), (48, 96, 40, 4, 6), (96, 48, 10, 9, 7), (1, 5, 2, 3, 8), (5, 1, 1, 2, 9),
    (3, 2, 2, 1, 10), (2, 5, 3, 4, 11), (64, 256, 26, 6, 12), (256, 64, 26, 6, 13), (40, 40, 1, 3, 14),
]

# (C, k, T, seed, scale, pattern)
TOPK_CASES = []
for C, ks in ((1, (1,)), (2, (1, 2)), (5, (1, 3, 5)), (8, (3,)), (33, (4, 17)), (100, (10, 50)),
              (768, (77,)), (3072, (307,))):
    for k in ks:
        for T in ((4.0, 0.5, 0.05, 1e-3, 1e-9) if C <= 768 else (4.0, 1e-3, 1e-9)):
            TOPK_CASES.append((C, k, T, 1000 + C + k, 1.0, "normal"))
TOPK_CASES += [
    (12, 4, 0.7, 7, 1.0, "ties"), (12, 4, 1e-9, 7, 1.0, "ties"), (9, 3, 0.3, 8, 1.0, "signed_zero"),
    (64, 8, 0.05, 9, 5.0, "normal"), (64, 60, 0.2, 10, 3.0, "normal"), (16, 16, 0.9, 11, 1.0, "normal"),
    (4, 2, 0.9, 12, 1.0, "uniform"),
]

# (in, out, sparsity, T, B, seed, alpha_noise)
LAYER_CASES = [
    (24, 32, 0.8, 0.7, 4, 1, 1.0), (32, 24, 0.8, 0.7, 4, 2, 1.0), (20, 20, 0.6, 0.7, 3, 3, 1.0),
    (48, 96, 0.5, 0.7, 5, 4, 1.0), (64, 256, 0.9, 0.05, 6, 5, 1.0), (256, 64, 0.9, 1e-3, 6, 6, 1.0),
    (16, 16, 0.75, 4.0, 2, 7, 0.0), (12, 12, 0.8, 1e-9, 3, 8, 2.0), (5, 7, 0.5, 0.9, 2, 9, 0.5),
]


def topk_alpha(C, seed, scale, pattern):
    rng = np.random.default_rng(seed)
    if pattern == "ties":
        return np.round(rng.standard_normal(C) * 2.0) / 2.0
    if pattern == "signed_zero":
        a = rng.standard_normal(C)
        a[[1, 4]] = -0.0
        a[[2, 6]] = 0.0
        return a
    if pattern == "uniform":
        return np.full(C, 0.3)
    return rng.standard_normal(C) * scale


def gen_spmm():
    out = {}
    for i, (M, N, K, B, seed) in enumerate(SPMM_CASES):
        rng = np.random.default_rng(seed)
        C = max(M, N)
        offs = np.sort(rng.choice(C, K, replace=False))
        vals = rng.standard_normal((K, min(M, N)))
        X = rng.standard_normal((N, B))
        m = diagcore.DiagSparseMatrix(diagcore.build_pattern(M, N, offs), vals)
        t = diagcore.transpose(m)
        U = rng.standard_normal((M, B))
        out[f"c{i}_shape"] = np.array([M, N, K, B])
        out[f"c{i}_offsets"] = offs
        out[f"c{i}_values"] = vals
        out[f"c{i}_X"] = X
        out[f"c{i}_Y"] = diagcore.reference_spmm(m, X)
        out[f"c{i}_dense"] = diagcore.materialize(m)
        out[f"c{i}_T_offsets"] = np.array(t.pattern.offsets)
        out[f"c{i}_T_values"] = t.values
        out[f"c{i}_U"] = U
        out[f"c{i}_TU"] = diagcore.reference_spmm(t, U)
    np.savez_compressed(OUT / "spmm.npz", n=len(SPMM_CASES), **out)


def gen_topk():
    out = {}
    for i, (C, k, T, seed, scale, pattern) in enumerate(TOPK_CASES):
        alpha = topk_alpha(C, seed, scale, pattern)
        up = np.random.default_rng(seed + 1).standard_normal(C)
        tilde, clamped = selection._waterfill(alpha / T, k)
        out[f"c{i}_meta"] = np.array([C, k, T])
        out[f"c{i}_alpha"] = alpha
        out[f"c{i}_up"] = up
        out[f"c{i}_soft"] = selection.soft_topk(alpha, k, T)
        out[f"c{i}_tilde"] = tilde
        out[f"c{i}_clamped"] = clamped
        out[f"c{i}_active"] = np.flatnonzero(tilde >= layers.EPS_ACTIVE)
        out[f"c{i}_hard"] = selection.select_hard(alpha, k)
        out[f"c{i}_grad"] = selection.soft_topk_grad(alpha, k, T, up)
        out[f"c{i}_l1grad"] = selection.l1_term(alpha, 1e-2)[1]
    np.savez_compressed(OUT / "topk.npz", n=len(TOPK_CASES), **out)


class _Dot:
    """Scalar loss sum(y * up) recorded on the reference tape as a custom op."""

    @staticmethod
    def apply(tape, y, up):
        out = autodiff.Tensor(float((y.value * up).sum()))
        return tape.record(out, (y,), lambda g: (float(g) * up,))


def gen_layers():
    out = {}
    for i, (n_in, n_out, s, T, B, seed, noise) in enumerate(LAYER_CASES):
        sched = selection.TemperatureSchedule("constant", T, T, 10)
        lyr = layers.DynaDiagLayer(n_in, n_out, s, t_schedule=sched, seed=seed, l1_coeff=1e-2)
        rng = np.random.default_rng(100 + seed)
        out[f"c{i}_values0"] = lyr.values.value.copy()
        out[f"c{i}_alpha0"] = lyr.alpha.value.copy()
        lyr.alpha.value = lyr.alpha.value + rng.standard_normal(lyr.candidates) * noise
        lyr.bias.value = rng.standard_normal(n_out) * 0.1
        x = autodiff.Tensor(rng.standard_normal((B, n_in)), requires_grad=True)
        up = rng.standard_normal((B, n_out))
        out[f"c{i}_meta"] = np.array([n_in, n_out, s, T, B, seed, noise, lyr.k])
        out[f"c{i}_alpha"] = lyr.alpha.value.copy()
        out[f"c{i}_bias"] = lyr.bias.value.copy()
        out[f"c{i}_x"] = x.value.copy()
        out[f"c{i}_up"] = up
        tape = autodiff.Tape()
        y = lyr.forward(x, tape, step=0)
        loss = _Dot.apply(tape, y, up)
        loss = tape.add(loss, lyr.penalty(tape))
        for p in (lyr.values, lyr.alpha, lyr.bias):
            p.zero_grad()
        tape.backward(loss)
        out[f"c{i}_y"] = y.value
        out[f"c{i}_active"] = lyr.active_set(0)
        out[f"c{i}_soft"] = lyr.soft_scores(0)
        out[f"c{i}_gx"] = x.grad
        out[f"c{i}_gvalues"] = lyr.values.grad
        out[f"c{i}_galpha"] = lyr.alpha.grad
        out[f"c{i}_gbias"] = lyr.bias.grad
        frozen = lyr.freeze()
        out[f"c{i}_frozen_offsets"] = np.array(frozen.weight.pattern.offsets)
        out[f"c{i}_frozen_values"] = frozen.weight.values
        out[f"c{i}_frozen_y"] = frozen.forward(x.value)
    np.savez_compressed(OUT / "layers.npz", n=len(LAYER_CASES), **out)


def gen_trajectory():
    """Five reference training steps of one layer: forward, backward (+l1),
    clip_global_norm, AdamW — masks and parameters after every step."""
    out = {}
    sched = selection.TemperatureSchedule("cosine", 2.0, 0.05, 5)
    lyr = layers.DynaDiagLayer(32, 48, 0.8, t_schedule=sched, seed=21, l1_coeff=1e-3)
    rng = np.random.default_rng(22)
    lyr.alpha.value = lyr.alpha.value + rng.standard_normal(lyr.candidates)
    params = lyr.parameters()
    cfg = training.OptimizerConfig(lr=5e-2)
    opt = training.AdamW(params, cfg)
    xs = rng.standard_normal((5, 6, 32))
    ups = rng.standard_normal((5, 6, 48))
    out["alpha_init"] = lyr.alpha.value.copy()
    out["xs"], out["ups"] = xs, ups
    for s in range(5):
        tape = autodiff.Tape()
        x = autodiff.Tensor(xs[s])
        y = lyr.forward(x, tape, step=s)
        loss = tape.add(_Dot.apply(tape, y, ups[s]), lyr.penalty(tape))
        opt.zero_grad()
        tape.backward(loss)
        norm = training.clip_global_norm(params, 1.0)
        opt.step(cfg.lr)
        out[f"s{s}_y"] = y.value
        out[f"s{s}_active"] = lyr.active_set(s)
        out[f"s{s}_norm"] = np.array(norm)
        out[f"s{s}_values"] = lyr.values.value.copy()
        out[f"s{s}_alpha"] = lyr.alpha.value.copy()
        out[f"s{s}_bias"] = lyr.bias.value.copy()
    np.savez_compressed(OUT / "trajectory.npz", **out)


def gen_misc():
    out = {}
    # adamw_step / clip_global_norm
    rng = np.random.default_rng(31)
    p0, g0 = rng.standard_normal(50), rng.standard_normal(50)
    p, g = p0.copy(), g0.copy()
    st = {"m": np.zeros(50), "v": np.zeros(50), "t": 0}
    seq = []
    for _ in range(3):
        p = training.adamw_step(p, g, st, lr=1e-2, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=5e-5)
        seq.append(p.copy())
        g = g * 0.5 + 0.1
    out["adamw_p0"], out["adamw_g0"] = p0, g0
    out["adamw_seq"] = np.array(seq)
    # diagheur_update
    h = layers.DiagHeurLayer(24, 40, 0.8, seed=41, prune_fraction=0.3)
    out["heur_active0"] = h.active.copy()
    out["heur_values0"] = h.values.value.copy()
    layers.diagheur_update(h, np.random.default_rng(42), step=10, total_steps=100)
    out["heur_active1"] = h.active.copy()
    out["heur_values1"] = h.values.value.copy()
    # K rule and budgets
    shapes = [(256, 784), (256, 256), (10, 256), (3072, 768), (768, 3072), (2304, 768), (768, 768)]
    out["k_rule"] = np.array([diagcore.required_diagonals(m, n, 0.9) for m, n in shapes])
    for meth in ("uniform", "erk", "compute_fraction"):
        out[f"budget_{meth}"] = np.array(
            selection.allocate_budgets(shapes, selection.BudgetAllocation(meth, 0.9)))
    tsched = selection.TemperatureSchedule("cosine", 4.0, 0.05, 100)
    out["t_cosine"] = np.array([selection.temperature_at(s, tsched) for s in range(0, 101, 5)])
    lsched = selection.TemperatureSchedule("linear", 4.0, 0.05, 100)
    out["t_linear"] = np.array([selection.temperature_at(s, lsched) for s in range(0, 101, 5)])
    ssched = selection.SparsitySchedule("cosine", 0.0, 0.9, 100)
    out["s_cosine"] = np.array([selection.sparsity_at(s, ssched) for s in range(0, 101, 5)])
    out["lr"] = np.array([training.lr_at(s, 100, 10, 1e-3, 1e-6) for s in range(0, 101, 5)])
    np.savez_compressed(OUT / "misc.npz", **out)


if __name__ == "__main__":
    gen_spmm()
    gen_topk()
    gen_layers()
    gen_trajectory()
    gen_misc()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)

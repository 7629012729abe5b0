"""Pin the CPU oracle against vectors produced by the reference itself (CPU only).

Fixtures: tests/golden/*.npz from tests/golden/make_golden.py (which imported
the reference read-only).  Masks, offsets and hard selections are compared
bit-for-bit; floats at the reference's own tolerances (1e-12 spmm, 1e-10 layer).
Also replays the reference's own known-answer tests for this path.
"""

import numpy as np
import pytest

import oracle
from oracle import layer as olayer
from oracle import topk as otopk
from diagtest_util import scaled_err


# ---------------------------------------------------------------- geometry KATs
def test_k_rule_reference_kats():
    # test_diagcore.py:47-59, test_training.py:621-622
    assert oracle.required_diagonals(768, 768, 0.90) == 77
    assert oracle.required_diagonals(4, 4, 0.0) == 4
    assert oracle.required_diagonals(10, 10, 0.9999) == 1
    assert oracle.required_diagonals(5, 5, 0.5) == 3
    assert oracle.required_diagonals(24, 32, 0.75) == 8
    with pytest.raises(ValueError):
        oracle.required_diagonals(4, 4, 1.0)


def test_entry_kats():
    # test_diagcore.py:69-81
    r, c = oracle.entry_coords(3, 2, [0])
    assert set(zip(r[0].tolist(), c[0].tolist())) == {(0, 0), (1, 1)}
    r, c = oracle.entry_coords(3, 2, [1])
    assert set(zip(r[0].tolist(), c[0].tolist())) == {(1, 0), (2, 1)}
    r, c = oracle.entry_coords(2, 5, [4])
    assert set(zip(r[0].tolist(), c[0].tolist())) == {(0, 4), (1, 0)}


def test_k_rule_and_budgets_golden(golden):
    g = golden["misc"]
    shapes = [(256, 784), (256, 256), (10, 256), (3072, 768), (768, 3072), (2304, 768), (768, 768)]
    assert [oracle.required_diagonals(m, n, 0.9) for m, n in shapes] == g["k_rule"].tolist()
    for meth in ("uniform", "erk", "compute_fraction"):
        np.testing.assert_array_equal(otopk.allocate_budgets(shapes, meth, 0.9), g[f"budget_{meth}"])


def test_schedules_golden(golden):
    g = golden["misc"]
    steps = range(0, 101, 5)
    np.testing.assert_array_equal([oracle.temperature_at(s, "cosine", 4.0, 0.05, 100) for s in steps],
                                  g["t_cosine"])
    np.testing.assert_array_equal([oracle.temperature_at(s, "linear", 4.0, 0.05, 100) for s in steps],
                                  g["t_linear"])
    np.testing.assert_array_equal([oracle.sparsity_at(s, "cosine", 0.0, 0.9, 100) for s in steps],
                                  g["s_cosine"])
    np.testing.assert_array_equal([olayer.lr_at(s, 100, 10, 1e-3, 1e-6) for s in steps], g["lr"])


# ---------------------------------------------------------------- spmm
def test_spmm_golden(golden):
    g = golden["spmm"]
    for i in range(int(g["n"])):
        M, N, K, B = g[f"c{i}_shape"].tolist()
        offs, vals = g[f"c{i}_offsets"], g[f"c{i}_values"]
        np.testing.assert_array_equal(oracle.dense_matrix(M, N, offs, vals), g[f"c{i}_dense"])
        Y = oracle.diag_spmm(M, N, offs, vals, g[f"c{i}_X"])
        assert scaled_err(Y, g[f"c{i}_Y"]) <= 1e-12, i
        Yc = oracle.csr_spmm(M, N, offs, vals, g[f"c{i}_X"])
        assert scaled_err(Yc, g[f"c{i}_Y"]) <= 1e-12, i
        to, tv = oracle.transpose_diagonals(M, N, offs, vals)
        np.testing.assert_array_equal(np.array(to), g[f"c{i}_T_offsets"])
        np.testing.assert_array_equal(tv, g[f"c{i}_T_values"])  # pure index remap: bitwise
        TU = oracle.diag_spmm(N, M, to, tv, g[f"c{i}_U"])
        assert scaled_err(TU, g[f"c{i}_TU"]) <= 1e-12, i


# ---------------------------------------------------------------- selection
def test_topk_golden(golden):
    g = golden["topk"]
    for i in range(int(g["n"])):
        C, k, T = g[f"c{i}_meta"]
        C, k = int(C), int(k)
        alpha = g[f"c{i}_alpha"]
        tilde, clamped, _, _ = otopk.waterfill(alpha / T, k)
        np.testing.assert_array_equal(clamped, g[f"c{i}_clamped"])
        np.testing.assert_array_equal(np.flatnonzero(tilde >= otopk.EPS_ACTIVE), g[f"c{i}_active"])
        np.testing.assert_array_equal(tilde, g[f"c{i}_tilde"])  # same numpy ops -> bitwise
        np.testing.assert_array_equal(oracle.select_hard(alpha, k), g[f"c{i}_hard"])
        np.testing.assert_allclose(oracle.soft_topk_grad(alpha, k, T, g[f"c{i}_up"]), g[f"c{i}_grad"],
                                   rtol=1e-12, atol=1e-14)
        np.testing.assert_array_equal(oracle.l1_term(alpha, 1e-2)[1], g[f"c{i}_l1grad"])


def test_topk_reference_kats():
    # test_selection.py:42-58, 151-156
    np.testing.assert_allclose(oracle.soft_topk(np.full(4, 7.5), 2, 0.9), 0.5, rtol=1e-12)
    a = np.array([2.0, 1.0, 0.0])
    np.testing.assert_allclose(oracle.soft_topk(a, 1, 1.0), np.exp(a) / np.exp(a).sum(), rtol=1e-12)
    np.testing.assert_array_equal(oracle.select_hard(np.array([0.5, 0.5, 0.1]), 1), [0])
    with pytest.raises(ValueError):
        oracle.soft_topk(np.zeros(3), 1, 0.0)
    with pytest.raises(ValueError):
        oracle.soft_topk(np.zeros(3), 4, 1.0)


# ---------------------------------------------------------------- layer op
def _oracle_layer_case(g, i):
    n_in, n_out, s, T, B, seed, noise, k = g[f"c{i}_meta"]
    lyr = olayer.OracleDiagLayer(int(n_in), int(n_out), float(s), t_kind="constant", t_init=float(T),
                                 t_final=float(T), t_total=10, l1_coeff=1e-2, seed=int(seed))
    return lyr, int(B), int(k)


def test_layer_init_parity_golden(golden):
    g = golden["layers"]
    for i in range(int(g["n"])):
        lyr, _, k = _oracle_layer_case(g, i)
        assert lyr.k == k
        np.testing.assert_array_equal(lyr.values, g[f"c{i}_values0"])
        np.testing.assert_array_equal(lyr.alpha, g[f"c{i}_alpha0"])


def test_layer_forward_backward_golden(golden):
    g = golden["layers"]
    for i in range(int(g["n"])):
        lyr, _, _ = _oracle_layer_case(g, i)
        lyr.alpha = g[f"c{i}_alpha"].copy()
        lyr.b = g[f"c{i}_bias"].copy()
        y, cache = lyr.forward(g[f"c{i}_x"], 0)
        np.testing.assert_array_equal(cache[3], g[f"c{i}_active"])
        assert scaled_err(y, g[f"c{i}_y"]) <= 1e-10
        grads = lyr.backward(g[f"c{i}_up"], cache)
        grads["alpha"] = grads["alpha"] + lyr.penalty_grad()[1]
        assert scaled_err(grads["x"], g[f"c{i}_gx"]) <= 1e-10
        assert scaled_err(grads["values"], g[f"c{i}_gvalues"]) <= 1e-10
        assert scaled_err(grads["alpha"], g[f"c{i}_galpha"]) <= 1e-10
        assert scaled_err(grads["bias"], g[f"c{i}_gbias"]) <= 1e-12
        inactive = np.setdiff1d(np.arange(lyr.C), g[f"c{i}_active"])
        assert np.all(grads["values"][inactive] == 0.0)
        offs, vals = lyr.freeze()
        np.testing.assert_array_equal(offs, g[f"c{i}_frozen_offsets"])
        assert scaled_err(vals, g[f"c{i}_frozen_values"]) <= 1e-12


def test_layer_trajectory_golden(golden):
    g = golden["trajectory"]
    lyr = olayer.OracleDiagLayer(32, 48, 0.8, t_kind="cosine", t_init=2.0, t_final=0.05, t_total=5,
                                 l1_coeff=1e-3, seed=21)
    lyr.alpha = g["alpha_init"].copy()
    state = {}
    for s in range(5):
        y, _ = olayer.layer_train_step(lyr, g["xs"][s], g["ups"][s], s, state, lr=5e-2)
        _, _, active = lyr.select(s)
        assert scaled_err(y, g[f"s{s}_y"]) <= 1e-10
        assert scaled_err(lyr.values, g[f"s{s}_values"]) <= 1e-9
        assert scaled_err(lyr.alpha, g[f"s{s}_alpha"]) <= 1e-9
        assert scaled_err(lyr.b, g[f"s{s}_bias"]) <= 1e-9
        # the mask after the update (what the next step will use) is exact
        np.testing.assert_array_equal(np.flatnonzero(oracle.soft_topk(lyr.alpha, lyr.k, lyr.temperature(s))
                                                     >= otopk.EPS_ACTIVE), g[f"s{s}_active"])


def test_adamw_and_diagheur_golden(golden):
    g = golden["misc"]
    p, gr = g["adamw_p0"].copy(), g["adamw_g0"].copy()
    st = {"m": np.zeros(50), "v": np.zeros(50), "t": 0}
    for j in range(3):
        p = olayer.adamw_update(p, gr, st, lr=1e-2, beta1=0.9, beta2=0.99, eps=1e-8, weight_decay=5e-5)
        np.testing.assert_array_equal(p, g["adamw_seq"][j])
        gr = gr * 0.5 + 0.1
    vals, act = olayer.diagheur_swap(g["heur_values0"], g["heur_active0"], len(g["heur_active0"]), 40,
                                     0.3, np.random.default_rng(42), step=10, total_steps=100)
    np.testing.assert_array_equal(act, g["heur_active1"])
    np.testing.assert_array_equal(vals, g["heur_values1"])

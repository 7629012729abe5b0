"""K4's top-k radix-select path (k < C, k <= 1024 < C: 8 histogram passes for the k-th
largest key, only the top k sorted, the rest folded into one fixed-order sum)
against the full-sort path and the CPU oracle on adversarial selections: ties
everywhere, tie groups straddling the k-th key, +0.0 / -0.0, k = 1, k = C - 1,
the k = 1024 boundary (1025 falls back to the full sort), every temperature
regime (4 ... 1e-9) and C up to 8192.  Bars: clamped / active sets bit-exact
(the reference's decisions), soft scores within 1e-12 relative of the full-sort
path (the tail sum uses a different fixed order) and of the oracle within 1e-9 or the
reference's own log-space rounding scale C ulp(|alpha| / T), whichever is larger."""

import numpy as np
import pytest
import torch

from oracle import topk as otopk

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_11449_b200 import ops


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _alpha(kind, C, rng):
    if kind == "random":
        return rng.standard_normal(C)
    if kind == "all_equal":
        return np.full(C, 0.37)
    if kind == "tie_groups":  # few distinct values: every threshold falls inside a tie group
        return rng.integers(0, 7, C).astype(np.float64) * 0.25
    if kind == "signed_zeros":
        a = rng.standard_normal(C)
        a[rng.choice(C, C // 3, replace=False)] = 0.0
        a[rng.choice(C, C // 5, replace=False)] = -0.0
        return a
    raise ValueError(kind)


def _run(alpha, k, T, radix, monkeypatch):
    monkeypatch.setenv("DIAGMM_K4_RADIX", "1" if radix else "0")
    sel = ops.soft_topk_select(torch.as_tensor(alpha, device="cuda"), k, T)
    torch.cuda.synchronize()
    n = int(sel.n_act.item())
    return (sel.alpha_soft.cpu().numpy(), sel.clamped.cpu().numpy().astype(bool), sel.active[:n].cpu().numpy())


CASES = ([(C, k) for C in (1025, 3072, 8192) for k in (1, C // 10, C - 1)] + [(4096, 1024), (4096, 1025), (2048, 1023)]
         + [(768, 77)])  # C <= 1024 takes the full sort either way


@pytest.mark.parametrize("kind", ["random", "all_equal", "tie_groups", "signed_zeros"])
@pytest.mark.parametrize("C,k", CASES)
@pytest.mark.parametrize("T", [4.0, 0.05, 1e-3, 1e-9])
def test_radix_path_matches_full_sort_and_oracle(kind, C, k, T, monkeypatch):
    rng = np.random.default_rng(C * 7 + k)
    alpha = _alpha(kind, C, rng)
    s_r, c_r, a_r = _run(alpha, k, T, True, monkeypatch)
    s_f, c_f, a_f = _run(alpha, k, T, False, monkeypatch)
    np.testing.assert_array_equal(c_r, c_f)
    np.testing.assert_array_equal(a_r, a_f)
    np.testing.assert_allclose(s_r, s_f, rtol=1e-12, atol=1e-300)
    ref = otopk.soft_topk(alpha, k, T)
    # the reference accumulates S sequentially in log space: at |z| = |alpha| / T its
    # rounding is ~C ulp(|z|) relative on the scores (1.2e-7 at T = 1e-9, all-equal)
    zmax = float(np.abs(alpha).max()) / T
    np.testing.assert_allclose(s_r, ref, rtol=max(1e-9, C * np.finfo(float).eps * zmax), atol=1e-300)
    np.testing.assert_array_equal(a_r, np.flatnonzero(ref >= 1e-3))

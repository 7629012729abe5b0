"""Host-side logic and the C-ABI library, CPU only (no compute calls)."""

import re
from pathlib import Path

import numpy as np
import pytest
import torch

from diagtest_util import ROOT, load_golden


def header_symbols():
    text = (ROOT / "include" / "diagmm.h").read_text()
    return sorted(set(re.findall(r"DIAGMM_API\s+[\w\s\*]+?\b(diagmm_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2506_11449_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} declared in diagmm.h but not bound in _lib.py"
    assert set(_lib.SIGNATURES) == set(syms)
    assert lib.diagmm_version().decode().endswith("sm_100a")
    assert lib.diagmm_status_string(1).decode() == "shape mismatch"


def test_library_is_sm100a_only():
    import subprocess

    so = ROOT / "paper_2506_11449_b200" / "_lib" / "libdiagmm.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_status_mapping_uses_reference_exceptions():
    from paper_2506_11449_b200 import _lib
    from paper_2506_11449_b200.errors import (DiagSparseError, NonPositiveTemperature, ShapeMismatch)

    with pytest.raises(ShapeMismatch):
        _lib.check(1, "x")
    with pytest.raises(NonPositiveTemperature):
        _lib.check(2, "x")
    with pytest.raises(ValueError):
        _lib.check(3, "x")
    assert issubclass(ShapeMismatch, DiagSparseError) and issubclass(DiagSparseError, ValueError)


def test_workspace_query_is_host_only():
    from paper_2506_11449_b200 import _lib

    lib = _lib.load()
    n = lib.diagmm_backward_weight_workspace(1, 3072, 768, 256, 307)
    assert n > 307 * 768 * 4
    assert lib.diagmm_backward_weight_workspace(1, 0, 768, 256, 0) == 0


def test_no_cpu_fallback():
    from paper_2506_11449_b200 import NativeLibraryError, ops

    a = torch.zeros(8, dtype=torch.float64)
    with pytest.raises(NativeLibraryError):
        ops.soft_topk_select(a, 2, 1.0)
    with pytest.raises(NativeLibraryError):
        ops.diag_forward(torch.zeros(2, 4), torch.zeros(6, 4), None, 6, 4)


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2506_11449_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
        assert "/root/reference" not in src, f


def test_schedules_and_budgets_match_reference(golden=None):
    from paper_2506_11449_b200 import selection as S
    from paper_2506_11449_b200.optim import lr_at

    g = load_golden("misc")
    steps = range(0, 101, 5)
    np.testing.assert_array_equal(
        [S.temperature_at(s, S.TemperatureSchedule("cosine", 4.0, 0.05, 100)) for s in steps], g["t_cosine"])
    np.testing.assert_array_equal(
        [S.temperature_at(s, S.TemperatureSchedule("linear", 4.0, 0.05, 100)) for s in steps], g["t_linear"])
    np.testing.assert_array_equal(
        [S.sparsity_at(s, S.SparsitySchedule("cosine", 0.0, 0.9, 100)) for s in steps], g["s_cosine"])
    np.testing.assert_allclose([lr_at(s, 100, 10, 1e-3, 1e-6) for s in steps], g["lr"], rtol=1e-15)
    shapes = [(256, 784), (256, 256), (10, 256), (3072, 768), (768, 3072), (2304, 768), (768, 768)]
    assert [S.required_diagonals(m, n, 0.9) for m, n in shapes] == g["k_rule"].tolist()
    for meth in ("uniform", "erk", "compute_fraction"):
        np.testing.assert_array_equal(S.allocate_budgets(shapes, S.BudgetAllocation(meth, 0.9)),
                                      g[f"budget_{meth}"])
    with pytest.raises(S.NonPositiveTemperature):
        S.TemperatureSchedule("cosine", 1.0, 0.0, 10)
    with pytest.raises(S.StepOutOfRange):
        S.temperature_at(11, S.TemperatureSchedule("cosine", 1.0, 0.1, 10))
    with pytest.raises(S.EmptyLayerList):
        S.allocate_budgets([], S.BudgetAllocation("erk", 0.9))


def test_vit_layer_k_values():
    """K at 90% for the ViT-B/16 and ViT-Tiny projections."""
    from paper_2506_11449_b200.selection import required_diagonals

    assert required_diagonals(2304, 768, 0.9) == 230
    assert required_diagonals(768, 768, 0.9) == 77
    assert required_diagonals(3072, 768, 0.9) == 307
    assert required_diagonals(768, 3072, 0.9) == 307
    assert required_diagonals(576, 192, 0.9) == 58
    assert required_diagonals(192, 192, 0.9) == 19


def test_vit_patchify_equals_conv():
    """The ViT caller's GEMM patch embedding equals the stride-16 convolution (CPU, fp64)."""
    import torch
    from paper_2506_11449_b200.vit import ViT, ViTConfig

    cfg = ViTConfig(image=32, patch=16, dim=24, depth=0, heads=2, classes=5)
    m = ViT(cfg, device="cpu").double()
    img = torch.randn(3, 3, 32, 32, dtype=torch.float64)
    ref = m.patch(img).flatten(2).transpose(1, 2)
    torch.testing.assert_close(m._patchify(img), ref, rtol=1e-12, atol=1e-12)


def test_diag_matrix_validates_offsets_like_the_reference():
    """DiagonalPattern's checks (diagcore.py:71-88) on the device matrix type:
    OffsetOutOfRange, DuplicateOffset, and unsorted offsets stored ascending."""
    import torch

    from paper_2506_11449_b200.errors import DuplicateOffset, OffsetOutOfRange
    from paper_2506_11449_b200.layer import DiagMatrix

    v = torch.arange(12, dtype=torch.float64).reshape(3, 4)
    with pytest.raises(OffsetOutOfRange):
        DiagMatrix(6, 4, torch.tensor([0, 2, 6]), v)
    with pytest.raises(OffsetOutOfRange):
        DiagMatrix(6, 4, torch.tensor([-1, 2, 3]), v)
    with pytest.raises(DuplicateOffset):
        DiagMatrix(6, 4, torch.tensor([1, 3, 1]), v)
    m = DiagMatrix(6, 4, torch.tensor([5, 0, 2]), v)
    assert m.offsets.tolist() == [0, 2, 5]
    assert m.values[:, 0].tolist() == [4.0, 8.0, 0.0]

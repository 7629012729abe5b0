"""Shared helpers for the test-suite (imported as a top-level module)."""

from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def load_golden(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def scaled_err(got, want) -> float:
    """max|got - want| / max(1, max|want|) — bench._validate's scale (bench.py:66-69)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if want.size == 0:
        return 0.0
    return float(np.abs(got - want).max() / max(1.0, float(np.abs(want).max())))

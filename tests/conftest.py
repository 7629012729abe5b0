"""Test configuration: the ``gpu`` marker and shared fixtures.

``-m "not gpu"``: oracle vs golden vectors, host logic, C-ABI exports (CPU only).
``-m gpu``: CUDA path vs the oracle / golden vectors (needs a B200).
"""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

from diagtest_util import load_golden  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdiagmm.so")


@pytest.fixture(scope="session")
def golden():
    return {n: load_golden(n) for n in ("spmm", "topk", "layers", "trajectory", "misc")}

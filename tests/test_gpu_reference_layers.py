"""The reference's OWN DynaDiagLayer, running its forward/backward through our GPU
op (``tape_adapter.record_diag_matmul`` swapped in for ``_record_diag_matmul``,
the one-assignment integration of INTEGRATION.md §1), checked the way the
reference's ``pkg/tests/test_layers.py`` checks its op:

* forward vs the dense oracle ``materialize(effective_matrix) @ x`` (test_layers.py:25-32);
* the full-layer central-difference ``grad_check`` <= 1e-5 (test_layers.py:80-106),
  i.e. the reference's own autodiff verifying our gradients;
* our backward vs the reference's backward (BCSR and reference paths) at rtol 1e-9
  (test_layers.py:108-135);
* inactive rows get exactly zero gradient (test_layers.py:137-149).

The reference package comes from ``baseline/_ref`` (the offline ``pip install
--target`` of /root/reference/pkg, git-ignored, shipped with the snapshot) or,
in the build container, /root/reference/pkg/src; without either the module skips.
"""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "diagsparse").is_dir() and str(cand) not in sys.path:
        sys.path.append(str(cand))
        break

pytestmark = pytest.mark.gpu
ref = pytest.importorskip("diagsparse")
from diagsparse import layers as rlayers  # noqa: E402
from diagsparse.autodiff import Tape, Tensor, grad_check  # noqa: E402
from diagsparse.diagcore import materialize  # noqa: E402
from diagsparse.selection import TemperatureSchedule  # noqa: E402

_REF_OP = rlayers._record_diag_matmul  # the reference's own op, captured before any monkeypatching


@pytest.fixture
def gpu_op(monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_11449_b200.tape_adapter import record_diag_matmul

    monkeypatch.setattr(rlayers, "_record_diag_matmul", record_diag_matmul)
    return record_diag_matmul


def make_layer(m=6, n=4, sparsity=0.5, seed=0, temperature=0.7, **kw):
    sched = TemperatureSchedule("constant", temperature, temperature, 10)
    return rlayers.DynaDiagLayer(n, m, sparsity, t_schedule=sched, seed=seed, **kw)


def test_reference_layer_forward_matches_dense_oracle(gpu_op):
    rng = np.random.default_rng(0)
    layer = make_layer(m=8, n=6, sparsity=0.4, seed=1)
    x = Tensor(rng.standard_normal((5, 6)))
    out = layer.forward(x, Tape(), step=0)
    W = materialize(layer.effective_matrix(0))
    np.testing.assert_allclose(out.value, x.value @ W.T + layer.bias.value, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("shape", [(6, 4), (4, 6), (5, 5)])
def test_reference_grad_check_through_gpu_op(gpu_op, shape):
    m, n = shape
    rng = np.random.default_rng(5)
    layer = make_layer(m=m, n=n, sparsity=0.5, seed=6, l1_coeff=0.01)
    layer.alpha.value += rng.standard_normal(layer.candidates) * 0.5
    x = Tensor(rng.standard_normal((3, n)), requires_grad=True)
    labels = rng.integers(0, m, 3)

    def f(xs, tape):
        out = layer.forward(xs[0], tape, step=0)
        loss = tape.softmax_cross_entropy(out, labels)
        return tape.add(loss, layer.penalty(tape))

    assert grad_check(f, [x, layer.values, layer.alpha, layer.bias]) <= 1e-5


@pytest.mark.parametrize("use_bcsr", [True, False])
def test_gpu_backward_matches_reference_backward(gpu_op, use_bcsr):
    rng = np.random.default_rng(9)
    layer = make_layer(m=24, n=16, sparsity=0.85, seed=10)
    x_val = rng.standard_normal((4, 16))
    labels = rng.integers(0, 24, 4)
    grads = {}
    for op in ("gpu", "ref"):
        tape = Tape()
        x = Tensor(x_val, requires_grad=True)
        layer.values.zero_grad()
        layer.alpha.zero_grad()
        a_soft = layer.soft_scores(0)
        active = np.flatnonzero(a_soft >= rlayers.EPS_ACTIVE)
        weights = a_soft[active, None] * layer.values.value[active]
        call = gpu_op if op == "gpu" else _REF_OP
        out = call(tape, x, layer.values, weights, active, layer._cache, use_bcsr=use_bcsr, alpha=layer.alpha,
                   alpha_soft=a_soft, k=layer.k, temperature=0.7)
        loss = tape.softmax_cross_entropy(out, labels)
        tape.backward(loss)
        grads[op] = (out.value.copy(), x.grad.copy(), layer.values.grad.copy(), layer.alpha.grad.copy())
    for got, want in zip(grads["gpu"], grads["ref"]):
        np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12)


def test_reference_inactive_values_get_zero_gradient(gpu_op):
    rng = np.random.default_rng(11)
    layer = make_layer(m=12, n=12, sparsity=0.8, temperature=1e-6, seed=12)
    x = Tensor(rng.standard_normal((3, 12)))
    tape = Tape()
    out = layer.forward(x, tape, step=0)
    loss = tape.mean(out)
    layer.values.zero_grad()
    tape.backward(loss)
    active = layer.active_set(0)
    inactive = np.setdiff1d(np.arange(layer.candidates), active)
    assert np.all(layer.values.grad[inactive] == 0.0)
    assert np.any(layer.values.grad[active] != 0.0)

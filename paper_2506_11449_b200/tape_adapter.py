"""Drop-in for the reference's custom tape op, backed by the sm_100a kernels.

``record_diag_matmul`` has exactly the signature, argument meaning, error
behaviour and gradient contract of the reference's ``_record_diag_matmul``
(``pkg/src/diagsparse/layers.py:108-170``): it takes the reference's float64
numpy ``Tensor`` objects (anything with a ``.value`` ndarray), computes
``y = x @ W^T`` for the matrix built from the ``active`` diagonals with the
given compact ``weights`` on the GPU, and records on ``tape`` a backward
closure returning ``(gx, g_values[, g_alpha])`` aligned to
``inputs = (x, values[, alpha])`` (``Tape.record``, ``autodiff.py:43-50``).

A reference user swaps it in with one assignment:

    from diagsparse import layers
    from paper_2506_11449_b200.tape_adapter import record_diag_matmul
    layers._record_diag_matmul = record_diag_matmul

``cache`` and ``use_bcsr`` are accepted for signature compatibility: the
BCSR plan cache (``layers.py:63-105``) and the dense-BLAS switch only change
how the reference computes the same numbers; the GPU path always runs the
diagonal kernels (K1/K2/K3), float64, on ``cuda:0``.  Host<->device copies
happen at this boundary because the reference's tensors live in host memory.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .errors import ShapeMismatch


def _dev():
    if not torch.cuda.is_available():
        raise ops._lib.NativeLibraryError("record_diag_matmul needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def record_diag_matmul(tape, x, values, weights, active, cache, use_bcsr, alpha=None, alpha_soft=None,
                       k=None, temperature=None):
    """layers.py:108-170 on the GPU (float64)."""
    M, N = int(cache.rows), int(cache.cols)
    xv = np.asarray(x.value, dtype=np.float64)
    if xv.ndim != 2 or xv.shape[1] != N:
        raise ShapeMismatch(f"input has shape {xv.shape}, expected (B, {N})")
    dev = _dev()
    C, L = ops.geometry(M, N)
    act = np.asarray(active, dtype=np.int64)
    n_act = act.size
    offs = torch.as_tensor(act, dtype=torch.int32, device=dev)
    sel = ops.selection_from_offsets(C, offs)
    sel.alpha_soft = None  # the compact weights already carry alpha_soft (layers.py:235)
    w_store = torch.zeros(C, L, dtype=torch.float64, device=dev)
    if n_act:
        w_store[offs.long()] = torch.as_tensor(np.asarray(weights, dtype=np.float64), device=dev)
    xt = torch.as_tensor(xv, device=dev)
    y = ops.diag_forward(xt, w_store, sel, M, N, max_act=max(n_act, 0)).cpu().numpy()
    out = type(x)(y) if _tensor_like(x) else y

    def backward(up):
        upt = torch.as_tensor(np.asarray(up, dtype=np.float64), device=dev)
        gx = ops.diag_backward_input(upt, w_store, sel, M, N, max_act=n_act).cpu().numpy()
        vals = torch.as_tensor(np.asarray(values.value, dtype=np.float64), device=dev)
        # unit scale: g_values rows = gw, g_soft = sum_t gw * values (layers.py:159-165)
        g_values, g_soft, _ = ops.diag_backward_weight(upt, xt, vals, sel, M, N, need_bias=False,
                                                       need_soft=alpha is not None, max_act=n_act)
        if alpha is None:
            return gx, g_values.cpu().numpy()
        a_soft = torch.as_tensor(np.asarray(alpha_soft, dtype=np.float64), device=dev)
        g_values = g_values * a_soft[:, None]
        a = torch.as_tensor(np.asarray(alpha.value, dtype=np.float64), device=dev)
        g_alpha = ops.soft_topk_grad(a, int(k), float(temperature), g_soft)
        return gx, g_values.cpu().numpy(), g_alpha.cpu().numpy()

    inputs = (x, values) if alpha is None else (x, values, alpha)
    return tape.record(out, inputs, backward)


def _tensor_like(x) -> bool:
    try:
        type(x)(np.zeros((1, 1)))
        return hasattr(x, "value")
    except Exception:  # noqa: BLE001
        return False

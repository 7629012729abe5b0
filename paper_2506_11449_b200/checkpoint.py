"""Frozen-model checkpoints in the reference's format (training.py:721-766).

``save_checkpoint`` freezes the model (``DiagLinear.freeze``: hard top-K, soft
scores baked in, layers.py:277-287; ``DiagHeurLinear``: its effective matrix;
dense layers as they are) and writes the reference's JSON bundle —
``{"config": ..., "layers": [{"kind": "frozen_diag", "weight": {rows, cols,
offsets, values}, "bias": ...} | {"kind": "dense", "weight": (in, out), "bias": ...}]}``
(diagcore.py:241-247 for the matrix document) — atomically (tmp file +
``os.replace``).  ``load_checkpoint`` reads such a file (ours or one the
reference wrote) into an ``InferenceModel`` of ``FrozenDiagLinear`` / dense
layers on the device, raising ``MalformedFile`` like the reference.  As in the
reference there is no optimizer state: a checkpoint is for inference, not for
resuming training.
"""

from __future__ import annotations

import json
import os

import numpy as np
import torch
from torch import nn

from .errors import DiagSparseError, MalformedFile, ShapeMismatch
from .layer import DiagHeurLinear, DiagLinear, DiagMatrix, FrozenDiagLinear


def _matrix_doc(m: DiagMatrix) -> dict:
    return {"rows": int(m.rows), "cols": int(m.cols), "offsets": [int(o) for o in m.offsets.cpu().tolist()],
            "values": m.values.detach().double().cpu().numpy().tolist()}


def _bias(b):
    return None if b is None else b.detach().double().cpu().numpy().tolist()


def _frozen_entry(layer) -> dict:
    if isinstance(layer, DiagLinear):
        fz = layer.freeze()
        return {"kind": "frozen_diag", "weight": _matrix_doc(fz.weight), "bias": _bias(fz.bias)}
    if isinstance(layer, FrozenDiagLinear):
        return {"kind": "frozen_diag", "weight": _matrix_doc(layer.weight), "bias": _bias(layer.bias)}
    if isinstance(layer, DiagHeurLinear):
        return {"kind": "frozen_diag", "weight": _matrix_doc(layer.effective_matrix()), "bias": _bias(layer.bias)}
    if isinstance(layer, nn.Linear):  # the reference's dense weight is (in, out): y = x @ W
        return {"kind": "dense", "weight": layer.weight.detach().double().t().cpu().numpy().tolist(),
                "bias": _bias(layer.bias)}
    raise TypeError(f"cannot checkpoint layer type {type(layer).__name__}")


def save_checkpoint(model: nn.Module, path: str, config: dict | None = None) -> None:
    """training.py:721-746 for an MLPModel-shaped model (``model.layers``)."""
    layers = getattr(model, "layers", None)
    if layers is None:
        raise TypeError("save_checkpoint takes an MLPModel-style model with a .layers list")
    payload = {"config": config or {}, "layers": [_frozen_entry(lyr) for lyr in layers]}
    tmp = f"{path}.tmp{os.getpid()}"
    with open(tmp, "w") as fh:
        json.dump(payload, fh)
    os.replace(tmp, path)


class _FrozenDense(nn.Module):
    def __init__(self, weight: torch.Tensor, bias: torch.Tensor | None):
        super().__init__()
        self.register_buffer("weight", weight)  # (in, out)
        self.register_buffer("bias", bias)

    def forward(self, x):
        y = x @ self.weight
        return y if self.bias is None else y + self.bias


class InferenceModel(nn.Module):
    """training.py:488-503: frozen layers joined by ReLU, on the device."""

    def __init__(self, layers: list):
        super().__init__()
        self.layers = nn.ModuleList(layers)

    def forward(self, h: torch.Tensor) -> torch.Tensor:
        for i, lyr in enumerate(self.layers):
            h = lyr(h)
            if i < len(self.layers) - 1:
                h = torch.relu(h)
        return h

    @torch.no_grad()
    def predict_logits(self, features, batch: int = 1024) -> torch.Tensor:
        dev = next(iter(self.buffers())).device
        x = torch.as_tensor(np.asarray(features), dtype=torch.float64, device=dev)
        return torch.cat([self(x[lo:lo + batch]) for lo in range(0, x.shape[0], batch)]) if x.shape[0] else \
            torch.empty(0, device=dev, dtype=torch.float64)

    def layer_matrices(self) -> list:
        return [lyr.weight if isinstance(lyr, FrozenDiagLinear) else None for lyr in self.layers]


def load_checkpoint(path: str, device="cuda", route: str = "auto"):
    """training.py:749-766 -> (InferenceModel, config dict)."""
    dev = torch.device(device)
    try:
        with open(path) as fh:
            payload = json.load(fh)
        layers = []
        for entry in payload["layers"]:
            bias = None if entry["bias"] is None else torch.as_tensor(np.asarray(entry["bias"], dtype=np.float64),
                                                                      device=dev)
            if entry["kind"] == "frozen_diag":
                doc = entry["weight"]
                rows, cols = int(doc["rows"]), int(doc["cols"])
                offs = torch.as_tensor(np.asarray([int(o) for o in doc["offsets"]], dtype=np.int64), device=dev)
                vals = torch.as_tensor(np.asarray(doc["values"], dtype=np.float64), device=dev)
                if vals.shape != (offs.numel(), min(rows, cols)):
                    raise ShapeMismatch(f"values {tuple(vals.shape)} vs {offs.numel()} offsets of {min(rows, cols)}")
                layers.append(FrozenDiagLinear(DiagMatrix(rows, cols, offs, vals), bias, route=route))
            elif entry["kind"] == "dense":
                layers.append(_FrozenDense(torch.as_tensor(np.asarray(entry["weight"], dtype=np.float64),
                                                           device=dev), bias))
            else:
                raise MalformedFile(f"unknown layer kind {entry['kind']!r}")
    except (OSError, KeyError, TypeError, ValueError, json.JSONDecodeError) as exc:
        if isinstance(exc, MalformedFile):
            raise
        if isinstance(exc, DiagSparseError):
            raise MalformedFile(f"bad checkpoint {path}: {exc}") from exc
        raise MalformedFile(f"bad checkpoint {path}: {exc}") from exc
    return InferenceModel(layers), payload.get("config", {})

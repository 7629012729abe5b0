"""Device-side optimizer for DiagLinear parameters (K6).

``AdamW`` mirrors the reference's ``AdamW`` (training.py:361-390): decoupled
weight decay applied only where the ParamSpec asks, moments for EVERY element
of the candidate store (inactive rows included), and ``clip_global_norm``
(training.py:406-417) computed on device and applied inside the AdamW kernel
(no host round trip).  ``lr_at`` restates the warmup + cosine LR schedule
(training.py:393-403).
"""

from __future__ import annotations

import math

import torch

from . import ops
from .layer import ParamSpec


def lr_at(step: int, total: int, warmup: float, lr_peak: float, lr_final: float = 0.0) -> float:
    """training.py:393-403."""
    if step > total:
        raise ValueError(f"step {step} beyond total {total}")
    if warmup > 0 and step < warmup:
        return lr_peak * step / warmup
    if total <= warmup:
        return lr_peak
    frac = (step - warmup) / (total - warmup)
    return lr_final + 0.5 * (lr_peak - lr_final) * (1.0 + math.cos(math.pi * frac))


class GlobalNormClipper:
    """clip_global_norm (training.py:406-417) as device scalars.

    ``compute(specs)`` enqueues sum(g^2) for every gradient into a fixed slot
    (deterministic order) and returns (norm, scale) device tensors; pass
    ``scale`` to ``AdamW.step(clip_scale=...)``.
    """

    def __init__(self, max_norm: float):
        self.max_norm = float(max_norm)
        self._buf = None
        self._scratch = None

    def compute(self, specs: list[ParamSpec]):
        grads = [s.tensor.grad for s in specs if s.tensor.grad is not None]
        dev = specs[0].tensor.device
        if self._buf is None or self._buf.numel() < max(1, len(grads)) or self._buf.device != dev:
            self._buf = torch.zeros(max(1, len(grads)), dtype=torch.float64, device=dev)
            self._scratch = ops.sumsq_scratch(dev)
        buf = self._buf[: max(1, len(grads))]
        buf.zero_()
        for i, g in enumerate(grads):
            ops.sumsq_into(g, buf[i:i + 1], self._scratch)
        return ops.clip_scale(buf, self.max_norm)


class AdamW:
    """Decoupled-weight-decay Adam over ParamSpecs, one fused kernel per tensor."""

    def __init__(self, specs: list[ParamSpec], lr: float = 1e-3, betas=(0.9, 0.99),
                 eps: float = 1e-8, weight_decay: float = 5e-5):
        self.specs = list(specs)
        self.lr, self.betas, self.eps, self.weight_decay = lr, tuple(betas), eps, weight_decay
        self.state = [
            {"m": torch.zeros_like(s.tensor), "v": torch.zeros_like(s.tensor), "t": 0}
            for s in self.specs
        ]

    @torch.no_grad()
    def step(self, lr: float | None = None, clip_scale: torch.Tensor | None = None) -> None:
        lr = self.lr if lr is None else lr
        b1, b2 = self.betas
        for spec, st in zip(self.specs, self.state):
            g = spec.tensor.grad
            if g is None:
                continue
            st["t"] += 1
            p = spec.tensor.data
            if g.dtype != p.dtype:
                g = g.to(p.dtype)
            ops.adamw_(p, g.contiguous(), st["m"], st["v"], st["t"], lr, b1, b2, self.eps,
                       self.weight_decay if spec.decay else 0.0, clip_scale)

    def zero_grad(self) -> None:
        for s in self.specs:
            s.tensor.grad = None


def model_param_specs(model: torch.nn.Module) -> list[ParamSpec]:
    """ParamSpecs for a whole model: DiagLinear/DiagHeur specs, plus dense params
    (weights decay, biases / norms do not — the reference's DenseLayer rule,
    layers.py:433-441)."""
    specs: list[ParamSpec] = []
    seen = set()
    for mod in model.modules():
        if hasattr(mod, "param_specs"):
            for s in mod.param_specs():
                specs.append(s)
                seen.add(id(s.tensor))
    for name, p in model.named_parameters():
        if id(p) in seen or not p.requires_grad:
            continue
        specs.append(ParamSpec(p, p.dim() >= 2, name))
    return specs

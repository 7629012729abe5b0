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

from . import _lib, ops  # noqa: F401
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


def _desc(p: torch.Tensor, g: torch.Tensor, m=None, v=None, step: int = 1, wd: float = 0.0):
    code = _lib.F64 if p.dtype == torch.float64 else _lib.F32
    return _lib.TensorDesc(code, int(step), p.numel(), p.data_ptr(), g.data_ptr(),
                           None if m is None else m.data_ptr(), None if v is None else v.data_ptr(),
                           float(wd))


class GlobalNormClipper:
    """clip_global_norm (training.py:406-417) as device scalars.

    ``compute(specs)`` reduces sum(g^2) over every gradient in one multi-tensor
    launch (fixed chunk order, deterministic), folds it with a fixed-order tree
    and returns (norm, scale) device tensors; pass ``scale`` to
    ``AdamW.step(clip_scale=...)``.  Nothing is read back to the host.
    """

    def __init__(self, max_norm: float):
        self.max_norm = float(max_norm)
        self._part = None

    def compute(self, specs: list[ParamSpec]):
        grads = [(s.tensor, s.tensor.grad) for s in specs if s.tensor.grad is not None]
        dev = specs[0].tensor.device
        keep = []
        descs = (_lib.TensorDesc * max(1, len(grads)))()
        for i, (p, g) in enumerate(grads):
            if g.dtype not in (torch.float32, torch.float64):
                g = g.float()
            g = g.contiguous()
            keep.append(g)
            descs[i] = _desc(g, g)
        lib = _lib.load()
        n_part = max(1, lib.diagmm_sumsq_multi_len(len(grads), descs))
        if self._part is None or self._part.numel() < n_part or self._part.device != dev:
            self._part = torch.empty(n_part, dtype=torch.float64, device=dev)
        part = self._part[:n_part]
        if not grads:
            part.zero_()
        stream = torch.cuda.current_stream(dev).cuda_stream
        if grads:
            _lib.call("diagmm_sumsq_multi", len(grads), descs, part.data_ptr(), n_part, stream)
        norm = torch.empty(1, dtype=torch.float64, device=dev)
        scale = torch.empty(1, dtype=torch.float64, device=dev)
        _lib.call("diagmm_clip_scale_tree", n_part, part.data_ptr(), self.max_norm, norm.data_ptr(),
                  scale.data_ptr(), stream)
        return norm, scale


class AdamW:
    """Decoupled-weight-decay Adam over ParamSpecs (training.py:361-390): every
    tensor updated by one multi-tensor launch (K6), clip scale read on device."""

    def __init__(self, specs: list[ParamSpec], lr: float = 1e-3, betas=(0.9, 0.99),
                 eps: float = 1e-8, weight_decay: float = 5e-5):
        self.specs = list(specs)
        self.lr, self.betas, self.eps, self.weight_decay = lr, tuple(betas), eps, weight_decay
        self.state = [
            {"m": torch.zeros_like(s.tensor), "v": torch.zeros_like(s.tensor), "t": 0}
            for s in self.specs
        ]

    @torch.no_grad()
    def step(self, lr: float | None = None, clip_scale: torch.Tensor | None = None,
             sched: torch.Tensor | None = None) -> None:
        """One AdamW update of every tensor.  ``sched``: a device float64 triple
        {lr, 1 - beta1^t, 1 - beta2^t} the kernel reads instead of ``lr`` and the
        host step count (schedule.DeviceSchedule writes it before each replay of a
        captured step)."""
        lr = self.lr if lr is None else lr
        b1, b2 = self.betas
        descs, keep = [], []
        stream = None
        for spec, st in zip(self.specs, self.state):
            g = spec.tensor.grad
            if g is None:
                continue
            p = spec.tensor.data
            if p.dtype not in (torch.float32, torch.float64) or not p.is_contiguous():
                raise TypeError(f"AdamW state must be contiguous float32/float64 ({spec.name})")
            st["t"] += 1
            if g.dtype != p.dtype or not g.is_contiguous():
                g = g.to(p.dtype).contiguous()
            keep.append(g)
            descs.append(_desc(p, g, st["m"], st["v"], st["t"], self.weight_decay if spec.decay else 0.0))
            stream = stream or torch.cuda.current_stream(p.device).cuda_stream
        if not descs:
            return
        arr = (_lib.TensorDesc * len(descs))(*descs)
        _lib.call("diagmm_adamw_multi", len(descs), arr, float(lr), float(b1), float(b2), float(self.eps),
                  None if clip_scale is None else clip_scale.data_ptr(),
                  None if sched is None else sched.data_ptr(), stream)

    def next_step(self) -> int:
        """The (1-based) step count of the next update (for host-computed bias corrections)."""
        return max((st["t"] for st in self.state), default=0) + 1

    def advance_steps(self) -> None:
        """Host bookkeeping after an update that ran inside a replayed CUDA graph."""
        for st in self.state:
            st["t"] += 1

    def zero_grad(self) -> None:
        for s in self.specs:
            s.tensor.grad = None


def model_param_specs(model: torch.nn.Module) -> list[ParamSpec]:
    """ParamSpecs for a whole model: DiagLinear/DiagHeur specs, plus dense params
    (weights decay, biases / norms do not — the reference's DenseLayer rule,
    layers.py:437-441)."""
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

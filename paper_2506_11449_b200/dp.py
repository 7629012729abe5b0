"""Data-parallel gradient exchange for DiagLinear models.

The batch is sharded across ranks; parameters, alpha and therefore the active
sets are replicated.  ``GradientAllReducer`` sums every gradient across ranks
and divides by the world size (the reference's batch-mean loss,
``autodiff.py:131``), one NCCL all-reduce per dtype bucket on the current
stream; inactive DiagLinear rows are exactly zero on every rank
(``layers.py:159-163``), so the average reproduces the single-process
gradient of the full batch.  Global-norm clipping runs AFTER this exchange
(``training.py:662``), so every replica applies the identical AdamW update.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class GradientAllReducer:
    """Flatten gradients into one contiguous bucket per dtype, all-reduce, scatter back."""

    def __init__(self, params, group=None):
        self.params = [p for p in params if p.requires_grad]
        self.group = group
        self._buckets: dict = {}

    def _layout(self, grads):
        key = tuple((g.dtype, g.numel()) for g in grads)
        lay = self._buckets.get(key)
        if lay is None:
            by_dt: dict = {}
            for i, g in enumerate(grads):
                by_dt.setdefault(g.dtype, []).append(i)
            lay = {dt: (idx, torch.empty(sum(grads[i].numel() for i in idx), dtype=dt, device=grads[idx[0]].device))
                   for dt, idx in by_dt.items()}
            self._buckets[key] = lay
        return lay

    @torch.no_grad()
    def __call__(self) -> None:
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        if world == 1:
            return
        live = [p for p in self.params if p.grad is not None]
        grads = [p.grad for p in live]
        for dt, (idx, flat) in self._layout(grads).items():
            off = 0
            for i in idx:
                n = grads[i].numel()
                flat[off:off + n].copy_(grads[i].reshape(-1))
                off += n
            dist.all_reduce(flat, group=self.group)
            flat.div_(world)
            off = 0
            for i in idx:
                n = grads[i].numel()
                grads[i].copy_(flat[off:off + n].view_as(grads[i]))
                off += n


def broadcast_parameters(module: torch.nn.Module, src: int = 0, group=None) -> None:
    """Make every replica start from rank ``src``'s parameters and buffers."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    with torch.no_grad():
        for t in list(module.parameters()) + list(module.buffers()):
            dist.broadcast(t.data, src, group=group)

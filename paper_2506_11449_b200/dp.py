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


class CompactGradExchange:
    """the compact, overlapped data-parallel gradient exchange.

    * Every DiagLinear gets a static bucket of ``cap = min(C, cap_factor * k)`` rows
      (the reference's sparse-path cap ``n_act <= 2K``, layers.py:243) that K3's
      finalize writes the active rows of g_values into while it writes g_values
      itself (diagmm_*backward_weight ``bucket``) — no pack pass.  Inactive rows
      are exactly zero on every rank (layers.py:159-163), so only
      ``[g_values[active] (n_act x L) | g_alpha (C) | g_bias (M)]`` crosses the
      wire; ViT-B: ~41 MB/step instead of the dense-equivalent ~350 MB.
    * Each parameter's all-reduce is launched from its post-accumulate-grad hook,
      i.e. as soon as the backward has produced that gradient, asynchronously
      (NCCL on its own stream): the exchange of layer l overlaps the backward of
      layers l-1 ... 0.
    * ``finish()`` (before the clip, training.py:662) waits for them, writes the
      averaged active rows back into ``values.grad`` and leaves every other
      gradient averaged in place (sum / world: the reference's batch-mean loss,
      autodiff.py:131).

    Gradients must start each step as None (``zero_grad`` sets them so); a layer
    whose active count exceeds its bucket falls back to all-reducing its full
    candidate gradient for that step (read from the forward's device count,
    already on the host by the time its backward runs).
    """

    def __init__(self, model: torch.nn.Module, group=None, cap_factor: int = 2):
        from .layer import DiagLinear

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.avg = dist.is_initialized() and dist.get_backend(group) == "nccl"
        self._work = []
        self.bytes_last = 0
        self._bytes = 0
        seen = set()
        self.layers = []
        for m in model.modules():
            if isinstance(m, DiagLinear) and id(m) not in seen:
                seen.add(id(m))
                cap = min(m.candidates, cap_factor * m.k)
                m._dp_bucket = torch.empty(cap, m.diag_len, dtype=m.values.dtype, device=m.values.device)
                self.layers.append(m)
        self._owner = {id(m.values): m for m in self.layers}
        self._handles = []
        if self.world > 1:
            for p in model.parameters():
                if p.requires_grad:
                    self._handles.append(p.register_post_accumulate_grad_hook(self._hook))

    def _reduce(self, t: torch.Tensor):
        op = dist.ReduceOp.AVG if self.avg else dist.ReduceOp.SUM
        self._bytes += t.numel() * t.element_size()
        return dist.all_reduce(t, op=op, group=self.group, async_op=True)

    def _scale(self, t: torch.Tensor) -> None:
        if not self.avg:
            t.div_(self.world)

    @torch.no_grad()
    def _hook(self, p: torch.Tensor) -> None:
        layer = self._owner.get(id(p))
        if layer is not None:
            spec = getattr(layer, "_last_spec", None)
            sel = getattr(spec, "sel", None)
            n = sel.host_count() if sel is not None else None
            if sel is not None and getattr(spec, "bucket", None) is not None and n <= layer._dp_bucket.shape[0]:
                rows = layer._dp_bucket[:n]
                work = self._reduce(rows)

                def fin(p=p, rows=rows, act=sel.active[:n]):
                    self._scale(rows)
                    p.grad.index_copy_(0, act.long(), rows)

                self._work.append((work, fin))
                return
        g = p.grad
        work = self._reduce(g)
        self._work.append((work, lambda g=g: self._scale(g)))

    @torch.no_grad()
    def finish(self) -> None:
        for work, fin in self._work:
            work.wait()
            fin()
        self._work.clear()
        self.bytes_last, self._bytes = self._bytes, 0

    def remove(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles.clear()
        for m in self.layers:
            m._dp_bucket = None

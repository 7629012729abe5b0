"""GPT-2 small with 90%-sparse DiagLinear layers (BASELINE config 4).

The paper sparsifies both the attention and the MLP projections of GPT-2
(PAPER.md:378): c_attn (d -> 3d), attn c_proj (d -> d), c_fc (d -> 4d) and mlp
c_proj (4d -> d) of every block are DiagLinear layers here.  Like ``vit.py``
this is a thin caller that drives DiagLinear at the config's shapes — pre-LN
blocks with causal attention (the same ``vit.Block`` with ``causal=True``:
qkv + cuDNN attention as one node, residual adds and GELU fused into the
tensor-core epilogues), token + position embeddings, final LayerNorm and an
LM head tied to the token embedding.  Everything that is not a DiagLinear is
stock PyTorch / library code.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
from torch import nn

from .layer import DiagLinear, dense_route_min_tokens, preselect
from .vit import _premat_enabled
from .selection import TemperatureSchedule
from .vit import Block, LayerNorm


@dataclass(frozen=True)
class GPT2Config:
    vocab: int = 50257
    ctx: int = 1024
    dim: int = 768
    depth: int = 12
    heads: int = 12
    mlp_ratio: int = 4
    sparsity: float = 0.9
    sparse_qkv: bool = True  # GPT-2 sparsifies attention too
    dense: str = ""          # "" DiagLinear; "cublas" / "tc": the dense-model arms (vit._sparse)


GPT2_SMALL = GPT2Config()


class GPT2(nn.Module):
    """GPT-2 (pre-LN, GELU-tanh MLP, tied LM head) with DiagLinear projections."""

    def __init__(self, cfg: GPT2Config = GPT2_SMALL, *, t_schedule: TemperatureSchedule | None = None,
                 route: str = "auto", device="cuda"):
        super().__init__()
        self.cfg = cfg
        t_schedule = t_schedule or TemperatureSchedule("constant", 1e-9, 1e-9, 1)
        with torch.device(device):
            self.wte = nn.Embedding(cfg.vocab, cfg.dim)
            self.wpe = nn.Embedding(cfg.ctx, cfg.dim)
            nn.init.normal_(self.wte.weight, std=0.02)
            nn.init.normal_(self.wpe.weight, std=0.01)
            self.blocks = nn.ModuleList(Block(cfg, i, t_schedule, route, causal=True) for i in range(cfg.depth))
            self.ln_f = LayerNorm(cfg.dim)

    def diag_layers(self):
        return [m for m in self.modules() if isinstance(m, DiagLinear)]

    def set_step(self, step: int) -> None:
        for m in self.diag_layers():
            m.step = step

    def forward(self, ids: torch.Tensor) -> torch.Tensor:
        """ids (B, S) int64 -> logits (B, S, vocab)."""
        diag = self.diag_layers()
        if diag:
            # one batched soft-TopK launch for all layers (+ one batched W_K build on the
            # tensor-core route)
            mat = (torch.bfloat16 if torch.is_autocast_enabled("cuda") and ids.is_cuda
                   and torch.get_autocast_dtype("cuda") == torch.bfloat16
                   and ids.numel() >= dense_route_min_tokens() and _premat_enabled() else None)
            preselect(diag, diag[0].step, materialize=mat)
        S = ids.shape[1]
        pos = torch.arange(S, device=ids.device)
        x = self.wte(ids) + self.wpe(pos)[None]
        if torch.is_autocast_enabled("cuda"):
            x = x.to(torch.get_autocast_dtype("cuda"))
        for blk in self.blocks:
            x = blk(x)
        x = self.ln_f(x)
        return torch.nn.functional.linear(x, self.wte.weight)  # tied LM head

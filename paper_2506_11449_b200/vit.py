"""Callers of the hot path used for measurement: ViT-B/16, ViT-Tiny/16, MLP.

The reference ships only an MLP of linear layers (training.py:423-475); the
paper's ViT experiments (BASELINE.json configs 2-3) sparsify the
attention projections and the MLP of every block with DiagLinear.  These thin
PyTorch models exist to drive ``DiagLinear`` at those shapes; everything that
is not a DiagLinear is stock PyTorch (LayerNorm, SDPA attention, GELU, the
patch-embedding conv and the classifier head).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F
from torch import nn

from . import _lib, ops
from .layer import DiagLinear, DiagMLP, FrozenDiagLinear, _tc_weight_grads, _w_k, dense_route_min_tokens, preselect
from .selection import TemperatureSchedule


try:  # library attention kernel for the caller (not the DiagLinear hot path)
    from flash_attn import flash_attn_qkvpacked_func as _flash_qkvpacked
except Exception:  # noqa: BLE001 - optional: SDPA is used without it
    _flash_qkvpacked = None


class PackedQKVAttention(torch.autograd.Function):
    """Attention on a packed (B, T, 3, H, hd) qkv tensor through cuDNN's fused
    SDPA kernels (library), with the three input gradients written straight
    back into one packed (B, T, 3, H, hd) gradient — the caller's attention
    around the qkv DiagLinear, without autograd's unbind/stack copies."""

    @staticmethod
    def forward(ctx, h, causal=False):
        # q, k, v: strided views of h made autograd leaves of their own, so the
        # library op's registered backward gives dq, dk, dv and nothing else
        qkv = [t.detach().requires_grad_(True) for t in h.permute(2, 0, 3, 1, 4).unbind(0)]
        with torch.enable_grad():
            out = torch.ops.aten._scaled_dot_product_cudnn_attention(*qkv, None, True, 0.0, bool(causal))[0]
        ctx.graph = (out, qkv)
        ctx.h_shape = h.shape
        return out.detach()

    @staticmethod
    def backward(ctx, g):
        out, qkv = ctx.graph
        grads = torch.autograd.grad(out, qkv, g)
        ctx.graph = None
        dh = torch.empty(ctx.h_shape, dtype=g.dtype, device=g.device)
        st = grads[0].stride()
        if (g.dtype == torch.bfloat16 and all(x.stride() == st and x.is_cuda for x in grads)
                and grads[0].stride(-1) == 1):
            B, T, _, H, hd = ctx.h_shape
            _lib.call("diagmm_pack_qkv_grad", B, T, H, hd, grads[0].data_ptr(), grads[1].data_ptr(),
                      grads[2].data_ptr(), st[0], st[1], st[2], dh.data_ptr(),
                      torch.cuda.current_stream(g.device).cuda_stream)
        else:
            dhv = dh.permute(2, 0, 3, 1, 4)  # (3, B, H, T, hd) view of the packed gradient
            for i in range(3):
                dhv[i].copy_(grads[i])
        return dh, None


class QKVAttentionFunction(torch.autograd.Function):
    """qkv DiagLinear (tensor-core route) + cuDNN attention as one autograd node.

    Forward: W_K materialized once, h = x W_K^T + b on our tcgen05 GEMM, cuDNN
    SDPA on the packed (B, T, 3, H, hd) h.  Backward: the attention gradients
    dq, dk, dv come back as three (B*T, d) row-major blocks (BSHD); the qkv
    input gradient (dx = [dq|dk|dv] W_K, W_K read MN-major) and the qkv weight
    gradient (diagonal gather + bias fused) read the three blocks directly, so
    the packed (B*T, 3d) gradient is never built.  Gradients are exactly those
    of DiagMMFunction (layers.py:143-167) for the qkv layer."""

    @staticmethod
    def forward(ctx, x, values, alpha, bias, spec, B, T, H, causal=False):
        M, N = spec.M, spec.N
        sel = spec.presel or ops.soft_topk_select(alpha.detach(), spec.k, spec.temperature, params=spec.params)
        spec.sel = sel
        vals = values.detach()
        W = _w_k(spec, x.dtype, vals, sel, M, N)
        h = ops.tc_gemm(x.contiguous(), W, None if bias is None else bias.detach())
        hd = N // H
        qkv = [t_.detach().requires_grad_(True) for t_ in h.view(B, T, 3, H, hd).permute(2, 0, 3, 1, 4).unbind(0)]
        with torch.enable_grad():
            out = torch.ops.aten._scaled_dot_product_cudnn_attention(*qkv, None, True, 0.0, bool(causal))[0]
        ctx.graph = (out, qkv)
        ctx.save_for_backward(x, values, alpha)
        ctx.sel, ctx.spec, ctx.W, ctx.has_bias, ctx.bth = sel, spec, W, bias is not None, (B, T, H)
        return out.detach()

    @staticmethod
    def backward(ctx, g):
        out, qkv = ctx.graph
        ctx.graph = None
        x, values, alpha = ctx.saved_tensors
        sel, spec, W = ctx.sel, ctx.spec, ctx.W
        ctx.W = None
        B, T, H = ctx.bth
        M, N = spec.M, spec.N
        grads = torch.autograd.grad(out, qkv, g)
        # (B, H, T, hd) with BSHD memory -> (B*T, d) views; copies only if cuDNN changes layout
        parts = [d.permute(0, 2, 1, 3).reshape(B * T, N) for d in grads]
        dx = ops.tc_gemm_nn_split(parts, W) if ctx.needs_input_grad[0] else None
        need_soft = alpha is not None and ctx.needs_input_grad[2]
        gv, gb, ga = _tc_weight_grads(spec, parts, x, values.detach(), sel, ctx.has_bias, need_soft, alpha)
        return dx, gv, ga, gb, None, None, None, None, None


class PatchEmbedFunction(torch.autograd.Function):
    """Patch embedding + cls token + position embedding as one node (caller-side).

    Forward: images -> patches by a 16-byte streaming kernel (diagmm_vit_patchify),
    the patch projection on cuBLAS bf16 (a plain dense GEMM, as F.linear under
    autocast), then [bf16(cls); y] + bf16(pos) in one pass (diagmm_vit_embed_fwd).
    Backward: one pass over the gradient gives the contiguous patch gradient and the
    pos / cls / bias sums (diagmm_vit_embed_bwd); the weight gradient is dy^T P in
    bf16.  Same roundings as the framework's cat + broadcast-add path it replaces."""

    @staticmethod
    def forward(ctx, images, weight, bias, cls, pos, patch):
        B, Cin, H, W = images.shape
        D = weight.shape[0]
        img = images.to(torch.bfloat16).contiguous()
        gh, gw = H // patch, W // patch
        T = gh * gw + 1
        st = torch.cuda.current_stream(images.device).cuda_stream
        P = torch.empty(B * gh * gw, Cin * patch * patch, dtype=torch.bfloat16, device=images.device)
        _lib.call("diagmm_vit_patchify", B, Cin, H, W, patch, img.data_ptr(), P.data_ptr(), st)
        w = weight.detach().reshape(D, -1).to(torch.bfloat16)
        b = None if bias is None else bias.detach().to(torch.bfloat16)
        with torch.autocast("cuda", enabled=False):
            y = F.linear(P, w, b)
        x = torch.empty(B, T, D, dtype=torch.bfloat16, device=images.device)
        clsf = cls.detach().float().reshape(D).contiguous()
        posf = pos.detach().float().reshape(T, D).contiguous()
        _lib.call("diagmm_vit_embed_fwd", B, T, D, y.data_ptr(), clsf.data_ptr(), posf.data_ptr(), x.data_ptr(), st)
        ctx.save_for_backward(P, w)
        ctx.meta = (B, T, D, weight.shape, bias is not None, cls.shape, pos.shape)
        return x

    @staticmethod
    def backward(ctx, gx):
        P, w = ctx.saved_tensors
        B, T, D, wshape, has_bias, cshape, pshape = ctx.meta
        g = gx.to(torch.bfloat16).contiguous()
        dev = g.device
        dy = torch.empty(B * (T - 1), D, dtype=torch.bfloat16, device=dev)
        dpos = torch.empty(T, D, dtype=torch.float32, device=dev)
        dcls = torch.empty(D, dtype=torch.float32, device=dev)
        dbias = torch.empty(D, dtype=torch.float32, device=dev) if has_bias else None
        nws = _lib.load().diagmm_vit_embed_bwd_workspace(T, D)
        ws = torch.empty(nws, dtype=torch.uint8, device=dev)
        _lib.call("diagmm_vit_embed_bwd", B, T, D, g.data_ptr(), dy.data_ptr(), dpos.data_ptr(), dcls.data_ptr(),
                  None if dbias is None else dbias.data_ptr(), ws.data_ptr(), nws,
                  torch.cuda.current_stream(dev).cuda_stream)
        dw = None
        if ctx.needs_input_grad[1]:
            with torch.autocast("cuda", enabled=False):
                dw = torch.mm(dy.t(), P).float().reshape(wshape)
        return (None, dw, dbias if ctx.needs_input_grad[2] else None, dcls.reshape(cshape),
                dpos.reshape(pshape), None)


def _embed_fusable(images, cfg) -> bool:
    import os

    bf16 = images.dtype == torch.bfloat16 or (torch.is_autocast_enabled("cuda")
                                               and torch.get_autocast_dtype("cuda") == torch.bfloat16)
    return (images.is_cuda and bf16 and cfg.patch % 8 == 0 and cfg.dim % 8 == 0
            and os.environ.get("DIAGMM_FUSE_EMBED", "1") != "0")


def _qkv_fusable(qkv, x2: torch.Tensor, H: int) -> bool:
    import os

    from .layer import dense_route_min_tokens

    return (isinstance(qkv, DiagLinear) and qkv.route == "auto" and x2.is_cuda and x2.dtype == torch.bfloat16
            and x2.shape[0] >= dense_route_min_tokens() and qkv.values.dtype == torch.float32
            and qkv.in_features % 128 == 0 and qkv.out_features == 3 * qkv.in_features
            and qkv.in_features % H == 0 and os.environ.get("DIAGMM_DENSE_BACKEND", "tc") != "cublas"
            and os.environ.get("DIAGMM_FUSE_QKV", "1") != "0")


def _attention_backend() -> str:
    import os

    return os.environ.get("DIAGMM_VIT_ATTENTION", "cudnn")


class LayerNorm(nn.LayerNorm):
    """nn.LayerNorm that runs the fused bf16 kernel (csrc/norm_kernels.cu) when
    the activations are bf16 (directly or under CUDA autocast); float32 params."""

    def _fused(self, x) -> bool:
        bf16 = x.dtype == torch.bfloat16 or (torch.is_autocast_enabled("cuda")
                                              and torch.get_autocast_dtype("cuda") == torch.bfloat16)
        D = x.shape[-1]
        return x.is_cuda and bf16 and self.elementwise_affine and D % 8 == 0 and D <= 1024

    def forward(self, x):
        if self._fused(x):
            return ops.layer_norm_bf16(x, self.weight, self.bias, self.eps)
        return super().forward(x)

    def forward_skip(self, x):
        """(norm(x), x) where x also feeds the block's skip connection: the two
        gradients of x are summed inside the LayerNorm backward kernel."""
        if self._fused(x) and x.dtype == torch.bfloat16:
            return ops.layer_norm_skip_bf16(x, self.weight, self.bias, self.eps)
        return self.forward(x), x


@dataclass(frozen=True)
class ViTConfig:
    image: int = 224
    patch: int = 16
    dim: int = 768
    depth: int = 12
    heads: int = 12
    mlp_ratio: int = 4
    classes: int = 1000
    sparsity: float = 0.9
    sparse_qkv: bool = True
    dense: str = ""  # "" DiagLinear projections; "cublas": nn.Linear; "tc": TCLinear (the dense-model arms)

    @property
    def tokens(self) -> int:
        return (self.image // self.patch) ** 2 + 1


VIT_B16 = ViTConfig()
VIT_TINY16 = ViTConfig(dim=192, depth=12, heads=3)


class _TCLinearFunction(torch.autograd.Function):
    """Dense y = x W^T + b on our tcgen05 GEMM (W cast to bf16 per call, as autocast
    does for nn.Linear); dX on the MN-major tcgen05 GEMM; dW / db on cuBLAS."""

    @staticmethod
    def forward(ctx, x, weight, bias):
        W = weight.detach().to(torch.bfloat16)
        x2 = x.reshape(-1, x.shape[-1]).to(torch.bfloat16).contiguous()
        y = ops.tc_gemm(x2, W, None if bias is None else bias.detach())
        ctx.save_for_backward(x2, W)
        ctx.has_bias, ctx.shape = bias is not None, x.shape
        return y.view(*x.shape[:-1], W.shape[0])

    @staticmethod
    def backward(ctx, dy):
        x2, W = ctx.saved_tensors
        g = dy.reshape(-1, W.shape[0]).to(torch.bfloat16).contiguous()
        dx = ops.tc_gemm_nn(g, W).view(ctx.shape)
        dW = torch.mm(g.t(), x2, out_dtype=torch.float32)
        db = g.sum(0, dtype=torch.float32) if ctx.has_bias else None
        return dx, dW, db


class TCLinear(nn.Linear):
    """nn.Linear whose bf16 products run on the repo's tcgen05 GEMM (dense-model arm)."""

    def forward(self, x):
        if x.is_cuda and self.in_features % 8 == 0 and self.out_features % 8 == 0:
            return _TCLinearFunction.apply(x, self.weight, self.bias)
        return super().forward(x)


class DenseMLP(nn.Module):
    """fc2(gelu_tanh(fc1(x))) (+ residual) with dense layers (the dense-model arms)."""

    def __init__(self, fc1: nn.Module, fc2: nn.Module):
        super().__init__()
        self.fc1, self.fc2 = fc1, fc2

    def forward(self, x, residual=None):
        y = self.fc2(F.gelu(self.fc1(x), approximate="tanh"))
        return y if residual is None else y + residual


def _sparse(n_in, n_out, cfg: ViTConfig, seed: int, t_schedule, route, dense: bool = False):
    if cfg.dense == "tc":
        return TCLinear(n_in, n_out)
    if dense or cfg.dense:
        return nn.Linear(n_in, n_out)
    return DiagLinear(n_in, n_out, cfg.sparsity, seed=seed, t_schedule=t_schedule, route=route,
                      dtype=torch.float32)


class Block(nn.Module):
    """Pre-LN transformer block: x + proj(attn(qkv(LN(x)))), then x + fc2(gelu(fc1(LN(x)))).
    ``causal`` masks the attention (GPT-2)."""

    def __init__(self, cfg, idx: int, t_schedule, route, causal: bool = False):
        super().__init__()
        d = cfg.dim
        self.heads = cfg.heads
        self.causal = bool(causal)
        self.norm1 = LayerNorm(d)
        self.qkv = _sparse(d, 3 * d, cfg, 4 * idx, t_schedule, route, dense=not cfg.sparse_qkv)
        self.proj = _sparse(d, d, cfg, 4 * idx + 1, t_schedule, route)
        self.norm2 = LayerNorm(d)
        self.fc1 = _sparse(d, cfg.mlp_ratio * d, cfg, 4 * idx + 2, t_schedule, route)
        self.fc2 = _sparse(cfg.mlp_ratio * d, d, cfg, 4 * idx + 3, t_schedule, route)
        if isinstance(self.fc1, DiagLinear):
            self.mlp = DiagMLP(self.fc1, self.fc2)  # GELU fused into the tensor-core epilogues
        else:
            self.mlp = DenseMLP(self.fc1, self.fc2)

    def forward(self, x):
        B, T, D = x.shape
        backend = _attention_backend()
        xn, x = self.norm1.forward_skip(x)  # x's skip and norm gradients meet in the LN backward
        x2 = xn.reshape(B * T, D)
        if x2.dtype == torch.float32 and torch.is_autocast_enabled("cuda"):
            x2 = x2.to(torch.get_autocast_dtype("cuda"))
        if backend == "cudnn" and _qkv_fusable(self.qkv, x2, self.heads):
            q = self.qkv
            step = q.step
            q.last_step = step
            a = QKVAttentionFunction.apply(x2, q.values, q.alpha, q.bias, q._make_spec(step), B, T, self.heads,
                                           self.causal)
            a = a.transpose(1, 2).reshape(B, T, D)
            x = self.proj(a, residual=x) if isinstance(self.proj, (DiagLinear, FrozenDiagLinear)) else x + self.proj(a)
            xn2, x = self.norm2.forward_skip(x)
            return self.mlp(xn2, residual=x)
        h = self.qkv(xn).view(B, T, 3, self.heads, D // self.heads)
        if backend == "cudnn" and h.is_cuda and h.dtype in (torch.bfloat16, torch.float16):
            a = PackedQKVAttention.apply(h, self.causal).transpose(1, 2).reshape(B, T, D)
        elif backend != "sdpa" and _flash_qkvpacked is not None and h.dtype in (torch.bfloat16, torch.float16):
            # packed q/k/v in, packed dq/dk/dv out: no unbind/stack copies
            a = _flash_qkvpacked(h, causal=self.causal).reshape(B, T, D)
        else:
            q, k, v = h.permute(2, 0, 3, 1, 4).unbind(0)
            a = F.scaled_dot_product_attention(q, k, v, is_causal=self.causal).transpose(1, 2).reshape(B, T, D)
        # skip connections fused into the proj / fc2 epilogues (DiagLinear residual=)
        x = self.proj(a, residual=x) if isinstance(self.proj, (DiagLinear, FrozenDiagLinear)) else x + self.proj(a)
        xn2, x = self.norm2.forward_skip(x)
        return self.mlp(xn2, residual=x)


class ViT(nn.Module):
    """ViT with DiagLinear qkv / proj / fc1 / fc2 in every block."""

    def __init__(self, cfg: ViTConfig = VIT_B16, *, t_schedule: TemperatureSchedule | None = None,
                 route: str = "auto", device="cuda"):
        super().__init__()
        self.cfg = cfg
        t_schedule = t_schedule or TemperatureSchedule("constant", 1e-9, 1e-9, 1)
        with torch.device(device):
            self.patch = nn.Conv2d(3, cfg.dim, cfg.patch, cfg.patch)
            self.cls = nn.Parameter(torch.zeros(1, 1, cfg.dim))
            self.pos = nn.Parameter(torch.randn(1, cfg.tokens, cfg.dim) * 0.02)
            self.blocks = nn.ModuleList(Block(cfg, i, t_schedule, route) for i in range(cfg.depth))
            self.norm = LayerNorm(cfg.dim)
            self.head = nn.Linear(cfg.dim, cfg.classes)

    def diag_layers(self):
        return [m for m in self.modules() if isinstance(m, DiagLinear)]

    def set_step(self, step: int) -> None:
        for m in self.diag_layers():
            m.step = step

    def _patchify(self, images):
        """Patch embedding as a GEMM: non-overlapping 16x16 patches are a pure
        reshape/permute of the image, so conv2d(stride=kernel) == unfold @ W^T
        (cuDNN's conv spends ~3 ms per step on layout transposes here)."""
        B, Cin, H, W = images.shape
        p = self.cfg.patch
        x = images.reshape(B, Cin, H // p, p, W // p, p).permute(0, 2, 4, 1, 3, 5).reshape(B, -1, Cin * p * p)
        w, b = self.patch.weight.reshape(self.cfg.dim, -1), self.patch.bias
        if not torch.is_autocast_enabled(x.device.type):
            w, b = w.to(x.dtype), None if b is None else b.to(x.dtype)
        return torch.nn.functional.linear(x, w, b)

    def forward(self, images):
        diag = self.diag_layers()
        if diag:
            # one batched soft-TopK launch for all layers (+ one batched W_K build when the
            # bf16 token count puts them on the tensor-core route)
            tokens = images.shape[0] * ((images.shape[-1] // self.cfg.patch) ** 2 + 1)
            mat = (torch.bfloat16 if torch.is_autocast_enabled("cuda") and images.is_cuda
                   and torch.get_autocast_dtype("cuda") == torch.bfloat16 and tokens >= dense_route_min_tokens()
                   and _premat_enabled() else None)
            preselect(diag, diag[0].step, materialize=mat)
        if _embed_fusable(images, self.cfg):
            x = PatchEmbedFunction.apply(images, self.patch.weight, self.patch.bias, self.cls, self.pos,
                                         self.cfg.patch)
        else:
            x = self._patchify(images)
            x = torch.cat([self.cls.expand(x.shape[0], -1, -1).to(x.dtype), x], dim=1) + self.pos.to(x.dtype)
        for blk in self.blocks:
            x = blk(x)
        return self.head(self.norm(x)[:, 0])


def _premat_enabled() -> bool:
    import os

    return os.environ.get("DIAGMM_PREMAT", "1") != "0"


class MLPModel(nn.Module):
    """training.py:423-475: DiagLinear / dense layers joined by ReLU."""

    def __init__(self, sizes=(784, 256, 256, 10), kinds=("dynadiag", "dynadiag", "dense"),
                 sparsity: float = 0.9, seeds=None, t_schedule=None, dtype=torch.float32, device="cuda"):
        super().__init__()
        seeds = seeds or list(range(len(kinds)))
        layers = []
        for (n_in, n_out), kind, seed in zip(zip(sizes[:-1], sizes[1:]), kinds, seeds):
            if kind == "dynadiag":
                layers.append(DiagLinear(n_in, n_out, sparsity, seed=int(seed), t_schedule=t_schedule,
                                         dtype=dtype, device=device))
            else:
                layers.append(nn.Linear(n_in, n_out, device=device, dtype=dtype))
        self.layers = nn.ModuleList(layers)

    def forward(self, x, step: int | None = None):
        diag = [m for m in self.layers if isinstance(m, DiagLinear)]
        if diag:
            preselect(diag, diag[0].step if step is None else step)
        for i, lyr in enumerate(self.layers):
            x = lyr(x, step) if isinstance(lyr, DiagLinear) else lyr(x)
            if i < len(self.layers) - 1:
                x = torch.relu(x)
        return x

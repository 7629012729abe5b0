"""compute-sanitizer workload for the round-2 kernels (3xTF32 products / dW, radix K4 + K5, LayerNorm
with the cp.async backward, the ViT patch-embedding kernels) on small ragged cases:
  compute-sanitizer --tool memcheck python tools/sanitize_new_kernels.py"""
import sys
sys.path.insert(0, ".")
import os
import numpy as np
import torch
from paper_2506_11449_b200 import ops, _lib
os.environ["DIAGMM_TF32X3_MIN_B"] = "1"
# 3xTF32 products + dW (ragged shape, non-multiple-of-4 widths)
for (M, N, B) in [(301, 603, 130), (600, 300, 257)]:
    C, L = max(M, N), min(M, N)
    rng = np.random.default_rng(0)
    offs = np.sort(rng.choice(C, C // 10, replace=False))
    vals = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    x = torch.randn(B, N, device="cuda"); dy = torch.randn(B, M, device="cuda")
    ops.diag_forward(x, vals, sel, M, N, torch.randn(M, device="cuda"), max_act=len(offs))
    ops.diag_backward_input(dy, vals, sel, M, N, max_act=len(offs))
    ops.diag_backward_weight(dy, x, vals, sel, M, N, max_act=len(offs))
os.environ.pop("DIAGMM_TF32X3_MIN_B")
# radix K4 (ties) + K5
for C, k in [(1025, 102), (3072, 307)]:
    a = torch.full((C,), 0.37, dtype=torch.float64, device="cuda")
    sel = ops.soft_topk_select(a, k, 1e-3)
    ops.soft_topk_grad(a, k, 1e-3, torch.randn(C, dtype=torch.float64, device="cuda"), clamped=sel.clamped)
# LayerNorm fwd/bwd (+ residual)
M, D = 1000, 768
x = torch.randn(M, D, device="cuda").to(torch.bfloat16).requires_grad_(True)
w = torch.randn(D, device="cuda", requires_grad=True); b = torch.randn(D, device="cuda", requires_grad=True)
y, xs = ops.layer_norm_skip_bf16(x, w, b, 1e-5) if hasattr(ops, "layer_norm_skip_bf16") else (ops.layer_norm_bf16(x, w, b), x)
(y.float().sum() + xs.float().sum()).backward()
# ViT embedding kernels
from paper_2506_11449_b200.vit import PatchEmbedFunction
img = torch.randn(2, 3, 64, 64, device="cuda").to(torch.bfloat16)
wt = torch.randn(128, 3, 16, 16, device="cuda", requires_grad=True); bt = torch.randn(128, device="cuda", requires_grad=True)
cls = torch.randn(1, 1, 128, device="cuda", requires_grad=True); pos = torch.randn(1, 17, 128, device="cuda", requires_grad=True)
out = PatchEmbedFunction.apply(img, wt, bt, cls, pos, 16)
out.float().sum().backward()
torch.cuda.synchronize()
print("sanitizer workload done")

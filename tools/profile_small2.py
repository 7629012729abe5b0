"""4096^2 90 % bf16 at B = 1 and B = 8: one warm fwd / dW call each (ncu target)."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops
from paper_2506_11449_b200.selection import required_diagonals

for B in (1, 8):
    M = N = C = L = 4096
    k = required_diagonals(M, N, 0.9)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    values = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    x = torch.randn(B, N, device="cuda").to(torch.bfloat16)
    dy = torch.randn(B, M, device="cuda").to(torch.bfloat16)
    for rep in range(2):
        ops.diag_forward(x, values, sel, M, N, max_act=k)
        ops.diag_backward_weight(dy, x, values, sel, M, N, need_bias=True, need_soft=True, max_act=k)
    torch.cuda.synchronize()

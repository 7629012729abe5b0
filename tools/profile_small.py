"""One warm call of K1 / K2 / K3 per shape (for an ncu launch list): config 1 fp32
and 4096^2 at 90 % with B = 1, 8, 64 (bf16)."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops
from paper_2506_11449_b200.selection import required_diagonals

cases = [(3072, 768, 256, torch.float32), (768, 3072, 256, torch.float32), (4096, 4096, 1, torch.bfloat16),
         (4096, 4096, 8, torch.bfloat16), (4096, 4096, 64, torch.bfloat16)]
for M, N, B, dt in cases:
    C, L = max(M, N), min(M, N)
    k = required_diagonals(M, N, 0.9)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    values = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    x = torch.randn(B, N, device="cuda").to(dt)
    dy = torch.randn(B, M, device="cuda").to(dt)
    for rep in range(3):
        torch.cuda.nvtx.range_push(f"{M}x{N}B{B}")
        ops.diag_forward(x, values, sel, M, N, max_act=k)
        ops.diag_backward_input(dy, values, sel, M, N, max_act=k)
        ops.diag_backward_weight(dy, x, values, sel, M, N, need_bias=True, need_soft=True, max_act=k)
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print(M, N, B, "done", flush=True)

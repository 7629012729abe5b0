"""4096^2 90 % bf16 B = 64 fwd (ncu target) and config 1 fp32 fwd."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops
from paper_2506_11449_b200.selection import required_diagonals

for (M, N, B, dt) in [(4096, 4096, 64, torch.bfloat16), (3072, 768, 256, torch.float32)]:
    C, L = max(M, N), min(M, N)
    k = required_diagonals(M, N, 0.9)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    values = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    x = torch.randn(B, N, device="cuda").to(dt)
    for rep in range(2):
        ops.diag_forward(x, values, sel, M, N, max_act=k)
    torch.cuda.synchronize()

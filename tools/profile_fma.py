"""ncu targets for the FMA product / dW kernels: one call per case after a warm-up.

  python tools/profile_fma.py b64      # 4096^2 90 % bf16 B = 64  fwd / dX / dW
  python tools/profile_fma.py cfg1     # 768 -> 3072 90 % fp32 B = 256 fwd / dX / dW
  python tools/profile_fma.py b1024s99 # 4096^2 99 % bf16 B = 1024 fwd / dX / dW
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops
from paper_2506_11449_b200.selection import required_diagonals

CASES = {"b64": (4096, 4096, 64, 0.9, torch.bfloat16), "cfg1": (3072, 768, 256, 0.9, torch.float32),
         "b1024s99": (4096, 4096, 1024, 0.99, torch.bfloat16), "b256": (4096, 4096, 256, 0.9, torch.bfloat16),
         "b8": (4096, 4096, 8, 0.9, torch.bfloat16), "b1": (4096, 4096, 1, 0.9, torch.bfloat16)}

for name in sys.argv[1:] or ["b64"]:
    M, N, B, s, dt = CASES[name]
    C, L = max(M, N), min(M, N)
    k = required_diagonals(M, N, s)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    values = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    x = torch.randn(B, N, device="cuda").to(dt)
    dy = torch.randn(B, M, device="cuda").to(dt)
    for rep in range(2):
        ops.diag_forward(x, values, sel, M, N, max_act=k)
        ops.diag_backward_input(dy, values, sel, M, N, max_act=k)
        ops.diag_backward_weight(dy, x, values, sel, M, N, max_act=k)
    torch.cuda.synchronize()
    print(name, "ok")

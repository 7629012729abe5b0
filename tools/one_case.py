"""Run K1/K2/K3 once on one shape (the ncu target): python tools/one_case.py M N B sparsity dtype"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops
from paper_2506_11449_b200.selection import required_diagonals

M, N, B = (int(a) for a in sys.argv[1:4])
s = float(sys.argv[4])
dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[sys.argv[5]]
C, L = max(M, N), min(M, N)
k = required_diagonals(M, N, s)
offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
values = torch.randn(C, L, device="cuda", dtype=ops.param_dtype_for(dt))
sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
x = torch.randn(B, N, device="cuda").to(dt)
dy = torch.randn(B, M, device="cuda").to(dt)
for _ in range(2):
    ops.diag_forward(x, values, sel, M, N, max_act=k)
    ops.diag_backward_input(dy, values, sel, M, N, max_act=k)
    ops.diag_backward_weight(dy, x, values, sel, M, N, need_bias=False, need_soft=False, max_act=k)
torch.cuda.synchronize()
print("ok")

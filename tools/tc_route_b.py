"""Tensor-core route of one 4096^2 90 % bf16 DiagLinear at B tokens: materialize, tcgen05
fwd, MN-major dX, fused-gather dW (ncu target).   python tools/tc_route_b.py 1024"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops
from paper_2506_11449_b200.selection import required_diagonals

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
M = N = 4096
C, L = M, N
k = required_diagonals(M, N, 0.9)
offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
values = torch.randn(C, L, device="cuda")
sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
x = torch.randn(B, N, device="cuda").to(torch.bfloat16)
dy = torch.randn(B, M, device="cuda").to(torch.bfloat16)
for _ in range(2):
    W = ops.materialize(values, sel, M, N, dtype=torch.bfloat16)
    ops.tc_gemm(x, W)
    ops.tc_gemm_nn(dy, W)
    ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=False, max_act=k)
torch.cuda.synchronize()

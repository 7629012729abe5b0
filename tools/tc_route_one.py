import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2506_11449_b200 import ops
M = N = 4096
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
k = 410
offs = np.sort(np.random.default_rng(0).choice(M, k, replace=False))
sel = ops.selection_from_offsets(M, torch.as_tensor(offs, device="cuda"))
values = torch.randn(M, N, device="cuda")
x = torch.randn(B, N, device="cuda").to(torch.bfloat16)
dy = torch.randn(B, M, device="cuda").to(torch.bfloat16)
for _ in range(2):
    W = ops.materialize(values, sel, M, N, dtype=torch.bfloat16)
    y = ops.tc_gemm(x, W)
    dx = ops.tc_gemm_nn(dy, W)
    ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=False, max_act=k)
torch.cuda.synchronize()

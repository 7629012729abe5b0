import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2506_11449_b200 import ops
T, M, N = 50432, 2304, 768
C, L = M, N
k = int(0.1 * M * N / L + 0.5)
offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
values = torch.randn(C, L, device="cuda")
dy = torch.randn(T, M, device="cuda").to(torch.bfloat16)
x = torch.randn(T, N, device="cuda").to(torch.bfloat16)
buf = torch.stack([dy[:, i * N:(i + 1) * N] for i in range(3)]).contiguous()
parts = [buf[0], buf[1], buf[2]]
for _ in range(2):
    ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True)
    ops.tc_backward_weight_split(parts, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True)
torch.cuda.synchronize()

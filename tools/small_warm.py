"""4096^2 90 % bf16, B = 1 / 8 / 64: fwd / dx / dw device time, warm L2 vs flushed
(graph replay of 20 calls)."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops, profiling
from paper_2506_11449_b200.selection import required_diagonals

flush = torch.empty(64 * 1024 * 1024, device="cuda")
for B in (1, 8, 64):
    M = N = C = L = 4096
    k = required_diagonals(M, N, 0.9)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    values = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    x = torch.randn(B, N, device="cuda").to(torch.bfloat16)
    dy = torch.randn(B, M, device="cuda").to(torch.bfloat16)
    gv = torch.empty(C, L, device="cuda")
    fns = {"fwd": lambda: ops.diag_forward(x, values, sel, M, N, max_act=k),
           "dx": lambda: ops.diag_backward_input(dy, values, sel, M, N, max_act=k),
           "dw": lambda: ops.diag_backward_weight(dy, x, values, sel, M, N, need_bias=True, need_soft=True,
                                                 max_act=k, g_values=gv),
           "dw_nobias": lambda: ops.diag_backward_weight(dy, x, values, sel, M, N, need_bias=False, need_soft=False,
                                                        max_act=k, g_values=gv),
           "zero64MB": lambda: gv.zero_()}
    out = []
    for nm, fn in fns.items():
        warm = profiling._time_call(fn, 20, None) * 1e3
        cold = profiling._time_call(fn, 20, flush) * 1e3
        out.append(f"{nm} {warm:.1f}/{cold:.1f}")
    print(f"B={B}: " + "  ".join(out) + "  (us warm/cold)", flush=True)

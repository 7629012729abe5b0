"""Warm (L2-resident, no flush) device time per op via CUDA-graph replay of 50 calls:
python tools/warm_ops.py  -> fwd / dX / dW us for 4096^2 90 % bf16 at several B."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops
from paper_2506_11449_b200.selection import required_diagonals


def graph_us(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


M = N = 4096
for s in (0.9, 0.99):
    for B in [int(a) for a in (sys.argv[1:] or ["1", "4", "8", "16", "32", "64"])]:
        C, L = max(M, N), min(M, N)
        k = required_diagonals(M, N, s)
        offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
        values = torch.randn(C, L, device="cuda")
        sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
        x = torch.randn(B, N, device="cuda").to(torch.bfloat16)
        dy = torch.randn(B, M, device="cuda").to(torch.bfloat16)
        w = (torch.randn(M, N, device="cuda") * 0.02).to(torch.bfloat16)
        tf = graph_us(lambda: ops.diag_forward(x, values, sel, M, N, max_act=k))
        tx = graph_us(lambda: ops.diag_backward_input(dy, values, sel, M, N, max_act=k))
        tw = graph_us(lambda: ops.diag_backward_weight(dy, x, values, sel, M, N, max_act=k))
        cf = graph_us(lambda: torch.nn.functional.linear(x, w))
        cx = graph_us(lambda: dy @ w)
        cw = graph_us(lambda: dy.t() @ x)
        print(f"s={s} B={B:4d}: ours fwd {tf:6.1f} dx {tx:6.1f} dw {tw:6.1f} = {tf + tx + tw:6.1f} | "
              f"cublas {cf:5.1f} {cx:5.1f} {cw:5.1f} = {cf + cx + cw:6.1f} | x{(cf + cx + cw) / (tf + tx + tw):.2f}",
              flush=True)

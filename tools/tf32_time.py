"""Warm device time of the fp32 products / dW (config 1 shape and neighbours) on
whatever route the library picks: run once with DIAGMM_TF32X3_MIN_B=0 (FMA
kernels) and once with the default (3xTF32 tensor cores for B >= 128).
  python tools/tf32_time.py [B ...]"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops


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


import os

SHAPES = [(3072, 768), (768, 3072), (4096, 4096)] if not os.environ.get("TF_SHAPE") else [tuple(map(int, os.environ["TF_SHAPE"].split("x")))]
for M, N in SHAPES:
    C, L = max(M, N), min(M, N)
    k = max(1, C // 10)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    vals = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    bias = torch.randn(M, device="cuda")
    for B in [int(a) for a in (sys.argv[1:] or ["64", "128", "256", "1024"])]:
        x = torch.randn(B, N, device="cuda")
        dy = torch.randn(B, M, device="cuda")
        tf = graph_us(lambda: ops.diag_forward(x, vals, sel, M, N, bias, max_act=k))
        tx = graph_us(lambda: ops.diag_backward_input(dy, vals, sel, M, N, max_act=k))
        tw = graph_us(lambda: ops.diag_backward_weight(dy, x, vals, sel, M, N, max_act=k))
        print(f"{M}x{N} B={B}: fwd {tf:.1f} dX {tx:.1f} dW {tw:.1f} us (sum {tf + tx + tw:.1f})", flush=True)

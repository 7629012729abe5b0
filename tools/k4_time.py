"""Warm device time of K4 (soft TopK re-selection) and K5 (its gradient) for one layer:
python tools/k4_time.py [C ...]"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import torch

from paper_2506_11449_b200 import ops
from warm_ops import graph_us

for C in [int(a) for a in (sys.argv[1:] or ["768", "2304", "3072", "4096", "8192"])]:
    k = max(1, C // 10)
    alpha = torch.randn(C, dtype=torch.float64, device="cuda")
    up = torch.randn(C, dtype=torch.float64, device="cuda")
    sel = ops.soft_topk_select(alpha, k, 1e-3)
    t4 = graph_us(lambda: ops.soft_topk_select(alpha, k, 1e-3, out=sel))
    t5 = graph_us(lambda: ops.soft_topk_grad(alpha, k, 1e-3, up, clamped=sel.clamped))
    print(f"C={C}: K4 {t4:.1f} us, K5 {t5:.1f} us", flush=True)

"""Tensor-core route of a 4096^2 90 % bf16 layer at 1024-4096 tokens, cold L2, per op, vs cuBLAS;
DIAGMM_TC_PAIR=1 (default: CTA pairs only when the 256 x 256 tiles fill the pairs) / 2 (always pairs)."""
import sys, os
sys.path.insert(0, ".")
import torch
from paper_2506_11449_b200 import profiling
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
peaks = {"hbm_gbs": 6558.1, "bf16_tflops": 1642.9}
for B in (1024, 2048, 4096):
    r = profiling.diag_case(4096, 4096, B, 0.9, torch.bfloat16, peaks, 72.4, flush=flush)
    print(os.environ.get("DIAGMM_TC_PAIR"), B, {k: round(v, 1) for k, v in r["tc_route_us"].items()}, "cublas", round(r["cublas_bf16_dense_us"]["total"], 1))

"""BASELINE config 5: DiagMM 4096x4096 at sparsity 50/80/90/95/99 % and batch 1..8192 (bf16),
our best route (diagonal FMA kernels or the tensor-core route) vs cuBLAS dense bf16, fwd+bwd
device time (cold L2, CUDA-graph replay; profiling.diag_case)."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import profiling

peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {"hbm_gbs": 6416.1}
flush = torch.empty(64 * 1024 * 1024, device="cuda")
print(f"{'sparsity':>8} {'B':>6} | {'FMA fwd+bwd us':>14} {'TC route us':>11} {'cuBLAS us':>10} | {'best/cuBLAS':>11} | FMA fwd TF, dW TF")
for s in (0.5, 0.8, 0.9, 0.95, 0.99):
    for B in (1, 8, 64, 512, 1024, 8192):
        r = profiling.diag_case(4096, 4096, B, s, torch.bfloat16, peaks, 72.4, reps=3, flush=flush)
        tc = r.get("tc_route_us", {}).get("total", float("nan"))
        cb = r["cublas_bf16_dense_us"]["total"]
        print(f"{s:8.2f} {B:6d} | {r['fwd_bwd_us']:14.1f} {tc:11.1f} {cb:10.1f} | "
              f"{r['speedup_vs_cublas_bf16_fwd_bwd']:11.2f} | {r['fwd']['tflops']:.1f}, {r['dw']['tflops']:.1f}", flush=True)

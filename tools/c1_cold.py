"""Config 1 (768 -> 3072, B = 256, fp32) per-op device time with L2 flushed before each
op, as bench.py measures it, on whichever route the library picks (set DIAGMM_TF32X3_MIN_B
to force / forbid the 3xTF32 route).  python tools/c1_cold.py"""
import sys, os
sys.path.insert(0, ".")
import torch
from paper_2506_11449_b200 import profiling
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
peaks = {"hbm_gbs": 6558.1, "bf16_tflops": 1642.9}
r = profiling.diag_case(3072, 768, 256, 0.9, torch.float32, peaks, 72.4, flush=flush, dense_cmp=False)
print(os.environ.get("DIAGMM_TF32X3_MIN_B"), {k: round(v["us"], 1) for k, v in r.items() if isinstance(v, dict) and "us" in v})

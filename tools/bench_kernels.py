"""Device time of K1/K2/K3 on a few shapes (L2 flushed, CUDA-graph replay)."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import profiling

peaks = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else {"hbm_gbs": 6416.1}
flush = torch.empty(64 * 1024 * 1024, device="cuda")
cases = [(3072, 768, 256, 0.9, torch.float32), (768, 3072, 256, 0.9, torch.float32),
         (3072, 768, 256, 0.9, torch.bfloat16), (3072, 768, 4096, 0.9, torch.bfloat16),
         (768, 3072, 4096, 0.9, torch.bfloat16), (4096, 4096, 1, 0.9, torch.bfloat16), (4096, 4096, 8, 0.9, torch.bfloat16),
         (4096, 4096, 16, 0.9, torch.bfloat16), (4096, 4096, 1, 0.99, torch.bfloat16),
         (4096, 4096, 64, 0.9, torch.bfloat16), (4096, 4096, 1024, 0.9, torch.bfloat16),
         (4096, 4096, 1024, 0.99, torch.bfloat16), (4096, 4096, 8192, 0.9, torch.bfloat16),
         (3072, 768, 50432, 0.9, torch.bfloat16)]
if len(sys.argv) > 1:
    cases = [cases[int(a)] for a in sys.argv[1:]]
for M, N, B, s, dt in cases:
    r = profiling.diag_case(M, N, B, s, dt, peaks, 72.4, reps=5, flush=flush)
    d = r.get("cublas_bf16_dense_us", {})
    print(f"{M}x{N} B={B} s={s} {str(dt)[6:]}: " + " ".join(
        f"{k}={r[k]['us']:.1f}us/{r[k]['tflops']:.1f}TF" for k in ("fwd", "dx", "dw")) +
        (f" | tc route {r['tc_route_us']['total']:.1f}us" if 'tc_route_us' in r else "") +
        f" | cublas bf16 fwd+bwd {d.get('total', 0):.1f}us, best-route speedup {r.get('speedup_vs_cublas_bf16_fwd_bwd', 0):.2f}",
        flush=True)

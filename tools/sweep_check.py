import sys, json
sys.path.insert(0, ".")
import torch
from paper_2506_11449_b200 import profiling
peaks = {"hbm_gbs": 6551.7}
cases = [(4096, 0.9, 1), (4096, 0.9, 64), (4096, 0.9, 1024), (4096, 0.99, 1024), (4096, 0.9, 8192)]
if len(sys.argv) > 1:
    cases = [cases[int(sys.argv[1])]]
for dim, s, B in cases:
    for dt in (torch.bfloat16, torch.float32):
        r = profiling.diag_case(dim, dim, B, s, dt, peaks, 72.4, reps=5, dense_cmp=False)
        torch.cuda.synchronize()
        print(dim, s, B, dt, {k: round(r[k]["us"], 1) for k in ("fwd", "dx", "dw")}, flush=True)

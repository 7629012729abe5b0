"""fp32 DiagLinear on the dense route (the reference's density >= 1/4 switch) — forward +
backward device time at config 1's shape, on the 3xTF32 kernel (default) or cuBLAS SGEMM
(DIAGMM_DENSE_BACKEND=cublas).  python tools/dense_fp32_time.py"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import DiagLinear, TemperatureSchedule

for B in (64, 256, 1024):
    torch.manual_seed(0)
    lyr = DiagLinear(768, 3072, 0.9, seed=0, dtype=torch.float32,
                     t_schedule=TemperatureSchedule("constant", 4.0, 4.0, 1), route="dense")
    x = torch.randn(B, 768, device="cuda", requires_grad=True)
    up = torch.randn(B, 3072, device="cuda")
    for _ in range(3):
        (lyr(x, step=0) * up).sum().backward()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        (lyr(x, step=0) * up).sum().backward()
    e.record()
    torch.cuda.synchronize()
    print(f"B={B}: {s.elapsed_time(e) / 20 * 1e3:.1f} us per eager fwd+bwd step (dense route, fp32)", flush=True)

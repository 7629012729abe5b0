"""Run BASELINE config 1 (DiagLinear 768->3072, 90%, B=256, fp32) fwd+bwd a few
times — the command profiled with ncu (profiles/r01_*)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2506_11449_b200 import DiagLinear, TemperatureSchedule

dt = torch.bfloat16 if "--bf16" in sys.argv else torch.float32
B = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 256
lyr = DiagLinear(768, 3072, 0.9, seed=0, dtype=torch.float32,
                 t_schedule=TemperatureSchedule("constant", 1e-9, 1e-9, 1))
x = torch.randn(B, 768, device="cuda").to(dt).requires_grad_(True)
dy = torch.randn(B, 3072, device="cuda").to(dt)
for _ in range(3):
    y = lyr(x, step=0)
    y.backward(dy)
torch.cuda.synchronize()
print("ok", y.shape, y.dtype)

import sys
sys.path.insert(0, ".")
import torch
from paper_2506_11449_b200 import ops
M, D = 50432, 768
x = torch.randn(M, D, device="cuda").to(torch.bfloat16).requires_grad_(True)
w = torch.ones(D, device="cuda", requires_grad=True)
b = torch.zeros(D, device="cuda", requires_grad=True)
g = torch.randn(M, D, device="cuda").to(torch.bfloat16)
def step():
    y = ops.layer_norm_bf16(x, w, b)
    y.backward(g)
for _ in range(3): step()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): step()
e.record(); torch.cuda.synchronize()
print(f"fused LN fwd+bwd {s.elapsed_time(e)/20*1e3:.1f} us")

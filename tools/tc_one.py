import sys
sys.path.insert(0, ".")
import torch
from paper_2506_11449_b200 import ops
M, N, K = (int(v) for v in sys.argv[1:4])
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
bias = torch.randn(N, device="cuda")
for _ in range(3):
    ops.tc_gemm(a, b, bias)
    torch.nn.functional.linear(a, b, bias.to(torch.bfloat16))
torch.cuda.synchronize()

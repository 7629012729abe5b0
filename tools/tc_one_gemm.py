"""One fc1-forward-shaped tcgen05 GEMM (50432 x 3072 x 768, bias epilogue) a few times (ncu target)."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import ops

a = torch.randn(50432, 768, device="cuda").to(torch.bfloat16)
b = (torch.randn(3072, 768, device="cuda") * 0.05).to(torch.bfloat16)
bias = torch.randn(3072, device="cuda")
for _ in range(3):
    ops.tc_gemm(a, b, bias)
torch.cuda.synchronize()

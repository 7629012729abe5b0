"""One fc1-shaped GEMM per epilogue (ncu target): python tools/tc_epi_one.py EPI"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import ops

epi = int(sys.argv[1])
T, n_out, k = 50432, 3072, 768
a = torch.randn(T, k, device="cuda").to(torch.bfloat16)
w = (torch.randn(n_out, k, device="cuda") * 0.05).to(torch.bfloat16)
bias = torch.randn(n_out, device="cuda")
pre = torch.randn(T, n_out, device="cuda").to(torch.bfloat16)
for _ in range(2):
    if epi == 0:
        ops.tc_gemm(a, w, bias)
    elif epi == 1:
        ops.tc_gemm_ex(a, w, bias, epilogue=1)
    else:
        ops.tc_gemm_ex(a, w, None, epilogue=2, aux=pre)
torch.cuda.synchronize()
print("ok")

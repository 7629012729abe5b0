"""tcgen05 GEMM timings at the ViT-B shapes (50 432 tokens): CTA-pair vs single-CTA
kernel (set DIAGMM_TC_PAIR=0/1 per run), vs cuBLAS.  L2 not flushed (operands > L2)."""
import os
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import ops


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


T = 50432
mode = os.environ.get("DIAGMM_TC_PAIR", "1")
for (N, K) in [(3072, 768), (768, 3072), (2304, 768), (768, 768)]:
    a = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    bt = b.t().contiguous()
    g = torch.randn(T, N, device="cuda").to(torch.bfloat16)
    fl = 2.0 * T * N * K
    us = t(lambda: ops.tc_gemm(a, b, bias))
    us_nn = t(lambda: ops.tc_gemm_nn(g, b))  # (T, N) @ (N, K) -> dx shape (T, K)
    us_cb = t(lambda: torch.nn.functional.linear(a, b))
    line = f"mode={mode} {T}x{N}x{K}: fwd {us:.1f}us {fl / us / 1e6:.0f}TF | nn {us_nn:.1f}us {fl / us_nn / 1e6:.0f}TF | cublas {us_cb:.1f}us {fl / us_cb / 1e6:.0f}TF"
    if K == 768 and N == 3072:
        us_g = t(lambda: ops.tc_gemm_ex(a, b, bias, epilogue=1))
        line += f" | gelu-epi {us_g:.1f}us {fl / us_g / 1e6:.0f}TF"
    if N == 768:
        r = torch.randn(T, N, device="cuda").to(torch.bfloat16)
        us_r = t(lambda: ops.tc_gemm_ex(a, b, bias, epilogue=3, aux=r))
        line += f" | resid-epi {us_r:.1f}us {fl / us_r / 1e6:.0f}TF"
    ref = a[:256].float() @ b.float().t() + bias
    err = ((ops.tc_gemm(a, b, bias)[:256].float() - ref).abs().max() / ref.abs().max()).item()
    ref2 = g[:256].float() @ b.float()
    err2 = ((ops.tc_gemm_nn(g, b)[:256].float() - ref2).abs().max() / ref2.abs().max()).item()
    print(line + f" | err {err:.1e} {err2:.1e}", flush=True)

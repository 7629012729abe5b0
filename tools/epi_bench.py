"""Time the tcgen05 GEMM epilogues on the ViT-B MLP shapes (50432 tokens):
epi 0 (+bias), 1 (+bias, gelu, pre-activation stored), 2 (x gelu'(aux)), vs
cuBLAS + a separate torch GELU pass."""
import sys

sys.path.insert(0, ".")
import torch
import torch.nn.functional as F

from paper_2506_11449_b200 import ops

T = 50432
dev = "cuda"


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


import os
shapes = [(3072, 768), (768, 3072), (2304, 768), (768, 768), (768, 2304)] if os.environ.get('EPI_ALL') else [(3072, 768), (768, 3072)]
for (n_out, k) in shapes:
    a = torch.randn(T, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(n_out, k, device=dev) * 0.05).to(torch.bfloat16)
    bias = torch.randn(n_out, device=dev)
    pre = torch.randn(T, n_out, device=dev).to(torch.bfloat16)
    t0 = timeit(lambda: ops.tc_gemm(a, w, bias))
    t1 = timeit(lambda: ops.tc_gemm_ex(a, w, bias, epilogue=1))
    t2 = timeit(lambda: ops.tc_gemm_ex(a, w, None, epilogue=2, aux=pre))
    tg = timeit(lambda: F.gelu(pre, approximate="tanh"))
    gb = timeit(lambda: torch.ops.aten.gelu_backward(pre, pre, approximate="tanh"))
    fl = 2.0 * T * n_out * k
    print(f"N={n_out} K={k}: epi0 {t0:.1f}us ({fl / t0 / 1e6:.0f} TF)  epi1 {t1:.1f}us  epi2 {t2:.1f}us | "
          f"torch gelu {tg:.1f}us, gelu_backward {gb:.1f}us", flush=True)

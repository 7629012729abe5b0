"""Correctness + speed of the tcgen05 GEMM (ops.tc_gemm) vs torch/cuBLAS."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import ops

torch.manual_seed(0)
for (M, N, K) in [(128, 256, 64), (256, 512, 128), (300, 200, 72), (1000, 3072, 768), (50432, 3072, 768),
                  (50432, 768, 3072), (50432, 2304, 768)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    out = ops.tc_gemm(a, b, bias)
    torch.cuda.synchronize()
    ref = (a.float() @ b.float().t() + bias)
    err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    for fn_name, fn in (("ours", lambda: ops.tc_gemm(a, b, bias)),
                        ("cublas", lambda: torch.nn.functional.linear(a, b, bias.to(torch.bfloat16)))):
        fn()
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / reps * 1e3
        print(f"{M}x{N}x{K} {fn_name}: {us:8.1f} us  {2 * M * N * K / us / 1e6:7.1f} TFLOP/s  rel_err {err:.2e}",
              flush=True)

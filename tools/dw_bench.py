"""dW: tensor-core diagonal-gather kernel vs cuBLAS fp32 dense dW + gather."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2506_11449_b200 import ops

def timeit(f, reps=10):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for (M, N) in [(3072, 768), (768, 3072), (2304, 768), (768, 768)]:
    B = 50432
    C, L = max(M, N), min(M, N)
    offs = np.sort(np.random.default_rng(0).choice(C, C // 10, replace=False))
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    vals = torch.randn(C, L, device="cuda")
    x = torch.randn(B, N, device="cuda").to(torch.bfloat16)
    dy = torch.randn(B, M, device="cuda").to(torch.bfloat16)
    t_tc = timeit(lambda: ops.tc_backward_weight(dy, x, vals, sel, M, N))
    t_tcb = timeit(lambda: ops.tc_backward_weight(dy, x, vals, sel, M, N, need_bias=True))
    t_bias = timeit(lambda: dy.sum(0, dtype=torch.float32))
    def ref():
        dW = torch.mm(dy.t(), x, out_dtype=torch.float32)
        return ops.gather_dense_grad(dW, vals, sel, M, N)
    t_cb = timeit(ref)
    t_mm = timeit(lambda: torch.mm(dy.t(), x, out_dtype=torch.float32))
    fl = 2.0 * M * N * B
    print(f"{M}x{N} B={B}: tc dW {t_tc:.1f}us ({fl/t_tc/1e6:.0f} TF), +fused bias {t_tcb:.1f}us | cublas+gather {t_cb:.1f}us "
          f"(mm alone {t_mm:.1f}us, {fl/t_mm/1e6:.0f} TF) + torch bias {t_bias:.1f}us", flush=True)

import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2506_11449_b200 import ops
T = 50432
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for (M, N) in [(3072, 768), (768, 3072), (768, 768)]:
    C, L = max(M, N), min(M, N)
    k = int(0.1 * M * N / L + 0.5)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    values = torch.randn(C, L, device="cuda")
    dy = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    x = torch.randn(T, N, device="cuda").to(torch.bfloat16)
    a = timeit(lambda: ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True))
    b = timeit(lambda: ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=False))
    g = timeit(lambda: torch.mm(dy.t(), x))
    print(f"dW {M}x{N}: with bias {a:.1f}us, no bias {b:.1f}us, cuBLAS dense dy^T x {g:.1f}us")

"""dX GEMM: K-major B (materialized W^T) vs MN-major B (W itself), ViT-B shapes (50 432 tokens);
tensor-core dW: one dy vs three column blocks."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import ops

T = 50432


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


for (M, N) in [(2304, 768), (768, 768), (3072, 768), (768, 3072)]:  # W (M_out, N_in); dx = dy (T, M) @ W
    dy = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    W = (torch.randn(M, N, device="cuda") * 0.05).to(torch.bfloat16)
    Wt = W.t().contiguous()
    t_nt = timeit(lambda: ops.tc_gemm(dy, Wt))
    t_nn = timeit(lambda: ops.tc_gemm_nn(dy, W))
    fl = 2.0 * T * M * N
    line = f"dX W {M}x{N}: NT {t_nt:.1f}us ({fl / t_nt / 1e6:.0f} TF)  NN {t_nn:.1f}us ({fl / t_nn / 1e6:.0f} TF)"
    if M == 3 * N:
        parts = [dy[:, i * N:(i + 1) * N].contiguous() for i in range(3)]
        t_sp = timeit(lambda: ops.tc_gemm_nn_split(parts, W))
        line += f"  NN split3 {t_sp:.1f}us"
    print(line, flush=True)

import numpy as np
for (M, N) in [(2304, 768), (768, 768), (3072, 768), (768, 3072)]:
    C, L = max(M, N), min(M, N)
    k = int(0.1 * M * N / L + 0.5)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    values = torch.randn(C, L, device="cuda")
    dy = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    x = torch.randn(T, N, device="cuda").to(torch.bfloat16)
    t1 = timeit(lambda: ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True))
    line = f"dW {M}x{N}: {t1:.1f}us ({2.0 * T * M * N / t1 / 1e6:.0f} TF dense-equiv)"
    if M == 3 * N:
        parts = [dy[:, i * N:(i + 1) * N].contiguous() for i in range(3)]
        t2 = timeit(lambda: ops.tc_backward_weight_split(parts, x, values, sel, M, N, need_soft=True, max_act=k,
                                                         need_bias=True))
        line += f"  split3 {t2:.1f}us"
    print(line, flush=True)

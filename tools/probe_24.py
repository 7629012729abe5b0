"""Probe: does 2:4 structured sparsity on the tensor cores (cuSPARSELt via
torch semi-structured) beat dense cuBLAS bf16 at the ViT DiagLinear shapes on
this B200?  Also: how many diagonals of a random 90% active set violate 2:4."""
import sys
import time

import numpy as np
import torch

dev = "cuda"
print(torch.__version__, torch.cuda.get_device_name())


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for (tok, n_in, n_out) in [(50432, 768, 3072), (50432, 3072, 768), (50432, 768, 2304), (4096, 4096, 4096)]:
    x = torch.randn(tok, n_in, device=dev, dtype=torch.bfloat16)
    W = torch.randn(n_out, n_in, device=dev, dtype=torch.bfloat16)
    mask = torch.tensor([1, 1, 0, 0], device=dev, dtype=torch.bool).repeat(n_out, n_in // 4)
    Ws = W * mask
    t_dense = timeit(lambda: torch.nn.functional.linear(x, W))
    line = f"{tok}x{n_in}->{n_out}: dense {t_dense:.1f}us"
    try:
        from torch.sparse import to_sparse_semi_structured, SparseSemiStructuredTensor
        for backend in ("cusparselt", "cutlass"):
            try:
                SparseSemiStructuredTensor._FORCE_CUTLASS = backend == "cutlass"
                Wss = to_sparse_semi_structured(Ws)
                t_sp = timeit(lambda: torch.nn.functional.linear(x, Wss))
                y1 = torch.nn.functional.linear(x, Wss)
                y0 = torch.nn.functional.linear(x, Ws)
                err = (y1.float() - y0.float()).abs().max().item()
                line += f" | 2:4 {backend} {t_sp:.1f}us ({t_dense / t_sp:.2f}x, err {err:.2e})"
            except Exception as exc:  # noqa: BLE001
                line += f" | 2:4 {backend} failed: {type(exc).__name__}: {str(exc)[:80]}"
    except Exception as exc:  # noqa: BLE001
        line += f" | semi-structured unavailable: {exc}"
    print(line, flush=True)

# 2:4 compatibility of random diagonal sets (tall, groups of 4 consecutive input columns)
rng = np.random.default_rng(0)
for C, K in [(3072, 307), (2304, 230), (768, 77), (4096, 410)]:
    bad = []
    for trial in range(20):
        offs = np.sort(rng.choice(C, K, replace=False))
        act = np.zeros(C, bool)
        act[offs] = True
        best = None
        for a in range(4):  # window alignment
            w = [act[(np.arange(4) + 4 * g + a) % C].sum() for g in range(C // 4)]
            nb = sum(1 for x in w if x > 2)
            best = nb if best is None else min(best, nb)
        bad.append(best)
    print(f"C={C} K={K}: aligned 4-windows with >2 active (best alignment): mean {np.mean(bad):.1f} max {max(bad)}")

"""Force v6 product plans (DIAGMM_V6_FORCE, read per call) and time fwd / dX per plan
(CUDA graph replay, L2 flushed before every call).   python tools/v6_sweep.py cfg1 b64"""
import itertools
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2506_11449_b200 import ops, profiling
from paper_2506_11449_b200.selection import required_diagonals

CASES = {"cfg1": (3072, 768, 256, 0.9, torch.float32), "b64": (4096, 4096, 64, 0.9, torch.bfloat16),
         "b256": (4096, 4096, 256, 0.9, torch.bfloat16), "b1024s99": (4096, 4096, 1024, 0.99, torch.bfloat16),
         "b32": (4096, 4096, 32, 0.9, torch.bfloat16)}
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for name in sys.argv[1:]:
    M, N, B, s, dt = CASES[name]
    C, L = max(M, N), min(M, N)
    k = required_diagonals(M, N, s)
    offs = np.sort(np.random.default_rng(0).choice(C, k, replace=False))
    values = torch.randn(C, L, device="cuda")
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device="cuda"))
    x = torch.randn(B, N, device="cuda").to(dt)
    dy = torch.randn(B, M, device="cuda").to(dt)
    plans = [None] + [f"{g},{nw},{pw},{ns}" for g, nw, pw, ns in itertools.product(
        (1, 2), (8, 16), (1, 2, 4, 8), (1, 2, 4)) if pw <= nw]
    res = []
    for pl in plans:
        if pl:
            os.environ["DIAGMM_V6_FORCE"] = pl
        else:
            os.environ.pop("DIAGMM_V6_FORCE", None)
        try:
            tf = profiling._time_call(lambda: ops.diag_forward(x, values, sel, M, N, max_act=k), 10, flush) * 1e3
            tx = profiling._time_call(lambda: ops.diag_backward_input(dy, values, sel, M, N, max_act=k), 10, flush) * 1e3
            res.append((pl or "auto", tf, tx))
            print(f"{name} {pl or 'auto':12s} fwd {tf:7.1f} us  dx {tx:7.1f} us", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name} {pl} ERR {str(e)[:120]}", flush=True)
            torch.cuda.synchronize()
    os.environ.pop("DIAGMM_V6_FORCE", None)
    bf = min(res, key=lambda r: r[1])
    bx = min(res, key=lambda r: r[2])
    print(f"## {name} best fwd {bf[0]} {bf[1]:.1f} us, best dx {bx[0]} {bx[2]:.1f} us (auto {res[0][1]:.1f} / {res[0][2]:.1f})")

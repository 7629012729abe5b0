"""Block fill of the reference's own BCSR route (row reorder + blocking, bcsr.py:161-313)
on the ViT-B DiagLinear shapes at 90 % with random active diagonals: how much of every
dense MMA tile a BCSR / band tensor-core path would actually use.  Runs the REFERENCE in
this container (CPU tool; reads /root/reference, never used by tests or the bench).

    python tools/bcsr_fill.py > profiles/r02_bcsr_block_fill.txt
"""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from diagsparse import bcsr, diagcore  # noqa: E402

rng = np.random.default_rng(0)
print("# reference reorder_rows + blocking_plan (bcsr.py:161-289) on random 90 %-sparse diagonal sets")
print("# fill = nnz / (num_blocks * br * bc): the useful fraction of the dense blocks a BCSR MMA path executes")
print(f"{'shape (M x N)':>14s} {'k':>5s} {'block':>7s} {'reorder':>8s} {'blocks':>8s} {'fill':>7s} {'dense-equiv':>12s} {'sec':>6s}")
for (M, N) in [(768, 768), (2304, 768), (3072, 768), (768, 3072)]:
    C, L = max(M, N), min(M, N)
    k = max(1, int(round(0.1 * C)))
    offs = tuple(int(o) for o in np.sort(rng.choice(C, k, replace=False)))
    p = diagcore.DiagonalPattern(M, N, offs)
    nnz = k * L
    for br, bc in [(8, 8), (16, 16), (64, 64), (128, 64)]:
        for alpha in (0.3,):
            t0 = time.perf_counter()
            plan = bcsr.blocking_plan(p, bcsr.BlockingConfig(alpha_blend=alpha, br=br, bc=bc))
            dt = time.perf_counter() - t0
            fill = nnz / (plan.num_blocks * br * bc)
            print(f"{M:>6d} x {N:<5d} {k:>5d} {br:>3d}x{bc:<3d} {'ref':>8s} {plan.num_blocks:>8d} {fill:7.3f} "
                  f"{plan.num_blocks * br * bc / (M * N):12.3f} {dt:6.1f}", flush=True)
        # identity row order, same blocks (what a band path without reordering sees)
        rows = np.concatenate([diagcore.diagonal_entries(M, N, o)[0] for o in offs])
        cols = np.concatenate([diagcore.diagonal_entries(M, N, o)[1] for o in offs])
        nb = np.unique((rows // br) * (-(-N // bc)) + cols // bc).size
        print(f"{M:>6d} x {N:<5d} {k:>5d} {br:>3d}x{bc:<3d} {'identity':>8s} {nb:>8d} {nnz / (nb * br * bc):7.3f} "
              f"{nb * br * bc / (M * N):12.3f} {'':>6s}", flush=True)

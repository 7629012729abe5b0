"""How far a random 10 %-diagonal active set is from 2:4 structure.

For row r of W_K, the 4 input columns of a 2:4 group hold the offsets
{r-4g-3 .. r-4g} (mod C), so 2:4 fails wherever 4 cyclically consecutive offsets
contain >= 3 active diagonals.  Counts such windows over all row phases and for
the best single phase (rows grouped by phase with their own K alignment)."""
import numpy as np


def windows(a, C, phase):
    return sum(1 for j in range(C // 4) if a[[(4 * j + phase - 3 + t) % C for t in range(4)]].sum() > 2)


rng = np.random.default_rng(0)
for C, k in [(3072, 307), (2304, 230), (768, 77)]:
    allp, best, zero = [], [], []
    for _ in range(20):
        a = np.zeros(C, bool)
        a[rng.choice(C, k, replace=False)] = True
        per = [windows(a, C, p) for p in range(4)]
        allp.append(sum(per))
        best.append(min(per))
        zero.append(min(per) == 0)
    print(f"C={C} k={k}: conflicting windows over all phases {np.mean(allp):.1f}, best single phase "
          f"{np.mean(best):.2f}, P(best phase clean) {np.mean(zero):.2f}")

import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2506_11449_b200 import ops
g = np.load('tests/golden/topk.npz')
for i in range(int(g['n'])):
    C, k, T = g[f'c{i}_meta']
    if int(C) == 9:
        a = g[f'c{i}_alpha']
print("alpha", a.tolist())
at = torch.as_tensor(a, device='cuda')
for k in range(1, 10):
    print(k, ops.select_hard(at, k).tolist(), np.sort(np.argsort(-a, kind='stable')[:k]).tolist())
for arr in ([0.0, 0.0, 0.0], [-0.0, 0.0], [0.0, -0.0], [1.0, 0.0, -0.0, 0.0], [0.5, 0.5, 0.1]):
    print(arr, ops.select_hard(torch.tensor(arr, dtype=torch.float64, device='cuda'), 1).tolist())

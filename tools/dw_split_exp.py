import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2506_11449_b200 import ops
T, M, N = 50432, 2304, 768
k = int(0.1 * M * N / N + 0.5)
offs = np.sort(np.random.default_rng(0).choice(M, k, replace=False))
sel = ops.selection_from_offsets(M, torch.as_tensor(offs, device="cuda"))
values = torch.randn(M, N, device="cuda")
dy = torch.randn(T, M, device="cuda").to(torch.bfloat16)
x = torch.randn(T, N, device="cuda").to(torch.bfloat16)
p0 = dy[:, :768].contiguous()
parts = [dy[:, i * N:(i + 1) * N].contiguous() for i in range(3)]
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
print("unsplit", timeit(lambda: ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True)))
print("split distinct", timeit(lambda: ops.tc_backward_weight_split(parts, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True)))
print("split same ptr", timeit(lambda: ops.tc_backward_weight_split([p0, p0, p0], x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True)))
big = torch.randn(T, 3 * 768, device="cuda").to(torch.bfloat16)
print("unsplit 2304-pitch other buffer", timeit(lambda: ops.tc_backward_weight(big, x, values, sel, M, N, need_soft=True, max_act=k, need_bias=True)))
# a 768-wide single matrix (M=768 layer) for reference x3
sel7 = ops.selection_from_offsets(768, torch.as_tensor(np.sort(np.random.default_rng(0).choice(768, 77, replace=False)), device="cuda"))
v7 = torch.randn(768, 768, device="cuda")
print("768x768 x3", 3 * timeit(lambda: ops.tc_backward_weight(p0, x, v7, sel7, 768, 768, need_soft=True, max_act=77, need_bias=True)))
for shift in (0, 64, 128, 512, 4096, 65536 + 4096):
    raw = torch.empty(T * 768 + shift, device="cuda", dtype=torch.bfloat16)
    xs = raw[shift:shift + T * 768].view(T, 768)
    xs.copy_(x)
    print("split, x shifted by", shift * 2, "B:", timeit(lambda: ops.tc_backward_weight_split(parts, xs, values, sel, M, N, need_soft=True, max_act=k, need_bias=True)))

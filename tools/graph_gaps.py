"""How much of the graphed ViT-B step is kernel time vs gaps between kernels:
the bench's own harness (bench.TrainHarness, whole step as one CUDA graph),
3 replays under torch.profiler (CUPTI traces graph-launched kernels) vs CUDA
events around the same replays.   python tools/graph_gaps.py [--model vit_b16]"""
import argparse
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import torch

import bench

p = argparse.ArgumentParser()
p.add_argument("--model", default="vit_b16")
a = p.parse_args()
args = bench.parse_args([]) if hasattr(bench, "parse_args") else None
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
wl = bench.Workload(a.model)
torch.manual_seed(1234)
model = wl.build(dev)
ns = argparse.Namespace(gpus=1, steps=3, warmup=3, graph="on", route="auto")
h = bench.TrainHarness(model, wl.batch(wl.default_batch, dev, 0), dev, 1, ns, wl.label_smoothing)
h.warm(3)
print(h.capture("on"))
for _ in range(3):
    h.train_step()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    h.train_step()
e.record()
torch.cuda.synchronize()
wall = s.elapsed_time(e) / 3
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        h.train_step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ker = sum(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total for e in ev) / 1e3 / 3
# busy time = union of kernel intervals (streams overlap)
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for st, en in iv:
    if cur_e is None or st > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = st, en
    else:
        cur_e = max(cur_e, en)
if cur_e is not None:
    busy += cur_e - cur_s
busy = busy / 1e3 / 3
n = len(ev) / 3
print(f"step (events) {wall:.2f} ms | kernels/step {n:.0f} | sum of kernel time {ker:.2f} ms | "
      f"busy (union) {busy:.2f} ms | idle {wall - busy:.2f} ms ({100 * (wall - busy) / wall:.1f} %)")
by = defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e.name[:70]
    by[k][0] += 1
    by[k][1] += (e.time_range.end - e.time_range.start) / 1e3 / 3
for k, v in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{v[1]:8.3f} ms  x{v[0] // 3:4d}  {k}")

# idle gaps: after each kernel, the time until the next kernel starts (union timeline of one replay)
iv = sorted((e.time_range.start, e.time_range.end, e.name[:60]) for e in ev)
third = len(iv) // 3
gaps = defaultdict(lambda: [0, 0.0])
cur_end = iv[0][1]
for k in range(1, third):
    st, en, nm = iv[k]
    if st > cur_end:
        gaps[nm][0] += 1
        gaps[nm][1] += (st - cur_end) / 1e3
    cur_end = max(cur_end, en)
print("idle before kernel (one replay): total %.3f ms" % sum(v[1] for v in gaps.values()))
for k, v in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"{v[1]:8.3f} ms  x{v[0]:4d}  {k}")

"""Which framework (aten) ops launch the non-DiagLinear kernels of an eager ViT-B
training step: torch.profiler op table sorted by device time.
  python tools/op_prof.py [--model vit_b16]"""
import argparse
import sys

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

import bench

p = argparse.ArgumentParser()
p.add_argument("--model", default="vit_b16")
a = p.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
wl = bench.Workload(a.model)
torch.manual_seed(1234)
model = wl.build(dev)
ns = argparse.Namespace(gpus=1, steps=3, warmup=3, graph="off", route="auto")
h = bench.TrainHarness(model, wl.batch(wl.default_batch, dev, 0), dev, 1, ns, wl.label_smoothing)
h.warm(3)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as prof:
    h.train_step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=60))
for e in prof.key_averages(group_by_input_shape=True):
    if e.key in ("aten::copy_", "aten::clone", "aten::add", "aten::sum", "aten::mul", "aten::cat", "aten::to", "aten::_to_copy") and e.device_time_total > 20:
        print(f"{e.key:16s} n={e.count:3d} cuda={e.device_time_total:9.1f}us shapes={str(e.input_shapes)[:150]}")

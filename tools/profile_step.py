"""Kernel-time breakdown of one ViT training step (torch.profiler / CUPTI).

    python tools/profile_step.py [--model vit_b16] [--route auto] [--batch 256]
"""
import argparse
import sys

sys.path.insert(0, ".")
import torch
import torch.nn.functional as F

from paper_2506_11449_b200 import AdamW, GlobalNormClipper, model_param_specs, penalties
from paper_2506_11449_b200.vit import VIT_B16, VIT_TINY16, ViT

p = argparse.ArgumentParser()
p.add_argument("--model", default="vit_b16")
p.add_argument("--route", default="auto")
p.add_argument("--batch", type=int, default=256)
p.add_argument("--rows", type=int, default=40)
a = p.parse_args()
cfg = VIT_B16 if a.model == "vit_b16" else VIT_TINY16
dev = torch.device("cuda")
model = ViT(cfg, route=a.route, device=dev)
specs = model_param_specs(model)
opt = AdamW(specs, lr=1e-3, betas=(0.9, 0.99), eps=1e-8, weight_decay=5e-5)
clip = GlobalNormClipper(1.0)
img = torch.randn(a.batch, 3, cfg.image, cfg.image, device=dev).to(torch.bfloat16)
lbl = torch.randint(0, cfg.classes, (a.batch,), device=dev)


def step(s):
    model.set_step(s)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model(img)
    loss = F.cross_entropy(logits.float(), lbl, label_smoothing=0.1)
    for pen in penalties(model, fused=True):
        loss = loss + pen
    loss.backward()
    _, sc = clip.compute(specs)
    opt.step(clip_scale=sc)
    opt.zero_grad()


for s in range(3):
    step(s)
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
step(3)
s1.record()
torch.cuda.synchronize()
print(f"step ms (events, unprofiled) {s0.elapsed_time(s1):.2f}")
import time
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step(3)
    t_host = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) * 1e3
    print(f"host enqueue ms {t_host:.2f}  enqueue+drain ms {t_all:.2f}")
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step(4)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=a.rows, max_name_column_width=70))
# kernels only, by self device time
ev = [e for e in prof.key_averages() if e.device_type.name == "CUDA" or getattr(e, "self_device_time_total", 0) > 0]
tot = sum(getattr(e, "self_device_time_total", 0) for e in ev)
print(f"\n# kernels by self device time (total {tot / 1e3:.2f} ms)")
for e in sorted(ev, key=lambda e: -getattr(e, "self_device_time_total", 0))[:a.rows]:
    t = getattr(e, "self_device_time_total", 0)
    if t <= 0:
        continue
    print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}% x{e.count:4d}  {e.key[:110]}")

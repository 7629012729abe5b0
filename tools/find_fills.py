"""Which ops launch fill/zero kernels inside a ViT training step (torch profiler, CPU op stacks)."""
import sys

sys.path.insert(0, ".")
import torch
import torch.nn.functional as F
from torch.profiler import ProfilerActivity, profile

from paper_2506_11449_b200 import AdamW, GlobalNormClipper, model_param_specs, penalties
from paper_2506_11449_b200.vit import VIT_B16, ViT

dev = torch.device("cuda")
model = ViT(VIT_B16, route="auto", device=dev)
specs = model_param_specs(model)
opt = AdamW(specs, lr=1e-3, betas=(0.9, 0.99), eps=1e-8, weight_decay=5e-5)
clip = GlobalNormClipper(1.0)
img = torch.randn(64, 3, 224, 224, device=dev).to(torch.bfloat16)
lbl = torch.randint(0, 1000, (64,), device=dev)


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
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
    step(4)
    torch.cuda.synchronize()
for ev in prof.key_averages(group_by_stack_n=6):
    if ev.key in ("aten::fill_", "aten::zero_", "aten::zeros", "aten::ones_like", "aten::zeros_like", "aten::add", "aten::add_", "aten::copy_"):
        print(ev.key, ev.count, f"{ev.device_time_total:.0f}us")
        for fr in ev.stack[:6]:
            print("    ", fr)

"""Which ATen ops launch the non-DiagLinear kernels of a ViT-B step (shapes)."""
import sys
sys.path.insert(0, ".")
import torch
import torch.nn.functional as F
from paper_2506_11449_b200 import AdamW, GlobalNormClipper, model_param_specs, penalties
from paper_2506_11449_b200.vit import VIT_B16, ViT
dev = torch.device("cuda")
model = ViT(VIT_B16, route="auto", device=dev)
specs = model_param_specs(model)
opt = AdamW(specs, lr=1e-3)
clip = GlobalNormClipper(1.0)
img = torch.randn(256, 3, 224, 224, device=dev).to(torch.bfloat16)
lbl = torch.randint(0, 1000, (256,), device=dev)
def step(s):
    model.set_step(s)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model(img)
    loss = F.cross_entropy(logits.float(), lbl, label_smoothing=0.1)
    for p in penalties(model, fused=True):
        loss = loss + p
    loss.backward()
    _, sc = clip.compute(specs)
    opt.step(clip_scale=sc)
    opt.zero_grad()
for s in range(3):
    step(s)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], record_shapes=True) as prof:
    step(4)
    torch.cuda.synchronize()
t = prof.key_averages(group_by_input_shape=True).table(sort_by="self_cuda_time_total", row_limit=30,
                                                       max_name_column_width=45, max_shapes_column_width=70)
print(t)

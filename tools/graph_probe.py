"""Can the ViT-B training step (fwd + bwd + clip + AdamW) be captured in one CUDA graph?"""
import sys
import time

sys.path.insert(0, ".")
import torch
import torch.nn.functional as F

from paper_2506_11449_b200 import AdamW, GlobalNormClipper, model_param_specs, penalties
from paper_2506_11449_b200.vit import VIT_B16, ViT

dev = torch.device("cuda")
model = ViT(VIT_B16, route="auto", device=dev)
specs = model_param_specs(model)
opt = AdamW(specs, lr=1e-3, betas=(0.9, 0.99), eps=1e-8, weight_decay=5e-5)
clip = GlobalNormClipper(1.0)
img = torch.randn(256, 3, 224, 224, device=dev).to(torch.bfloat16)
lbl = torch.randint(0, 1000, (256,), device=dev)


def fwd_bwd():
    model.set_step(0)
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        logits = model(img)
    loss = F.cross_entropy(logits.float(), lbl, label_smoothing=0.1)
    for pen in penalties(model, fused=True):
        loss = loss + pen
    loss.backward()
    return loss


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        fwd_bwd()
        for sp in specs:
            sp.tensor.grad = None
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g):
        loss = fwd_bwd()
    print("captured fwd+bwd OK")
except Exception as e:  # noqa: BLE001
    import traceback; traceback.print_exc(limit=12)
    sys.exit(0)
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph fwd+bwd ms {e0.elapsed_time(e1) / 10:.2f}")
e0.record()
for _ in range(10):
    fwd_bwd()
    for sp in specs:
        sp.tensor.grad = None
e1.record()
torch.cuda.synchronize()
print(f"eager fwd+bwd ms {e0.elapsed_time(e1) / 10:.2f}")

"""Probe LayerNorm variants at ViT-B token counts (fwd+bwd device time)."""
import torch
import torch.nn.functional as F

dev = "cuda"
M, D = 50432, 768


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


x0 = torch.randn(M, D, device=dev, dtype=torch.bfloat16)
g = torch.randn(M, D, device=dev, dtype=torch.bfloat16)
w = torch.ones(D, device=dev, requires_grad=True)
b = torch.zeros(D, device=dev, requires_grad=True)


def autocast_fp32():
    x = x0.detach().requires_grad_(True)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        y = F.layer_norm(x, (D,), w, b)
    y.backward(g.float() if y.dtype == torch.float32 else g)


def bf16_ln():
    x = x0.detach().requires_grad_(True)
    with torch.autocast("cuda", enabled=False):
        y = F.layer_norm(x, (D,), w.to(torch.bfloat16), b.to(torch.bfloat16))
    y.backward(g)


def bf16_ln_fp32w():
    x = x0.detach().requires_grad_(True)
    with torch.autocast("cuda", enabled=False):
        y = F.layer_norm(x, (D,), w, b)
    y.backward(g)


for name, fn in [("autocast fp32 LN", autocast_fp32), ("bf16 LN bf16 weights", bf16_ln),
                 ("bf16 input fp32 weights", bf16_ln_fp32w)]:
    try:
        print(f"{name}: {timeit(fn):.1f} us fwd+bwd")
    except Exception as exc:  # noqa: BLE001
        print(f"{name}: failed {exc}")

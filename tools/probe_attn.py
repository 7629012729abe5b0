"""Probe attention variants for the ViT-B block at 256 images (197 tokens, 12 heads)."""
import torch
import torch.nn.functional as F

B, T, H, hd = 256, 197, 12, 64
dev = "cuda"


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


h0 = torch.randn(B, T, 3, H, hd, device=dev, dtype=torch.bfloat16)
g = torch.randn(B, T, H * hd, device=dev, dtype=torch.bfloat16)


def sdpa_unbind():
    h = h0.detach().requires_grad_(True)
    q, k, v = h.permute(2, 0, 3, 1, 4).unbind(0)
    a = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(B, T, H * hd)
    a.backward(g)


print(f"sdpa+unbind: {timeit(sdpa_unbind):.0f} us")
try:
    from flash_attn import flash_attn_qkvpacked_func

    def fa_packed():
        h = h0.detach().requires_grad_(True)
        a = flash_attn_qkvpacked_func(h).reshape(B, T, H * hd)
        a.backward(g)

    print(f"flash_attn qkvpacked: {timeit(fa_packed):.0f} us")
except Exception as exc:  # noqa: BLE001
    print("flash_attn failed:", type(exc).__name__, str(exc)[:200])

"""The ViT caller's fused patch embedding (diagmm_vit_patchify / _embed_fwd / _embed_bwd,
PatchEmbedFunction) against the framework path it replaces (permute-copy + linear + cat +
broadcast add): the patches and the embedded tokens bit for bit, the gradients of the
patch weight / bias, cls and pos to the bf16 rounding of their sums (needs a B200)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_11449_b200 import _lib
    from paper_2506_11449_b200.vit import ViT, ViTConfig


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_patchify_kernel_bitwise():
    g = torch.Generator(device="cuda").manual_seed(3)
    img = torch.randn(3, 3, 64, 48, device="cuda", generator=g).to(torch.bfloat16)
    p = 16
    out = torch.empty(3 * 4 * 3, 3 * p * p, dtype=torch.bfloat16, device="cuda")
    _lib.call("diagmm_vit_patchify", 3, 3, 64, 48, p, img.data_ptr(), out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    ref = img.reshape(3, 3, 4, p, 3, p).permute(0, 2, 4, 1, 3, 5).reshape(-1, 3 * p * p)
    assert torch.equal(out, ref)


def _vit_run(fuse: str, monkeypatch):
    monkeypatch.setenv("DIAGMM_FUSE_EMBED", fuse)
    torch.manual_seed(0)
    model = ViT(ViTConfig(dim=256, depth=1, heads=4, classes=10), device="cuda")
    with torch.no_grad():
        model.cls.normal_()
        model.patch.bias.normal_()
    g = torch.Generator(device="cuda").manual_seed(9)
    img = torch.randn(6, 3, 224, 224, device="cuda", generator=g).to(torch.bfloat16)
    model.set_step(0)
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        tokens = model._embed(img) if hasattr(model, "_embed") else None
        logits = model(img)
    logits.float().square().sum().backward()
    torch.cuda.synchronize()
    grads = {n: p.grad.detach().clone() for n, p in model.named_parameters()
             if n.startswith(("patch.", "cls", "pos"))}
    return logits.detach().clone(), grads


def test_fused_embedding_matches_framework_path(monkeypatch):
    ref_logits, ref = _vit_run("0", monkeypatch)
    got_logits, got = _vit_run("1", monkeypatch)
    assert torch.equal(got_logits, ref_logits)  # identical forward roundings
    for name, r in ref.items():
        a = got[name]
        scale = float(r.abs().max())
        # sums over 6 x 196 tokens re-associated: within a few bf16 ulps of the largest entry
        assert float((a - r).abs().max()) <= 2 ** -6 * scale + 1e-12, name

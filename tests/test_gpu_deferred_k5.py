"""Deferred, batched K5 and tensor-core dW finalize (every layer's g_values / g_bias /
g_soft fold and soft-TopK gradient in one launch each after the backward,
``deferred_topk_grads``) against the per-layer path: bit-identical values / bias / alpha
gradients on the tensor-core route (ViT blocks: plain DiagLinear, the fused MLP and
the fused qkv-attention node), on the FMA route, with gradient accumulation, and
inside a captured CUDA graph (needs a B200)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import torch.nn.functional as F

    from paper_2506_11449_b200 import DiagLinear, TemperatureSchedule, deferred_topk_grads, penalties
    from paper_2506_11449_b200.graphed import GraphedStep
    from paper_2506_11449_b200.vit import ViT, ViTConfig


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _vit_grads(deferred: bool, accumulate: bool = False):
    torch.manual_seed(0)
    cfg = ViTConfig(dim=256, depth=2, heads=4, classes=10)
    model = ViT(cfg, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    img = torch.randn(4, 3, 224, 224, device="cuda", generator=g).to(torch.bfloat16)
    lbl = torch.randint(0, 10, (4,), device="cuda", generator=g)
    for _ in range(2 if accumulate else 1):
        model.set_step(0)
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            logits = model(img)
        loss = F.cross_entropy(logits.float(), lbl)
        for pen in penalties(model, fused=True):
            loss = loss + pen
        if deferred:
            with deferred_topk_grads():
                loss.backward()
        else:
            loss.backward()
    torch.cuda.synchronize()
    return [p.grad.detach().clone() if p.grad is not None else None for p in model.parameters()]


@pytest.mark.parametrize("accumulate", [False, True])
def test_deferred_k5_bitwise_equal_tensor_core_route(accumulate):
    ref = _vit_grads(False, accumulate)
    got = _vit_grads(True, accumulate)
    assert len(ref) == len(got) > 0
    for a, b in zip(ref, got):
        assert (a is None) == (b is None)
        assert a is None or torch.equal(a, b)


def test_deferred_k5_fma_route_and_graph():
    sched = TemperatureSchedule("constant", 0.05, 0.05, 1)

    def build():
        torch.manual_seed(0)
        return [DiagLinear(256, 512, 0.9, seed=1, dtype=torch.float32, t_schedule=sched, l1_coeff=1e-4),
                DiagLinear(512, 256, 0.9, seed=2, dtype=torch.float32, t_schedule=sched, l1_coeff=1e-4)]

    x = torch.randn(48, 256, device="cuda")
    up = torch.randn(48, 256, device="cuda")

    def run(layers, deferred):
        def fwd_bwd(inp, u):
            loss = (layers[1](layers[0](inp, step=0), step=0) * u).sum()
            for pen in penalties(torch.nn.ModuleList(layers), fused=True):
                loss = loss + pen
            if deferred:
                with deferred_topk_grads():
                    loss.backward()
            else:
                loss.backward()
            return loss
        return fwd_bwd

    ref_layers = build()
    run(ref_layers, False)(x, up)
    ref = [m.alpha.grad.clone() for m in ref_layers]
    eager_layers = build()
    run(eager_layers, True)(x, up)
    for m, r in zip(eager_layers, ref):
        assert torch.equal(m.alpha.grad, r)
    graph_layers = build()
    params = [p for m in graph_layers for p in m.parameters()]
    gs = GraphedStep(run(graph_layers, True), params, x.clone(), up.clone())
    gs.step(x, up)
    torch.cuda.synchronize()
    for m, r in zip(graph_layers, ref):
        assert torch.equal(m.alpha.grad, r)


def test_batched_w_k_prepass_bitwise_equal(monkeypatch):
    """preselect(materialize=bf16): every layer's W_K built in one launch before the forward
    gives the same logits and gradients, bit for bit, as the per-layer builds."""
    def run(premat: str):
        monkeypatch.setenv("DIAGMM_PREMAT", premat)
        torch.manual_seed(0)
        model = ViT(ViTConfig(dim=256, depth=2, heads=4, classes=10), device="cuda")
        g = torch.Generator(device="cuda").manual_seed(7)
        img = torch.randn(4, 3, 224, 224, device="cuda", generator=g).to(torch.bfloat16)
        model.set_step(0)
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            logits = model(img)
        logits.float().square().sum().backward()
        torch.cuda.synchronize()
        return [logits.detach().clone()] + [p.grad.detach().clone() for p in model.parameters() if p.grad is not None]

    ref, got = run("0"), run("1")
    assert len(ref) == len(got)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)

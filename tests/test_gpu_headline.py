"""The bench's headline configuration against the float64 oracle (needs a B200).

BENCH times ViT-B/16 at 256 images per GPU, i.e. every DiagLinear call sees
50 432 tokens and runs the bf16 tensor-core route: W_K materialized once, the
tcgen05 GEMM for y and dX (dX reads W_K MN-major), the fused-gather tcgen05 dW
with split-K over tokens, and the caller fusions — qkv's input and weight
gradients reading cuDNN's dq / dk / dv blocks in place, proj's residual add in
the epilogue, fc1's GELU and fc2's GELU' in the epilogues.  Every one of those
is checked here at that token count against the float64 oracle on the same
bf16 inputs:

* selections (offsets, clamped set) from ``oracle.topk`` — bit-exact;
* W_K from ``oracle.dense_matrix`` and entry coordinates from
  ``oracle.entry_coords``; y and dX on 64 sampled rows also straight from
  ``oracle.diag_spmm`` (the bulk float64 products run as torch float64 GEMMs on
  the same device, library code independent of our kernels, tied to the oracle
  by the sampled rows);
* g_values / g_soft / g_bias in full from the float64 dyᵀx gathered at the
  oracle's coordinates, g_alpha from ``oracle.soft_topk_grad``.

Tolerances (max|got − ref| / max(1, max|ref|), bench._validate's scale):
``BF16_TOL`` = 5e-3 for bf16 outputs (the output rounding alone is up to
2^-9 ≈ 2e-3 of max|y|, W_K's bf16 rounding adds ≈ 1e-3); ``DW_TOL`` = 1e-4 for
the weight / bias gradients of one layer (exact bf16 products, float32
accumulation over 50 432 tokens).
"""

import numpy as np
import pytest
import torch

import oracle
from diagtest_util import scaled_err

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_11449_b200 import DiagLinear, DiagMLP, TemperatureSchedule, ops

BF16_TOL = 5e-3
DW_TOL = 1e-4
DEV = "cuda"
TOKENS = 256 * 197  # ViT-B/16, 256 images per GPU
SAMPLE_ROWS = 64


MEASURED: dict = {}  # test -> the largest scaled error each check saw (written to gpurun_out/)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    import json
    import os
    from pathlib import Path

    out = Path(os.environ.get("GRAFT_REPO_ROOT", Path(__file__).resolve().parents[1])) / "gpurun_out"
    if out.is_dir() and MEASURED:
        (out / "headline_parity_errors.json").write_text(json.dumps(MEASURED, indent=1, sort_keys=True))


@pytest.fixture(autouse=True)
def _name(request):
    global _CUR
    _CUR = request.node.name
    yield


_CUR = "?"


def _layer(n_in, n_out, seed, T):
    """A ViT-B-shaped DiagLinear on the tensor-core route, alpha perturbed so the
    soft selection is non-trivial, random bias."""
    lyr = DiagLinear(n_in, n_out, 0.9, seed=seed, l1_coeff=0.0, route="auto",
                     t_schedule=TemperatureSchedule("constant", T, T, 1))
    rng = np.random.default_rng(seed + 100)
    with torch.no_grad():
        lyr.alpha.add_(torch.as_tensor(rng.standard_normal(lyr.candidates), device=DEV))
        lyr.bias.copy_(torch.as_tensor(rng.standard_normal(n_out) * 0.1, device=DEV))
    return lyr


class _Ref:
    """float64 reference of one layer at its current selection (oracle geometry)."""

    def __init__(self, lyr, T):
        M, N = lyr.out_features, lyr.in_features
        self.M, self.N, self.T, self.k = M, N, T, lyr.k
        self.alpha = lyr.alpha.detach().cpu().numpy()
        self.values = lyr.values.detach().double().cpu().numpy()
        self.soft = oracle.soft_topk(self.alpha, lyr.k, T)
        self.active = np.flatnonzero(self.soft >= oracle.EPS_ACTIVE)
        self.weights = self.soft[self.active, None] * self.values[self.active]
        self.W = torch.as_tensor(oracle.dense_matrix(M, N, self.active, self.weights), device=DEV)
        self.bias = lyr.bias.detach().double()
        r, c = oracle.entry_coords(M, N, self.active)
        self.r = torch.as_tensor(r, device=DEV)
        self.c = torch.as_tensor(c, device=DEV)

    def forward(self, x64):
        return x64 @ self.W.t() + self.bias

    def input_grad(self, dy64):
        return dy64 @ self.W

    def grads(self, dy64, x64):
        """(g_values, g_soft, g_alpha, g_bias) of layers.py:149-167 in float64."""
        gw = (dy64.t() @ x64)[self.r, self.c].cpu().numpy()
        C = self.values.shape[0]
        g_values = np.zeros_like(self.values)
        g_values[self.active] = self.soft[self.active, None] * gw
        g_soft = np.zeros(C)
        g_soft[self.active] = (gw * self.values[self.active]).sum(axis=1)
        g_alpha = oracle.soft_topk_grad(self.alpha, self.k, self.T, g_soft)
        return g_values, g_soft, g_alpha, dy64.sum(0).cpu().numpy()

    def check_rows(self, x_rows64, y_rows64):
        """The bulk float64 product equals the oracle's own diagonal product on sampled rows."""
        want = oracle.diag_spmm(self.M, self.N, self.active, self.weights, x_rows64.cpu().numpy().T).T
        assert scaled_err(y_rows64.cpu().numpy() - self.bias.cpu().numpy(), want) < 1e-10


def _rows(n):
    rng = np.random.default_rng(n)
    return torch.as_tensor(np.sort(rng.choice(n, SAMPLE_ROWS, replace=False)), device=DEV)


def _bf16(shape, seed, scale=1.0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return (torch.randn(*shape, device=DEV, generator=g) * scale).to(torch.bfloat16)


def _err(got, want):
    e = scaled_err(got.double().cpu().numpy() if torch.is_tensor(got) else got,
                   want.cpu().numpy() if torch.is_tensor(want) else want)
    MEASURED.setdefault(_CUR, []).append(e)
    return e


def _check_layer_grads(lyr, ref, dy64, x64, tol_w=DW_TOL):
    g_values, g_soft, g_alpha, g_bias = ref.grads(dy64, x64)
    assert _err(lyr.values.grad, g_values) <= tol_w
    assert _err(lyr.bias.grad, g_bias) <= tol_w
    assert _err(lyr.alpha.grad, g_alpha) <= tol_w
    inactive = torch.as_tensor(np.setdiff1d(np.arange(lyr.candidates), ref.active), device=DEV)
    assert not lyr.values.grad[inactive].any()  # layers.py:159-163: exactly zero


@pytest.mark.parametrize("T", [0.05, 1e-9])
def test_proj_residual_epilogue_vs_oracle(T):
    """proj (768 -> 768) with the block's residual add fused into the tcgen05 epilogue."""
    lyr = _layer(768, 768, 1, T)
    ref = _Ref(lyr, T)
    x = _bf16((TOKENS, 768), 1).requires_grad_(True)
    r = _bf16((TOKENS, 768), 2).requires_grad_(True)
    dy = _bf16((TOKENS, 768), 3)
    y = lyr(x, step=0, residual=r)
    y.backward(dy)
    np.testing.assert_array_equal(lyr.active_set(0).cpu().numpy(), ref.active)  # bit-exact offsets
    rows = _rows(TOKENS)
    x64, dy64 = x.detach().double(), dy.double()
    y_ref = ref.forward(x64[rows]) + r.detach().double()[rows]
    ref.check_rows(x64[rows], ref.forward(x64[rows]))
    assert _err(y.detach()[rows], y_ref) <= BF16_TOL
    assert _err(x.grad[rows], ref.input_grad(dy64[rows])) <= BF16_TOL
    assert torch.equal(r.grad, dy)  # d residual = dy, untouched
    _check_layer_grads(lyr, ref, dy64, x64)


@pytest.mark.parametrize("shape", [(768, 3072), (3072, 768)])
def test_mlp_shapes_plain_route_vs_oracle(shape):
    """fc1 / fc2 shapes through DiagMMFunction's tensor-core route (no fusion),
    split-K dW at 50 432 tokens, every gradient in full."""
    n_in, n_out = shape
    T = 0.05
    lyr = _layer(n_in, n_out, 2, T)
    ref = _Ref(lyr, T)
    x = _bf16((TOKENS, n_in), 4).requires_grad_(True)
    dy = _bf16((TOKENS, n_out), 5)
    y = lyr(x, step=0)
    y.backward(dy)
    rows = _rows(TOKENS)
    x64, dy64 = x.detach().double(), dy.double()
    ref.check_rows(x64[rows], ref.forward(x64[rows]))
    assert _err(y.detach()[rows], ref.forward(x64[rows])) <= BF16_TOL
    assert _err(x.grad[rows], ref.input_grad(dy64[rows])) <= BF16_TOL
    _check_layer_grads(lyr, ref, dy64, x64)


def _gelu64(p):
    return torch.nn.functional.gelu(p, approximate="tanh")


def _gelu_grad64(p):
    k0, k1 = 0.7978845608028654, 0.044715
    t = torch.tanh(k0 * (p + k1 * p ** 3))
    return 0.5 * (1 + t) + 0.5 * p * (1 - t * t) * k0 * (1 + 3 * k1 * p * p)


def test_mlp_gelu_epilogues_vs_oracle():
    """ViT-B MLP (768 -> 3072 -> GELU -> 768) + residual through DiagMLPFunction:
    fc1's epilogue writes the pre-activation and gelu(pre), fc2's input-gradient
    epilogue multiplies by gelu'(pre).  The float64 reference rounds at the same
    stage boundaries the bf16 path stores tensors (pre, act, d_pre are bf16)."""
    T = 0.05
    f1, f2 = _layer(768, 3072, 3, T), _layer(3072, 768, 4, T)
    r1, r2 = _Ref(f1, T), _Ref(f2, T)
    mlp = DiagMLP(f1, f2)
    x = _bf16((TOKENS, 768), 6).requires_grad_(True)
    res = _bf16((TOKENS, 768), 7).requires_grad_(True)
    dy = _bf16((TOKENS, 768), 8)
    assert mlp._fusable(x.detach())
    y = mlp(x, step=0, residual=res)
    y.backward(dy)

    bf = lambda t_: t_.to(torch.bfloat16).double()  # noqa: E731 - a stored bf16 tensor
    x64, dy64 = x.detach().double(), dy.double()
    pre = bf(r1.forward(x64))
    act = bf(_gelu64(pre))
    y_ref = act @ r2.W.t() + r2.bias + res.detach().double()
    d_pre = bf((dy64 @ r2.W) * _gelu_grad64(pre))
    dx_ref = d_pre @ r1.W
    rows = _rows(TOKENS)
    r1.check_rows(x64[rows], r1.forward(x64[rows]))
    assert _err(y.detach()[rows], y_ref[rows]) <= BF16_TOL
    assert _err(x.grad[rows], dx_ref[rows]) <= BF16_TOL
    assert torch.equal(res.grad, dy)
    # weight gradients through rounded intermediates: one bf16 ulp on a fraction of
    # the stored activations moves a token sum by ~2^-9 of its size -> BF16_TOL
    _check_layer_grads(f2, r2, dy64, act, tol_w=BF16_TOL)
    _check_layer_grads(f1, r1, d_pre, x64, tol_w=BF16_TOL)


def test_qkv_split_gradient_path_vs_oracle():
    """qkv (768 -> 2304): the three calls QKVAttentionFunction makes — h = x W_K^T + b
    on the tcgen05 GEMM, dx = [dq|dk|dv] W_K with the three (tokens x 768) blocks
    selected per k-block, and the split dW reading them per m-block (bias fused) —
    against the oracle on the concatenated gradient."""
    T = 0.05
    lyr = _layer(768, 2304, 5, T)
    ref = _Ref(lyr, T)
    sel = lyr.selection(0)
    np.testing.assert_array_equal(sel.active_offsets().cpu().numpy(), ref.active)
    x = _bf16((TOKENS, 768), 9)
    parts = [_bf16((TOKENS, 768), 10 + i) for i in range(3)]
    vals = lyr.values.detach()
    W = ops.materialize(vals, sel, 2304, 768, dtype=torch.bfloat16)
    h = ops.tc_gemm(x, W, lyr.bias.detach())
    dx = ops.tc_gemm_nn_split(parts, W)
    gv, gs, gb = ops.tc_backward_weight_split(parts, x, vals, sel, 2304, 768, need_soft=True, need_bias=True)
    ga = ops.soft_topk_grad(lyr.alpha.detach(), lyr.k, T, gs, clamped=sel.clamped)
    rows = _rows(TOKENS)
    x64 = x.double()
    dh64 = torch.cat([p.double() for p in parts], dim=1)
    ref.check_rows(x64[rows], ref.forward(x64[rows]))
    assert _err(h[rows], ref.forward(x64[rows])) <= BF16_TOL
    assert _err(dx[rows], ref.input_grad(dh64[rows])) <= BF16_TOL
    g_values, g_soft, g_alpha, g_bias = ref.grads(dh64, x64)
    assert _err(gv, g_values) <= DW_TOL
    assert _err(gs, g_soft) <= DW_TOL
    assert _err(ga, g_alpha) <= DW_TOL
    assert _err(gb, g_bias) <= DW_TOL
    # the single-matrix dW on the concatenated gradient is the same reduction, bit for bit
    gv1, gs1, gb1 = ops.tc_backward_weight(dh64.to(torch.bfloat16), x, vals, sel, 2304, 768, need_soft=True,
                                           need_bias=True)
    assert torch.equal(gv1, gv) and torch.equal(gb1, gb)


def test_vit_depth2_step_vs_fp32_reference_model():
    """One ViT-B-width (768, 12 heads) depth-2 training step of the bf16 model
    (tensor-core route, split qkv, fused MLP / residual / LayerNorm nodes, fused
    l1) against a plain PyTorch float32 model whose linear layers carry the
    oracle's dense W_K (oracle.dense_matrix at the oracle's selection): the loss,
    every DiagLinear gradient (values / alpha / bias, alpha through
    oracle.soft_topk_grad + l1) and the dense parameters' gradients."""
    import torch.nn.functional as F

    from paper_2506_11449_b200 import penalties
    from paper_2506_11449_b200.vit import ViT, ViTConfig

    T = 0.05
    cfg = ViTConfig(dim=768, depth=2, heads=12, classes=1000)
    torch.manual_seed(0)
    model = ViT(cfg, t_schedule=TemperatureSchedule("constant", T, T, 1), device=DEV)
    for i, m in enumerate(model.diag_layers()):
        rng = np.random.default_rng(200 + i)
        with torch.no_grad():
            m.alpha.add_(torch.as_tensor(rng.standard_normal(m.candidates), device=DEV))
            m.bias.copy_(torch.as_tensor(rng.standard_normal(m.out_features) * 0.05, device=DEV))
    g = torch.Generator(device=DEV).manual_seed(1)
    B = 8  # 1576 tokens: the tensor-core route (>= 512 tokens)
    img = torch.randn(B, 3, 224, 224, device=DEV, generator=g).to(torch.bfloat16)
    lbl = torch.randint(0, 1000, (B,), device=DEV, generator=g)
    model.set_step(0)
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        logits = model(img)
    loss = F.cross_entropy(logits.float(), lbl, label_smoothing=0.1)
    for p in penalties(model, fused=True):
        loss = loss + p
    loss.backward()

    # ---- float32 reference model, same parameters, oracle W_K
    refs = {id(m): _Ref(m, T) for m in model.diag_layers()}
    Wleaf = {k: r.W.float().clone().requires_grad_(True) for k, r in refs.items()}
    bleaf = {id(m): m.bias.detach().float().clone().requires_grad_(True) for m in model.diag_layers()}
    dense = {n: p.detach().float().clone().requires_grad_(True) for n, p in model.named_parameters()
             if not any(n.endswith(s) for s in (".values", ".alpha")) and "qkv.bias" not in n
             and "proj.bias" not in n and "fc1.bias" not in n and "fc2.bias" not in n}

    def lin(m, x):
        return x @ Wleaf[id(m)].t() + bleaf[id(m)]

    x = img.float()
    p = cfg.patch
    xp = x.reshape(B, 3, 14, p, 14, p).permute(0, 2, 4, 1, 3, 5).reshape(B, -1, 3 * p * p)
    h = xp @ dense["patch.weight"].reshape(cfg.dim, -1).t() + dense["patch.bias"]
    h = torch.cat([dense["cls"].expand(B, -1, -1), h], dim=1) + dense["pos"]
    for i, blk in enumerate(model.blocks):
        pre = f"blocks.{i}."
        hn = F.layer_norm(h, (cfg.dim,), dense[pre + "norm1.weight"], dense[pre + "norm1.bias"], 1e-5)
        qkv = lin(blk.qkv, hn).view(B, -1, 3, cfg.heads, cfg.dim // cfg.heads).permute(2, 0, 3, 1, 4)
        a = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2]).transpose(1, 2).reshape(B, -1, cfg.dim)
        h = h + lin(blk.proj, a)
        hn = F.layer_norm(h, (cfg.dim,), dense[pre + "norm2.weight"], dense[pre + "norm2.bias"], 1e-5)
        h = h + lin(blk.fc2, F.gelu(lin(blk.fc1, hn), approximate="tanh"))
    hn = F.layer_norm(h, (cfg.dim,), dense["norm.weight"], dense["norm.bias"], 1e-5)
    ref_logits = hn[:, 0] @ dense["head.weight"].t() + dense["head.bias"]
    ref_loss = F.cross_entropy(ref_logits, lbl, label_smoothing=0.1)
    pen = sum(m.l1_coeff * float(np.abs(refs[id(m)].alpha).sum()) for m in model.diag_layers())
    ref_loss.backward()

    assert abs(loss.item() - (ref_loss.item() + pen)) <= 1e-2 * abs(ref_loss.item() + pen)
    MODEL_TOL = 1e-2  # whole bf16 model vs float32 (measured <= 2.6e-3 on B200, profiles/r02_headline_parity_errors.json)
    for m in model.diag_layers():
        r = refs[id(m)]
        dW = Wleaf[id(m)].grad.double()
        gw = dW[r.r, r.c].cpu().numpy()
        g_values = np.zeros_like(r.values)
        g_values[r.active] = r.soft[r.active, None] * gw
        g_soft = np.zeros(r.values.shape[0])
        g_soft[r.active] = (gw * r.values[r.active]).sum(axis=1)
        g_alpha = oracle.soft_topk_grad(r.alpha, r.k, T, g_soft) + oracle.l1_term(r.alpha, m.l1_coeff)[1]
        assert _err(m.values.grad, g_values) <= MODEL_TOL
        assert _err(m.alpha.grad, g_alpha) <= MODEL_TOL
        assert _err(m.bias.grad, bleaf[id(m)].grad) <= MODEL_TOL
    for n in ("patch.weight", "head.weight", "blocks.0.norm1.weight"):
        got = dict(model.named_parameters())[n].grad
        assert _err(got.float(), dense[n].grad.double()) <= MODEL_TOL, n


def _diag_grads_ref(m, r, dW, T):
    """g_values / g_alpha of a DiagLinear from the reference model's dense dW (layers.py:149-167)."""
    gw = dW.double()[r.r, r.c].cpu().numpy()
    g_values = np.zeros_like(r.values)
    g_values[r.active] = r.soft[r.active, None] * gw
    g_soft = np.zeros(r.values.shape[0])
    g_soft[r.active] = (gw * r.values[r.active]).sum(axis=1)
    g_alpha = oracle.soft_topk_grad(r.alpha, r.k, T, g_soft) + oracle.l1_term(r.alpha, m.l1_coeff)[1]
    return g_values, g_alpha


def test_gpt2_block_step_vs_fp32_reference_model():
    """GPT-2 small geometry (768, 12 heads, seq 1024, causal), one block, all four
    projections DiagLinear at 90 %: loss and every gradient of the
    bf16 model (tensor-core route, qkv + causal cuDNN attention node, fused MLP /
    residual epilogues) against a float32 PyTorch model carrying the oracle's W_K."""
    import torch.nn.functional as F

    from paper_2506_11449_b200 import penalties
    from paper_2506_11449_b200.gpt2 import GPT2, GPT2Config

    T = 0.05
    cfg = GPT2Config(vocab=512, depth=1)
    torch.manual_seed(0)
    model = GPT2(cfg, t_schedule=TemperatureSchedule("constant", T, T, 1), device=DEV)
    for i, m in enumerate(model.diag_layers()):
        rng = np.random.default_rng(300 + i)
        with torch.no_grad():
            m.alpha.add_(torch.as_tensor(rng.standard_normal(m.candidates), device=DEV))
            m.bias.copy_(torch.as_tensor(rng.standard_normal(m.out_features) * 0.05, device=DEV))
    g = torch.Generator(device=DEV).manual_seed(2)
    ids = torch.randint(0, cfg.vocab, (1, cfg.ctx), device=DEV, generator=g)
    lbl = torch.randint(0, cfg.vocab, (1, cfg.ctx), device=DEV, generator=g)
    model.set_step(0)
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        logits = model(ids)
    loss = F.cross_entropy(logits.float().reshape(-1, cfg.vocab), lbl.reshape(-1))
    for p in penalties(model, fused=True):
        loss = loss + p
    loss.backward()

    refs = {id(m): _Ref(m, T) for m in model.diag_layers()}
    W = {k: r.W.float().clone().requires_grad_(True) for k, r in refs.items()}
    b = {id(m): m.bias.detach().float().clone().requires_grad_(True) for m in model.diag_layers()}
    P = {n: p.detach().float().clone().requires_grad_(True) for n, p in model.named_parameters()
         if "wte" in n or "wpe" in n or "ln" in n or "norm" in n}
    lin = lambda m, x: x @ W[id(m)].t() + b[id(m)]  # noqa: E731
    blk = model.blocks[0]
    h = P["wte.weight"][ids] + P["wpe.weight"][None, : cfg.ctx]
    hn = F.layer_norm(h, (cfg.dim,), P["blocks.0.norm1.weight"], P["blocks.0.norm1.bias"], 1e-5)
    qkv = lin(blk.qkv, hn).view(1, cfg.ctx, 3, cfg.heads, cfg.dim // cfg.heads).permute(2, 0, 3, 1, 4)
    a = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], is_causal=True).transpose(1, 2).reshape(1, -1, cfg.dim)
    h = h + lin(blk.proj, a)
    hn = F.layer_norm(h, (cfg.dim,), P["blocks.0.norm2.weight"], P["blocks.0.norm2.bias"], 1e-5)
    h = h + lin(blk.fc2, F.gelu(lin(blk.fc1, hn), approximate="tanh"))
    hn = F.layer_norm(h, (cfg.dim,), P["ln_f.weight"], P["ln_f.bias"], 1e-5)
    ref_loss = F.cross_entropy((hn @ P["wte.weight"].t()).reshape(-1, cfg.vocab), lbl.reshape(-1))
    pen = sum(m.l1_coeff * float(np.abs(refs[id(m)].alpha).sum()) for m in model.diag_layers())
    ref_loss.backward()

    assert abs(loss.item() - (ref_loss.item() + pen)) <= 1e-2 * abs(ref_loss.item() + pen)
    MODEL_TOL = 2e-3  # measured <= 1.5e-4 on B200 (profiles/r02_headline_parity_errors.json)
    for m in model.diag_layers():
        g_values, g_alpha = _diag_grads_ref(m, refs[id(m)], W[id(m)].grad, T)
        assert _err(m.values.grad, g_values) <= MODEL_TOL
        assert _err(m.alpha.grad, g_alpha) <= MODEL_TOL
        assert _err(m.bias.grad, b[id(m)].grad) <= MODEL_TOL
    got = dict(model.named_parameters())
    for n in ("wte.weight", "wpe.weight", "blocks.0.norm1.weight"):
        assert _err(got[n].grad.float(), P[n].grad.double()) <= MODEL_TOL, n

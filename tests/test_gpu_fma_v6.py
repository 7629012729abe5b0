"""The v6 FMA kernels (k_product6 with its interleaved weight ring and the three
staged-row modes, k_dw6 with packed operands and bulk-copy double buffering)
against the CPU oracle, through the C ABI (needs a B200).

Cases are chosen to hit every v6 branch: gather rows (wide forward / tall dX),
circular scatter rows (square and near-square C < L + 128), guard-band scatter
rows (tall forward / wide dX, C >= L + 128), widths that are not multiples of
the 8-element vector (scalar staging and packing paths), ragged batches (B not a
multiple of the 8-row unit), 90 % and 99 % sparsity (spread offsets: full-row dW
windows), and both bf16 (products + dW) and fp32 (dW) activations.  Batches of
1-16 (bf16) / 1-8 (fp32) take the packed-direct kernels (k_product_pk, k_dw_pk).
Bars: bf16 outputs 5e-3 of max(1, max|ref|) against the oracle on the same
bf16-rounded inputs; dW (exact bf16 products, fp32 accumulation) 1e-4; fp32 1e-5.
"""

import numpy as np
import pytest
import torch

import oracle
from oracle import layer as olayer
from diagtest_util import scaled_err

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_11449_b200 import ops

BF16_TOL = 5e-3
DW_BF16_TOL = 1e-4
F32_TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _case(M, N, B, sparsity, seed):
    rng = np.random.default_rng(seed)
    C, L = max(M, N), min(M, N)
    k = max(1, int(round((1 - sparsity) * C)))
    offs = np.sort(rng.choice(C, k, replace=False))
    values = rng.standard_normal((C, L))
    asoft = np.zeros(C)
    asoft[offs] = rng.uniform(0.2, 1.0, k)
    bias = rng.standard_normal(M)
    x = rng.standard_normal((B, N))
    dy = rng.standard_normal((B, M))
    return C, L, offs, values, asoft, bias, x, dy


def _gpu(a, dtype):
    return torch.as_tensor(np.asarray(a), dtype=dtype, device="cuda")


def _gw_ref(M, N, offs, x, dy):
    r_idx, c_idx = oracle.entry_coords(M, N, offs)
    return np.stack([(dy[:, r_idx[j]] * x[:, c_idx[j]]).sum(axis=0) for j in range(len(offs))])


SHAPES = [(512, 512), (1024, 256), (256, 1024), (320, 256), (256, 320), (600, 296), (296, 600), (600, 300), (300, 600)]


@pytest.mark.parametrize("M,N", SHAPES)
@pytest.mark.parametrize("B,sparsity", [(64, 0.9), (37, 0.9), (100, 0.99), (1, 0.9), (5, 0.9), (16, 0.99)])
def test_v6_bf16_products_and_dw_vs_oracle(M, N, B, sparsity):
    C, L, offs, values, asoft, bias, x, dy = _case(M, N, B, sparsity, seed=M * 7 + N + B)
    xb = _gpu(x, torch.float32).to(torch.bfloat16)
    dyb = _gpu(dy, torch.float32).to(torch.bfloat16)
    x_r = xb.double().cpu().numpy()
    dy_r = dyb.double().cpu().numpy()
    vals = _gpu(values, torch.float32)
    v32 = vals.double().cpu().numpy()
    sel = ops.selection_from_offsets(C, _gpu(offs, torch.int64), _gpu(asoft, torch.float64))
    # the bf16 products multiply bf16 weights (one rounding of alpha_soft * values, like the
    # kernel's pre-scale): the oracle gets the same rounded weights, so the bar covers the
    # bf16 output rounding and the fp32 accumulation order only
    w_ref = torch.as_tensor(asoft[offs, None] * v32[offs]).to(torch.bfloat16).double().numpy()
    w_exact = asoft[offs, None] * v32[offs]
    y = ops.diag_forward(xb, vals, sel, M, N, _gpu(bias, torch.float32), max_act=len(offs))
    y_ref = olayer.diag_matmul_forward(x_r, w_ref, offs, M, N) + bias
    assert scaled_err(y.double().cpu().numpy(), y_ref) <= BF16_TOL
    dx = ops.diag_backward_input(dyb, vals, sel, M, N, max_act=len(offs))
    gx_ref, _ = olayer.diag_matmul_backward(dy_r, x_r, v32, w_ref, offs, M, N)
    assert np.abs(w_ref - w_exact).max() <= 2.0 ** -8 * np.abs(w_exact).max()
    assert scaled_err(dx.double().cpu().numpy(), gx_ref) <= BF16_TOL
    # weight gradient: exact bf16 products accumulated in fp32
    gv, gs, gb = ops.diag_backward_weight(dyb, xb, vals, sel, M, N, max_act=len(offs))
    gw = _gw_ref(M, N, offs, x_r, dy_r)
    gv_ref = np.zeros((C, L))
    gv_ref[offs] = asoft[offs, None] * gw
    gs_ref = np.zeros(C)
    gs_ref[offs] = (gw * v32[offs]).sum(axis=1)
    assert scaled_err(gv.double().cpu().numpy(), gv_ref) <= DW_BF16_TOL
    assert scaled_err(gs.cpu().numpy(), gs_ref) <= DW_BF16_TOL
    assert scaled_err(gb.double().cpu().numpy(), dy_r.sum(axis=0)) <= DW_BF16_TOL
    inactive = np.setdiff1d(np.arange(C), offs)
    assert not gv[torch.as_tensor(inactive, device="cuda")].any(), "inactive rows must be exact zeros"


@pytest.mark.parametrize("M,N", [(3072, 768), (768, 3072), (512, 512), (600, 300)])
@pytest.mark.parametrize("B,sparsity", [(256, 0.9), (45, 0.99), (3, 0.9), (8, 0.99)])
def test_v6_fp32_dw_vs_oracle(M, N, B, sparsity):
    C, L, offs, values, asoft, bias, x, dy = _case(M, N, B, sparsity, seed=M + 3 * N + B)
    x32, dy32, vals = _gpu(x, torch.float32), _gpu(dy, torch.float32), _gpu(values, torch.float32)
    x_r, dy_r, v32 = x32.double().cpu().numpy(), dy32.double().cpu().numpy(), vals.double().cpu().numpy()
    sel = ops.selection_from_offsets(C, _gpu(offs, torch.int64), _gpu(asoft, torch.float64))
    gv, gs, gb = ops.diag_backward_weight(dy32, x32, vals, sel, M, N, max_act=len(offs))
    gw = _gw_ref(M, N, offs, x_r, dy_r)
    gv_ref = np.zeros((C, L))
    gv_ref[offs] = asoft[offs, None] * gw
    gs_ref = np.zeros(C)
    gs_ref[offs] = (gw * v32[offs]).sum(axis=1)
    assert scaled_err(gv.double().cpu().numpy(), gv_ref) <= F32_TOL
    assert scaled_err(gs.cpu().numpy(), gs_ref) <= F32_TOL
    assert scaled_err(gb.double().cpu().numpy(), dy_r.sum(axis=0)) <= F32_TOL


def test_v6_deterministic():
    """Two calls of the v6 path on the same inputs are bitwise identical (fixed
    reduction orders: no atomics, deterministic folds)."""
    M, N, B = 1024, 256, 96
    C, L, offs, values, asoft, bias, x, dy = _case(M, N, B, 0.9, seed=5)
    xb = _gpu(x, torch.float32).to(torch.bfloat16)
    dyb = _gpu(dy, torch.float32).to(torch.bfloat16)
    vals = _gpu(values, torch.float32)
    sel = ops.selection_from_offsets(C, _gpu(offs, torch.int64), _gpu(asoft, torch.float64))
    outs = []
    for _ in range(2):
        y = ops.diag_forward(xb, vals, sel, M, N, max_act=len(offs))
        dx = ops.diag_backward_input(dyb, vals, sel, M, N, max_act=len(offs))
        gv, gs, _ = ops.diag_backward_weight(dyb, xb, vals, sel, M, N, max_act=len(offs))
        outs.append((y.clone(), dx.clone(), gv.clone(), gs.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_fp32_fma_route_step_graph_capturable():
    """A float32 DiagLinear model on the FMA kernels captured as one CUDA graph
    (forward + backward: no host read of the active count inside the capture, grids
    bounded by C) gives the eager step's gradients."""
    from paper_2506_11449_b200 import DiagLinear, TemperatureSchedule
    from paper_2506_11449_b200.graphed import GraphedStep

    torch.manual_seed(0)
    sched = TemperatureSchedule("constant", 0.05, 0.05, 1)
    layers = [DiagLinear(256, 512, 0.9, seed=1, dtype=torch.float32, t_schedule=sched),
              DiagLinear(512, 256, 0.9, seed=2, dtype=torch.float32, t_schedule=sched)]
    x = torch.randn(48, 256, device="cuda")
    up = torch.randn(48, 256, device="cuda")
    params = [p for m in layers for p in m.parameters()]

    def fwd_bwd(inp, u):
        h = layers[1](layers[0](inp, step=0), step=0)
        loss = (h * u).sum()
        loss.backward()
        return loss

    fwd_bwd(x, up)
    eager = [p.grad.detach().clone() for p in params]
    for p in params:
        p.grad = None
    gs = GraphedStep(fwd_bwd, params, x.clone(), up.clone())
    gs.step(x, up)
    torch.cuda.synchronize()
    for p, g in zip(params, eager):
        assert torch.allclose(p.grad, g, rtol=1e-5, atol=1e-6 * float(g.abs().max())), p.shape


@pytest.mark.parametrize("B", [1, 5, 16, 64])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_empty_active_set_every_plan(B, dtype):
    """No active diagonal (the reference's empty pattern is rejected, but a soft TopK can
    leave n_act = 0 on the device): every product plan returns the bias, dX is zero, and
    dW writes exact zero rows with the bias gradient intact."""
    M, N = 512, 256
    C, L = max(M, N), min(M, N)
    sel = ops.selection_from_offsets(C, torch.tensor([3], device="cuda"))
    sel.n_act.zero_()  # the device count the kernels read
    sel.n_act_host = None
    vals = torch.randn(C, L, device="cuda")
    bias = torch.randn(M, device="cuda")
    x = torch.randn(B, N, device="cuda").to(dtype)
    dy = torch.randn(B, M, device="cuda").to(dtype)
    y = ops.diag_forward(x, vals, sel, M, N, bias, max_act=1)
    assert torch.equal(y.float(), bias.expand(B, M).to(dtype).float())
    dx = ops.diag_backward_input(dy, vals, sel, M, N, max_act=1)
    assert not dx.any()
    gv, gs, gb = ops.diag_backward_weight(dy, x, vals, sel, M, N, max_act=1)
    assert not gv.any() and not gs.any()
    assert torch.allclose(gb, dy.float().sum(0), rtol=1e-4, atol=1e-3)

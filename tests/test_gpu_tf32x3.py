"""The fp32 tensor-core route (3xTF32 on tcgen05: hi*hi + hi*lo + lo*hi, fp32
accumulation in TMEM; tf32_kernels.cu) against the fp64 oracle at the fp32 bar
(1e-5 of max(1, max|ref|)), through the C ABI (needs a B200).

Covers both product orientations (gather / scatter rows: wide and tall layers,
forward and dX), widths that are not multiples of 4 (padded operand rows, TMA
zero fill along K), ragged batches (tiles cut in M and split-K ranges cut in
K), 90 % and 99 % sparsity, the dW gather onto the active diagonals with the
shared finalize (exact zero rows, g_soft, bias gradient), and bitwise
run-to-run determinism.  BASELINE config 1 (768 -> 3072, B = 256) is a case."""

import numpy as np
import pytest
import torch

import oracle
from oracle import layer as olayer
from diagtest_util import scaled_err

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_11449_b200 import ops

F32_TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(autouse=True)
def _force_tf32x3(monkeypatch):
    """Every fp32 call with B >= 1 takes the 3xTF32 route (the library reads the
    switch per call; unset, it picks the route by its measured rule)."""
    monkeypatch.setenv("DIAGMM_TF32X3_MIN_B", "1")


def _gpu(a, dtype=torch.float32):
    return torch.as_tensor(np.asarray(a), dtype=dtype, device="cuda")


@pytest.mark.parametrize("M,N", [(3072, 768), (768, 3072), (512, 512), (600, 300), (301, 603), (1000, 1000)])
@pytest.mark.parametrize("B,sparsity", [(256, 0.9), (130, 0.9), (517, 0.99), (9, 0.9)])
def test_tf32x3_products_and_dw_vs_oracle(M, N, B, sparsity):
    rng = np.random.default_rng(M * 31 + N + B)
    C, L = max(M, N), min(M, N)
    k = max(1, int(round((1 - sparsity) * C)))
    offs = np.sort(rng.choice(C, k, replace=False))
    values = rng.standard_normal((C, L))
    asoft = np.zeros(C)
    asoft[offs] = rng.uniform(0.2, 1.0, k)
    bias = rng.standard_normal(M)
    x32, dy32, vals = _gpu(rng.standard_normal((B, N))), _gpu(rng.standard_normal((B, M))), _gpu(values)
    x_r, dy_r, v32 = x32.double().cpu().numpy(), dy32.double().cpu().numpy(), vals.double().cpu().numpy()
    sel = ops.selection_from_offsets(C, _gpu(offs, torch.int64), _gpu(asoft, torch.float64))
    w = asoft[offs, None] * v32[offs]
    y = ops.diag_forward(x32, vals, sel, M, N, _gpu(bias), max_act=k)
    assert scaled_err(y.double().cpu().numpy(), olayer.diag_matmul_forward(x_r, w, offs, M, N) + bias) <= F32_TOL
    dx = ops.diag_backward_input(dy32, vals, sel, M, N, max_act=k)
    gx_ref, _ = olayer.diag_matmul_backward(dy_r, x_r, v32, w, offs, M, N)
    assert scaled_err(dx.double().cpu().numpy(), gx_ref) <= F32_TOL
    gv, gs, gb = ops.diag_backward_weight(dy32, x32, vals, sel, M, N, max_act=k)
    r_idx, c_idx = oracle.entry_coords(M, N, offs)
    gw = np.stack([(dy_r[:, r_idx[j]] * x_r[:, c_idx[j]]).sum(axis=0) for j in range(k)])
    gv_ref = np.zeros((C, L))
    gv_ref[offs] = asoft[offs, None] * gw
    gs_ref = np.zeros(C)
    gs_ref[offs] = (gw * v32[offs]).sum(axis=1)
    assert scaled_err(gv.double().cpu().numpy(), gv_ref) <= F32_TOL
    assert scaled_err(gs.cpu().numpy(), gs_ref) <= F32_TOL
    assert scaled_err(gb.double().cpu().numpy(), dy_r.sum(axis=0)) <= F32_TOL
    inactive = np.setdiff1d(np.arange(C), offs)
    assert not gv[torch.as_tensor(inactive, device="cuda")].any(), "inactive rows must be exact zeros"


def test_tf32x3_deterministic_and_beats_1xtf32():
    """Bitwise repeatable; and the error is far below a single-pass tf32 product's
    (the hi/lo split is doing its job: 1xTF32 would sit near 2^-11 relative)."""
    M, N, B = 3072, 768, 256
    rng = np.random.default_rng(3)
    C, L = M, N
    offs = np.sort(rng.choice(C, 307, replace=False))
    vals = _gpu(rng.standard_normal((C, L)))
    sel = ops.selection_from_offsets(C, _gpu(offs, torch.int64))
    x = _gpu(rng.standard_normal((B, N)))
    outs = [ops.diag_forward(x, vals, sel, M, N, max_act=len(offs)).clone() for _ in range(2)]
    assert torch.equal(outs[0], outs[1])
    ref = olayer.diag_matmul_forward(x.double().cpu().numpy(), vals.double().cpu().numpy()[offs], offs, M, N)
    err = scaled_err(outs[0].double().cpu().numpy(), ref)
    assert err < 2e-6, err


def test_tf32x3_graph_capture_and_default_rule(monkeypatch):
    """The route captures into a CUDA graph (tensor maps are kernel parameters, the
    workspace is fixed) and replays to the eager result; with the switch unset a
    B = 1024 call takes the route on its own (same bits as forced)."""
    M, N, B = 768, 3072, 1024
    rng = np.random.default_rng(11)
    C, L = N, M
    offs = np.sort(rng.choice(C, 307, replace=False))
    vals = _gpu(rng.standard_normal((C, L)))
    sel = ops.selection_from_offsets(C, _gpu(offs, torch.int64))
    x = _gpu(rng.standard_normal((B, N)))
    eager = ops.diag_forward(x, vals, sel, M, N, max_act=len(offs)).clone()
    out = torch.empty_like(eager)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        out.copy_(ops.diag_forward(x, vals, sel, M, N, max_act=len(offs)))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    monkeypatch.delenv("DIAGMM_TF32X3_MIN_B")
    assert torch.equal(ops.diag_forward(x, vals, sel, M, N, max_act=len(offs)), eager)


def test_diaglinear_fp32_training_step_on_tf32_route(monkeypatch):
    """A float32 DiagLinear step at B = 512 (the route's default range) through the public
    module: y, dx, d values, d alpha, d bias equal the FMA-route step's to the fp32 bar
    (both against the same fp64-accurate arithmetic), and the step replays from a graph."""
    from paper_2506_11449_b200 import DiagLinear, TemperatureSchedule
    from paper_2506_11449_b200.graphed import GraphedStep

    sched = TemperatureSchedule("constant", 0.05, 0.05, 1)
    x = torch.randn(512, 768, device="cuda")
    up = torch.randn(512, 3072, device="cuda")

    def step(route_min_b):
        monkeypatch.setenv("DIAGMM_TF32X3_MIN_B", route_min_b)
        torch.manual_seed(0)
        lyr = DiagLinear(768, 3072, 0.9, seed=3, dtype=torch.float32, t_schedule=sched, l1_coeff=1e-4)
        xi = x.clone().requires_grad_(True)
        y = lyr(xi, step=0)
        (y * up).sum().backward()
        torch.cuda.synchronize()
        return lyr, [y.detach(), xi.grad, lyr.values.grad, lyr.alpha.grad, lyr.bias.grad]

    _, fma = step("0")
    lyr, tf = step("1")
    for a, b in zip(tf, fma):
        scale = max(1.0, float(b.abs().max()))
        assert float((a.double() - b.double()).abs().max()) <= F32_TOL * scale
    params = list(lyr.parameters())
    for p in params:
        p.grad = None

    def fwd_bwd(inp, u):
        loss = (lyr(inp, step=0) * u).sum()
        loss.backward()
        return loss

    gs = GraphedStep(fwd_bwd, params, x.clone(), up.clone())
    gs.step(x, up)
    torch.cuda.synchronize()
    for p, ref in zip([lyr.values, lyr.alpha, lyr.bias], tf[2:]):
        scale = max(1.0, float(ref.abs().max()))
        assert float((p.grad.double() - ref.double()).abs().max()) <= F32_TOL * scale


@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize("trans_b", [False, True])
@pytest.mark.parametrize("M,N,K", [(64, 3072, 768), (301, 257, 603), (1000, 70, 5)])
def test_dense_tf32x3_gemm_vs_fp64(trans_a, trans_b, M, N, K):
    """diagmm_tf32x3_gemm (the float32 layers' dense route) against an fp64 product at the
    fp32 bar, every operand orientation, sizes that are not multiples of 4 or of a tile."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn((K, M) if trans_a else (M, K), device="cuda", generator=g)
    b = torch.randn((K, N) if trans_b else (N, K), device="cuda", generator=g)
    bias = torch.randn(N, device="cuda", generator=g)
    out = ops.tf32x3_gemm(a, b, trans_a=trans_a, trans_b=trans_b, bias=bias)
    A = (a.t() if trans_a else a).double()
    Bm = (b.t() if trans_b else b).double()
    ref = (A @ Bm.t() + bias.double()).cpu().numpy()
    assert scaled_err(out.double().cpu().numpy(), ref) <= F32_TOL

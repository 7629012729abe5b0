"""DiagLinear: the reference's DynaDiag layer as a PyTorch module on sm_100a kernels.

``DiagLinear`` mirrors ``DynaDiagLayer`` (reference ``layers.py:173-287``):
same constructor arguments, same parameter layout (a dense-equivalent
candidate store ``values (C, L)``, selection logits ``alpha (C,)`` float64,
``bias (M,)``), same host-side initialisation stream
(``np.random.default_rng(seed)``: values U(±sqrt(1/N)), then alpha N(0, 0.01),
layers.py:199-208) so a layer built with the same seed starts bit-identical,
and the same DST API (``set_k``, ``soft_scores``, ``active_set``,
``active_count``, ``effective_matrix``, ``penalty``, ``freeze``).

``DiagMMFunction`` is the ``torch.autograd.Function`` that replaces the
reference's custom tape op ``_record_diag_matmul`` (layers.py:108-170): the
forward runs K4 (soft TopK, device) then K1; the backward runs K2 (dX through
the transpose), K3 (per-diagonal dW, g_values, g_soft, g_bias) and K5
(soft-TopK gradient).  Gradients follow the reference exactly: inactive rows of
``values.grad`` are 0, ``alpha.grad`` flows only through unclamped candidates.
"""

from __future__ import annotations

import contextlib

from dataclasses import dataclass
from math import ceil, sqrt

import numpy as np
import torch
import torch.nn.functional as F
from torch import nn

from . import ops
from .errors import ShapeMismatch
from .selection import (
    EPS_ACTIVE,
    TemperatureSchedule,
    candidate_count,
    required_diagonals,
    temperature_at,
)

ROUTES = ("diag", "dense", "auto")


@dataclass
class ParamSpec:
    """One trainable tensor plus its optimizer treatment (layers.py:44-50)."""

    tensor: torch.Tensor
    decay: bool
    name: str


@dataclass
class DiagMatrix:
    """Device counterpart of ``DiagSparseMatrix`` (diagcore.py:124-150).

    offsets (K,) int64 ascending, values (K, min(M, N)).
    """

    rows: int
    cols: int
    offsets: torch.Tensor
    values: torch.Tensor

    def __post_init__(self):
        """DiagonalPattern's checks (diagcore.py:71-88): offsets in [0, max(M, N)),
        no duplicates; stored ascending (values permuted with them)."""
        offs = ops.validate_offsets(max(self.rows, self.cols), self.offsets)
        if not torch.equal(offs, self.offsets.to(offs.dtype)):
            order = torch.argsort(self.offsets)
            self.values = self.values[order]
        self.offsets = offs.to(self.offsets.dtype)

    def store(self) -> torch.Tensor:
        """Candidate-store layout (C, L) with zeros on unused offsets."""
        C, L = ops.geometry(self.rows, self.cols)
        st = torch.zeros(C, L, dtype=self.values.dtype, device=self.values.device)
        st[self.offsets] = self.values
        return st

    def selection(self) -> ops.Selection:
        C, _ = ops.geometry(self.rows, self.cols)
        return ops.selection_from_offsets(C, self.offsets)

    def dense(self, dtype: torch.dtype | None = None) -> torch.Tensor:
        """materialize (diagcore.py:153-159) on device."""
        return ops.materialize(self.store(), self.selection(), self.rows, self.cols, dtype)


@dataclass
class _OpSpec:
    M: int
    N: int
    k: int
    temperature: float
    route: str
    fixed: ops.Selection | None = None
    presel: ops.Selection | None = None
    l1: float = 0.0  # set by penalties(fused=True): the l1 gradient is added inside K5
    bucket: torch.Tensor | None = None  # dp.CompactGradExchange: K3 also writes the active rows here
    params: torch.Tensor | None = None  # schedule.DeviceSchedule: device {T, k} read by K4 / K5
    sel: ops.Selection | None = None    # the selection the forward used (set by the forward)
    alpha_param: torch.Tensor | None = None  # the layer's alpha Parameter (deferred K5 writes its .grad)
    prew: torch.Tensor | None = None    # W_K materialized by preselect's batched pre-pass (same selection)
    values_param: torch.Tensor | None = None  # the layer's values / bias Parameters (deferred finalize)
    bias_param: torch.Tensor | None = None


def _use_dense(spec: _OpSpec, sel: ops.Selection, B: int, act_dtype: torch.dtype) -> bool:
    if spec.route == "dense":
        return True
    if spec.route == "diag":
        return False
    # "auto": the B200 cost model first — with bf16
    # activations and enough tokens the tensor cores run the dense-equivalent
    # product faster than the FMA pipe runs the diagonal one, and this branch
    # needs no host read of n_act; below that the reference's own switch
    # (diagcore.py:226, layers.py:150): dense once the structural density of
    # the active set reaches 1/4 (one host read of the device count).
    if act_dtype == torch.bfloat16 and B >= dense_route_min_tokens():
        return True
    L = min(spec.M, spec.N)
    if torch.cuda.is_current_stream_capturing():
        # inside a CUDA-graph capture the device count cannot be read (and a host value
        # would be baked into the graph): the switch uses the TopK budget k instead; both
        # routes give the reference's results, and the kernels bound their grids by C
        return 4 * spec.k * L >= spec.M * spec.N
    return 4 * sel.host_count() * L >= spec.M * spec.N


def _tc_ok(x: torch.Tensor, M: int, N: int) -> bool:
    """The tcgen05 route takes bf16 activations with 16-byte rows (M, N % 8 == 0).
    DIAGMM_DENSE_BACKEND=cublas selects the library GEMM instead (A/B comparisons)."""
    import os

    return (x.dtype == torch.bfloat16 and M % 8 == 0 and N % 8 == 0
            and os.environ.get("DIAGMM_DENSE_BACKEND", "tc") != "cublas")


def _tf32_dense(t: torch.Tensor) -> bool:
    """float32 dense-route GEMMs on the 3xTF32 kernel (DIAGMM_DENSE_BACKEND=cublas: the library)."""
    import os

    return t.dtype == torch.float32 and t.is_cuda and os.environ.get("DIAGMM_DENSE_BACKEND", "tc") != "cublas"


def dense_route_min_tokens() -> int:
    """Token count from which the bf16 tensor-core route beats the FMA route
    (measured on B200, profiles/r01_*; override with DIAGMM_DENSE_MIN_TOKENS)."""
    import os

    return int(os.environ.get("DIAGMM_DENSE_MIN_TOKENS", "512"))


def _accumulate(param: torch.Tensor, g: torch.Tensor) -> None:
    """What autograd's AccumulateGrad does for a dense gradient."""
    if param.grad is None:
        param.grad = g
    else:
        param.grad.add_(g)


class _K5Queue:
    """Work queued by the backwards inside ``deferred_topk_grads()``: tensor-core dW
    finalizes (``fin``) and K5 jobs (``jobs``)."""

    def __init__(self):
        self.jobs = []
        self.fin = []

    def flush(self) -> None:
        """ONE batched finalize launch for every deferred tensor-core dW (g_values, g_soft,
        g_bias), then ONE batched K5 launch for every queued layer (layers whose alpha
        appears more than once go in later launches, so each accumulation sees the
        previous one)."""
        if self.fin:
            fin, self.fin = self.fin, []
            outs = ops.dw_finalize_many([f[0] for f in fin])
            for (_, vp, bp, k5), (gv, gs, gb) in zip(fin, outs):
                if vp.requires_grad:
                    _accumulate(vp, gv)
                if bp is not None and gb is not None and bp.requires_grad:
                    _accumulate(bp, gb)
                if k5 is not None:
                    alpha_param, k, T, clamped, l1, params = k5
                    self.jobs.append((alpha_param, k, T, gs, clamped, l1, params))
        pending = self.jobs
        self.jobs = []
        while pending:
            batch, rest, seen = [], [], set()
            for job in pending:
                (rest if id(job[0]) in seen else batch).append(job)
                seen.add(id(job[0]))
            calls = []
            for alpha, k, T, g_soft, clamped, l1, params in batch:
                acc = alpha.grad is not None
                calls.append((alpha.detach(), k, T, g_soft, clamped, l1, alpha.grad if acc else None, acc, params))
            outs = ops.soft_topk_grad_many(calls)
            for (alpha, *_), g in zip(batch, outs):
                if alpha.grad is None:
                    alpha.grad = g
            pending = rest


_K5_QUEUE: "_K5Queue | None" = None  # module-wide: autograd runs CUDA backwards on its own device thread


@contextlib.contextmanager
def deferred_topk_grads():
    """Inside this context the DiagLinear backwards queue their soft-TopK gradients (K5)
    instead of launching one kernel per layer, and return no alpha gradient to autograd;
    on exit ONE batched launch writes every layer's g_alpha into ``alpha.grad``
    (accumulating, as autograd would).  Results are bit-identical to the per-layer path.
    Single-process use (the data-parallel exchange hooks alpha's autograd accumulation)."""
    global _K5_QUEUE
    prev, q = _K5_QUEUE, _K5Queue()
    _K5_QUEUE = q
    try:
        yield q
    finally:
        _K5_QUEUE = prev
    q.flush()


def _k5(spec: "_OpSpec", alpha: torch.Tensor, g_soft: torch.Tensor, sel: ops.Selection):
    """g_alpha of one layer now, or queued for the batched launch (returns None then)."""
    q = _K5_QUEUE
    if q is not None and spec.alpha_param is not None:
        q.jobs.append((spec.alpha_param, spec.k, spec.temperature, g_soft, sel.clamped, spec.l1, spec.params))
        return None
    return ops.soft_topk_grad(alpha.detach(), spec.k, spec.temperature, g_soft, clamped=sel.clamped,
                              l1_coeff=spec.l1, params=spec.params)


def _tc_weight_grads(spec: "_OpSpec", dy_parts, x: torch.Tensor, vals: torch.Tensor, sel: ops.Selection,
                     has_bias: bool, need_soft: bool, alpha):
    """(g_values, g_bias, g_alpha) of a tensor-core layer (fused-gather dW + bias gradient +
    K5) — or (None, None, None) inside ``deferred_topk_grads()``, where only the dW GEMM runs
    now and the finalize / K5 join the batched launches after the backward."""
    M, N = spec.M, spec.N
    q = _K5_QUEUE
    if q is not None and spec.bucket is None and spec.values_param is not None and spec.alpha_param is not None:
        rec = ops.tc_backward_weight_begin(dy_parts, x, vals, sel, M, N, need_bias=has_bias, need_soft=need_soft)
        k5 = (spec.alpha_param, spec.k, spec.temperature, sel.clamped, spec.l1, spec.params) if need_soft else None
        q.fin.append((rec, spec.values_param, spec.bias_param if has_bias else None, k5))
        return None, None, None
    if isinstance(dy_parts, (list, tuple)):
        gv, gs, gb = ops.tc_backward_weight_split(list(dy_parts), x, vals, sel, M, N, need_soft=need_soft,
                                                  need_bias=True, bucket=spec.bucket)
    else:
        gv, gs, gb = ops.tc_backward_weight(dy_parts, x, vals, sel, M, N, need_soft=need_soft, need_bias=True,
                                            bucket=spec.bucket)
    ga = _k5(spec, alpha, gs, sel) if need_soft else None
    return gv, (gb if has_bias else None), ga


def _w_k(spec: "_OpSpec", dtype: torch.dtype, values, sel, M: int, N: int) -> torch.Tensor:
    """W_K for this forward: the pre-pass's (preselect(materialize=...)) when it was built
    for this selection and dtype, else materialized now."""
    W, spec.prew = spec.prew, None
    if W is not None and W.dtype == dtype and tuple(W.shape) == (M, N):
        return W
    return ops.materialize(values, sel, M, N, dtype=dtype)


class DiagMMFunction(torch.autograd.Function):
    """y = x @ W_K^T + bias for the soft-selected diagonals (layers.py:108-170, 230-251)."""

    @staticmethod
    def forward(ctx, x, values, alpha, bias, spec: _OpSpec, residual=None):
        M, N = spec.M, spec.N
        if alpha is not None:
            sel = spec.presel or ops.soft_topk_select(alpha.detach(), spec.k, spec.temperature,
                                                      params=spec.params)
        else:
            sel = spec.fixed
        spec.sel = sel
        dense = _use_dense(spec, sel, x.shape[0], x.dtype)
        vals = values.detach()
        W = None
        tc = dense and _tc_ok(x, M, N)
        if tc:
            # tensor-core route: our tcgen05 GEMM on the dense-equivalent W_K (bias fused);
            # W_K is kept for the input gradient (read MN-major there: no W_K^T is built)
            W = _w_k(spec, x.dtype, vals, sel, M, N)
            bz = None if bias is None else bias.detach()
            if residual is not None and residual.dtype == x.dtype:
                # the caller's residual add fused into the epilogue (one rounding)
                y, _ = ops.tc_gemm_ex(x.contiguous(), W, bz, epilogue=3, aux=residual.detach())
                residual = None
            else:
                y = ops.tc_gemm(x.contiguous(), W, bz)
        elif dense:
            W = _w_k(spec, x.dtype, vals, sel, M, N)
            if _tf32_dense(x):  # float32: our 3xTF32 tensor-core GEMM, fp32-accurate
                y = ops.tf32x3_gemm(x.contiguous(), W, bias=None if bias is None else bias.detach())
            else:  # float64: the reference's own BLAS switch on a library DGEMM
                y = F.linear(x, W, None if bias is None else bias.detach().to(x.dtype))
        else:
            y = ops.diag_forward(x, vals, sel, M, N, None if bias is None else bias.detach(),
                                 max_act=sel.known_count())
        if residual is not None:
            y = y + residual.detach()
        ctx.save_for_backward(x, values, alpha)
        ctx.sel, ctx.spec, ctx.W, ctx.has_bias, ctx.tc = sel, spec, W, bias is not None, tc
        return y

    @staticmethod
    def backward(ctx, dy):
        x, values, alpha = ctx.saved_tensors
        sel, spec, W = ctx.sel, ctx.spec, ctx.W
        ctx.W = None
        d_res = dy if len(ctx.needs_input_grad) > 5 and ctx.needs_input_grad[5] else None
        M, N = spec.M, spec.N
        dy = dy.contiguous()
        vals = values.detach()
        dx = g_alpha = None
        need_soft = alpha is not None and ctx.needs_input_grad[2]
        if W is not None or ctx.tc:
            dy = dy.to(x.dtype)
            if ctx.needs_input_grad[0]:
                if ctx.tc:  # dx = dy @ W_K on the tensor cores, W_K staged MN-major
                    dx = ops.tc_gemm_nn(dy, W)
                elif _tf32_dense(dy):  # dx = dy @ W_K = dy . (W_K^T)^T
                    dx = ops.tf32x3_gemm(dy, W, trans_b=True)
                else:
                    dx = dy @ W
            out_dt = vals.dtype
            if ctx.tc and M % 64 == 0 and N % 64 == 0:
                # tensor-core dW with the diagonal gather and the bias gradient fused (dy read once,
                # no dense dW written); K5 included
                g_values, g_bias, g_alpha = _tc_weight_grads(spec, dy, x.to(dy.dtype), vals, sel, ctx.has_bias,
                                                             need_soft, alpha)
                return dx, g_values, g_alpha, g_bias, None, d_res
            else:
                spec.bucket = None  # this branch does not fill the exchange bucket (dp falls back to full)
                if dy.dtype == torch.bfloat16:
                    dW = torch.mm(dy.t(), x.to(dy.dtype), out_dtype=out_dt)
                elif _tf32_dense(dy):  # dW = dy^T x = (dy^T) . (x^T)^T
                    dW = ops.tf32x3_gemm(dy, x.to(dy.dtype).contiguous(), trans_a=True, trans_b=True)
                else:
                    dW = (dy.t() @ x.to(dy.dtype)).to(out_dt)
                g_values, g_soft = ops.gather_dense_grad(dW, vals, sel, M, N, need_soft=need_soft)
                g_bias = dy.sum(0, dtype=out_dt) if ctx.has_bias else None
        else:
            ma = sel.known_count()
            if ctx.needs_input_grad[0]:
                dx = ops.diag_backward_input(dy, vals, sel, M, N, max_act=ma)
            g_values, g_soft, g_bias = ops.diag_backward_weight(
                dy, x, vals, sel, M, N, need_bias=ctx.has_bias, need_soft=need_soft, bucket=spec.bucket,
                max_act=ma)
        if need_soft:
            g_alpha = _k5(spec, alpha, g_soft, sel)
        return dx, g_values, g_alpha, g_bias, None, d_res


class DiagMLPFunction(torch.autograd.Function):
    """fc2(gelu_tanh(fc1(x))) for two DiagLinear layers on the tensor-core route
    with the GELU fused into the GEMM epilogues: fc1's epilogue writes the
    pre-activation and gelu(pre); fc2's input-gradient epilogue multiplies by
    gelu'(pre) — no separate GELU kernels, forward or backward.  Gradients per
    layer are exactly those of DiagMMFunction (layers.py:143-167)."""

    @staticmethod
    def forward(ctx, x, v1, a1, b1, v2, a2, b2, s1: _OpSpec, s2: _OpSpec, fuse_fwd: bool = True, residual=None):
        sel1 = s1.presel or ops.soft_topk_select(a1.detach(), s1.k, s1.temperature, params=s1.params)
        sel2 = s2.presel or ops.soft_topk_select(a2.detach(), s2.k, s2.temperature, params=s2.params)
        s1.sel, s2.sel = sel1, sel2
        x = x.contiguous()
        W1 = _w_k(s1, x.dtype, v1.detach(), sel1, s1.M, s1.N)
        if fuse_fwd:
            act, pre = ops.tc_gemm_ex(x, W1, None if b1 is None else b1.detach(), epilogue=1)
        else:
            pre = ops.tc_gemm(x, W1, None if b1 is None else b1.detach())
            act = F.gelu(pre, approximate="tanh")
        W2 = _w_k(s2, x.dtype, v2.detach(), sel2, s2.M, s2.N)
        bz2 = None if b2 is None else b2.detach()
        if residual is not None and residual.dtype == x.dtype:  # residual add fused into fc2's epilogue
            y, _ = ops.tc_gemm_ex(act, W2, bz2, epilogue=3, aux=residual.detach())
        else:
            y = ops.tc_gemm(act, W2, bz2)
            if residual is not None:
                y = y + residual.detach()
        ctx.save_for_backward(x, pre, act, v1, a1, v2, a2)
        ctx.sels, ctx.specs, ctx.has_bias = (sel1, sel2), (s1, s2), (b1 is not None, b2 is not None)
        ctx.W = (W1, W2)  # read MN-major by the input-gradient products (no W^T materialized)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, pre, act, v1, a1, v2, a2 = ctx.saved_tensors
        (sel1, sel2), (s1, s2) = ctx.sels, ctx.specs
        dy0 = dy
        dy = dy.to(x.dtype).contiguous()
        v1d, v2d = v1.detach(), v2.detach()
        # fc2: input gradient straight to d(pre) through gelu', then dW2 (+ bias) from act
        W1, W2 = ctx.W
        ctx.W = None
        d_pre = ops.tc_gemm_nn(dy, W2, None, epilogue=2, aux=pre)
        gv2, gb2, ga2 = _tc_weight_grads(s2, dy, act, v2d, sel2, True, True, a2)
        # fc1
        dx = ops.tc_gemm_nn(d_pre, W1)
        gv1, gb1, ga1 = _tc_weight_grads(s1, d_pre, x, v1d, sel1, True, True, a1)
        hb1, hb2 = ctx.has_bias
        d_res = dy0 if ctx.needs_input_grad[10] else None
        return (dx, gv1, ga1, gb1 if hb1 else None, gv2, ga2, gb2 if hb2 else None, None, None, None, d_res)


def _flatten(x: torch.Tensor, width: int) -> torch.Tensor:
    if x.dim() < 1 or x.shape[-1] != width:
        raise ShapeMismatch(f"input has shape {tuple(x.shape)}, expected (..., {width})")
    return x.reshape(-1, width)


class DiagLinear(nn.Module):
    """Linear layer on soft-selected wrap-around diagonals (layers.py:173-287).

    Computes y = x W^T + bias, W = sum over active diagonals of
    alpha_soft_j P_j diag(V_j); active = candidates with soft score >= 1e-3.
    ``forward(x, step=None)`` accepts any leading dims (tokens are flattened
    into the batch, as rank-2 is all the reference supports,
    autodiff.py:26-27).  ``step`` defaults to ``self.step``.
    """

    def __init__(self, in_features: int, out_features: int, sparsity: float = 0.9, *,
                 t_schedule: TemperatureSchedule | None = None, l1_coeff: float = 1e-4,
                 bias: bool = True, seed: int = 0, blocking=None, device=None,
                 dtype: torch.dtype = torch.float32, route: str = "diag"):
        super().__init__()
        if route not in ROUTES:
            raise ValueError(f"route must be one of {ROUTES}")
        self.in_features, self.out_features = int(in_features), int(out_features)
        M, N = self.out_features, self.in_features
        self.candidates = candidate_count(M, N)
        self.diag_len = min(M, N)
        self.k = required_diagonals(M, N, sparsity)
        self.t_schedule = t_schedule or TemperatureSchedule()
        self.l1_coeff = l1_coeff
        self.route = route
        pdt = torch.float64 if dtype == torch.float64 else torch.float32
        rng = np.random.default_rng(seed)
        bound = sqrt(1.0 / N)
        vals = rng.uniform(-bound, bound, (self.candidates, self.diag_len))
        alpha = rng.normal(0.0, 0.01, self.candidates)
        device = torch.device(device) if device is not None else torch.device("cuda")
        self.values = nn.Parameter(torch.from_numpy(vals).to(device=device, dtype=pdt))
        self.alpha = nn.Parameter(torch.from_numpy(alpha).to(device=device, dtype=torch.float64))
        self.bias = nn.Parameter(torch.zeros(M, device=device, dtype=pdt)) if bias else None
        self.step = 0
        self.last_step = 0
        self._presel = None

    # ---- DST mask-update API (layers.py:212-228, 268-287) --------------------
    def set_k(self, k: int) -> None:
        if not 1 <= k <= self.candidates:
            raise ValueError(f"k={k} outside [1, {self.candidates}]")
        self.k = int(k)

    def temperature(self, step: int) -> float:
        """layers.py:217-219: past the horizon the layer keeps training at t_final."""
        return temperature_at(min(step, self.t_schedule.total_steps), self.t_schedule)

    def selection(self, step: int) -> ops.Selection:
        return ops.soft_topk_select(self.alpha.detach(), self.k, self.temperature(step))

    def soft_scores(self, step: int) -> torch.Tensor:
        return self.selection(step).alpha_soft

    def active_set(self, step: int) -> torch.Tensor:
        return self.selection(step).active_offsets().long()

    def active_count(self, step: int) -> int:
        return self.selection(step).host_count()

    def effective_matrix(self, step: int) -> DiagMatrix:
        """layers.py:268-275: the active-set matrix exactly as forward uses it."""
        sel = self.selection(step)
        act = sel.active_offsets().long()
        vals = sel.alpha_soft[act].to(self.values.dtype)[:, None] * self.values.detach()[act]
        return DiagMatrix(self.out_features, self.in_features, act, vals)

    def penalty(self) -> torch.Tensor:
        """layers.py:253-257: l1_coeff * sum|alpha| (grad l1 * sign(alpha), sign(0)=0)."""
        return self.l1_coeff * self.alpha.abs().sum()

    def param_specs(self) -> list[ParamSpec]:
        """layers.py:259-266: values decay, alpha and bias do not."""
        specs = [ParamSpec(self.values, True, "values"), ParamSpec(self.alpha, False, "alpha")]
        if self.bias is not None:
            specs.append(ParamSpec(self.bias, False, "bias"))
        return specs

    def freeze(self) -> "FrozenDiagLinear":
        """layers.py:277-287: hard top-K at t_final, soft scores baked into V."""
        sel = ops.select_hard(self.alpha.detach(), self.k)
        a_soft = ops.soft_topk(self.alpha.detach(), self.k, self.t_schedule.t_final)
        vals = a_soft[sel].to(self.values.dtype)[:, None] * self.values.detach()[sel]
        w = DiagMatrix(self.out_features, self.in_features, sel, vals)
        return FrozenDiagLinear(w, None if self.bias is None else self.bias.detach().clone(), route=self.route)

    # ---- forward ----------------------------------------------------------------
    def forward(self, x: torch.Tensor, step: int | None = None, residual: torch.Tensor | None = None) -> torch.Tensor:
        """y = x W_K^T + bias (+ residual: the caller's skip connection, fused into the
        tensor-core epilogue when it can be)."""
        step = self.step if step is None else int(step)
        self.last_step = step
        lead = x.shape[:-1]
        x2 = _flatten(x, self.in_features)
        if x2.dtype != torch.float64 and self.values.dtype == torch.float64:
            x2 = x2.double()
        elif x2.dtype == torch.float32 and torch.is_autocast_enabled("cuda"):
            x2 = x2.to(torch.get_autocast_dtype("cuda"))  # like nn.Linear under autocast
        spec = self._make_spec(step)
        r2 = None if residual is None else _flatten(residual, self.out_features)
        y = DiagMMFunction.apply(x2, self.values, self.alpha, self.bias, spec, r2)
        return y.reshape(*lead, self.out_features)

    def _make_spec(self, step: int) -> "_OpSpec":
        T = self.temperature(step)
        spec = _OpSpec(self.out_features, self.in_features, self.k, T, self.route,
                       presel=self._take_preselection(step, T), bucket=getattr(self, "_dp_bucket", None),
                       params=getattr(self, "_sched_params", None), alpha_param=self.alpha,
                       values_param=self.values, bias_param=self.bias)
        spec.prew = self._take_premat(step, T) if spec.presel is not None else None
        self._last_spec = spec
        return spec

    def _take_preselection(self, step: int, T: float):
        ps, self._presel = self._presel, None
        if ps is not None and ps[0] == (step, self.k, T):
            return ps[1]
        return None

    def _take_premat(self, step: int, T: float):
        pm, self._premat = getattr(self, "_premat", None), None
        if pm is not None and pm[0] == (step, self.k, T):
            return pm[1]
        return None

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, k={self.k}, "
                f"candidates={self.candidates}, route={self.route}")


class DiagMLP(nn.Module):
    """fc1 -> GELU (tanh) -> fc2 with two DiagLinear layers (the ViT / GPT MLP).

    On the tensor-core route (bf16, >= dense_route_min_tokens tokens, dims multiple
    of 64) the GELU is fused into the GEMM epilogues (DiagMLPFunction): gelu in
    fc1's epilogue (which also stores the pre-activation) and gelu' in fc2's
    input-gradient epilogue, so the two elementwise GELU passes over the
    (tokens x 4d) activation disappear.  DIAGMM_FUSE_MLP selects it: "1" (default)
    both, "bwd" backward only, "0" the unfused fc2(gelu(fc1(x))).  The epilogues
    take tanh from the SFU; with a full-precision tanhf the short-K (768) GEMMs
    were epilogue-bound and the fused step was slower."""

    def __init__(self, fc1: "DiagLinear", fc2: "DiagLinear"):
        super().__init__()
        if fc1.out_features != fc2.in_features:
            raise ShapeMismatch("fc1.out_features must equal fc2.in_features")
        self.fc1, self.fc2 = fc1, fc2

    def _fusable(self, x2: torch.Tensor) -> bool:
        import os

        layers = (self.fc1, self.fc2)
        return (x2.dtype == torch.bfloat16 and x2.shape[0] >= dense_route_min_tokens()
                and all(m.route == "auto" and m.out_features % 64 == 0 and m.in_features % 64 == 0 for m in layers)
                and all(m.values.dtype == torch.float32 for m in layers)
                and os.environ.get("DIAGMM_DENSE_BACKEND", "tc") != "cublas"
                and os.environ.get("DIAGMM_FUSE_MLP", "1") != "0")

    def forward(self, x: torch.Tensor, step: int | None = None, residual: torch.Tensor | None = None) -> torch.Tensor:
        f1, f2 = self.fc1, self.fc2
        lead = x.shape[:-1]
        x2 = _flatten(x, f1.in_features)
        if x2.dtype == torch.float32 and torch.is_autocast_enabled("cuda"):
            x2 = x2.to(torch.get_autocast_dtype("cuda"))
        r2 = None if residual is None else _flatten(residual, f2.out_features)
        if isinstance(f1, FrozenDiagLinear) and isinstance(f2, FrozenDiagLinear):  # inference (freeze())
            return f2(f1.forward_gelu(x2), residual=r2).reshape(*lead, f2.out_features)
        if not self._fusable(x2):
            h = F.gelu(f1(x2, step), approximate="tanh")
            return f2(h, step, residual=r2).reshape(*lead, f2.out_features)
        step1 = f1.step if step is None else int(step)
        step2 = f2.step if step is None else int(step)
        f1.last_step, f2.last_step = step1, step2
        import os

        fuse_fwd = os.environ.get("DIAGMM_FUSE_MLP", "1") in ("1", "both", "fwd")
        y = DiagMLPFunction.apply(x2, f1.values, f1.alpha, f1.bias, f2.values, f2.alpha, f2.bias,
                                  f1._make_spec(step1), f2._make_spec(step2), fuse_fwd, r2)
        return y.reshape(*lead, f2.out_features)


class FrozenDiagLinear(nn.Module):
    """Inference layer over a fixed diagonal matrix (layers.py:290-310).

    ``route`` as for DiagLinear: "auto" multiplies bf16 batches of >= 512 tokens
    with the dense-equivalent matrix on the tensor cores (materialized once per
    dtype and cached: the weights are frozen) and smaller batches with the
    diagonal kernel (K1)."""

    def __init__(self, weight: DiagMatrix, bias: torch.Tensor | None = None, route: str = "auto"):
        super().__init__()
        if route not in ROUTES:
            raise ValueError(f"route must be one of {ROUTES}")
        self.weight = weight
        self.route = route
        self.in_features, self.out_features = weight.cols, weight.rows
        self.register_buffer("store", weight.store())
        self.register_buffer("bias", bias)
        self._sel = weight.selection()
        self._dense = {}

    def _dense_weight(self, dtype: torch.dtype) -> torch.Tensor:
        W = self._dense.get(dtype)
        if W is None:
            W = ops.materialize(self.store, self._sel, self.out_features, self.in_features, dtype)
            self._dense[dtype] = W
        return W

    def _prep(self, x: torch.Tensor) -> torch.Tensor:
        x2 = _flatten(x, self.in_features)
        if self.store.dtype == torch.float64:
            x2 = x2.double()
        elif x2.dtype == torch.float32 and torch.is_autocast_enabled("cuda"):
            x2 = x2.to(torch.get_autocast_dtype("cuda"))
        return x2

    def _tc(self, x2: torch.Tensor) -> bool:
        dense = self.route == "dense" or (self.route == "auto" and x2.dtype == torch.bfloat16
                                          and x2.shape[0] >= dense_route_min_tokens())
        return dense and _tc_ok(x2, self.out_features, self.in_features)

    def forward(self, x: torch.Tensor, step: int | None = None, residual: torch.Tensor | None = None) -> torch.Tensor:
        """y = x W^T + bias (+ residual, fused into the tensor-core epilogue); ``step``
        is accepted for call compatibility with DiagLinear and ignored (frozen)."""
        lead = x.shape[:-1]
        x2 = self._prep(x)
        r2 = None if residual is None else _flatten(residual, self.out_features)
        dense = self.route == "dense" or (self.route == "auto" and x2.dtype == torch.bfloat16
                                          and x2.shape[0] >= dense_route_min_tokens())
        if self._tc(x2):
            if r2 is not None and r2.dtype == x2.dtype:
                y, _ = ops.tc_gemm_ex(x2.contiguous(), self._dense_weight(x2.dtype), self.bias, epilogue=3, aux=r2)
                r2 = None
            else:
                y = ops.tc_gemm(x2.contiguous(), self._dense_weight(x2.dtype), self.bias)
        elif dense:
            y = F.linear(x2, self._dense_weight(x2.dtype), None if self.bias is None else self.bias.to(x2.dtype))
        else:
            y = ops.diag_forward(x2, self.store, self._sel, self.out_features, self.in_features, self.bias)
        if r2 is not None:
            y = y + r2
        return y.reshape(*lead, self.out_features)

    def forward_gelu(self, x: torch.Tensor) -> torch.Tensor:
        """gelu_tanh(x W^T + bias), fused into the tensor-core epilogue when it can be
        (the frozen MLP's fc1)."""
        lead = x.shape[:-1]
        x2 = self._prep(x)
        if self._tc(x2):
            act, _ = ops.tc_gemm_ex(x2.contiguous(), self._dense_weight(x2.dtype), self.bias, epilogue=1)
            return act.reshape(*lead, self.out_features)
        return F.gelu(self.forward(x), approximate="tanh")


class DiagHeurLinear(nn.Module):
    """Magnitude-prune / random-regrow baseline over whole diagonals (layers.py:313-378).

    The active set lives on the device (a Selection: active / slot / n_act) and
    ``diagheur_update`` swaps it in place with one kernel; ``active`` reads it
    back as a sorted numpy array (the reference's attribute)."""

    def __init__(self, in_features: int, out_features: int, sparsity: float = 0.9, *,
                 update_every: int = 100, prune_fraction: float = 0.3, bias: bool = True,
                 seed: int = 0, blocking=None, device=None, dtype: torch.dtype = torch.float32):
        super().__init__()
        if not 0.0 < prune_fraction < 1.0:
            raise ValueError("prune_fraction must lie in (0, 1)")
        self.in_features, self.out_features = int(in_features), int(out_features)
        M, N = self.out_features, self.in_features
        self.candidates = candidate_count(M, N)
        self.diag_len = min(M, N)
        self.k = required_diagonals(M, N, sparsity)
        self.update_every, self.prune_fraction = update_every, prune_fraction
        pdt = torch.float64 if dtype == torch.float64 else torch.float32
        rng = np.random.default_rng(seed)
        bound = sqrt(1.0 / N)
        vals = rng.uniform(-bound, bound, (self.candidates, self.diag_len))
        device = torch.device(device) if device is not None else torch.device("cuda")
        self.values = nn.Parameter(torch.from_numpy(vals).to(device=device, dtype=pdt))
        self.bias = nn.Parameter(torch.zeros(M, device=device, dtype=pdt)) if bias else None
        self._sel = ops.selection_from_offsets(
            self.candidates, torch.as_tensor(np.sort(rng.choice(self.candidates, self.k, replace=False)),
                                             device=device))

    @property
    def active(self) -> np.ndarray:
        """Sorted active offsets (host copy of the device set)."""
        return self._sel.active[: self.k].cpu().numpy().astype(np.int64)

    @active.setter
    def active(self, offsets) -> None:
        offs = np.sort(np.asarray(offsets, dtype=np.int64))
        if offs.size != self.k:
            raise ValueError(f"DiagHeur keeps exactly k={self.k} diagonals")
        self._sel = ops.selection_from_offsets(self.candidates, torch.as_tensor(offs, device=self.values.device))

    def _selection(self) -> ops.Selection:
        return self._sel

    def forward(self, x: torch.Tensor, step: int = 0) -> torch.Tensor:
        lead = x.shape[:-1]
        x2 = _flatten(x, self.in_features)
        if self.values.dtype == torch.float64:
            x2 = x2.double()
        spec = _OpSpec(self.out_features, self.in_features, self.k, 1.0, "diag", self._selection())
        y = DiagMMFunction.apply(x2, self.values, None, self.bias, spec, None)
        return y.reshape(*lead, self.out_features)

    def param_specs(self) -> list[ParamSpec]:
        specs = [ParamSpec(self.values, True, "values")]
        if self.bias is not None:
            specs.append(ParamSpec(self.bias, False, "bias"))
        return specs

    def effective_matrix(self, step: int = 0) -> DiagMatrix:
        act = self._sel.active[: self.k].long()
        return DiagMatrix(self.out_features, self.in_features, act, self.values.detach()[act])


def diagheur_update(layer: DiagHeurLinear, rng: np.random.Generator, step: int | None = None,
                    total_steps: int | None = None) -> DiagHeurLinear:
    """layers.py:381-413: prune the ceil(frac*k) weakest diagonals (L2 norm, ties ->
    smaller offset), regrow as many uniformly random inactive ones with zero values.
    Everything runs on the device (diagmm_diagheur_update); the host only draws the
    regrowth indices from the reference's RNG stream (rng.choice(pool, n) ==
    pool[rng.choice(len(pool), n)]) — no device-to-host copy."""
    frac = layer.prune_fraction
    if step is not None and total_steps:
        frac = frac * 0.5 * (1.0 + np.cos(np.pi * min(step, total_steps) / total_steps))
    n = min(ceil(frac * layer.k), layer.candidates - layer.k)
    if n <= 0:
        return layer
    idx = rng.choice(layer.candidates - layer.k, n, replace=False)
    sel = layer._sel
    dev = layer.values.device
    grow = torch.as_tensor(idx.astype(np.int32)).pin_memory().to(dev, non_blocking=True)
    code = 0 if layer.values.dtype == torch.float64 else 1
    from . import _lib

    with torch.no_grad():
        _lib.call("diagmm_diagheur_update", code, layer.candidates, layer.diag_len, layer.k, sel.active.data_ptr(),
                  sel.slot.data_ptr(), sel.n_act.data_ptr(), layer.values.data_ptr(), int(n), grow.data_ptr(),
                  torch.cuda.current_stream(dev).cuda_stream)
    sel.n_act_host = torch.full((1,), layer.k, dtype=torch.int32)
    sel.event = torch.cuda.Event()
    sel.event.record(torch.cuda.current_stream(dev))
    layer._keep = grow  # the copy is stream-ordered; keep its source alive until it ran
    return layer


def preselect(layers, step: int, materialize: torch.dtype | None = None) -> None:
    """Run the soft TopK of every layer for ``step`` in ONE launch (batched K4)
    and hand each layer its selection for its next forward at that step.
    Call it right before the model's forward (alpha and values must not change
    between the two); a layer whose forward does not match (step, k, T) re-selects
    on its own, so the result never differs from the per-layer path.
    ``materialize``: also build every auto-route layer's dense W_K of that dtype in
    ONE launch (the tensor-core route's operand; identical to the per-layer build)."""
    layers = [m for m in layers if isinstance(m, DiagLinear)]
    if not layers:
        return
    temps = [m.temperature(step) for m in layers]
    sels = ops.soft_topk_select_many([m.alpha.detach() for m in layers], [m.k for m in layers], temps,
                                     params=[getattr(m, "_sched_params", None) for m in layers])
    for m, T, sel in zip(layers, temps, sels):
        m._presel = ((step, m.k, T), sel)
    if materialize is not None:
        todo = [(m, T, sel) for m, T, sel in zip(layers, temps, sels)
                if m.route == "auto" and m.values.dtype == torch.float32]
        Ws = ops.materialize_many([(m.values.detach(), sel, m.out_features, m.in_features) for m, _, sel in todo],
                                  materialize)
        for (m, T, _), W in zip(todo, Ws):
            m._premat = ((step, m.k, T), W)


def penalties(model: nn.Module, fused: bool = False) -> list[torch.Tensor]:
    """MLPModel.penalties (training.py:439-444) for any module tree.

    ``fused=True`` (after the forward): returns ONE scalar, sum of l1_coeff * |alpha|_1
    over the layers (the loss value is identical), computed without autograd;
    its gradient l1_coeff * sign(alpha) (selection.py:217-222) is instead added
    by each layer's soft-TopK gradient kernel (K5) in the backward of the
    forward that just ran — one fused launch per layer instead of an autograd
    chain of elementwise kernels."""
    layers = [m for m in model.modules() if isinstance(m, DiagLinear) and m.l1_coeff > 0]
    if not fused:
        return [m.penalty() for m in layers]
    if not layers:
        return []
    for m in layers:
        spec = getattr(m, "_last_spec", None)
        if spec is None:
            raise RuntimeError("penalties(fused=True) must follow the forward of every DiagLinear")
        spec.l1 = float(m.l1_coeff)
    with torch.no_grad():
        norms = torch._foreach_norm([m.alpha.detach() for m in layers], 1)
        # scalar coefficients (no host-to-device copy: the step stays CUDA-graph capturable)
        scaled = torch._foreach_mul(norms, [float(m.l1_coeff) for m in layers])
        return [torch.stack(scaled).sum()]


__all__ = [
    "DiagLinear", "DiagMMFunction", "DiagMLP", "DiagMLPFunction", "FrozenDiagLinear", "DiagHeurLinear", "DiagMatrix",
    "ParamSpec", "diagheur_update", "penalties", "preselect", "EPS_ACTIVE", "deferred_topk_grads",
]

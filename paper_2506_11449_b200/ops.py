"""Tensor-level wrappers over the C ABI (device buffers in, device buffers out).

Every function here launches sm_100a kernels from ``_lib/libdiagmm.so`` on the
current CUDA stream of the tensors' device.  Shapes and dtypes are validated
before launch with the reference's exception types.  There is no CPU path:
CPU tensors are rejected.

Dtype policy (include/diagmm.h): activations float64 -> parameters float64;
activations float32 or bfloat16 -> parameters float32 (fp32 accumulation).
Selection state (alpha, alpha_soft) is always float64.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .errors import DuplicateOffset, OffsetOutOfRange, ShapeMismatch

_ACT_CODES = {torch.float64: _lib.F64, torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}


def _code(act_dtype: torch.dtype) -> int:
    try:
        return _ACT_CODES[act_dtype]
    except KeyError:
        raise TypeError(f"unsupported activation dtype {act_dtype}") from None


def param_dtype_for(act_dtype: torch.dtype) -> torch.dtype:
    return torch.float64 if act_dtype == torch.float64 else torch.float32


def _p(t):
    return None if t is None else t.data_ptr()


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise _lib.NativeLibraryError(
                "DiagLinear kernels run on CUDA tensors only (no CPU fallback); got a CPU tensor"
            )


def _contig(t):
    return None if t is None else t.contiguous()


def geometry(M: int, N: int) -> tuple[int, int]:
    """(C, L) = (max, min) — candidate count and diagonal length (diagcore.py:22-26)."""
    return max(M, N), min(M, N)


@dataclass
class Selection:
    """Device-resident result of one soft TopK (K4) for a layer.

    alpha_soft (C,) f64, clamped (C,) u8, active (C,) i32 (first n_act valid,
    ascending), slot (C,) i32 (index in active or -1), n_act (1,) i32.
    ``n_act_host`` is a pinned copy filled asynchronously; call
    ``host_count()`` to read it (waits only on this selection's event).
    """

    alpha_soft: torch.Tensor
    clamped: torch.Tensor
    active: torch.Tensor
    slot: torch.Tensor
    n_act: torch.Tensor
    k: int
    temperature: float
    n_act_host: torch.Tensor | None = None
    event: torch.cuda.Event | None = None
    _alpha_keepalive: torch.Tensor | None = None

    @property
    def C(self) -> int:
        return self.slot.numel()

    def start_host_copy(self) -> None:
        self.n_act_host = torch.empty(1, dtype=torch.int32, pin_memory=True)
        self.n_act_host.copy_(self.n_act, non_blocking=True)
        self.event = torch.cuda.Event()
        self.event.record(torch.cuda.current_stream(self.n_act.device))

    def host_count(self) -> int:
        if self.n_act_host is None:
            self.start_host_copy()
        self.event.synchronize()
        return int(self.n_act_host.item())

    def known_count(self) -> int | None:
        """The active count if its host copy has already landed (no wait, and never
        while a CUDA graph is being captured: a count baked into a graph would be
        stale on replay), else None.  Used as the kernels' grid / plan bound
        ``max_act`` (they process min(device count, max_act) diagonals), so the
        FMA kernels are planned for the real count instead of C."""
        if self.n_act_host is None or self.event is None or torch.cuda.is_current_stream_capturing():
            return None
        if not self.event.query():
            return None
        return max(1, int(self.n_act_host.item()))

    def active_offsets(self) -> torch.Tensor:
        return self.active[: self.host_count()]


def new_selection(C: int, device, k: int = 1, temperature: float = 1.0) -> Selection:
    return Selection(
        alpha_soft=torch.empty(C, dtype=torch.float64, device=device),
        clamped=torch.empty(C, dtype=torch.uint8, device=device),
        active=torch.empty(C, dtype=torch.int32, device=device),
        slot=torch.empty(C, dtype=torch.int32, device=device),
        n_act=torch.empty(1, dtype=torch.int32, device=device),
        k=k,
        temperature=temperature,
    )


def soft_topk_select(alpha: torch.Tensor, k: int, temperature: float,
                     out: Selection | None = None, host_copy: bool = False,
                     params: torch.Tensor | None = None) -> Selection:
    """K4: soft_topk + clamped set + active set (selection.py:100-142, layers.py:234).

    Nothing is read back to the host unless ``host_copy`` (or a later
    ``host_count()``) asks for the active count.  ``params``: a device float64
    pair {T, k} the kernel reads instead of (temperature, k) — set per step by
    schedule.DeviceSchedule, so a captured CUDA graph replays an annealing run."""
    return soft_topk_select_many([alpha], [k], [temperature], [out], host_copy=host_copy,
                                 params=[params])[0]


def soft_topk_select_many(alphas, ks, temperatures, outs=None, host_copy: bool = False, params=None) -> list:
    """Batched K4: every selection in ONE launch (one CTA each) — the per-step
    re-selection of all DiagLinear layers of a model (layers.py:233 per layer)."""
    n = len(alphas)
    if not (len(ks) == len(temperatures) == n):
        raise ValueError("alphas, ks and temperatures must have the same length")
    outs = list(outs) if outs is not None else [None] * n
    params = list(params) if params is not None else [None] * n
    jobs = (_lib.TopkJob * max(1, n))()
    sels = []
    stream = None
    for i, (alpha, k, T, out, prm) in enumerate(zip(alphas, ks, temperatures, outs, params)):
        _need_cuda(alpha)
        if alpha.dtype != torch.float64 or alpha.dim() != 1:
            raise ShapeMismatch("alpha must be a float64 vector")
        a = alpha if alpha.is_contiguous() else alpha.contiguous()
        C = a.numel()
        sel = out if out is not None else new_selection(C, a.device)
        sel.k, sel.temperature = int(k), float(T)
        sel._alpha_keepalive = a
        if prm is not None and (prm.dtype != torch.float64 or prm.numel() != 2 or not prm.is_cuda):
            raise ShapeMismatch("params must be a device float64 pair {T, k}")
        jobs[i] = _lib.TopkJob(C, int(k), float(T), _p(a), _p(sel.alpha_soft), _p(sel.clamped),
                               _p(sel.active), _p(sel.slot), _p(sel.n_act), _p(prm))
        stream = _stream(a) if stream is None else stream
        sels.append(sel)
    if n:
        _lib.call("diagmm_topk_waterfill_batched", n, jobs, stream)
    for sel in sels:
        sel.n_act_host = None
        if host_copy:
            sel.start_host_copy()
    return sels


def soft_topk(alpha: torch.Tensor, k: int, temperature: float) -> torch.Tensor:
    """Device soft_topk (selection.py:127-142) returning alpha_soft only."""
    return soft_topk_select(alpha, k, temperature, host_copy=False).alpha_soft


def soft_topk_grad(alpha: torch.Tensor, k: int, temperature: float, upstream: torch.Tensor,
                   clamped: torch.Tensor | None = None, l1_coeff: float = 0.0,
                   out: torch.Tensor | None = None, accumulate: bool = False,
                   params: torch.Tensor | None = None) -> torch.Tensor:
    """K5: soft_topk_grad (selection.py:145-173) [+ l1 * sign(alpha)]; ``params`` as for
    soft_topk_select."""
    _need_cuda(alpha, upstream)
    a = alpha.contiguous()
    up = upstream.to(torch.float64).contiguous()
    if up.shape != a.shape:
        raise ValueError("upstream must match alpha's shape")
    if clamped is None:
        clamped = soft_topk_select(a, k, temperature, host_copy=False, params=params).clamped
    g = out if out is not None else torch.empty_like(a)
    _lib.call("diagmm_topk_grad", a.numel(), int(k), float(temperature), _p(a), _p(clamped), _p(up),
              float(l1_coeff), _p(g), int(bool(accumulate)), _p(params), _stream(a))
    return g


def soft_topk_grad_many(jobs) -> list:
    """Batched K5: ``jobs`` = [(alpha, k, T, upstream, clamped, l1, out, accumulate, params)];
    every layer's soft TopK gradient in ONE launch (one CTA each) — bit-identical to
    calling ``soft_topk_grad`` per layer.  Returns the ``out`` tensors (allocated when None)."""
    n = len(jobs)
    if n == 0:
        return []
    arr = (_lib.TopkGradJob * n)()
    outs, keep = [], []
    stream = None
    for i, (alpha, k, T, up, clamped, l1, out, acc, prm) in enumerate(jobs):
        _need_cuda(alpha, up)
        a = alpha.contiguous()
        u = up.to(torch.float64).contiguous()
        if u.shape != a.shape or clamped is None:
            raise ValueError("batched K5 needs the upstream at alpha's shape and the clamped set")
        g = out if out is not None else torch.empty_like(a)
        keep += [a, u, clamped, g]
        arr[i] = _lib.TopkGradJob(a.numel(), int(k), float(T), _p(a), _p(clamped), _p(u), float(l1), _p(g),
                                  int(bool(acc)), _p(prm))
        outs.append(g)
        stream = _stream(a) if stream is None else stream
    _lib.call("diagmm_topk_grad_batched", n, arr, stream)
    return outs


def select_hard(alpha: torch.Tensor, k: int) -> torch.Tensor:
    """select_hard (selection.py:176-186): int64 indices, ascending."""
    _need_cuda(alpha)
    a = alpha.to(torch.float64).contiguous()
    idx = torch.empty(int(k), dtype=torch.int32, device=a.device)
    _lib.call("diagmm_select_hard", a.numel(), int(k), _p(a), _p(idx), _stream(a))
    return idx.long()


def validate_offsets(C: int, offsets: torch.Tensor) -> torch.Tensor:
    """DiagonalPattern's checks (diagcore.py:71-88), one host read at construction
    time: every offset in [0, C) (OffsetOutOfRange), none twice (DuplicateOffset).
    Returns the offsets sorted ascending (the reference stores them sorted)."""
    h = offsets.detach().to("cpu", torch.int64).reshape(-1)
    if h.numel() and (int(h.min()) < 0 or int(h.max()) >= C):
        bad = int(h[(h < 0) | (h >= C)][0])
        raise OffsetOutOfRange(f"offset {bad} outside [0, {C})")
    s = torch.sort(h).values
    if s.numel() > 1 and bool((s[1:] == s[:-1]).any()):
        dup = int(s[1:][s[1:] == s[:-1]][0])
        raise DuplicateOffset(f"offset {dup} given twice")
    return s.to(offsets.device)


def selection_from_offsets(C: int, offsets: torch.Tensor, alpha_soft: torch.Tensor | None = None
                           ) -> Selection:
    """Selection for an explicit offset list (DiagHeur / frozen layers): validated
    like the reference's DiagonalPattern and sorted ascending."""
    _need_cuda(offsets)
    offs = validate_offsets(C, offsets).to(torch.int32).contiguous()
    n = offs.numel()
    dev = offs.device
    sel = new_selection(C, dev, k=n)
    sel.active[:n].copy_(offs)
    if alpha_soft is None:
        sel.alpha_soft = None
    else:
        sel.alpha_soft.copy_(alpha_soft)
    _lib.call("diagmm_active_from_list", C, n, _p(offs), _p(sel.slot), _p(sel.n_act), _stream(offs))
    sel.n_act_host = torch.full((1,), n, dtype=torch.int32)
    sel.event = torch.cuda.Event()
    sel.event.record(torch.cuda.current_stream(dev))
    return sel


_WORKSPACE: dict = {}


def _workspace(device, nbytes: int) -> torch.Tensor:
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    ws = _WORKSPACE.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WORKSPACE[key] = ws
    return ws


def _check_product(x: torch.Tensor, width: int, values: torch.Tensor, M: int, N: int):
    _need_cuda(x, values)
    if x.dim() != 2 or x.shape[1] != width:
        raise ShapeMismatch(f"input has shape {tuple(x.shape)}, expected (B, {width})")
    C, L = geometry(M, N)
    if tuple(values.shape) != (C, L):
        raise ShapeMismatch(f"values shape {tuple(values.shape)} does not match {(C, L)}")
    if values.dtype != param_dtype_for(x.dtype):
        raise TypeError(f"values dtype {values.dtype} incompatible with activations {x.dtype}")


def diag_forward(x: torch.Tensor, values: torch.Tensor, sel: Selection, M: int, N: int,
                 bias: torch.Tensor | None = None, max_act: int | None = None) -> torch.Tensor:
    """K1: y = x @ W_K^T (+ bias), x (B, N) -> y (B, M)."""
    _check_product(x, N, values, M, N)
    C, _ = geometry(M, N)
    x = x.contiguous()
    values = values.contiguous()
    bias = _contig(bias)
    y = torch.empty(x.shape[0], M, dtype=x.dtype, device=x.device)
    ma = C if max_act is None else int(max_act)
    code = _code(x.dtype)
    ws = _workspace(x.device, _lib.load().diagmm_forward_workspace(code, M, N, x.shape[0], ma))
    _lib.call("diagmm_forward", code, M, N, x.shape[0], _p(x), _p(values), _p(sel.alpha_soft),
              _p(sel.active), _p(sel.n_act), ma, _p(bias), _p(y), _p(ws), ws.numel(), _stream(x))
    return y


def diag_backward_input(dy: torch.Tensor, values: torch.Tensor, sel: Selection, M: int, N: int,
                        max_act: int | None = None) -> torch.Tensor:
    """K2: dx = dy @ W_K through the never-materialized transpose."""
    _check_product(dy, M, values, M, N)
    C, _ = geometry(M, N)
    dy = dy.contiguous()
    dx = torch.empty(dy.shape[0], N, dtype=dy.dtype, device=dy.device)
    ma = C if max_act is None else int(max_act)
    code = _code(dy.dtype)
    ws = _workspace(dy.device, _lib.load().diagmm_backward_input_workspace(code, M, N, dy.shape[0], ma))
    _lib.call("diagmm_backward_input", code, M, N, dy.shape[0], _p(dy), _p(values.contiguous()),
              _p(sel.alpha_soft), _p(sel.active), _p(sel.n_act), ma, _p(dx), _p(ws), ws.numel(), _stream(dy))
    return dx


def diag_backward_weight(dy: torch.Tensor, x: torch.Tensor, values: torch.Tensor, sel: Selection,
                         M: int, N: int, need_bias: bool = True, need_soft: bool = True,
                         max_act: int | None = None, g_values: torch.Tensor | None = None,
                         bucket: torch.Tensor | None = None):
    """K3: (g_values (C, L), g_soft (C,) f64 | None, g_bias (M,) | None).  ``bucket``
    (rows, L) in the values' dtype: active row j (< rows) is also written there (the
    data-parallel exchange buffer, dp.CompactGradExchange)."""
    _check_product(dy, M, values, M, N)
    _check_product(x, N, values, M, N)
    if dy.shape[0] != x.shape[0]:
        raise ShapeMismatch("dy and x disagree on the batch size")
    C, L = geometry(M, N)
    if max_act is None:  # grid sized by the candidate count, the device count bounds the work: no host sync
        max_act = C
    B = x.shape[0]
    dy = dy.contiguous()
    x = x.contiguous().to(dy.dtype)
    code = _code(dy.dtype)
    lib = _lib.load()
    nbytes = lib.diagmm_backward_weight_workspace(code, M, N, B, int(max_act))
    ws = _workspace(dy.device, nbytes)
    if g_values is None:
        g_values = torch.empty(C, L, dtype=values.dtype, device=dy.device)
    g_soft = torch.empty(C, dtype=torch.float64, device=dy.device) if need_soft else None
    g_bias = torch.empty(M, dtype=values.dtype, device=dy.device) if need_bias else None
    _lib.call("diagmm_backward_weight", code, M, N, B, _p(dy), _p(x), _p(values.contiguous()),
              _p(sel.alpha_soft), _p(sel.active), _p(sel.slot), _p(sel.n_act), int(max_act),
              _p(g_values), _p(g_soft), _p(g_bias), _p(ws), ws.numel(), *_bucket_args(bucket, values, L),
              _stream(dy))
    return g_values, g_soft, g_bias


def _bucket_args(bucket, values, L):
    if bucket is None:
        return None, 0
    if bucket.dtype != values.dtype or bucket.dim() != 2 or bucket.shape[1] != L or not bucket.is_contiguous():
        raise ShapeMismatch(f"bucket must be a contiguous (rows, {L}) {values.dtype} tensor")
    return bucket.data_ptr(), bucket.shape[0]


def materialize(values: torch.Tensor, sel: Selection, M: int, N: int,
                dtype: torch.dtype | None = None, transposed: bool = False) -> torch.Tensor:
    """Dense W_K (M, N) — or W_K^T (N, M) — of the active diagonals
    (diagcore.py:153-159 + layers.py:235)."""
    _need_cuda(values)
    C, L = geometry(M, N)
    if tuple(values.shape) != (C, L):
        raise ShapeMismatch(f"values shape {tuple(values.shape)} does not match {(C, L)}")
    dtype = dtype or values.dtype
    if param_dtype_for(dtype) != values.dtype:
        raise TypeError(f"cannot materialize {values.dtype} values as {dtype}")
    W = torch.empty((N, M) if transposed else (M, N), dtype=dtype, device=values.device)
    _lib.call("diagmm_materialize_transposed" if transposed else "diagmm_materialize", _code(dtype), M, N,
              _p(values.contiguous()), _p(sel.alpha_soft), _p(sel.active), _p(sel.slot), _p(sel.n_act), C, _p(W),
              _stream(values))
    return W


def tc_backward_weight_begin(dy_parts, x: torch.Tensor, values: torch.Tensor, sel: Selection, M: int, N: int,
                             need_bias: bool = True, need_soft: bool = True, max_act: int | None = None) -> dict:
    """First half of ``tc_backward_weight`` / ``tc_backward_weight_split`` for a deferred
    finalize: only the dW GEMM (split-K partials + bias column partials, into a workspace
    owned by the returned record).  ``dw_finalize_many`` completes it later; together they
    are bit-identical to the one-call path.  ``dy_parts``: dy, or its 1-3 column blocks."""
    parts = list(dy_parts) if isinstance(dy_parts, (list, tuple)) else [dy_parts]
    if any(p.dtype != torch.bfloat16 for p in parts) or x.dtype != torch.bfloat16:
        raise TypeError("tc_backward_weight_begin takes bfloat16 dy and x (the TMA maps are bf16)")
    C, L = geometry(M, N)
    if tuple(values.shape) != (C, L) or values.dtype != torch.float32:
        raise ShapeMismatch(f"values {tuple(values.shape)} {values.dtype} for a ({M}, {N}) layer")
    B = x.shape[0]
    ms = parts[0].shape[1] if len(parts) > 1 else 0
    if ms == 0 and parts[0].shape != (B, M):
        raise ShapeMismatch(f"dy {tuple(parts[0].shape)} vs ({B}, {M})")
    ma = C if max_act is None else int(max_act)
    lib = _lib.load()
    ws = torch.empty(max(16, lib.diagmm_tc_backward_weight_workspace(M, N, B, ma)), dtype=torch.uint8,
                     device=x.device)
    ps = [p.contiguous() for p in parts]
    x = x.contiguous()
    _lib.call("diagmm_tc_backward_weight_partials", M, N, B, _p(ps[0]), _p(ps[1] if len(ps) > 1 else None),
              _p(ps[2] if len(ps) > 2 else None), ms, _p(x), _p(sel.slot), _p(sel.n_act), ma, int(bool(need_bias)),
              _p(ws), ws.numel(), _stream(x))
    ks = lib.diagmm_tc_dw_splits(M, N, B)
    pbytes = (ks * max(ma, 1) * L * 4 + 15) // 16 * 16
    return {"M": M, "N": N, "parts": ks, "ws": ws, "colsum_off": pbytes if need_bias else None, "max_act": ma,
            "sel": sel, "values": values.contiguous(), "need_soft": need_soft, "keep": ps + [x]}


def dw_finalize_many(records) -> list:
    """Complete ``tc_backward_weight_begin`` records in ONE launch; returns
    [(g_values (C, L), g_soft (C,) | None, g_bias (M,) | None)]."""
    n = len(records)
    if n == 0:
        return []
    arr = (_lib.DwFinalizeJob * n)()
    outs = []
    stream = None
    for i, r in enumerate(records):
        M, N = r["M"], r["N"]
        C, L = geometry(M, N)
        v = r["values"]
        gv = torch.empty(C, L, dtype=v.dtype, device=v.device)
        gs = torch.empty(C, dtype=torch.float64, device=v.device) if r["need_soft"] else None
        gb = torch.empty(M, dtype=v.dtype, device=v.device) if r["colsum_off"] is not None else None
        ws = r["ws"]
        colsum = ws.data_ptr() + r["colsum_off"] if r["colsum_off"] is not None else None
        sel = r["sel"]
        arr[i] = _lib.DwFinalizeJob(M, N, r["parts"], _p(ws), colsum, r["max_act"], _p(sel.slot), _p(sel.n_act),
                                    _p(sel.alpha_soft), _p(v), _p(gv), _p(gs), _p(gb), None, 0)
        outs.append((gv, gs, gb))
        stream = _stream(v) if stream is None else stream
    _lib.call("diagmm_tc_dw_finalize_batched", n, arr, stream)
    return outs


def materialize_many(items, dtype: torch.dtype) -> list:
    """Every layer's dense W_K in ONE launch: ``items`` = [(values, sel, M, N)] (float32
    stores), W of ``dtype`` (bf16 / fp32) — identical to ``materialize`` per layer."""
    n = len(items)
    if n == 0:
        return []
    code = _code(dtype)
    arr = (_lib.MaterializeJob * n)()
    outs, keep = [], []
    stream = None
    for i, (values, sel, M, N) in enumerate(items):
        _need_cuda(values)
        C, L = geometry(M, N)
        if tuple(values.shape) != (C, L) or values.dtype != torch.float32:
            raise ShapeMismatch(f"values {tuple(values.shape)} {values.dtype} for a batched ({M}, {N}) W")
        v = values.contiguous()
        W = torch.empty((M, N), dtype=dtype, device=values.device)
        keep.append(v)
        arr[i] = _lib.MaterializeJob(M, N, _p(v), _p(sel.alpha_soft), _p(sel.slot), _p(sel.n_act), C, _p(W))
        outs.append(W)
        stream = _stream(values) if stream is None else stream
    _lib.call("diagmm_materialize_batched", code, n, arr, stream)
    return outs


def gather_dense_grad(dW: torch.Tensor, values: torch.Tensor, sel: Selection, M: int, N: int,
                      need_soft: bool = True):
    """g_values / g_soft from a dense dW (M, N) (the dense branch of layers.py:150-153)."""
    _need_cuda(dW, values)
    C, L = geometry(M, N)
    dW = dW.to(values.dtype).contiguous()
    g_values = torch.empty(C, L, dtype=values.dtype, device=values.device)
    g_soft = torch.empty(C, dtype=torch.float64, device=values.device) if need_soft else None
    code = _lib.F64 if values.dtype == torch.float64 else _lib.F32
    _lib.call("diagmm_gather_dense_grad", code, M, N, _p(dW), _p(values.contiguous()), _p(sel.alpha_soft),
              _p(sel.active), _p(sel.slot), _p(sel.n_act), _p(g_values), _p(g_soft), _stream(values))
    return g_values, g_soft


def adamw_(param: torch.Tensor, grad: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: int,
           lr: float, beta1: float, beta2: float, eps: float, weight_decay: float,
           clip_scale: torch.Tensor | None = None) -> None:
    """K6: in-place AdamW (training.py:346-358) over every element of param."""
    _need_cuda(param, grad, m, v)
    for t in (grad, m, v):
        if t.shape != param.shape or t.dtype != param.dtype or not t.is_contiguous():
            raise ShapeMismatch("param, grad, m, v must share shape/dtype and be contiguous")
    if not param.is_contiguous():
        raise ShapeMismatch("param must be contiguous")
    code = _lib.F64 if param.dtype == torch.float64 else _lib.F32
    if param.dtype not in (torch.float64, torch.float32):
        raise TypeError("AdamW state must be float32 or float64")
    _lib.call("diagmm_adamw", code, param.numel(), _p(param), _p(grad), _p(m), _p(v), int(step),
              float(lr), float(beta1), float(beta2), float(eps), float(weight_decay), _p(clip_scale),
              _stream(param))


def sumsq_into(x: torch.Tensor, out: torch.Tensor, scratch: torch.Tensor) -> None:
    """out[0] = sum(x^2) in float64 with a fixed reduction order."""
    _need_cuda(x)
    code = _lib.F64 if x.dtype == torch.float64 else _lib.F32
    if x.dtype not in (torch.float64, torch.float32):
        x = x.float()
    x = x.contiguous()
    _lib.call("diagmm_sumsq", code, x.numel(), _p(x), _p(out), _p(scratch), _stream(x))


def sumsq_scratch(device) -> torch.Tensor:
    return torch.empty(_lib.load().diagmm_sumsq_scratch_len(), dtype=torch.float64, device=device)


def clip_scale(partials: torch.Tensor, max_norm: float):
    """(norm, scale) device scalars of clip_global_norm (training.py:406-417)."""
    norm = torch.empty(1, dtype=torch.float64, device=partials.device)
    scale = torch.empty(1, dtype=torch.float64, device=partials.device)
    _lib.call("diagmm_clip_scale", partials.numel(), _p(partials.contiguous()), float(max_norm), _p(norm),
              _p(scale), _stream(partials))
    return norm, scale


class FusedLayerNorm(torch.autograd.Function):
    """LayerNorm over the last dim for bf16 activations with float32 affine
    parameters (csrc/norm_kernels.cu) — the ViT caller's norm around DiagLinear."""

    @staticmethod
    def forward(ctx, x, weight, bias, eps):
        _need_cuda(x, weight, bias)
        D = x.shape[-1]
        x2 = x.reshape(-1, D).to(torch.bfloat16).contiguous()
        M = x2.shape[0]
        y = torch.empty_like(x2)
        mean = torch.empty(M, dtype=torch.float32, device=x.device)
        rstd = torch.empty(M, dtype=torch.float32, device=x.device)
        w = weight.detach().float().contiguous()
        b = bias.detach().float().contiguous()
        _lib.call("diagmm_layernorm_fwd", M, D, float(eps), _p(x2), _p(w), _p(b), _p(y), _p(mean), _p(rstd),
                  _stream(x2))
        ctx.save_for_backward(x2, w, mean, rstd)
        ctx.shape, ctx.in_dtype = x.shape, x.dtype
        return y.view(x.shape)

    @staticmethod
    def backward(ctx, dy):
        x2, w, mean, rstd = ctx.saved_tensors
        M, D = x2.shape
        g = dy.reshape(M, D).to(torch.bfloat16).contiguous()
        dx = torch.empty_like(x2)
        dw = torch.empty(D, dtype=torch.float32, device=x2.device)
        db = torch.empty(D, dtype=torch.float32, device=x2.device)
        ws = _workspace(x2.device, _lib.load().diagmm_layernorm_bwd_workspace(M, D))
        _lib.call("diagmm_layernorm_bwd", M, D, _p(x2), _p(g), _p(w), _p(mean), _p(rstd), _p(dx), _p(dw), _p(db),
                  _p(ws), ws.numel(), _stream(x2))
        return dx.view(ctx.shape).to(ctx.in_dtype), dw, db, None


def layer_norm_bf16(x, weight, bias, eps: float = 1e-5):
    return FusedLayerNorm.apply(x, weight, bias, eps)


class FusedLayerNormSkip(torch.autograd.Function):
    """(LayerNorm(x), x) as ONE autograd node: when x also feeds the block's skip
    connection, both of its gradient contributions arrive in this backward and the
    kernel sums them (diagmm_layernorm_bwd_res) — no separate gradient add."""

    @staticmethod
    def forward(ctx, x, weight, bias, eps):
        _need_cuda(x, weight, bias)
        D = x.shape[-1]
        x2 = x.reshape(-1, D).to(torch.bfloat16).contiguous()
        M = x2.shape[0]
        y = torch.empty_like(x2)
        mean = torch.empty(M, dtype=torch.float32, device=x.device)
        rstd = torch.empty(M, dtype=torch.float32, device=x.device)
        w = weight.detach().float().contiguous()
        b = bias.detach().float().contiguous()
        _lib.call("diagmm_layernorm_fwd", M, D, float(eps), _p(x2), _p(w), _p(b), _p(y), _p(mean), _p(rstd),
                  _stream(x2))
        ctx.save_for_backward(x2, w, mean, rstd)
        ctx.shape, ctx.in_dtype = x.shape, x.dtype
        return y.view(x.shape), x

    @staticmethod
    def backward(ctx, dy, dskip):
        x2, w, mean, rstd = ctx.saved_tensors
        M, D = x2.shape
        g = dy.reshape(M, D).to(torch.bfloat16).contiguous()
        r = None if dskip is None else dskip.reshape(M, D).to(torch.bfloat16).contiguous()
        dx = torch.empty_like(x2)
        dw = torch.empty(D, dtype=torch.float32, device=x2.device)
        db = torch.empty(D, dtype=torch.float32, device=x2.device)
        ws = _workspace(x2.device, _lib.load().diagmm_layernorm_bwd_workspace(M, D))
        _lib.call("diagmm_layernorm_bwd_res", M, D, _p(x2), _p(g), _p(r), _p(w), _p(mean), _p(rstd), _p(dx),
                  _p(dw), _p(db), _p(ws), ws.numel(), _stream(x2))
        return dx.view(ctx.shape).to(ctx.in_dtype), dw, db, None


def layer_norm_skip_bf16(x, weight, bias, eps: float = 1e-5):
    """(layer_norm(x), x) with the skip connection's gradient summed in the LN backward."""
    return FusedLayerNormSkip.apply(x, weight, bias, eps)


def tf32x3_gemm(a: torch.Tensor, b: torch.Tensor, trans_a: bool = False, trans_b: bool = False,
                bias: torch.Tensor | None = None) -> torch.Tensor:
    """out = op(a) @ op(b).T (+ bias) in float32 on the 3xTF32 tensor-core kernel
    (fp32-accurate; tf32_kernels.cu): op(a) = a (M, K), or a.T for a given as (K, M)
    with ``trans_a``; op(b) = b (N, K), or b.T for b given as (K, N) with ``trans_b``.
    The float32 layers' dense route (the reference's density >= 1/4 switch,
    diagcore.py:226-228 / layers.py:150-153) runs its three GEMMs here."""
    _need_cuda(a, b)
    if a.dtype != torch.float32 or b.dtype != torch.float32 or a.dim() != 2 or b.dim() != 2:
        raise TypeError("tf32x3_gemm takes 2-D float32 operands")
    a, b = a.contiguous(), b.contiguous()
    M, K = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    N, Kb = (b.shape[1], b.shape[0]) if trans_b else (b.shape[0], b.shape[1])
    if K != Kb:
        raise ShapeMismatch(f"inner dims differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    out = torch.empty(M, N, dtype=torch.float32, device=a.device)
    nws = _lib.load().diagmm_tf32x3_gemm_workspace(M, N, K, int(trans_a), int(trans_b))
    ws = _workspace(a.device, nws)
    bz = None if bias is None else bias.float().contiguous()
    _lib.call("diagmm_tf32x3_gemm", M, N, K, _p(a), a.shape[1], int(trans_a), _p(b), b.shape[1], int(trans_b),
              _p(bz), _p(out), N, _p(ws), nws, _stream(a))
    return out


def tc_gemm(a: torch.Tensor, b: torch.Tensor, bias: torch.Tensor | None = None) -> torch.Tensor:
    """out = a @ b.T (+ bias) on the tcgen05 tensor cores (bf16 in/out, fp32 accumulate)."""
    _need_cuda(a, b)
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or a.dim() != 2 or b.dim() != 2:
        raise TypeError("tc_gemm takes 2-D bfloat16 operands")
    if a.shape[1] != b.shape[1]:
        raise ShapeMismatch(f"inner dims differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    a, b = a.contiguous(), b.contiguous()
    out = torch.empty(a.shape[0], b.shape[0], dtype=torch.bfloat16, device=a.device)
    bz = None if bias is None else bias.float().contiguous()
    _lib.call("diagmm_tc_gemm_bf16", a.shape[0], b.shape[0], a.shape[1], _p(a), _p(b), _p(bz), _p(out), out.shape[1],
              _stream(a))
    return out


def tc_gemm_nn(a: torch.Tensor, b: torch.Tensor, bias: torch.Tensor | None = None, epilogue: int = 0,
               aux: torch.Tensor | None = None):
    """out = a @ b (+ bias) with b (K, N) row-major, staged MN-major (diagmm_tc_gemm_bf16_nn):
    the dense-equivalent input gradient dx = dy @ W_K straight from the forward's W_K.
    epilogue 2 (aux = pre-activation) returns (a @ b) * gelu'(aux)."""
    _need_cuda(a, b)
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or a.dim() != 2 or b.dim() != 2:
        raise TypeError("tc_gemm_nn takes 2-D bfloat16 operands")
    if a.shape[1] != b.shape[0] or b.shape[1] % 8:
        raise ShapeMismatch(f"tc_gemm_nn: {tuple(a.shape)} @ {tuple(b.shape)} (N must be a multiple of 8)")
    if epilogue not in (0, 2):
        raise ValueError("tc_gemm_nn supports epilogue 0 or 2")
    a, b = a.contiguous(), b.contiguous()
    out = torch.empty(a.shape[0], b.shape[1], dtype=torch.bfloat16, device=a.device)
    if epilogue == 2 and (aux is None or tuple(aux.shape) != tuple(out.shape) or aux.dtype != torch.bfloat16):
        raise ShapeMismatch("epilogue 2 needs the (M, N) bf16 pre-activation as aux")
    ax = None if epilogue == 0 else aux.contiguous()
    bz = None if bias is None else bias.float().contiguous()
    _lib.call("diagmm_tc_gemm_bf16_nn", a.shape[0], b.shape[1], a.shape[1], _p(a), _p(b), _p(bz), _p(out),
              out.shape[1], _p(ax), int(epilogue), _stream(a))
    return out


def tc_backward_weight(dy: torch.Tensor, x: torch.Tensor, values: torch.Tensor, sel: Selection, M: int, N: int,
                       need_soft: bool = True, max_act: int | None = None, need_bias: bool = False,
                       bucket: torch.Tensor | None = None):
    """K3 on the tensor cores (bf16): (g_values (C, L) f32, g_soft (C,) f64 | None[, g_bias (M,) f32])."""
    if dy.dtype != torch.bfloat16 or x.dtype != torch.bfloat16:
        raise TypeError("tc_backward_weight takes bfloat16 dy and x (the TMA maps are bf16)")
    _check_product(dy, M, values, M, N)
    _check_product(x, N, values, M, N)
    C, L = geometry(M, N)
    ma = C if max_act is None else int(max_act)
    B = x.shape[0]
    dy = dy.contiguous()
    x = x.contiguous()
    ws = _workspace(dy.device, _lib.load().diagmm_tc_backward_weight_workspace(M, N, B, ma))
    g_values = torch.empty(C, L, dtype=values.dtype, device=dy.device)
    g_soft = torch.empty(C, dtype=torch.float64, device=dy.device) if need_soft else None
    g_bias = torch.empty(M, dtype=values.dtype, device=dy.device) if need_bias else None
    _lib.call("diagmm_tc_backward_weight", M, N, B, _p(dy), _p(x), _p(values.contiguous()), _p(sel.alpha_soft),
              _p(sel.slot), _p(sel.n_act), ma, _p(g_values), _p(g_soft), _p(g_bias), _p(ws), ws.numel(),
              *_bucket_args(bucket, values, L), _stream(dy))
    return (g_values, g_soft, g_bias) if need_bias else (g_values, g_soft)


def tc_gemm_nn_split(parts: list[torch.Tensor], b: torch.Tensor) -> torch.Tensor:
    """out = cat(parts, dim=1) @ b without the concatenation (diagmm_tc_gemm_bf16_nn_split):
    2-3 row-major (M, ks) bf16 blocks, b (len(parts)*ks, N)."""
    if not 2 <= len(parts) <= 3:
        raise ValueError("tc_gemm_nn_split takes 2 or 3 column blocks")
    _need_cuda(b, *parts)
    M, ks = parts[0].shape
    if any(p.shape != (M, ks) or p.dtype != torch.bfloat16 for p in parts) or b.dtype != torch.bfloat16:
        raise ShapeMismatch("tc_gemm_nn_split: equal (M, ks) bf16 blocks")
    if b.shape[0] != ks * len(parts) or b.shape[1] % 8 or ks % 64:
        raise ShapeMismatch(f"tc_gemm_nn_split: blocks of {ks} columns against b {tuple(b.shape)}")
    ps = [p.contiguous() for p in parts] + [None] * (3 - len(parts))
    b = b.contiguous()
    out = torch.empty(M, b.shape[1], dtype=torch.bfloat16, device=b.device)
    _lib.call("diagmm_tc_gemm_bf16_nn_split", M, b.shape[1], b.shape[0], _p(ps[0]), _p(ps[1]), _p(ps[2]), ks,
              _p(b), None, _p(out), out.shape[1], _stream(b))
    return out


def tc_backward_weight_split(dy_parts: list[torch.Tensor], x: torch.Tensor, values: torch.Tensor, sel: Selection,
                             M: int, N: int, need_soft: bool = True, max_act: int | None = None,
                             need_bias: bool = False, bucket: torch.Tensor | None = None):
    """tc_backward_weight with dy = cat(dy_parts, dim=1) read block by block (no concatenation)."""
    if not 2 <= len(dy_parts) <= 3:
        raise ValueError("tc_backward_weight_split takes 2 or 3 column blocks")
    if any(p.dtype != torch.bfloat16 for p in dy_parts) or x.dtype != torch.bfloat16:
        raise TypeError("tc_backward_weight_split takes bfloat16 dy blocks and x (the TMA maps are bf16)")
    B, ms = dy_parts[0].shape
    if any(p.shape != (B, ms) for p in dy_parts) or ms * len(dy_parts) != M or ms % 128:
        raise ShapeMismatch("tc_backward_weight_split: equal (B, ms) blocks with ms*len == M, ms % 128 == 0")
    _check_product(x, N, values, M, N)
    C, L = geometry(M, N)
    ma = C if max_act is None else int(max_act)
    ps = [p.contiguous() for p in dy_parts] + [None] * (3 - len(dy_parts))
    x = x.contiguous()
    ws = _workspace(x.device, _lib.load().diagmm_tc_backward_weight_workspace(M, N, B, ma))
    g_values = torch.empty(C, L, dtype=values.dtype, device=x.device)
    g_soft = torch.empty(C, dtype=torch.float64, device=x.device) if need_soft else None
    g_bias = torch.empty(M, dtype=values.dtype, device=x.device) if need_bias else None
    _lib.call("diagmm_tc_backward_weight_split", M, N, B, _p(ps[0]), _p(ps[1]), _p(ps[2]), ms, _p(x),
              _p(values.contiguous()), _p(sel.alpha_soft), _p(sel.slot), _p(sel.n_act), ma, _p(g_values),
              _p(g_soft), _p(g_bias), _p(ws), ws.numel(), *_bucket_args(bucket, values, L), _stream(x))
    return (g_values, g_soft, g_bias) if need_bias else (g_values, g_soft)


def tc_gemm_ex(a: torch.Tensor, b: torch.Tensor, bias: torch.Tensor | None = None, epilogue: int = 1,
               aux: torch.Tensor | None = None):
    """Tensor-core GEMM with a fused GELU (tanh) epilogue (diagmm_tc_gemm_bf16_ex):
    epilogue 1 -> (gelu(a b^T + bias), pre-activation);  epilogue 2 (aux = pre) ->
    ((a b^T) * gelu'(aux), aux);  epilogue 3 (aux = residual) -> (a b^T + bias + aux, aux)."""
    _need_cuda(a, b)
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or a.shape[1] != b.shape[1]:
        raise ShapeMismatch("tc_gemm_ex takes bf16 operands with equal inner dims")
    a, b = a.contiguous(), b.contiguous()
    out = torch.empty(a.shape[0], b.shape[0], dtype=torch.bfloat16, device=a.device)
    if epilogue == 1:
        aux = torch.empty_like(out)
    elif epilogue in (2, 3):
        if aux is None or tuple(aux.shape) != tuple(out.shape) or aux.dtype != torch.bfloat16:
            raise ShapeMismatch(f"epilogue {epilogue} needs an (M, N) bf16 aux tensor")
        aux = aux.contiguous()
    else:
        raise ValueError("epilogue must be 1, 2 or 3")
    bz = None if bias is None else bias.float().contiguous()
    _lib.call("diagmm_tc_gemm_bf16_ex", a.shape[0], b.shape[0], a.shape[1], _p(a), _p(b), _p(bz), _p(out),
              out.shape[1], _p(aux), int(epilogue), _stream(a))
    return out, aux

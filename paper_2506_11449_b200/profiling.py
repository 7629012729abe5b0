"""Measurement helpers: per-C-ABI-call CUDA-event timing, algorithmic work
 and roofline fractions, and the DiagMM kernel section of bench.py.

Algorithmic work per call (nnz = n_act * L, s = activation element size):
    forward / backward_input : 2 nnz B FLOP; s B (M + N) + 4 nnz + 12 n_act bytes
    backward_weight          : 2 nnz B FLOP; s B (M + N) + 4 C L (full g_values) + 4 nnz bytes
    materialize              : s_w M N + 4 nnz bytes
    gather_dense_grad        : 4 nnz (gathered dW) + 4 C L + 4 nnz bytes
    adamw                    : 7 p n bytes (read p, g, m, v; write p, m, v)
The roofline time is max(FLOP / P_fma, bytes / HBM) with P_fma the measured
FFMA peak and HBM the measured copy bandwidth (MEASURED_PEAKS.json).
"""

from __future__ import annotations

import torch

from . import _lib

_ELT = {0: 8, 1: 4, 2: 2}

# C-ABI entry points that implement SURVEY §8 (a) rows (the roofline candidates)
SECTION8_KERNELS = {
    "diagmm_forward", "diagmm_backward_input", "diagmm_backward_weight", "diagmm_topk_waterfill",
    "diagmm_topk_waterfill_batched", "diagmm_topk_grad", "diagmm_adamw", "diagmm_adamw_multi",
    "diagmm_sumsq_multi", "diagmm_materialize", "diagmm_gather_dense_grad", "diagmm_tc_gemm_bf16",
    "diagmm_tc_backward_weight",
}


# C-ABI entry points that launch the same kernel with another epilogue / operand
# layout are one kernel family for the roofline (k_tc_gemm, k_tc_dw)
FAMILY = {
    "diagmm_tc_gemm_bf16_ex": "diagmm_tc_gemm_bf16", "diagmm_tc_gemm_bf16_nn": "diagmm_tc_gemm_bf16",
    "diagmm_tc_gemm_bf16_nn_split": "diagmm_tc_gemm_bf16",
    "diagmm_tc_backward_weight_split": "diagmm_tc_backward_weight",
}


def family(name: str) -> str:
    return FAMILY.get(name, name)


def measured_traffic(name: str):
    """dram bytes (read + write) per launch of ``name`` from the committed ncu
    --set full capture (profiles/*traffic*.json), or None."""
    import json
    from pathlib import Path

    for f in sorted(Path(__file__).resolve().parents[1].glob("profiles/*traffic*.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
        except (OSError, ValueError):
            continue
        if name in d:
            return d[name]
    return None


class CallTimer:
    """Context manager: CUDA events around every C-ABI call (or only ``only``)."""

    def __init__(self, only=None):
        self.only = {only} if isinstance(only, str) else (set(only) if only is not None else None)
        self.records = []

    def _hook(self, name, args, fn):
        if self.only is not None and name not in self.only:
            return fn(*args)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        out = fn(*args)
        e.record()
        self.records.append((name, args, s, e))
        return out

    def __enter__(self):
        _lib.set_hook(self._hook)
        return self

    def __exit__(self, *exc):
        _lib.set_hook(None)

    def totals_ms(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for name, _, s, e in self.records:
            out[name] = out.get(name, 0.0) + s.elapsed_time(e)
        return out


def _n_act(args, name, nact_of):
    if name in ("diagmm_forward", "diagmm_backward_input", "diagmm_backward_weight"):
        M, N = args[1], args[2]
    elif name in ("diagmm_materialize", "diagmm_gather_dense_grad"):
        M, N = args[1], args[2]
    else:
        return None
    return nact_of.get((M, N)) if nact_of else None


TC_FORWARD = ("diagmm_tc_gemm_bf16", "diagmm_tc_gemm_bf16_ex")
TC_PRODUCTS = TC_FORWARD + ("diagmm_tc_gemm_bf16_nn", "diagmm_tc_gemm_bf16_nn_split")
TC_DW = ("diagmm_tc_backward_weight", "diagmm_tc_backward_weight_split")


def tc_layer_shape(name, args):
    """(M, N) of the DiagLinear layer a tensor-core call belongs to: the forward
    GEMM is (tokens x M) = (tokens x N) W_K^T, the input gradient (tokens x N) =
    (tokens x M) W_K, dW takes (M, N) directly."""
    if name in TC_DW:
        return args[0], args[1]
    Md, Nd, K = args[0], args[1], args[2]
    return (Nd, K) if name in TC_FORWARD else (K, Nd)


def tc_work(name, args, nact_of=None, dense_equivalent=False):
    """(flops, bytes) of one tensor-core call.  Default: SURVEY §8(d)'s algorithmic
    work of the DiagLinear op the call implements — 2 nnz B FLOP with nnz = n_act L,
    bytes s B (M + N) + s_w nnz (+ the fused epilogue's extra (B x M) tensor, + the
    full fp32 candidate gradient C L written by dW).  ``dense_equivalent``: the
    dense GEMM the tensor cores actually execute (2 M N B) — reported separately,
    never as the roofline."""
    M, N = tc_layer_shape(name, args)
    C, L = max(M, N), min(M, N)
    if name in TC_DW:
        B = args[2]
        n = (nact_of or {}).get((M, N), C)
        flops = 2.0 * (M * N if dense_equivalent else n * L) * B
        return flops, 2.0 * B * (M + N) + 4.0 * C * L + 4.0 * n * L
    B = args[0]
    n = (nact_of or {}).get((M, N), C)
    aux = 2.0 * B * args[1] if name in ("diagmm_tc_gemm_bf16_ex", "diagmm_tc_gemm_bf16_nn") and args[9] else 0.0
    flops = 2.0 * (M * N if dense_equivalent else n * L) * B
    return flops, 2.0 * B * (M + N) + 2.0 * n * L + 8.0 * n + aux


def work(name, args, nact_of=None):
    """(flops, bytes) of one call, or None when not modelled."""
    if name in ("diagmm_forward", "diagmm_backward_input", "diagmm_backward_weight"):
        dt, M, N, B = args[0], args[1], args[2], args[3]
        C, L = max(M, N), min(M, N)
        n = _n_act(args, name, nact_of) or args[9 if name != "diagmm_backward_weight" else 11]
        s = _ELT[dt]
        p = 8 if dt == 0 else 4
        flops = 2.0 * n * L * B
        if name == "diagmm_backward_weight":
            byts = s * B * (M + N) + p * C * L + p * n * L
        else:
            byts = s * B * (M + N) + p * n * L + 12 * n
        return flops, byts
    if name == "diagmm_materialize":
        dt, M, N = args[0], args[1], args[2]
        n = _n_act(args, name, nact_of) or args[8]
        return 0.0, _ELT[dt] * M * N + 4 * n * min(M, N)
    if name == "diagmm_gather_dense_grad":
        dt, M, N = args[0], args[1], args[2]
        n = _n_act(args, name, nact_of) or max(M, N)
        p = 8 if dt == 0 else 4
        return 0.0, p * n * min(M, N) * 2 + p * max(M, N) * min(M, N)
    if name in TC_PRODUCTS or name in TC_DW:
        return tc_work(name, args, nact_of)
    if name == "diagmm_adamw_multi":
        n, descs = args[0], args[1]
        return 0.0, float(sum(7 * (8 if descs[i].dtype == 0 else 4) * descs[i].n for i in range(n)))
    if name == "diagmm_sumsq_multi":
        n, descs = args[0], args[1]
        return 0.0, float(sum((8 if descs[i].dtype == 0 else 4) * descs[i].n for i in range(n)))
    if name == "diagmm_topk_waterfill_batched":
        n, jobs = args[0], args[1]
        # alpha read, alpha_soft written (f64), clamped (u8), active + slot (i32) per candidate
        return 0.0, float(sum(25 * jobs[i].C for i in range(n)))
    if name == "diagmm_topk_waterfill":
        return 0.0, 25.0 * args[0]
    if name == "diagmm_topk_grad":
        # alpha, g_soft read and g_alpha written (f64), clamped (u8); + g_alpha read if accumulating
        return 0.0, (25.0 + 8.0 * bool(args[8])) * args[0]
    if name == "diagmm_adamw":
        dt, n = args[0], args[1]
        return 0.0, 7 * (8 if dt == 0 else 4) * n
    if name == "diagmm_sumsq":
        dt, n = args[0], args[1]
        return 0.0, (8 if dt == 0 else 4) * n
    return None


def roofline(records, peaks: dict, peaks_kind: str, fma_tflops: float, nact_of=None):
    """Roofline object for the timed calls of one function (bench JSON contract)."""
    if not records:
        return None
    torch.cuda.synchronize()
    name = records[0][0]
    tot_ms, tot_f, tot_b = 0.0, 0.0, 0.0
    for nm, args, s, e in records:
        w = work(nm, args, nact_of)
        if w is None:
            return {"kernel": name, "note": "work not modelled"}
        tot_ms += s.elapsed_time(e)
        tot_f += w[0]
        tot_b += w[1]
    n = len(records)
    sec = tot_ms / 1e3
    hbm = float(peaks["hbm_gbs"])
    name = family(name)
    if name.startswith("diagmm_tc_"):
        # tensor-core family: the roofline is SURVEY §8(d)'s algorithmic work (2 nnz B
        # FLOP at the bf16 tensor peak vs the algorithmic bytes at HBM bandwidth); the
        # dense-equivalent rate the tensor cores run at is reported beside it
        tpk = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1400.0)))
        dense_f = sum(tc_work(nm, a, nact_of, dense_equivalent=True)[0] for nm, a, _, _ in records)
        t_tc, t_hbm = tot_f / (tpk * 1e12), tot_b / (hbm * 1e9)
        common = {"kernel": name, "traffic": None, "launches": n, "avg_launch_us": tot_ms * 1e3 / n,
                  "algorithmic_flops_per_launch": tot_f / n, "algorithmic_bytes_per_launch": tot_b / n,
                  "work_model": "SURVEY 8(d): 2*n_act*L*B FLOP; s*B*(M+N) + s_w*nnz (+ fused epilogue tensor) bytes",
                  "dense_equivalent": {"flops_per_launch": dense_f / n, "tflops": dense_f / sec / 1e12,
                                       "frac_of_bf16_peak": dense_f / sec / 1e12 / tpk,
                                       "note": "the dense GEMM the tcgen05 route executes (W_K materialized); "
                                               "not the roofline"}}
        if t_tc >= t_hbm:
            achieved = tot_f / sec / 1e12
            return {**common, "bound": "tensor", "achieved": achieved, "peak": tpk, "unit": "TFLOP/s",
                    "frac": achieved / tpk,
                    "peak_source": f"{peaks_kind} bf16_tflops_sustained (MEASURED_PEAKS.json)"}
        achieved = tot_b / sec / 1e9
        return {**common, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_source": f"{peaks_kind} hbm_gbs (MEASURED_PEAKS.json)"}
    t_fma = tot_f / (fma_tflops * 1e12)
    t_hbm = tot_b / (hbm * 1e9)
    if t_fma > t_hbm:
        achieved = tot_f / sec / 1e12
        return {"kernel": name, "bound": "fma", "achieved": achieved, "peak": fma_tflops, "unit": "TFLOP/s",
                "frac": achieved / fma_tflops, "traffic": None, "launches": n,
                "avg_launch_us": tot_ms * 1e3 / n, "algorithmic_bytes_per_launch": tot_b / n,
                "algorithmic_flops_per_launch": tot_f / n,
                "peak_source": "measured FFMA (profiles/r01_microbench_fma_lds.txt)",
                "hbm_gbs_achieved": tot_b / sec / 1e9}
    achieved = tot_b / sec / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "launches": n, "avg_launch_us": tot_ms * 1e3 / n,
            "algorithmic_bytes_per_launch": tot_b / n, "peak_source": f"{peaks_kind} (MEASURED_PEAKS.json)"}


# ------------------------------------------------------------------ kernel section
def _time_call(fn, reps: int, flush: torch.Tensor | None):
    """Device time of one call of ``fn`` (ms): ``reps`` calls, each preceded by an
    L2 flush (a READ of a 256 MB buffer: it evicts L2 without leaving dirty lines
    whose write-back would compete with the timed kernel), captured in a CUDA
    graph and replayed, minus a graph of the flushes alone — so neither
    Python/ctypes launch overhead nor the flush is counted, and every call
    starts from a cold L2."""
    fn()
    torch.cuda.synchronize()
    g_work, g_flush = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    sink = torch.empty(1, device=flush.device) if flush is not None else None
    with torch.cuda.graph(g_work):
        for _ in range(reps):
            if flush is not None:
                torch.amax(flush, dim=0, keepdim=True, out=sink)
            fn()
    with torch.cuda.graph(g_flush):
        for _ in range(reps):
            if flush is not None:
                torch.amax(flush, dim=0, keepdim=True, out=sink)

    def timed(g):
        g.replay()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        best = float("inf")
        for _ in range(3):
            s.record()
            g.replay()
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        return best

    return max(timed(g_work) - timed(g_flush), 1e-6) / reps


def diag_case(M, N, B, sparsity, act_dtype, peaks, fma_tflops, seed=0, reps=20, flush=None, dense_cmp=True):
    """Time K1/K2/K3 (and the cuBLAS dense bf16 equivalent) on one shape."""
    import numpy as np

    from . import ops
    from .selection import required_diagonals

    dev = torch.device("cuda")
    C, L = max(M, N), min(M, N)
    k = required_diagonals(M, N, sparsity)
    rng = np.random.default_rng(seed)
    offs = np.sort(rng.choice(C, k, replace=False))
    values = torch.randn(C, L, device=dev, dtype=ops.param_dtype_for(act_dtype))
    sel = ops.selection_from_offsets(C, torch.as_tensor(offs, device=dev))
    x = torch.randn(B, N, device=dev).to(act_dtype)
    dy = torch.randn(B, M, device=dev).to(act_dtype)
    out = {}
    fns = {
        "fwd": lambda: ops.diag_forward(x, values, sel, M, N, max_act=k),
        "dx": lambda: ops.diag_backward_input(dy, values, sel, M, N, max_act=k),
        "dw": lambda: ops.diag_backward_weight(dy, x, values, sel, M, N, need_bias=False, need_soft=False,
                                              max_act=k),
    }
    s = x.element_size()
    for nm, fn in fns.items():
        fn()
        ms = _time_call(fn, reps, flush)
        flops = 2.0 * k * L * B
        byts = s * B * (M + N) + 4 * k * L + (4 * C * L if nm == "dw" else 0)
        t_roof = max(flops / (fma_tflops * 1e12), byts / (peaks["hbm_gbs"] * 1e9))
        out[nm] = {"us": ms * 1e3, "tflops": flops / (ms / 1e3) / 1e12, "gbs": byts / (ms / 1e3) / 1e9,
                   "roofline_frac": t_roof / (ms / 1e3)}
    tot = sum(out[n]["us"] for n in fns)
    res = {"shape": {"M": M, "N": N, "B": B, "sparsity": sparsity, "k": k, "dtype": str(act_dtype)},
           **out, "fwd_bwd_us": tot}
    if act_dtype == torch.bfloat16 and M % 64 == 0 and N % 64 == 0:
        # the tensor-core route of the same framework (materialize + tcgen05 GEMMs, fused-gather dW)
        # the layer's route: W_K materialized once in the forward and read MN-major by dX
        W = ops.materialize(values, sel, M, N, dtype=act_dtype)
        tc = {
            "fwd": lambda: ops.tc_gemm(x, ops.materialize(values, sel, M, N, dtype=act_dtype)),
            "dx": lambda: ops.tc_gemm_nn(dy, W),
            "dw": lambda: ops.tc_backward_weight(dy, x, values, sel, M, N, need_soft=False, max_act=k),
        }
        res["tc_route_us"] = {}
        for nm, fn in tc.items():
            fn()
            res["tc_route_us"][nm] = _time_call(fn, reps, flush) * 1e3
        res["tc_route_us"]["total"] = sum(res["tc_route_us"][n] for n in tc)
        res["best_route_us"] = min(tot, res["tc_route_us"]["total"])
    if dense_cmp:
        W = torch.randn(M, N, device=dev, dtype=torch.bfloat16)
        xb, dyb = x.to(torch.bfloat16), dy.to(torch.bfloat16)
        f = lambda: xb @ W.t()  # noqa: E731
        b1 = lambda: dyb @ W  # noqa: E731
        b2 = lambda: dyb.t() @ xb  # noqa: E731
        for fn in (f, b1, b2):
            fn()
        dense = [_time_call(fn, reps, flush) * 1e3 for fn in (f, b1, b2)]
        res["cublas_bf16_dense_us"] = {"fwd": dense[0], "dx": dense[1], "dw": dense[2], "total": sum(dense)}
        res["speedup_vs_cublas_bf16_fwd_bwd"] = sum(dense) / res.get("best_route_us", tot)
        if act_dtype == torch.float32:
            # the same-precision baseline for float32 layers: cuBLAS SGEMM with TF32 off
            prev = torch.backends.cuda.matmul.allow_tf32
            torch.backends.cuda.matmul.allow_tf32 = False
            try:
                W32 = W.float()
                f32 = [lambda: x @ W32.t(), lambda: dy @ W32, lambda: dy.t() @ x]
                for fn in f32:
                    fn()
                d32 = [_time_call(fn, reps, flush) * 1e3 for fn in f32]
            finally:
                torch.backends.cuda.matmul.allow_tf32 = prev
            res["cublas_fp32_dense_us"] = {"fwd": d32[0], "dx": d32[1], "dw": d32[2], "total": sum(d32),
                                           "note": "cuBLAS SGEMM, TF32 off: the same-precision dense baseline"}
            res["speedup_vs_cublas_fp32_fwd_bwd"] = sum(d32) / res.get("best_route_us", tot)
    return res


def layer_step_case(n_in=768, n_out=3072, B=256, T=1e-3, reps=20, flush=None):
    """BASELINE config 1 as the reference times it: one DiagLinear step — soft TopK
    re-selection (K4), forward, backward (dX, dW, g_values / g_soft, K5 + l1) — through
    the public module (eager autograd), float32, device time per step (CUDA events
    around each step, L2 flushed before each; median)."""
    import numpy as np

    from .layer import DiagLinear
    from .selection import TemperatureSchedule

    lyr = DiagLinear(n_in, n_out, 0.9, seed=0, dtype=torch.float32,
                     t_schedule=TemperatureSchedule("constant", T, T, 1))
    rng = np.random.default_rng(0)
    with torch.no_grad():
        lyr.alpha.add_(torch.as_tensor(rng.standard_normal(lyr.candidates), device="cuda"))
    x = torch.randn(B, n_in, device="cuda", requires_grad=True)
    dy = torch.randn(B, n_out, device="cuda")
    sink = torch.empty(1, device="cuda")

    def step():
        lyr.values.grad = lyr.alpha.grad = lyr.bias.grad = x.grad = None
        lyr(x, step=0).backward(dy)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            torch.amax(flush, dim=0, keepdim=True, out=sink)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        step()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    eager_us = ts[len(ts) // 2] * 1e3
    # the same step captured as one CUDA graph (the FMA route needs no host read inside a
    # capture): device time without the eager autograd / Python launch overhead
    from .graphed import GraphedStep

    def fwd_bwd(inp, up):
        lyr(inp, step=0).backward(up)
        return up

    params = [lyr.values, lyr.alpha, lyr.bias, x]
    gs = GraphedStep(fwd_bwd, params, x, dy)
    gts = []
    for _ in range(reps):
        if flush is not None:
            torch.amax(flush, dim=0, keepdim=True, out=sink)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gs.step(x, dy)
        e.record()
        torch.cuda.synchronize()
        gts.append(s.elapsed_time(e))
    gts.sort()
    return {"us": eager_us, "graphed_us": gts[len(gts) // 2] * 1e3, "n_act": lyr.active_count(0), "k": lyr.k,
            "T": T, "what": "K4 + fwd + dX + dW + K5 through DiagLinear, fp32, B=256: eager autograd (us) and "
                            "the same step replayed as one CUDA graph (graphed_us); L2 flushed before each"}


def diagmm_config1(peaks, peaks_kind, fma_tflops):
    """BASELINE config 1 (DiagLinear 768->3072, 90%, B=256, fp32) + a few sweep points."""
    flush = torch.empty(64 * 1024 * 1024, device="cuda")  # 256 MB > 126 MB L2
    cfg1 = diag_case(3072, 768, 256, 0.9, torch.float32, peaks, fma_tflops, flush=flush)
    cfg1["layer_step"] = layer_step_case(flush=flush)
    sweep = []
    for (dim, s, B) in [(4096, 0.9, 1), (4096, 0.9, 8), (4096, 0.9, 64), (4096, 0.9, 1024), (4096, 0.99, 1),
                        (4096, 0.99, 8), (4096, 0.99, 64), (4096, 0.99, 1024), (4096, 0.9, 8192)]:
        sweep.append(diag_case(dim, dim, B, s, torch.bfloat16, peaks, fma_tflops, reps=10, flush=flush))
    # the ViT-B/16 MLP shape at its per-step token count (256 images x 197 tokens)
    vit = diag_case(3072, 768, 50432, 0.9, torch.bfloat16, peaks, fma_tflops, reps=5, flush=flush)
    return {"config1": cfg1, "sweep_4096": sweep, "vit_fc1_50432_tokens": vit, "hbm_peak_gbs": peaks["hbm_gbs"],
            "fma_peak_tflops": fma_tflops, "peaks": peaks_kind,
            "note": "L2 flushed (256 MB read) before every timed launch; mean of reps, CUDA-graph replay minus flush-only replay"}

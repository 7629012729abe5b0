"""ctypes binding of the C ABI in ``include/diagmm.h`` (``_lib/libdiagmm.so``).

This is the only place the package touches native code.  There is no CPU
fallback: if the library is missing or fails to load, every op raises
``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import STATUS_EXCEPTIONS, NativeLibraryError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libdiagmm.so"

F64, F32, BF16 = 0, 1, 2

_vp, _i, _d, _sz = C.c_void_p, C.c_int, C.c_double, C.c_size_t

# name -> (restype, argtypes); mirrors include/diagmm.h one to one.
SIGNATURES = {
    "diagmm_version": (C.c_char_p, []),
    "diagmm_status_string": (C.c_char_p, [_i]),
    "diagmm_last_error": (C.c_char_p, []),
    "diagmm_launch_count": (C.c_ulonglong, []),
    "diagmm_forward_workspace": (_sz, [_i, _i, _i, _i, _i]),
    "diagmm_forward": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _sz, _vp]),
    "diagmm_backward_input_workspace": (_sz, [_i, _i, _i, _i, _i]),
    "diagmm_backward_input": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _sz, _vp]),
    "diagmm_backward_weight_workspace": (_sz, [_i, _i, _i, _i, _i]),
    "diagmm_backward_weight": (
        _i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _sz, _vp, _i, _vp]),
    "diagmm_topk_waterfill": (_i, [_i, _i, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "diagmm_topk_grad": (_i, [_i, _i, _d, _vp, _vp, _vp, _d, _vp, _i, _vp, _vp]),
    "diagmm_select_hard": (_i, [_i, _i, _vp, _vp, _vp]),
    "diagmm_diagheur_update": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp]),
    "diagmm_active_from_list": (_i, [_i, _i, _vp, _vp, _vp, _vp]),
    "diagmm_adamw": (_i, [_i, _sz, _vp, _vp, _vp, _vp, _i, _d, _d, _d, _d, _d, _vp, _vp]),
    "diagmm_sumsq_scratch_len": (_i, []),
    "diagmm_sumsq": (_i, [_i, _sz, _vp, _vp, _vp, _vp]),
    "diagmm_clip_scale": (_i, [_i, _vp, _d, _vp, _vp, _vp]),
    "diagmm_materialize": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp]),
    "diagmm_materialize_transposed": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp]),
    "diagmm_gather_dense_grad": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
}



class TopkJob(C.Structure):
    """diagmm_topk_job (include/diagmm.h)."""

    _fields_ = [("C", C.c_int), ("k", C.c_int), ("temperature", C.c_double), ("alpha", _vp),
                ("alpha_soft", _vp), ("clamped", _vp), ("active", _vp), ("slot", _vp), ("n_act", _vp),
                ("params", _vp)]


class TensorDesc(C.Structure):
    """diagmm_tensor (include/diagmm.h)."""

    _fields_ = [("dtype", C.c_int), ("step", C.c_int), ("n", C.c_size_t), ("param", _vp), ("grad", _vp),
                ("m", _vp), ("v", _vp), ("weight_decay", C.c_double)]


class TopkGradJob(C.Structure):
    """diagmm_topk_grad_job (include/diagmm.h)."""

    _fields_ = [("C", C.c_int), ("k", C.c_int), ("temperature", C.c_double), ("alpha", _vp), ("clamped", _vp),
                ("g_soft", _vp), ("l1_coeff", C.c_double), ("g_alpha", _vp), ("accumulate", C.c_int),
                ("params", _vp)]


class MaterializeJob(C.Structure):
    """diagmm_materialize_job (include/diagmm.h)."""

    _fields_ = [("M", C.c_int), ("N", C.c_int), ("values", _vp), ("alpha_soft", _vp), ("slot", _vp),
                ("n_act", _vp), ("max_act", C.c_int), ("w", _vp)]


class DwFinalizeJob(C.Structure):
    """diagmm_dw_finalize_job (include/diagmm.h)."""

    _fields_ = [("M", C.c_int), ("N", C.c_int), ("parts", C.c_int), ("partial", _vp), ("colsum", _vp),
                ("max_act", C.c_int), ("slot", _vp), ("n_act", _vp), ("alpha_soft", _vp), ("values", _vp),
                ("g_values", _vp), ("g_soft", _vp), ("g_bias", _vp), ("bucket", _vp), ("bucket_rows", C.c_int)]


SIGNATURES["diagmm_materialize_batched"] = (_i, [_i, _i, C.POINTER(MaterializeJob), _vp])
SIGNATURES["diagmm_tc_dw_splits"] = (_i, [_i, _i, _i])
SIGNATURES["diagmm_tc_backward_weight_partials"] = (
    _i, [_i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _vp, _sz, _vp])
SIGNATURES["diagmm_tc_dw_finalize_batched"] = (_i, [_i, C.POINTER(DwFinalizeJob), _vp])
SIGNATURES["diagmm_topk_waterfill_batched"] = (_i, [_i, C.POINTER(TopkJob), _vp])
SIGNATURES["diagmm_topk_grad_batched"] = (_i, [_i, C.POINTER(TopkGradJob), _vp])
SIGNATURES["diagmm_adamw_multi"] = (_i, [_i, C.POINTER(TensorDesc), _d, _d, _d, _d, _vp, _vp, _vp])
SIGNATURES["diagmm_sumsq_multi_len"] = (_i, [_i, C.POINTER(TensorDesc)])
SIGNATURES["diagmm_sumsq_multi"] = (_i, [_i, C.POINTER(TensorDesc), _vp, _i, _vp])
SIGNATURES["diagmm_clip_scale_tree"] = (_i, [_i, _vp, _d, _vp, _vp, _vp])
SIGNATURES["diagmm_tc_backward_weight_workspace"] = (_sz, [_i, _i, _i, _i])
SIGNATURES["diagmm_tc_backward_weight"] = (
    _i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _sz, _vp, _i, _vp])
SIGNATURES["diagmm_tc_gemm_bf16"] = (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp])
SIGNATURES["diagmm_tc_gemm_bf16_ex"] = (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _i, _vp])
SIGNATURES["diagmm_tc_gemm_bf16_nn"] = (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _i, _vp])
SIGNATURES["diagmm_tc_gemm_bf16_nn_split"] = (_i, [_i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp])
SIGNATURES["diagmm_tc_backward_weight_split"] = (
    _i, [_i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _sz, _vp, _i, _vp])
SIGNATURES["diagmm_pack_qkv_grad"] = (_i, [_i, _i, _i, _i, _vp, _vp, _vp, C.c_longlong, C.c_longlong, C.c_longlong,
                                           _vp, _vp])
SIGNATURES["diagmm_tf32x3_gemm_workspace"] = (_sz, [_i, _i, _i, _i, _i])
SIGNATURES["diagmm_tf32x3_gemm"] = (_i, [_i, _i, _i, _vp, _i, _i, _vp, _i, _i, _vp, _vp, _i, _vp, _sz, _vp])
SIGNATURES["diagmm_vit_patchify"] = (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp])
SIGNATURES["diagmm_vit_embed_fwd"] = (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp])
SIGNATURES["diagmm_vit_embed_bwd_workspace"] = (_sz, [_i, _i])
SIGNATURES["diagmm_vit_embed_bwd"] = (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp])
SIGNATURES["diagmm_layernorm_fwd"] = (_i, [_i, _i, C.c_float, _vp, _vp, _vp, _vp, _vp, _vp, _vp])
SIGNATURES["diagmm_layernorm_bwd_workspace"] = (_sz, [_i, _i])
SIGNATURES["diagmm_layernorm_bwd"] = (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp])
SIGNATURES["diagmm_layernorm_bwd_res"] = (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp])

_LIB = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle with typed signatures."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeLibraryError(
            f"{p} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the DiagLinear path has no CPU fallback)"
        )
    try:
        lib = C.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - environment failure
        raise NativeLibraryError(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def check(status: int, what: str) -> None:
    if status == 0:
        return
    lib = load()
    msg = lib.diagmm_status_string(status).decode()
    if status == 6:  # DIAGMM_ECUDA: name the CUDA error behind it
        msg += f" ({lib.diagmm_last_error().decode()})"
    exc = STATUS_EXCEPTIONS.get(status, NativeLibraryError)
    raise exc(f"{what}: {msg}")


_HOOK = None


def set_hook(hook) -> None:
    """Install ``hook(name, args, fn)`` around every call (profiling.CallTimer)."""
    global _HOOK
    _HOOK = hook


def call(name: str, *args) -> int:
    fn = getattr(load(), name)
    status = fn(*args) if _HOOK is None else _HOOK(name, args, fn)
    check(status, name)
    return status

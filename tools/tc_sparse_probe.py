"""Throughput probe: 2:4-sparse tcgen05.mma.sp vs dense tcgen05 at the ViT shapes."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch

from paper_2506_11449_b200 import _lib, ops

lib = _lib.load()
fn = lib.diagmm_internal_tc_sparse_probe
fn.restype = C.c_int
fn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]


def timeit(f, reps=10):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for (M, N, K) in [(3072, 50432, 768), (768, 50432, 3072), (2304, 50432, 768)]:
    # sparse orientation: A = W (M_out x K) compressed, B = x (tokens x K), out (M_out x tokens)
    Ac = torch.randn(M, K // 2, device="cuda").to(torch.bfloat16)
    Ad = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Bm = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    t_sp = timeit(lambda: fn(M, N, K, Ac.data_ptr(), Bm.data_ptr(), out.data_ptr(), st))
    t_dn = timeit(lambda: ops.tc_gemm(Ad, Bm))
    t_cb = timeit(lambda: torch.nn.functional.linear(Ad, Bm))
    fl = 2.0 * M * N * K
    print(f"{M}x{N}x{K}: sparse {t_sp:.1f}us ({fl / t_sp / 1e6:.0f} logical TF) | dense ours {t_dn:.1f}us "
          f"({fl / t_dn / 1e6:.0f} TF) | cublas {t_cb:.1f}us | sparse/dense speedup {t_dn / t_sp:.2f}", flush=True)

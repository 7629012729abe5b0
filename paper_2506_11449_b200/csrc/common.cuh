// common.cuh — shared types and helpers for the sm_100a DiagLinear kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../../include/diagmm.h"

namespace diagmm {

// Storage type T of activations -> parameter type P and accumulator type A.
template <typename T> struct Traits;
template <> struct Traits<double> { using P = double; using A = double; };
template <> struct Traits<float> { using P = float; using A = float; };
template <> struct Traits<__nv_bfloat16> { using P = float; using A = float; };

template <typename A> __device__ __forceinline__ A to_acc(double v) { return (A)v; }
template <typename A> __device__ __forceinline__ A to_acc(float v) { return (A)v; }
template <typename A> __device__ __forceinline__ A to_acc(__nv_bfloat16 v) {
  return (A)__bfloat162float(v);
}
template <typename T> __device__ __forceinline__ T from_acc(double v);
template <> __device__ __forceinline__ double from_acc<double>(double v) { return v; }
template <typename T> __device__ __forceinline__ T from_acc(float v);
template <> __device__ __forceinline__ float from_acc<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

constexpr int kWarp = 32;

// Number of kernels this library has launched (diagmm_launch_count()).
void note_launch(int n = 1);

// Largest index in [0, n) whose sorted value is < key, +1  (lower_bound).
__device__ __forceinline__ int lower_bound_i32(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier -------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Wait for phase `parity` of an mbarrier.  A bounded spin: if the expected bytes
// never arrive (a programming error) the kernel traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (long long spins = 0; !done; ++spins) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (spins > (1LL << 26)) __trap();
  }
}
// generic-proxy accesses before a buffer is refilled by the async proxy
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// the CUDA error behind the last DIAGMM_ECUDA of this host thread (diagmm_last_error)
inline const char*& last_cuda_error() {
  static thread_local const char* msg = "no error";
  return msg;
}

inline int status_from_cuda() {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return DIAGMM_OK;
  last_cuda_error() = cudaGetErrorString(e);
  return DIAGMM_ECUDA;
}

inline int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace diagmm

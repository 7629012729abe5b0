// Microbenchmarks for the bf16 DiagMM design on B200 (sm_100a):
// FHFMA.BF16 (fma.rn.f32.bf16: fp32 accumulate, bf16 multiplicands taken from
// halves of packed registers) vs FFMA 3-register form, and LDS.128 with
// lane-contiguous (conflict-free) addressing at several occupancies.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ void mfma(float& d, unsigned a, unsigned b, int ha, int hb) {
  // d += bf16(a.h[ha]) * bf16(b.h[hb])
  if (ha == 0 && hb == 0)
    asm volatile("{.reg .b16 a0,a1,b0,b1; mov.b32 {a0,a1},%1; mov.b32 {b0,b1},%2; fma.rn.f32.bf16 %0,a0,b0,%0;}" : "+f"(d) : "r"(a), "r"(b));
  else if (ha == 1 && hb == 0)
    asm volatile("{.reg .b16 a0,a1,b0,b1; mov.b32 {a0,a1},%1; mov.b32 {b0,b1},%2; fma.rn.f32.bf16 %0,a1,b0,%0;}" : "+f"(d) : "r"(a), "r"(b));
  else if (ha == 0 && hb == 1)
    asm volatile("{.reg .b16 a0,a1,b0,b1; mov.b32 {a0,a1},%1; mov.b32 {b0,b1},%2; fma.rn.f32.bf16 %0,a0,b1,%0;}" : "+f"(d) : "r"(a), "r"(b));
  else
    asm volatile("{.reg .b16 a0,a1,b0,b1; mov.b32 {a0,a1},%1; mov.b32 {b0,b1},%2; fma.rn.f32.bf16 %0,a1,b1,%0;}" : "+f"(d) : "r"(a), "r"(b));
}

__global__ void fhfma_kernel(float* out, int iters) {
  float acc[16];
  unsigned x[4], y[2];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 0.001f + i;
#pragma unroll
  for (int i = 0; i < 4; i++) x[i] = 0x3f803f80u + i + threadIdx.x;
  y[0] = 0x3f7f3f7fu; y[1] = 0x3f7e3f7eu;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      mfma(acc[i * 4 + 0], x[i], y[0], 0, 0);
      mfma(acc[i * 4 + 1], x[i], y[0], 1, 1);
      mfma(acc[i * 4 + 2], x[i], y[1], 0, 0);
      mfma(acc[i * 4 + 3], x[i], y[1], 1, 1);
    }
#pragma unroll
    for (int i = 0; i < 4; i++) x[i] ^= 0x00010001u;
  }
  float s = 0; for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}

__global__ void ffma3_kernel(float* out, int iters) {
  float acc[16], x[4], y[4];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 0.001f + i;
#pragma unroll
  for (int i = 0; i < 4; i++) { x[i] = 1.0001f + i * 1e-4f + threadIdx.x * 1e-7f; y[i] = 0.9999f - i * 1e-4f; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) acc[i * 4 + j] = fmaf(x[i], y[j], acc[i * 4 + j]);
#pragma unroll
    for (int i = 0; i < 4; i++) x[i] = __int_as_float(__float_as_int(x[i]) ^ 1);
  }
  float s = 0; for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}

// LDS.128 lane-contiguous, 8 FHFMA per load (the bf16 DiagMM inner loop shape)
__global__ void lds_fhfma_kernel(float* out, int iters, int stride) {
  __shared__ __align__(16) unsigned sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0x3f803f80u ^ i;
  __syncthreads();
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = 0.f;
  const unsigned v = 0x3f7f3f7fu;
  int base = (threadIdx.x & 31) * 4;
  for (int it = 0; it < iters; it++) {
    const int off = ((it * stride) & 63) * 128;
    uint4 q = *reinterpret_cast<const uint4*>(&sm[off + base]);
    mfma(acc[0], q.x, v, 0, 0); mfma(acc[1], q.x, v, 1, 0);
    mfma(acc[2], q.y, v, 0, 1); mfma(acc[3], q.y, v, 1, 1);
    mfma(acc[4], q.z, v, 0, 0); mfma(acc[5], q.z, v, 1, 0);
    mfma(acc[6], q.w, v, 0, 1); mfma(acc[7], q.w, v, 1, 1);
  }
  float s = 0; for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float* d; CK(cudaMalloc(&d, 4));
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d clock(kHz) %d\n", sms, clk);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int thr : {256, 512, 1024}) {
    for (int w = 0; w < 2; w++) {
      int blocks = sms * 2;
      (w ? fhfma_kernel : ffma3_kernel)<<<blocks, thr>>>(d, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      (w ? fhfma_kernel : ffma3_kernel)<<<blocks, thr>>>(d, iters);
      cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      double fl = 2.0 * 16 * iters * (double)blocks * thr;
      printf("%-12s thr=%4d: %.1f TFLOP/s\n", w ? "FHFMA.BF16" : "FFMA 3reg", thr, fl / ms / 1e9);
    }
  }
  for (int thr : {256, 512, 1024}) {
    int blocks = sms * 2;
    lds_fhfma_kernel<<<blocks, thr>>>(d, 100, 7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    lds_fhfma_kernel<<<blocks, thr>>>(d, iters, 7);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 8 * iters * (double)blocks * thr;
    double lds = (double)iters * blocks * thr / 32;
    printf("LDS.128+8xFHFMA thr=%4d: %.1f TFLOP/s, %.3f LDS.128/clk/SM\n", thr, fl / ms / 1e9,
           lds / (ms * 1e-3) / (clk * 1e3) / sms);
  }
  return 0;
}

// Microbenchmarks that size the DiagMM kernel design on B200 (sm_100a):
// FFMA vs FFMA2 issue rate, LDS.128 broadcast vs conflict-free throughput.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void ffma_kernel(float* out, float a, float b, int iters) {
  float r[16];
  #pragma unroll
  for (int i = 0; i < 16; i++) r[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 16; i++) r[i] = fmaf(r[i], a, b);
  }
  float s = 0; for (int i = 0; i < 16; i++) s += r[i];
  if (s == 1234.5f) out[0] = s;
}
__global__ void ffma3_kernel(float* out, int iters) {
  // 3-distinct-register-source form: acc += x*y with x,y varying registers
  float acc[16], x[4], y[4];
  #pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = threadIdx.x * 0.001f + i;
  #pragma unroll
  for (int i = 0; i < 4; i++) { x[i] = 1.0001f + i*1e-4f + threadIdx.x*1e-7f; y[i] = 0.9999f - i*1e-4f; }
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 4; i++)
      #pragma unroll
      for (int j = 0; j < 4; j++) acc[i*4+j] = fmaf(x[i], y[j], acc[i*4+j]);
    #pragma unroll
    for (int i = 0; i < 4; i++) { x[i] = x[i]*0.99999f; }
  }
  float s = 0; for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}
__device__ __forceinline__ void fma2(float2& d, float2 a, float2 b) {
  unsigned long long dd = *reinterpret_cast<unsigned long long*>(&d);
  unsigned long long aa = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long bb = *reinterpret_cast<unsigned long long*>(&b);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(aa), "l"(bb));
  d = *reinterpret_cast<float2*>(&dd);
}
__global__ void ffma2_kernel(float* out, int iters) {
  float2 acc[16], x[4], y[4];
  #pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = make_float2(threadIdx.x * 0.001f + i, i);
  #pragma unroll
  for (int i = 0; i < 4; i++) { x[i] = make_float2(1.0001f + i*1e-4f, 1.0f); y[i] = make_float2(0.9999f - i*1e-4f, 0.5f); }
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < 4; i++)
      #pragma unroll
      for (int j = 0; j < 4; j++) fma2(acc[i*4+j], x[i], y[j]);
  }
  float s = 0; for (int i = 0; i < 16; i++) s += acc[i].x + acc[i].y;
  if (s == 1234.5f) out[0] = s;
}
// LDS.128: each lane reads float4 at (lane*stride + it*? ) ; broadcast = all lanes same address
template <int MODE>
__global__ void lds_kernel(float* out, int iters) {
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i+1, i+2, i+3);
  __syncthreads();
  float4 acc = make_float4(0,0,0,0);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int idx = (MODE == 0) ? (w * 37) & 2047 : (w * 32 + lane) & 2047;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int u = 0; u < 8; u++) {
      float4 v = sm[(idx + u * 64 + it) & 2047];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}
__global__ void lds32_kernel(float* out, int iters) {
  __shared__ float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float acc = 0, acc2 = 0;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int idx = (w * 32 + lane);
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int u = 0; u < 8; u++) { acc += sm[(idx + u * 256 + it) & 8191]; }
  }
  if (acc + acc2 == 1234.5f) out[0] = acc;
}

int main() {
  float* d; CK(cudaMalloc(&d, 16));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock(kHz) %d\n", sms, clk);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    ffma_kernel<<<blocks, threads>>>(d, 1.0001f, 0.5f, 100);
    cudaEventRecord(a); ffma_kernel<<<blocks, threads>>>(d, 1.0001f, 0.5f, iters); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 16 * iters * (double)blocks * threads;
    printf("FFMA imm-ish  thr=%d: %.1f TFLOP/s\n", threads, fl / ms / 1e9);
    cudaEventRecord(a); ffma3_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("FFMA 3reg     thr=%d: %.1f TFLOP/s\n", threads, fl / ms / 1e9);
    cudaEventRecord(a); ffma2_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("FFMA2 f32x2   thr=%d: %.1f TFLOP/s\n", threads, 2 * fl / ms / 1e9);
  }
  int blocks = sms * 2, threads = 1024; iters = 20000;
  double bytes;
  cudaEventRecord(a); lds_kernel<0><<<blocks, threads>>>(d, iters); cudaEventRecord(b);
  CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
  double instr = 8.0 * iters * blocks * threads / 32;  // warp instructions
  printf("LDS.128 broadcast: %.2f warp-instr/clk/SM\n", instr / (ms * 1e-3) / sms / (clk * 1e3));
  cudaEventRecord(a); lds_kernel<1><<<blocks, threads>>>(d, iters); cudaEventRecord(b);
  CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
  bytes = instr * 512;
  printf("LDS.128 conflict-free: %.2f warp-instr/clk/SM, %.1f B/clk/SM\n", instr / (ms * 1e-3) / sms / (clk * 1e3), bytes / (ms*1e-3) / sms / (clk*1e3));
  cudaEventRecord(a); lds32_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(b);
  CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
  printf("LDS.32 conflict-free: %.2f warp-instr/clk/SM\n", instr / (ms * 1e-3) / sms / (clk * 1e3));
  return 0;
}

// Debug: bitonic (key desc, idx asc) sort of a signed-zero input, printed.
#include <cstdio>
#include <cuda_runtime.h>
#include <math_constants.h>
__device__ __forceinline__ double canon(double v) { return v == 0.0 ? 0.0 : v; }
__device__ __forceinline__ bool before(double ka, int ia, double kb, int ib) {
  return ka > kb || (!(ka < kb) && !(ka > kb) && ia < ib);
}
__global__ void k(const double* a, int C, double* ok, int* oi) {
  __shared__ double key[16];
  __shared__ int idx[16];
  int NP = 16;
  for (int i = threadIdx.x; i < NP; i += blockDim.x) { key[i] = i < C ? canon(a[i]) : -CUDART_INF; idx[i] = i < C ? i : 0x7fffffff; }
  __syncthreads();
  for (int kk = 2; kk <= NP; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < NP; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          double ka = key[i], kb = key[ixj]; int ia = idx[i], ib = idx[ixj];
          bool up = (i & kk) == 0;
          bool sw = up ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
          if (sw) { key[i] = kb; key[ixj] = ka; idx[i] = ib; idx[ixj] = ia; }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < NP; i += blockDim.x) { ok[i] = key[i]; oi[i] = idx[i]; }
}
int main() {
  double h[9] = {-1.738266398496882, -0.0, 0.0, -0.35161713127840977, -0.0, -0.18889719608460778, 0.0, 0.8936001849299788, 0.956847237579234};
  double *d, *ok; int* oi;
  cudaMalloc(&d, 72); cudaMalloc(&ok, 128); cudaMalloc(&oi, 64);
  cudaMemcpy(d, h, 72, cudaMemcpyHostToDevice);
  for (int nt : {1024, 32, 16}) {
    k<<<1, nt>>>(d, 9, ok, oi);
    double hk[16]; int hi[16];
    cudaMemcpy(hk, ok, 128, cudaMemcpyDeviceToHost); cudaMemcpy(hi, oi, 64, cudaMemcpyDeviceToHost);
    printf("threads %d:", nt); for (int i = 0; i < 9; i++) printf(" (%g,%d)", hk[i], hi[i]); printf("\n");
  }
  return 0;
}

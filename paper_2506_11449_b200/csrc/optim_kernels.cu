// optim_kernels.cu — K6: AdamW over the full candidate store and device-side
// global-norm clipping (training.py:346-358, 406-417).
//
// The reference updates EVERY candidate row each step (inactive rows carry a
// zero gradient, so their moments decay and weight decay still applies,
// layers.py:429-433 + training.py:354-358); the kernel is therefore a plain
// HBM-bound streaming update: per element it reads param, grad, m, v and
// writes param, m, v (7 words).  Clipping never leaves the device: sumsq
// partials -> clip_scale -> adamw reads *clip_scale.
#include "common.cuh"

namespace diagmm {

template <typename P>
__global__ void __launch_bounds__(256)
k_adamw(size_t n, P* __restrict__ param, const P* __restrict__ grad, P* __restrict__ m,
        P* __restrict__ v, P lr, P b1, P b2, P eps, P wd, P bc1, P bc2,
        const double* __restrict__ clip_scale) {
  const P s = clip_scale ? (P)(*clip_scale) : P(1);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const P g = grad[i] * s;
    const P mi = b1 * m[i] + (P(1) - b1) * g;
    const P vi = b2 * v[i] + (P(1) - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    const P mh = mi / bc1, vh = vi / bc2;
    const P p = param[i];
    param[i] = p - lr * (mh / (sqrt(vh) + eps) + wd * p);
  }
}

// sum(x^2) with a fixed reduction tree: per-block partials in a static order,
// then one block folds them (deterministic run to run).
template <typename P>
__global__ void __launch_bounds__(256)
k_sumsq_partial(size_t n, const P* __restrict__ x, double* __restrict__ part) {
  __shared__ double red[256];
  double acc = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = (double)x[i];
    acc += v * v;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_sum_to(int n, const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

__global__ void k_clip_scale(int n, const double* __restrict__ partial, double max_norm,
                             double* __restrict__ norm, double* __restrict__ scale) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double total = 0.0;
    for (int i = 0; i < n; ++i) total += partial[i];
    const double nrm = sqrt(total);
    if (norm) *norm = nrm;
    if (scale) *scale = (nrm > max_norm && nrm > 0.0) ? max_norm / nrm : 1.0;
  }
}

template <typename P>
int run_adamw(size_t n, void* param, const void* grad, void* m, void* v, int step, double lr,
              double b1, double b2, double eps, double wd, const double* clip_scale, cudaStream_t st) {
  if (step < 1) return DIAGMM_ESHAPE;
  if (n == 0) return DIAGMM_OK;
  const double bc1 = 1.0 - pow(b1, (double)step), bc2 = 1.0 - pow(b2, (double)step);
  long long blocks = (long long)((n + 255) / 256);
  const long long cap = 8LL * num_sms();
  if (blocks > cap) blocks = cap;
  k_adamw<P><<<(int)blocks, 256, 0, st>>>(n, static_cast<P*>(param), static_cast<const P*>(grad),
                                          static_cast<P*>(m), static_cast<P*>(v), (P)lr, (P)b1, (P)b2,
                                          (P)eps, (P)wd, (P)bc1, (P)bc2, clip_scale);
  note_launch();
  return status_from_cuda();
}

constexpr int kSumsqBlocks = 296;

template <typename P>
int run_sumsq(size_t n, const void* x, double* out, double* scratch, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > kSumsqBlocks) blocks = kSumsqBlocks;
  if (blocks < 1) blocks = 1;
  k_sumsq_partial<P><<<blocks, 256, 0, st>>>(n, static_cast<const P*>(x), scratch);
  note_launch();
  k_sum_to<<<1, 32, 0, st>>>(blocks, scratch, out);
  note_launch();
  return status_from_cuda();
}

int run_clip_scale(int n, const double* partial, double max_norm, double* norm, double* scale,
                   cudaStream_t st) {
  k_clip_scale<<<1, 32, 0, st>>>(n, partial, max_norm, norm, scale);
  note_launch();
  return status_from_cuda();
}

template int run_adamw<double>(size_t, void*, const void*, void*, void*, int, double, double, double,
                               double, double, const double*, cudaStream_t);
template int run_adamw<float>(size_t, void*, const void*, void*, void*, int, double, double, double,
                              double, double, const double*, cudaStream_t);
template int run_sumsq<double>(size_t, const void*, double*, double*, cudaStream_t);
template int run_sumsq<float>(size_t, const void*, double*, double*, cudaStream_t);

}  // namespace diagmm

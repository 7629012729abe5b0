// optim_kernels.cu — K6: AdamW over the full candidate store and device-side
// global-norm clipping (training.py:346-358, 406-417).
//
// The reference updates EVERY candidate row each step (inactive rows carry a
// zero gradient, so their moments decay and weight decay still applies,
// layers.py:159-163 + training.py:354-358); the kernel is therefore a plain
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


// ---------------------------------------------------------------- multi-tensor
// One launch updates (or reduces) a whole list of tensors: the per-tensor
// launch sequence of the reference loop (training.py:372-386) becomes a grid
// of fixed-size chunks; block b finds its tensor in the cumulative chunk table.
constexpr int kMtMax = 40;          // tensors per launch (kernel-parameter budget)
constexpr int kMtChunk = 8192;      // elements per block
struct MtTable {
  int n;
  int first[kMtMax + 1];            // first chunk of tensor t; first[n] = total chunks
  diagmm_tensor t[kMtMax];
  double bc1[kMtMax], bc2[kMtMax];  // Adam bias corrections 1 - beta^step (host-computed)
};

__device__ __forceinline__ int mt_find(const MtTable& T, int b) {
  int lo = 0, hi = T.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (T.first[mid] <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <typename P> struct Vec4;
template <> struct Vec4<float> { using t = float4; };
template <> struct Vec4<double> { using t = double2; };  // 16-byte vectors

template <typename P>
__device__ __forceinline__ void adamw_elem(P& p, P g, P& m, P& v, P lr, P b1, P b2, P eps, P wd, P bc1, P bc2) {
  const P mi = b1 * m + (P(1) - b1) * g;
  const P vi = b2 * v + (P(1) - b2) * g * g;
  m = mi;
  v = vi;
  const P mh = mi / bc1, vh = vi / bc2;
  p = p - lr * (mh / (sqrt(vh) + eps) + wd * p);
}

// fp32 stores: the bias corrections as reciprocals (one IEEE division per element
// instead of three; the kernel was issue-bound at 66 % SM / 48 % DRAM throughput)
__device__ __forceinline__ void adamw_elem_f32(float& p, float g, float& m, float& v, float lr, float b1, float b2,
                                               float eps, float wd, float ibc1, float ibc2) {
  const float mi = b1 * m + (1.f - b1) * g;
  const float vi = b2 * v + (1.f - b2) * g * g;
  m = mi;
  v = vi;
  p = p - lr * ((mi * ibc1) / (sqrtf(vi * ibc2) + eps) + wd * p);
}

template <typename P>
__device__ __forceinline__ void adamw_range(const diagmm_tensor& d, size_t i0, size_t i1, P lr, P b1, P b2,
                                            P eps, P s, double bc1d, double bc2d) {
  P* __restrict__ param = static_cast<P*>(d.param);
  const P* __restrict__ grad = static_cast<const P*>(d.grad);
  P* __restrict__ m = static_cast<P*>(d.m);
  P* __restrict__ v = static_cast<P*>(d.v);
  const P bc1 = (P)bc1d, bc2 = (P)bc2d, wd = (P)d.weight_decay;
  constexpr int W = 16 / sizeof(P);
  const bool vec = ((reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(grad) |
                     reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  size_t i = i0;
  if (vec) {
    using V = typename Vec4<P>::t;
    for (size_t q = i0 / W + threadIdx.x; (q + 1) * W <= i1; q += blockDim.x) {
      V pp = reinterpret_cast<V*>(param)[q], gg = reinterpret_cast<const V*>(grad)[q];
      V mm = reinterpret_cast<V*>(m)[q], vv = reinterpret_cast<V*>(v)[q];
      P* pe = reinterpret_cast<P*>(&pp); P* ge = reinterpret_cast<P*>(&gg);
      P* me = reinterpret_cast<P*>(&mm); P* ve = reinterpret_cast<P*>(&vv);
      if constexpr (sizeof(P) == 4) {
        const float ibc1 = (float)(1.0 / bc1d), ibc2 = (float)(1.0 / bc2d);
#pragma unroll
        for (int e = 0; e < W; ++e) adamw_elem_f32(pe[e], ge[e] * s, me[e], ve[e], lr, b1, b2, eps, wd, ibc1, ibc2);
      } else {
#pragma unroll
        for (int e = 0; e < W; ++e) adamw_elem<P>(pe[e], ge[e] * s, me[e], ve[e], lr, b1, b2, eps, wd, bc1, bc2);
      }
      reinterpret_cast<V*>(param)[q] = pp;
      reinterpret_cast<V*>(m)[q] = mm;
      reinterpret_cast<V*>(v)[q] = vv;
    }
    i = i0 + (i1 - i0) / W * W;  // chunks start at multiples of kMtChunk (a multiple of W)
  }
  for (size_t k = i + threadIdx.x; k < i1; k += blockDim.x) {
    P pk = param[k], mk = m[k], vk = v[k];
    adamw_elem<P>(pk, grad[k] * s, mk, vk, lr, b1, b2, eps, wd, bc1, bc2);
    param[k] = pk; m[k] = mk; v[k] = vk;
  }
}

__global__ void __launch_bounds__(256)
k_adamw_multi(const __grid_constant__ MtTable T, double lr, double b1, double b2, double eps,
              const double* __restrict__ clip_scale, const double* __restrict__ sched) {
  const int t = mt_find(T, blockIdx.x);
  const diagmm_tensor& d = T.t[t];
  const size_t i0 = (size_t)(blockIdx.x - T.first[t]) * kMtChunk;
  const size_t i1 = i0 + kMtChunk < d.n ? i0 + kMtChunk : d.n;
  const double s = clip_scale ? *clip_scale : 1.0;
  // sched (device {lr, 1 - b1^t, 1 - b2^t}, host-computed): a CUDA-graph replay of the step
  const double bc1 = sched ? sched[1] : T.bc1[t], bc2 = sched ? sched[2] : T.bc2[t];
  if (sched) lr = sched[0];
  if (d.dtype == DIAGMM_F64)
    adamw_range<double>(d, i0, i1, lr, b1, b2, eps, s, bc1, bc2);
  else
    adamw_range<float>(d, i0, i1, (float)lr, (float)b1, (float)b2, (float)eps, (float)s, bc1, bc2);
}

// per-chunk sum of squares of the gradients, written to part[first_out + block]
__global__ void __launch_bounds__(256)
k_sumsq_multi(const __grid_constant__ MtTable T, double* __restrict__ part, int part_base) {
  __shared__ double red[256];
  const int t = mt_find(T, blockIdx.x);
  const diagmm_tensor& d = T.t[t];
  const size_t i0 = (size_t)(blockIdx.x - T.first[t]) * kMtChunk;
  const size_t i1 = i0 + kMtChunk < d.n ? i0 + kMtChunk : d.n;
  double acc = 0.0;
  if (d.dtype == DIAGMM_F64) {
    const double* g = static_cast<const double*>(d.grad);
    for (size_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) acc += g[i] * g[i];
  } else {
    const float* g = static_cast<const float*>(d.grad);
    if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
      // 16-byte loads, two independent accumulators per thread (fixed order: deterministic)
      const float4* g4 = reinterpret_cast<const float4*>(g);
      double a0 = 0.0, a1 = 0.0;
      const size_t q1 = i1 / 4;  // chunks start at multiples of kMtChunk (a multiple of 4)
      for (size_t q = i0 / 4 + threadIdx.x; q < q1; q += blockDim.x) {
        const float4 v = __ldcs(g4 + q);
        a0 += (double)v.x * (double)v.x + (double)v.y * (double)v.y;
        a1 += (double)v.z * (double)v.z + (double)v.w * (double)v.w;
      }
      acc = a0 + a1;
      for (size_t i = q1 * 4 + threadIdx.x; i < i1; i += blockDim.x) acc += (double)g[i] * (double)g[i];
    } else {
      for (size_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) acc += (double)g[i] * (double)g[i];
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[part_base + blockIdx.x] = red[0];
}

// fixed-order block fold of n partials: norm = sqrt(sum), scale = clip factor
__global__ void __launch_bounds__(1024)
k_clip_scale_tree(int n, const double* __restrict__ partial, double max_norm, double* __restrict__ norm,
                  double* __restrict__ scale) {
  __shared__ double red[1024];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double nrm = sqrt(red[0]);
    if (norm) *norm = nrm;
    if (scale) *scale = (nrm > max_norm && nrm > 0.0) ? max_norm / nrm : 1.0;
  }
}

static int mt_check(int n, const diagmm_tensor* ts) {
  if (n < 0 || (n > 0 && ts == nullptr)) return DIAGMM_ESHAPE;
  for (int i = 0; i < n; ++i) {
    if (ts[i].dtype != DIAGMM_F64 && ts[i].dtype != DIAGMM_F32) return DIAGMM_EDTYPE;
    if (ts[i].n > 0 && ts[i].grad == nullptr) return DIAGMM_ESHAPE;
  }
  return DIAGMM_OK;
}

// Calls fn(table, total_chunks_before) for consecutive batches of <= kMtMax tensors.
template <typename F>
static void mt_batches(int n, const diagmm_tensor* ts, F&& fn) {
  int i = 0, base = 0;
  while (i < n) {
    MtTable T{};
    int chunks = 0;
    while (i < n && T.n < kMtMax) {
      if (ts[i].n == 0) { ++i; continue; }
      T.first[T.n] = chunks;
      T.t[T.n] = ts[i];
      chunks += (int)((ts[i].n + kMtChunk - 1) / kMtChunk);
      ++T.n;
      ++i;
    }
    T.first[T.n] = chunks;
    if (T.n) fn(T, chunks, base);
    base += chunks;
  }
}

int mt_sumsq_parts(int n, const diagmm_tensor* ts) {
  long long c = 0;
  for (int i = 0; i < n; ++i) c += (long long)((ts[i].n + kMtChunk - 1) / kMtChunk);
  return (int)c;
}

int run_adamw_multi(int n, const diagmm_tensor* ts, double lr, double b1, double b2, double eps,
                    const double* clip_scale, const double* sched, cudaStream_t st) {
  if (int e = mt_check(n, ts)) return e;
  for (int i = 0; i < n; ++i)
    if (ts[i].step < 1 || ts[i].param == nullptr || ts[i].m == nullptr || ts[i].v == nullptr)
      return DIAGMM_ESHAPE;
  mt_batches(n, ts, [&](MtTable& T, int chunks, int) {
    for (int i = 0; i < T.n; ++i) {
      T.bc1[i] = 1.0 - pow(b1, (double)T.t[i].step);
      T.bc2[i] = 1.0 - pow(b2, (double)T.t[i].step);
    }
    k_adamw_multi<<<chunks, 256, 0, st>>>(T, lr, b1, b2, eps, clip_scale, sched);
    note_launch();
  });
  return status_from_cuda();
}

int run_sumsq_multi(int n, const diagmm_tensor* ts, double* partial, int partial_len, cudaStream_t st) {
  if (int e = mt_check(n, ts)) return e;
  if (partial_len < mt_sumsq_parts(n, ts)) return DIAGMM_EWORKSPACE;
  mt_batches(n, ts, [&](MtTable& T, int chunks, int base) {
    k_sumsq_multi<<<chunks, 256, 0, st>>>(T, partial, base);
    note_launch();
  });
  return status_from_cuda();
}

int run_clip_scale_tree(int n, const double* partial, double max_norm, double* norm, double* scale,
                        cudaStream_t st) {
  k_clip_scale_tree<<<1, 1024, 0, st>>>(n, partial, max_norm, norm, scale);
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

// diagmm_kernels.cu — sm_100a kernels for the DiagLinear products (K1 forward,
// K2 input gradient, K3 per-diagonal weight gradient) and the dense-equivalent
// helpers (materialize / gather of a dense dW).
//
// Exact math (verified against the reference):
//   W is M x N, C = max(M,N), L = min(M,N), active offsets o_j ascending,
//   V[j,t] = s_j * values[o_j, t]  with s_j = alpha_soft[o_j].
//   "gather" form  (G): out[b,t] = sum_j V[j,t] * in[b, (o_j + t) mod C],  t < L
//        = wide forward (diagcore.py:234-237) and tall/square dX (the transpose
//          of diagcore.py:162-191 read "by own index, +o").
//   "scatter" form (S): out[b,r] = sum_j [c=(r-o_j) mod C < L] V[j,c]*in[b,c], r < C
//        = tall/square forward (diagcore.py:230-233) and wide dX.
//   dW: gw[j,t] = sum_b Aop[b,(o_j+t) mod C] * Bop[b,t]   (layers.py:419-428)
//        tall: Aop = dy, Bop = x;   wide: Aop = x, Bop = dy.
//
// Design notes (B200): one CTA owns a tile of batch rows and a range of output
// positions; the CTA's batch rows of the gathered operand are staged once in
// shared memory (whole rows: every output tile touches almost every column at
// 10% density), so each FMA costs one conflict-free LDS from consecutive
// lanes; the diagonal values are read with coalesced LDG (lane = output
// position) and reused across the BT rows held in registers.  The measured
// smem delivery (128 B/clk/SM, profiles/r01_microbench_fma_lds.txt) bounds
// this design at ~32 fp32 FMA/clk/SM; see DESIGN.md.
#include "common.cuh"

namespace diagmm {

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Copy rows [b0, b0+nb) of a (B, W) row-major matrix into smem (nb, W),
// zero-filling rows past B.
template <typename T>
__device__ __forceinline__ void stage_rows(T* __restrict__ dst, const T* __restrict__ src,
                                           int b0, int nb, int B, int W) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const size_t row_bytes = (size_t)W * sizeof(T);
  const bool vec = (row_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  if (vec) {
    const int per_row = (int)(row_bytes / 16);
    const int total = nb * per_row;
    for (int i = tid; i < total; i += nt) {
      int b = i / per_row, q = i - b * per_row;
      int4 v = make_int4(0, 0, 0, 0);
      if (b0 + b < B) v = __ldg(reinterpret_cast<const int4*>(src + (size_t)(b0 + b) * W) + q);
      reinterpret_cast<int4*>(dst + (size_t)b * W)[q] = v;
    }
  } else {
    for (int b = 0; b < nb; ++b) {
      const bool in_range = b0 + b < B;
      for (int c = tid; c < W; c += nt)
        dst[(size_t)b * W + c] = in_range ? src[(size_t)(b0 + b) * W + c] : T(0);
    }
  }
}

template <typename T>
__device__ __forceinline__ void stage_diagonals(int* __restrict__ offs,
                                                typename Traits<T>::A* __restrict__ scl,
                                                const int32_t* __restrict__ active,
                                                const double* __restrict__ asoft, int n_act) {
  using A = typename Traits<T>::A;
  for (int j = threadIdx.x; j < n_act; j += blockDim.x) {
    int o = active[j];
    offs[j] = o;
    scl[j] = asoft ? (A)asoft[o] : (A)1;
  }
}

// ---------------------------------------------------------------- form G
template <typename T, int BT>
__global__ void __launch_bounds__(256)
k_gather(int B, int C, int L, const T* __restrict__ in, const typename Traits<T>::P* __restrict__ vals,
         const double* __restrict__ asoft, const int32_t* __restrict__ active,
         const int32_t* __restrict__ n_act_p, int max_act,
         const typename Traits<T>::P* __restrict__ bias, T* __restrict__ out) {
  using A = typename Traits<T>::A;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n_act = min(*n_act_p, max_act);
  A* scl = reinterpret_cast<A*>(smem);
  int* offs = reinterpret_cast<int*>(smem + align16((size_t)max_act * sizeof(A)));
  T* xs = reinterpret_cast<T*>(smem + align16((size_t)max_act * sizeof(A)) +
                               align16((size_t)max_act * sizeof(int)));
  const int b0 = blockIdx.y * BT;
  stage_diagonals<T>(offs, scl, active, asoft, n_act);
  stage_rows<T>(xs, in, b0, BT, B, C);
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L) return;
  A acc[BT];
#pragma unroll
  for (int b = 0; b < BT; ++b) acc[b] = A(0);
  const auto* vcol = vals + t;
#pragma unroll 2
  for (int j = 0; j < n_act; ++j) {
    const int o = offs[j];
    const A v = scl[j] * (A)__ldg(vcol + (size_t)o * L);
    int c = o + t;
    c = (c >= C) ? c - C : c;
    const T* xp = xs + c;
#pragma unroll
    for (int b = 0; b < BT; ++b) acc[b] = fma(v, to_acc<A>(xp[(size_t)b * C]), acc[b]);
  }
  const A bb = bias ? (A)bias[t] : A(0);
#pragma unroll
  for (int b = 0; b < BT; ++b)
    if (b0 + b < B) out[(size_t)(b0 + b) * L + t] = from_acc<T>(acc[b] + bb);
}

// ---------------------------------------------------------------- form S
template <typename T, int BT>
__global__ void __launch_bounds__(256)
k_scatter(int B, int C, int L, const T* __restrict__ in, const typename Traits<T>::P* __restrict__ vals,
          const double* __restrict__ asoft, const int32_t* __restrict__ active,
          const int32_t* __restrict__ n_act_p, int max_act,
          const typename Traits<T>::P* __restrict__ bias, T* __restrict__ out) {
  using A = typename Traits<T>::A;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n_act = min(*n_act_p, max_act);
  A* scl = reinterpret_cast<A*>(smem);
  int* offs = reinterpret_cast<int*>(smem + align16((size_t)max_act * sizeof(A)));
  T* xs = reinterpret_cast<T*>(smem + align16((size_t)max_act * sizeof(A)) +
                               align16((size_t)max_act * sizeof(int)));
  const int b0 = blockIdx.y * BT;
  stage_diagonals<T>(offs, scl, active, asoft, n_act);
  stage_rows<T>(xs, in, b0, BT, B, L);
  __syncthreads();
  const int r0 = blockIdx.x * blockDim.x + (threadIdx.x & ~(kWarp - 1));
  if (r0 >= C) return;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  // Diagonals that can touch this warp's 32 rows: o in cyclic [r0-L+1, r0+31].
  int lo1 = 0, hi1 = n_act, lo2 = 0, hi2 = 0;
  if (L + kWarp - 1 < C) {
    const int lo = r0 - L + 1, hi = r0 + kWarp - 1;
    if (lo < 0) {
      lo1 = lower_bound_i32(offs, n_act, lo + C); hi1 = n_act;
      lo2 = 0; hi2 = lower_bound_i32(offs, n_act, hi + 1);
    } else if (hi >= C) {
      lo1 = lower_bound_i32(offs, n_act, lo); hi1 = n_act;
      lo2 = 0; hi2 = lower_bound_i32(offs, n_act, hi - C + 1);
    } else {
      lo1 = lower_bound_i32(offs, n_act, lo); hi1 = lower_bound_i32(offs, n_act, hi + 1);
    }
  }
  A acc[BT];
#pragma unroll
  for (int b = 0; b < BT; ++b) acc[b] = A(0);
  const bool row_ok = r < C;
  for (int pass = 0; pass < 2; ++pass) {
    const int jb = pass ? lo2 : lo1, je = pass ? hi2 : hi1;
#pragma unroll 2
    for (int j = jb; j < je; ++j) {
      const int o = offs[j];
      int c = r - o;
      c = (c < 0) ? c + C : c;
      const bool ok = row_ok && (c < L);
      const int ci = ok ? c : 0;
      const A v = ok ? scl[j] * (A)__ldg(vals + (size_t)o * L + ci) : A(0);
      const T* xp = xs + ci;
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b] = fma(v, to_acc<A>(xp[(size_t)b * L]), acc[b]);
    }
  }
  if (!row_ok) return;
  const A bb = bias ? (A)bias[r] : A(0);
#pragma unroll
  for (int b = 0; b < BT; ++b)
    if (b0 + b < B) out[(size_t)(b0 + b) * C + r] = from_acc<T>(acc[b] + bb);
}

// ---------------------------------------------------------------- dW partials
template <typename T, int TJ>
__global__ void __launch_bounds__(128)
k_dw_partial(int B, int C, int L, const T* __restrict__ aop, const T* __restrict__ bop,
             const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p,
             int rows_per_part, typename Traits<T>::A* __restrict__ partial, int max_act) {
  using A = typename Traits<T>::A;
  __shared__ int so[TJ];
  const int n_act = min(*n_act_p, max_act);
  const int j0 = blockIdx.y * TJ;
  if (j0 >= n_act) return;
  const int nj = min(TJ, n_act - j0);
  if (threadIdx.x < TJ) so[threadIdx.x] = threadIdx.x < nj ? active[j0 + threadIdx.x] : 0;
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L) return;
  int cc[TJ];
#pragma unroll
  for (int jj = 0; jj < TJ; ++jj) {
    int c = so[jj] + t;
    cc[jj] = c >= C ? c - C : c;
  }
  A acc[TJ];
#pragma unroll
  for (int jj = 0; jj < TJ; ++jj) acc[jj] = A(0);
  const int bb = blockIdx.z * rows_per_part;
  const int be = min(B, bb + rows_per_part);
  for (int b = bb; b < be; ++b) {
    const A bm = to_acc<A>(__ldg(bop + (size_t)b * L + t));
    const T* arow = aop + (size_t)b * C;
#pragma unroll
    for (int jj = 0; jj < TJ; ++jj) acc[jj] = fma(to_acc<A>(__ldg(arow + cc[jj])), bm, acc[jj]);
  }
#pragma unroll
  for (int jj = 0; jj < TJ; ++jj)
    if (jj < nj) partial[((size_t)blockIdx.z * max_act + j0 + jj) * L + t] = acc[jj];
}

// Deterministic block sum of one double per thread (fixed tree order).
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double tot = 0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) tot += red[i];
  }
  return tot;  // valid in thread 0
}

// Reduce dW partials over parts (fixed order), scale into g_values rows,
// zero inactive rows, and form g_soft.
template <typename T>
__global__ void __launch_bounds__(256)
k_dw_finalize(int C, int L, int nparts, const typename Traits<T>::A* __restrict__ partial, int max_act,
              const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p,
              const double* __restrict__ asoft, const typename Traits<T>::P* __restrict__ vals,
              typename Traits<T>::P* __restrict__ g_values, double* __restrict__ g_soft) {
  using P = typename Traits<T>::P;
  using A = typename Traits<T>::A;
  __shared__ double red[32];
  const int i = blockIdx.x;
  const int n_act = min(*n_act_p, max_act);
  const int s = slot[i];
  P* grow = g_values + (size_t)i * L;
  if (s < 0 || s >= n_act) {
    for (int t = threadIdx.x; t < L; t += blockDim.x) grow[t] = P(0);
    if (g_soft && threadIdx.x == 0) g_soft[i] = 0.0;
    return;
  }
  const double sc = asoft ? asoft[i] : 1.0;
  double local = 0.0;
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    A gw = A(0);
    for (int p = 0; p < nparts; ++p) gw += partial[((size_t)p * max_act + s) * L + t];
    grow[t] = (P)(sc * (double)gw);
    local += (double)gw * (double)vals[(size_t)i * L + t];
  }
  if (g_soft) {
    double tot = block_sum(local, red);
    if (threadIdx.x == 0) g_soft[i] = tot;
  }
}

// Column sums of dy (bias gradient), two levels for determinism.
template <typename T>
__global__ void __launch_bounds__(256)
k_colsum_partial(int B, int M, const T* __restrict__ dy, int rows_per_part,
                 typename Traits<T>::A* __restrict__ part) {
  using A = typename Traits<T>::A;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  const int bb = blockIdx.y * rows_per_part, be = min(B, bb + rows_per_part);
  A acc = A(0);
  for (int b = bb; b < be; ++b) acc += to_acc<A>(dy[(size_t)b * M + r]);
  part[(size_t)blockIdx.y * M + r] = acc;
}
template <typename T>
__global__ void k_colsum_final(int M, int nparts, const typename Traits<T>::A* __restrict__ part,
                               typename Traits<T>::P* __restrict__ g_bias) {
  using A = typename Traits<T>::A;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  A acc = A(0);
  for (int p = 0; p < nparts; ++p) acc += part[(size_t)p * M + r];
  g_bias[r] = (typename Traits<T>::P)acc;
}

// ---------------------------------------------------------------- dense route
template <typename T>
__global__ void k_materialize(int M, int N, const typename Traits<T>::P* __restrict__ vals,
                              const double* __restrict__ asoft, const int32_t* __restrict__ active,
                              const int32_t* __restrict__ n_act_p, int max_act, T* __restrict__ w) {
  using A = typename Traits<T>::A;
  const int j = blockIdx.y;
  const int n_act = min(*n_act_p, max_act);
  if (j >= n_act) return;
  const int L = min(M, N);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L) return;
  const int o = active[j];
  const A sc = asoft ? (A)asoft[o] : A(1);
  int r, c;
  if (M >= N) { r = (o + t) % M; c = t; } else { r = t; c = (o + t) % N; }
  w[(size_t)r * N + c] = from_acc<T>(sc * (A)vals[(size_t)o * L + t]);
}

template <typename P>
__global__ void __launch_bounds__(256)
k_gather_dense(int M, int N, const P* __restrict__ dW, const P* __restrict__ vals,
               const double* __restrict__ asoft, const int32_t* __restrict__ slot,
               const int32_t* __restrict__ n_act_p, P* __restrict__ g_values, double* __restrict__ g_soft) {
  __shared__ double red[32];
  const int i = blockIdx.x;
  const int L = min(M, N);
  const int s = slot[i];
  P* grow = g_values + (size_t)i * L;
  if (s < 0 || s >= *n_act_p) {
    for (int t = threadIdx.x; t < L; t += blockDim.x) grow[t] = P(0);
    if (g_soft && threadIdx.x == 0) g_soft[i] = 0.0;
    return;
  }
  const double sc = asoft ? asoft[i] : 1.0;
  double local = 0.0;
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    int r, c;
    if (M >= N) { r = (i + t) % M; c = t; } else { r = t; c = (i + t) % N; }
    const double gw = (double)dW[(size_t)r * N + c];
    grow[t] = (P)(sc * gw);
    local += gw * (double)vals[(size_t)i * L + t];
  }
  if (g_soft) {
    double tot = block_sum(local, red);
    if (threadIdx.x == 0) g_soft[i] = tot;
  }
}

// ================================================================ host side
struct ProductPlan {
  int bt, tpb, grid_x, grid_y;
  size_t smem;
};

template <typename T>
static size_t product_smem(int max_act, int bt, int width) {
  using A = typename Traits<T>::A;
  return align16((size_t)max_act * sizeof(A)) + align16((size_t)max_act * sizeof(int)) +
         (size_t)bt * width * sizeof(T);
}

// Pick rows-per-CTA (bt) and threads-per-CTA so that shared memory fits and the
// grid covers the 148 SMs at least twice when the problem allows it.
template <typename T>
static ProductPlan plan_product(int B, int out_w, int in_w, int max_act) {
  const size_t kSmemMax = 220 * 1024;
  const int target = 2 * num_sms();
  ProductPlan p{};
  int bts[] = {16, 8, 4, 2, 1};
  for (int tpb : {256, 128, 64}) {
    for (int bt : bts) {
      if (sizeof(T) == 8 && bt > 8) continue;
      size_t sm = product_smem<T>(max_act, bt, in_w);
      if (sm > kSmemMax) continue;
      int gx = ceil_div(out_w, tpb), gy = ceil_div(B, bt);
      p = {bt, tpb, gx, gy, sm};
      if ((long long)gx * gy >= target) return p;
    }
  }
  if (p.bt == 0) p = {1, 64, ceil_div(out_w, 64), B, product_smem<T>(max_act, 1, in_w)};
  return p;
}

template <typename T, int BT>
static void launch_form(bool gather, const ProductPlan& p, cudaStream_t st, int B, int C, int L,
                        const T* in, const typename Traits<T>::P* vals, const double* asoft,
                        const int32_t* active, const int32_t* n_act, int max_act,
                        const typename Traits<T>::P* bias, T* out) {
  dim3 grid(p.grid_x, p.grid_y);
  if (gather) {
    auto k = k_gather<T, BT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    k<<<grid, p.tpb, p.smem, st>>>(B, C, L, in, vals, asoft, active, n_act, max_act, bias, out);
    note_launch();
  } else {
    auto k = k_scatter<T, BT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    k<<<grid, p.tpb, p.smem, st>>>(B, C, L, in, vals, asoft, active, n_act, max_act, bias, out);
    note_launch();
  }
}

// One product in either form.  gather: out width L, in width C.
// scatter: out width C, in width L.
template <typename T>
int run_product(bool gather, int B, int C, int L, const void* in, const void* vals,
                const double* asoft, const int32_t* active, const int32_t* n_act, int max_act,
                const void* bias, void* out, cudaStream_t st) {
  using P = typename Traits<T>::P;
  if (B == 0) return DIAGMM_OK;
  const int out_w = gather ? L : C, in_w = gather ? C : L;
  ProductPlan p = plan_product<T>(B, out_w, in_w, max_act);
  if (p.smem > 227 * 1024) return DIAGMM_ETOOLARGE;
  auto tin = static_cast<const T*>(in);
  auto tv = static_cast<const P*>(vals);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
  switch (p.bt) {
    case 16: launch_form<T, 16>(gather, p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to); break;
    case 8: launch_form<T, 8>(gather, p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to); break;
    case 4: launch_form<T, 4>(gather, p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to); break;
    case 2: launch_form<T, 2>(gather, p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to); break;
    default: launch_form<T, 1>(gather, p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to); break;
  }
  return status_from_cuda();
}

constexpr int kTJ = 16;
constexpr int kDwThreads = 128;

static void dw_parts(int B, int L, int max_act, int* parts, int* rows_per_part) {
  const int tiles = ceil_div(L, kDwThreads) * ceil_div(max_act > 0 ? max_act : 1, kTJ);
  int p = ceil_div(2 * num_sms(), tiles);
  p = p < 1 ? 1 : p;
  const int max_p = ceil_div(B, 32);
  if (p > max_p) p = max_p;
  if (p < 1) p = 1;
  *rows_per_part = ceil_div(B, p);
  *parts = ceil_div(B, *rows_per_part);
}

template <typename T>
size_t dw_workspace(int M, int N, int B, int max_act) {
  using A = typename Traits<T>::A;
  const int L = M < N ? M : N;
  int parts, rpp;
  dw_parts(B > 0 ? B : 1, L, max_act, &parts, &rpp);
  int cparts = ceil_div(B > 0 ? B : 1, 256);
  return align16((size_t)parts * max_act * L * sizeof(A)) + align16((size_t)cparts * M * sizeof(A));
}

template <typename T>
int run_dw(int M, int N, int B, const void* dy, const void* x, const void* vals, const double* asoft,
           const int32_t* active, const int32_t* slot, const int32_t* n_act, int max_act,
           void* g_values, double* g_soft, void* g_bias, void* ws, size_t ws_bytes, cudaStream_t st) {
  using P = typename Traits<T>::P;
  using A = typename Traits<T>::A;
  const int C = M > N ? M : N, L = M < N ? M : N;
  if (ws_bytes < dw_workspace<T>(M, N, B, max_act)) return DIAGMM_EWORKSPACE;
  int parts, rpp;
  dw_parts(B > 0 ? B : 1, L, max_act, &parts, &rpp);
  A* partial = static_cast<A*>(ws);
  const bool tall = M >= N;
  const T* aop = static_cast<const T*>(tall ? dy : x);
  const T* bop = static_cast<const T*>(tall ? x : dy);
  if (B > 0 && max_act > 0) {
    dim3 grid(ceil_div(L, kDwThreads), ceil_div(max_act, kTJ), parts);
    k_dw_partial<T, kTJ><<<grid, kDwThreads, 0, st>>>(B, C, L, aop, bop, active, n_act, rpp, partial, max_act);
    note_launch();
  } else {
    parts = 0;
  }
  k_dw_finalize<T><<<C, 256, 0, st>>>(C, L, parts, partial, max_act, slot, n_act, asoft,
                                       static_cast<const P*>(vals), static_cast<P*>(g_values), g_soft);
  note_launch();
  if (g_bias) {
    A* cpart = reinterpret_cast<A*>(static_cast<char*>(ws) + align16((size_t)parts * max_act * L * sizeof(A)));
    const int cparts = ceil_div(B > 0 ? B : 1, 256);
    const int crpp = ceil_div(B > 0 ? B : 1, cparts);
    if (B > 0) {
      k_colsum_partial<T><<<dim3(ceil_div(M, 256), cparts), 256, 0, st>>>(
          B, M, static_cast<const T*>(dy), crpp, cpart);
      note_launch();
      k_colsum_final<T><<<ceil_div(M, 256), 256, 0, st>>>(M, cparts, cpart, static_cast<P*>(g_bias));
      note_launch();
    } else {
      cudaMemsetAsync(g_bias, 0, (size_t)M * sizeof(P), st);
    }
  }
  return status_from_cuda();
}

template <typename T>
int run_materialize(int M, int N, const void* vals, const double* asoft, const int32_t* active,
                    const int32_t* n_act, int max_act, void* w, cudaStream_t st) {
  using P = typename Traits<T>::P;
  const int L = M < N ? M : N;
  cudaMemsetAsync(w, 0, (size_t)M * N * sizeof(T), st);
  if (max_act > 0) {
    dim3 grid(ceil_div(L, 256), max_act);
    k_materialize<T><<<grid, 256, 0, st>>>(M, N, static_cast<const P*>(vals), asoft, active, n_act,
                                            max_act, static_cast<T*>(w));
    note_launch();
  }
  return status_from_cuda();
}

template <typename P>
int run_gather_dense(int M, int N, const void* dW, const void* vals, const double* asoft,
                     const int32_t* slot, const int32_t* n_act, void* g_values, double* g_soft,
                     cudaStream_t st) {
  const int C = M > N ? M : N;
  k_gather_dense<P><<<C, 256, 0, st>>>(M, N, static_cast<const P*>(dW), static_cast<const P*>(vals),
                                       asoft, slot, n_act, static_cast<P*>(g_values), g_soft);
  note_launch();
  return status_from_cuda();
}

// explicit instantiations used by capi.cu
#define DIAGMM_INST(T)                                                                          \
  template int run_product<T>(bool, int, int, int, const void*, const void*, const double*,     \
                              const int32_t*, const int32_t*, int, const void*, void*,          \
                              cudaStream_t);                                                    \
  template size_t dw_workspace<T>(int, int, int, int);                                          \
  template int run_dw<T>(int, int, int, const void*, const void*, const void*, const double*,   \
                         const int32_t*, const int32_t*, const int32_t*, int, void*, double*,   \
                         void*, void*, size_t, cudaStream_t);                                   \
  template int run_materialize<T>(int, int, const void*, const double*, const int32_t*,         \
                                  const int32_t*, int, void*, cudaStream_t);
DIAGMM_INST(double)
DIAGMM_INST(float)
DIAGMM_INST(__nv_bfloat16)
template int run_gather_dense<double>(int, int, const void*, const void*, const double*, const int32_t*,
                                      const int32_t*, void*, double*, cudaStream_t);
template int run_gather_dense<float>(int, int, const void*, const void*, const double*, const int32_t*,
                                     const int32_t*, void*, double*, cudaStream_t);

}  // namespace diagmm

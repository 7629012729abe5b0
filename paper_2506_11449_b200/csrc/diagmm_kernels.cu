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
// B200 design (profiles/r01_*):
//  * A CTA (8 warps) owns 128 consecutive output positions x BT batch rows.
//    The gathered operand's BT rows are staged ONCE in shared memory in a
//    column-major tile xs[c][b] (a circular halo of 128 columns removes the
//    per-element `mod`), so for one (diagonal, position) a lane fetches the BT
//    rows of its column with 16-byte LDS and reuses its diagonal value BT times.
//  * The 8 warps split the diagonal list (warp w takes j = w, w+8, ...) and
//    reduce through shared memory in a fixed order at the end (deterministic);
//    the offsets and scales of the next 32 diagonals sit in a per-lane cache
//    (shuffled out), and the diagonal values of diagonal q+1 are loaded while
//    diagonal q is being multiplied, so the dependent-load latency that bounded
//    the first version (ncu: long-scoreboard stalls) is hidden.
//  * Small batches split the diagonal list across CTAs too (grid.z), with a
//    fixed-order reduction kernel, so even B = 1 fills the 148 SMs.
//  * Lanes take positions t0 + lane + 32u (u < 4): every diagonal-value LDG is a
//    coalesced 128-byte warp access and every smem access is bank-conflict free
//    for any offset, wrap or alignment.
//  The shared-memory bandwidth (128 B/clk/SM, profiles/r01_microbench_fma_lds)
//  then bounds fp32 at 32 FMA/clk/SM (4 bytes per FMA) and bf16 at 64.
#include "common.cuh"

namespace diagmm {

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / kWarp;
constexpr int kTile = 128;  // output positions per CTA
constexpr int kU = kTile / kWarp;

// Load BT consecutive T values from shared memory (16-byte aligned) as A.
template <typename T, int BT, typename A>
__device__ __forceinline__ void load_col(const T* __restrict__ p, A (&v)[BT]) {
  static_assert((BT * sizeof(T)) % 16 == 0, "BT * sizeof(T) must be a multiple of 16");
  constexpr int kVec = BT * sizeof(T) / 16;
  constexpr int kPer = 16 / sizeof(T);
  const int4* q = reinterpret_cast<const int4*>(p);
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
    int4 w = q[i];
    const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
    for (int k = 0; k < kPer; ++k) v[i * kPer + k] = to_acc<A>(e[k]);
  }
}

// Stage rows [b0, b0+BT) of a row-major (B, W) matrix, columns c = 0 .. cols-1
// taken circularly (c mod W), into the column-major tile dst[c * BT + b].
template <typename T, int BT>
__device__ __forceinline__ void stage_tile(T* __restrict__ dst, const T* __restrict__ src, int b0, int B,
                                           int W, int cols) {
  for (int i = threadIdx.x; i < BT * cols; i += blockDim.x) {
    const int b = i / cols, c = i - b * cols;
    const int cc = c < W ? c : c % W;
    dst[(size_t)c * BT + b] = (b0 + b < B) ? src[(size_t)(b0 + b) * W + cc] : T(0);
  }
}

// --------------------------------------------------------------------------- K1/K2
// GATHER: out width L (positions t), in width C, smem columns C + kTile (halo).
// !GATHER: out width C (positions r), in width L, smem columns L.
template <typename T, int BT, bool GATHER>
__global__ void __launch_bounds__(kThreads, 2)
k_product(int B, int C, int L, const T* __restrict__ in, const typename Traits<T>::P* __restrict__ vals,
          const double* __restrict__ asoft, const int32_t* __restrict__ active,
          const int32_t* __restrict__ n_act_p, int max_act, const typename Traits<T>::P* __restrict__ bias,
          T* __restrict__ out, typename Traits<T>::A* __restrict__ part, int nsplit) {
  using A = typename Traits<T>::A;
  extern __shared__ __align__(16) unsigned char smem[];
  T* xs = reinterpret_cast<T*>(smem);
  A* red = reinterpret_cast<A*>(smem);  // reused after the main loop
  const int n_act = min(*n_act_p, max_act);
  const int in_w = GATHER ? C : L;
  const int out_w = GATHER ? L : C;
  const int cols = GATHER ? C + kTile : L;
  const int t0 = blockIdx.x * kTile;
  const int b0 = blockIdx.y * BT;
  const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;

  stage_tile<T, BT>(xs, in, b0, B, in_w, cols);

  // The CTA's diagonal list as up to two ranges of the ascending active list.
  int lo1 = 0, hi1 = n_act, lo2 = 0, hi2 = 0;
  if (!GATHER && L + kTile - 1 < C) {
    // (r - o) mod C < L for some r in [t0, t0+128)  <=>  o in cyclic [t0-L+1, t0+127]
    const int lo = t0 - L + 1, hi = t0 + kTile - 1;
    if (lo < 0) {
      lo1 = lower_bound_i32(active, n_act, lo + C); hi1 = n_act;
      hi2 = lower_bound_i32(active, n_act, hi + 1);
    } else if (hi >= C) {
      lo1 = lower_bound_i32(active, n_act, lo); hi1 = n_act;
      hi2 = lower_bound_i32(active, n_act, hi - C + 1);
    } else {
      lo1 = lower_bound_i32(active, n_act, lo); hi1 = lower_bound_i32(active, n_act, hi + 1);
    }
  }
  const int len1 = hi1 - lo1, total = len1 + (hi2 - lo2);
  // split z of nsplit takes a contiguous chunk of the virtual list
  const int per = (total + nsplit - 1) / nsplit;
  const int vb = min(total, (int)blockIdx.z * per), ve = min(total, vb + per);
  __syncthreads();

  A acc[BT][kU];
#pragma unroll
  for (int b = 0; b < BT; ++b)
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[b][u] = A(0);

  // warp-strided walk of [vb, ve): v = vb + warp + kWarps * q
  const int nq = ve - vb - warp > 0 ? (ve - vb - warp + kWarps - 1) / kWarps : 0;
  int o_cache = 0;
  A s_cache = A(0);
  auto fill = [&](int q0) {
    const int v = vb + warp + kWarps * (q0 + lane);
    if (q0 + lane < nq) {
      const int j = v < len1 ? lo1 + v : lo2 + (v - len1);
      o_cache = active[j];
      s_cache = asoft ? (A)asoft[o_cache] : A(1);
    }
  };
  auto fetch = [&](int o, A s, A (&vv)[kU], int (&ci)[kU]) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = t0 + lane + kWarp * u;
      if (GATHER) {
        const bool ok = p < L;
        vv[u] = ok ? s * (A)__ldg(vals + (size_t)o * L + p) : A(0);
        int base = o + t0;
        base = base >= C ? base - C : base;
        ci[u] = base + lane + kWarp * u;
      } else {
        int c = p - o;
        c = c < 0 ? c + C : c;
        const bool ok = p < C && c < L;
        vv[u] = ok ? s * (A)__ldg(vals + (size_t)o * L + c) : A(0);
        ci[u] = ok ? c : 0;
      }
    }
  };
  A vcur[kU], vnxt[kU];
  int ccur[kU], cnxt[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) { vcur[u] = vnxt[u] = A(0); ccur[u] = cnxt[u] = 0; }
  if (nq > 0) {
    fill(0);
    const int o = __shfl_sync(0xffffffffu, o_cache, 0);
    const A s = __shfl_sync(0xffffffffu, s_cache, 0);
    fetch(o, s, vcur, ccur);
  }
  for (int q = 0; q < nq; ++q) {
    if (q + 1 < nq) {
      if (((q + 1) & (kWarp - 1)) == 0) fill(q + 1);
      const int o = __shfl_sync(0xffffffffu, o_cache, (q + 1) & (kWarp - 1));
      const A s = __shfl_sync(0xffffffffu, s_cache, (q + 1) & (kWarp - 1));
      fetch(o, s, vnxt, cnxt);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      A xv[BT];
      load_col<T, BT, A>(xs + (size_t)ccur[u] * BT, xv);
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b][u] = fma(vcur[u], xv[b], acc[b][u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) { vcur[u] = vnxt[u]; ccur[u] = cnxt[u]; }
  }

  // fixed-order cross-warp reduction
  __syncthreads();
#pragma unroll
  for (int b = 0; b < BT; ++b)
#pragma unroll
    for (int u = 0; u < kU; ++u) red[((size_t)warp * BT + b) * kTile + lane + kWarp * u] = acc[b][u];
  __syncthreads();
  for (int i = threadIdx.x; i < BT * kTile; i += kThreads) {
    const int b = i / kTile, tt = i - b * kTile;
    const int p = t0 + tt;
    if (b0 + b >= B || p >= out_w) continue;
    A s = A(0);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[((size_t)w * BT + b) * kTile + tt];
    if (nsplit == 1) {
      if (bias) s += (A)bias[p];
      out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(s);
    } else {
      part[((size_t)blockIdx.z * B + b0 + b) * out_w + p] = s;
    }
  }
}

// Fixed-order sum of the split partials (+ bias).
template <typename T>
__global__ void __launch_bounds__(256)
k_split_reduce(int B, int out_w, int nsplit, const typename Traits<T>::A* __restrict__ part,
               const typename Traits<T>::P* __restrict__ bias, T* __restrict__ out) {
  using A = typename Traits<T>::A;
  const size_t n = (size_t)B * out_w;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    A s = A(0);
    for (int z = 0; z < nsplit; ++z) s += part[(size_t)z * n + i];
    if (bias) s += (A)bias[i % out_w];
    out[i] = from_acc<T>(s);
  }
}

// --------------------------------------------------------------------------- K3
// CTA: 128 positions x (kWarps * JQ) diagonals x one batch part; walks its rows in
// chunks of RB staged column-major in smem: the Aop window the tile's diagonals
// read (offsets ascend, so a tile of consecutive diagonals reads one short
// circular window of each row) and the Bop columns of the tile.
template <typename T, int RB, int JQ>
__global__ void __launch_bounds__(kThreads, 2)
k_dw(int B, int C, int L, const T* __restrict__ aop, const T* __restrict__ bop,
     const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act, int win_cap,
     int rows_per_part, typename Traits<T>::A* __restrict__ partial) {
  using A = typename Traits<T>::A;
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int kJ = kWarps * JQ;
  const int n_act = min(*n_act_p, max_act);
  const int j0 = blockIdx.y * kJ;
  if (j0 >= n_act) return;
  const int nj = min(kJ, n_act - j0);
  const int t0 = blockIdx.x * kTile;
  const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;
  const int o_first = active[j0], o_last = active[j0 + nj - 1];
  // window of Aop columns: [ws, ws + wcols) taken circularly
  int ws, wcols;
  if (o_last - o_first + kTile <= win_cap) {
    ws = o_first + t0;
    ws = ws >= C ? ws - C : ws;
    wcols = o_last - o_first + kTile;
  } else {
    ws = 0;
    wcols = C + kTile;
  }
  T* as = reinterpret_cast<T*>(smem);  // wcols x RB
  T* bs = reinterpret_cast<T*>(smem + align16((size_t)win_cap * RB * sizeof(T)));  // kTile x RB
  // window column of (diagonal q, position u) = rel[q] + lane + 32u
  int rel[JQ];
#pragma unroll
  for (int q = 0; q < JQ; ++q) {
    const int j = j0 + warp + kWarps * q;
    int r = 0;
    if (j < j0 + nj) {
      const int o = active[j];
      if (ws == 0 && wcols == C + kTile) {
        r = o + t0;
        r = r >= C ? r - C : r;
      } else {
        r = o - o_first;  // offsets ascend inside the tile
      }
    }
    rel[q] = r;
  }
  A acc[JQ][kU];
#pragma unroll
  for (int q = 0; q < JQ; ++q)
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[q][u] = A(0);

  const int rb = blockIdx.z * rows_per_part, re = min(B, rb + rows_per_part);
  for (int c0 = rb; c0 < re; c0 += RB) {
    __syncthreads();
    for (int i = threadIdx.x; i < RB * wcols; i += kThreads) {
      const int b = i / wcols, c = i - b * wcols;
      int cc = ws + c;
      while (cc >= C) cc -= C;
      as[(size_t)c * RB + b] = (c0 + b < re) ? aop[(size_t)(c0 + b) * C + cc] : T(0);
    }
    for (int i = threadIdx.x; i < RB * kTile; i += kThreads) {
      const int b = i / kTile, c = i - b * kTile;
      bs[(size_t)c * RB + b] = (c0 + b < re && t0 + c < L) ? bop[(size_t)(c0 + b) * L + t0 + c] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      A bv[RB];
      load_col<T, RB, A>(bs + (size_t)(lane + kWarp * u) * RB, bv);
#pragma unroll
      for (int q = 0; q < JQ; ++q) {
        A av[RB];
        load_col<T, RB, A>(as + (size_t)(rel[q] + lane + kWarp * u) * RB, av);
#pragma unroll
        for (int b = 0; b < RB; ++b) acc[q][u] = fma(av[b], bv[b], acc[q][u]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < JQ; ++q) {
    const int j = j0 + warp + kWarps * q;
    if (j >= j0 + nj) continue;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = t0 + lane + kWarp * u;
      if (t < L) partial[((size_t)blockIdx.z * max_act + j) * L + t] = acc[q][u];
    }
  }
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

// Column sums of dy (bias gradient): 32-row partials, then a fixed-order fold.
constexpr int kColRows = 32;
template <typename T>
__global__ void __launch_bounds__(256)
k_colsum_partial(int B, int M, const T* __restrict__ dy, typename Traits<T>::A* __restrict__ part) {
  using A = typename Traits<T>::A;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  const int bb = blockIdx.y * kColRows, be = min(B, bb + kColRows);
  A acc = A(0);
  for (int b = bb; b < be; ++b) acc += to_acc<A>(dy[(size_t)b * M + r]);
  part[(size_t)blockIdx.y * M + r] = acc;
}
template <typename T>
__global__ void __launch_bounds__(256)
k_colsum_final(int M, int nparts, const typename Traits<T>::A* __restrict__ part,
               typename Traits<T>::P* __restrict__ g_bias) {
  using A = typename Traits<T>::A;
  __shared__ A red[8][33];
  // 32 columns per CTA, the 8 warps split the parts, fixed-order fold
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + lane;
  A acc = A(0);
  if (r < M)
    for (int p = w; p < nparts; p += 8) acc += part[(size_t)p * M + r];
  red[w][lane] = acc;
  __syncthreads();
  if (w == 0 && r < M) {
    A s = A(0);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += red[i][lane];
    g_bias[r] = (typename Traits<T>::P)s;
  }
}

// --------------------------------------------------------------------------- dense route
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
  if (M >= N) { r = o + t; r = r >= M ? r - M : r; c = t; } else { r = t; c = o + t; c = c >= N ? c - N : c; }
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
    if (M >= N) { r = i + t; r = r >= M ? r - M : r; c = t; } else { r = t; c = i + t; c = c >= N ? c - N : c; }
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
  int bt, gx, gy, nsplit;
  size_t smem;
};

template <typename T>
static size_t product_smem(int bt, int cols) {
  using A = typename Traits<T>::A;
  const size_t tile = (size_t)bt * cols * sizeof(T);
  const size_t red = (size_t)kWarps * bt * kTile * sizeof(A);
  return align16(tile > red ? tile : red);
}

template <typename T>
static void row_choices(int (&v)[3]) {
  if (sizeof(T) == 8) { v[0] = 8; v[1] = 4; v[2] = 2; }
  else if (sizeof(T) == 4) { v[0] = 16; v[1] = 8; v[2] = 4; }
  else { v[0] = 16; v[1] = 8; v[2] = 8; }
}

template <typename T>
static ProductPlan plan_product(int B, int out_w, int cols, int max_act) {
  const size_t kSmem2 = 113 * 1024, kSmem1 = 220 * 1024;
  const int sms = num_sms();
  const int gx = ceil_div(out_w, kTile);
  int choices[3];
  row_choices<T>(choices);
  ProductPlan best{0, 0, 0, 1, 0};
  for (size_t cap : {kSmem2, kSmem1}) {
    for (int bt : choices) {
      const size_t sm = product_smem<T>(bt, cols);
      if (sm > cap) continue;
      const int gy = ceil_div(B, bt);
      // largest row tile that still gives every SM a CTA; else the smallest tile
      best = {bt, gx, gy, 1, sm};
      if ((long long)gx * gy >= sms) break;
    }
    if (best.bt != 0) break;
  }
  if (best.bt == 0) return best;
  const long long ctas = (long long)best.gx * best.gy;
  if (ctas < 2LL * sms) {
    const int ns = (int)ceil_div(2LL * sms, ctas);
    const int max_ns = max_act / 32 > 1 ? max_act / 32 : 1;
    best.nsplit = ns < max_ns ? ns : max_ns;
  }
  return best;
}

template <typename T, int BT, bool G>
static void launch_product(const ProductPlan& p, cudaStream_t st, int B, int C, int L, const T* in,
                           const typename Traits<T>::P* vals, const double* asoft, const int32_t* active,
                           const int32_t* n_act, int max_act, const typename Traits<T>::P* bias, T* out,
                           typename Traits<T>::A* part) {
  auto k = k_product<T, BT, G>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  k<<<dim3(p.gx, p.gy, p.nsplit), kThreads, p.smem, st>>>(B, C, L, in, vals, asoft, active, n_act, max_act,
                                                          bias, out, part, p.nsplit);
  note_launch();
}

template <typename T>
size_t product_workspace(bool gather, int B, int C, int L, int max_act) {
  using A = typename Traits<T>::A;
  const int out_w = gather ? L : C, cols = gather ? C + kTile : L;
  ProductPlan p = plan_product<T>(B > 0 ? B : 1, out_w, cols, max_act);
  return p.nsplit > 1 ? (size_t)p.nsplit * B * out_w * sizeof(A) : 0;
}

template <typename T>
int run_product(bool gather, int B, int C, int L, const void* in, const void* vals, const double* asoft,
                const int32_t* active, const int32_t* n_act, int max_act, const void* bias, void* out,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  using P = typename Traits<T>::P;
  using A = typename Traits<T>::A;
  if (B == 0) return DIAGMM_OK;
  const int out_w = gather ? L : C, cols = gather ? C + kTile : L;
  ProductPlan p = plan_product<T>(B, out_w, cols, max_act);
  if (p.bt == 0) return DIAGMM_ETOOLARGE;
  if (p.nsplit > 1 && (ws == nullptr || ws_bytes < (size_t)p.nsplit * B * out_w * sizeof(A))) p.nsplit = 1;
  auto tin = static_cast<const T*>(in);
  auto tv = static_cast<const P*>(vals);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
  auto part = static_cast<A*>(ws);
#define DIAGMM_LAUNCH(BT)                                                                           \
  if (p.bt == BT) {                                                                                 \
    if (gather)                                                                                     \
      launch_product<T, BT, true>(p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to, part); \
    else                                                                                            \
      launch_product<T, BT, false>(p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to, part); \
  }
  if constexpr (sizeof(T) == 8) {
    DIAGMM_LAUNCH(8) DIAGMM_LAUNCH(4) DIAGMM_LAUNCH(2)
  } else if constexpr (sizeof(T) == 4) {
    DIAGMM_LAUNCH(16) DIAGMM_LAUNCH(8) DIAGMM_LAUNCH(4)
  } else {
    DIAGMM_LAUNCH(16) DIAGMM_LAUNCH(8)
  }
#undef DIAGMM_LAUNCH
  if (p.nsplit > 1) {
    const size_t n = (size_t)B * out_w;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    k_split_reduce<T><<<blocks, 256, 0, st>>>(B, out_w, p.nsplit, part, tb, to);
    note_launch();
  }
  return status_from_cuda();
}

// dW tiling: rows per staged chunk (16-byte column loads) and diagonals per warp
template <typename T> struct DwRows;
template <> struct DwRows<double> { static constexpr int RB = 4; };
template <> struct DwRows<float> { static constexpr int RB = 8; };
template <> struct DwRows<__nv_bfloat16> { static constexpr int RB = 16; };
constexpr int kJQ = 4;
constexpr int kDwJ = kWarps * kJQ;

template <typename T>
static int dw_win_cap(int C) {
  // Room for a full circular row (C + 128 columns): a tile whose offsets span
  // more than that falls back to staging whole rows.  Up to C ~ 3300 the tiles
  // still fit two CTAs per SM.
  return C + kTile;
}

template <typename T>
static size_t dw_smem(int C) {
  constexpr int RB = DwRows<T>::RB;
  return align16((size_t)dw_win_cap<T>(C) * RB * sizeof(T)) + (size_t)kTile * RB * sizeof(T);
}

static void dw_parts(int B, int L, int max_act, int rb, int* parts, int* rows_per_part) {
  const long long tiles = (long long)ceil_div(L, kTile) * ceil_div(max_act > 0 ? max_act : 1, kDwJ);
  long long p = ceil_div(2LL * num_sms(), tiles);
  if (p < 1) p = 1;
  const long long max_p = ceil_div(B, rb);
  if (p > max_p) p = max_p;
  if (p < 1) p = 1;
  int rpp = ceil_div(B, p);
  rpp = ceil_div(rpp, rb) * rb;
  *rows_per_part = rpp;
  *parts = ceil_div(B, rpp);
}

template <typename T>
size_t dw_workspace(int M, int N, int B, int max_act) {
  using A = typename Traits<T>::A;
  const int L = M < N ? M : N;
  const int C = M > N ? M : N;
  int parts, rpp;
  dw_parts(B > 0 ? B : 1, L, max_act, DwRows<T>::RB, &parts, &rpp);
  const int cparts = ceil_div(B > 0 ? B : 1, kColRows);
  const size_t prod_f = product_workspace<T>(M < N, B, C, L, max_act);
  const size_t prod_b = product_workspace<T>(M >= N, B, C, L, max_act);
  const size_t dw = align16((size_t)parts * max_act * L * sizeof(A)) + align16((size_t)cparts * M * sizeof(A));
  size_t ws = dw > prod_f ? dw : prod_f;
  return ws > prod_b ? ws : prod_b;
}

template <typename T>
int run_dw(int M, int N, int B, const void* dy, const void* x, const void* vals, const double* asoft,
           const int32_t* active, const int32_t* slot, const int32_t* n_act, int max_act, void* g_values,
           double* g_soft, void* g_bias, void* ws, size_t ws_bytes, cudaStream_t st) {
  using P = typename Traits<T>::P;
  using A = typename Traits<T>::A;
  constexpr int RB = DwRows<T>::RB;
  const int C = M > N ? M : N, L = M < N ? M : N;
  if (ws_bytes < dw_workspace<T>(M, N, B, max_act)) return DIAGMM_EWORKSPACE;
  int parts, rpp;
  dw_parts(B > 0 ? B : 1, L, max_act, RB, &parts, &rpp);
  A* partial = static_cast<A*>(ws);
  const bool tall = M >= N;
  const T* aop = static_cast<const T*>(tall ? dy : x);
  const T* bop = static_cast<const T*>(tall ? x : dy);
  if (B > 0 && max_act > 0) {
    const size_t sm = dw_smem<T>(C);
    if (sm > 227 * 1024) return DIAGMM_ETOOLARGE;
    auto k = k_dw<T, RB, kJQ>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid(ceil_div(L, kTile), ceil_div(max_act, kDwJ), parts);
    k<<<grid, kThreads, sm, st>>>(B, C, L, aop, bop, active, n_act, max_act, dw_win_cap<T>(C), rpp, partial);
    note_launch();
  } else {
    parts = 0;
  }
  k_dw_finalize<T><<<C, 256, 0, st>>>(C, L, parts, partial, max_act, slot, n_act, asoft,
                                       static_cast<const P*>(vals), static_cast<P*>(g_values), g_soft);
  note_launch();
  if (g_bias) {
    A* cpart = reinterpret_cast<A*>(static_cast<char*>(ws) + align16((size_t)parts * max_act * L * sizeof(A)));
    if (B > 0) {
      const int cparts = ceil_div(B, kColRows);
      k_colsum_partial<T><<<dim3(ceil_div(M, 256), cparts), 256, 0, st>>>(B, M, static_cast<const T*>(dy), cpart);
      note_launch();
      k_colsum_final<T><<<ceil_div(M, 32), 256, 0, st>>>(M, cparts, cpart, static_cast<P*>(g_bias));
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
    k_materialize<T><<<grid, 256, 0, st>>>(M, N, static_cast<const P*>(vals), asoft, active, n_act, max_act,
                                            static_cast<T*>(w));
    note_launch();
  }
  return status_from_cuda();
}

template <typename P>
int run_gather_dense(int M, int N, const void* dW, const void* vals, const double* asoft, const int32_t* slot,
                     const int32_t* n_act, void* g_values, double* g_soft, cudaStream_t st) {
  const int C = M > N ? M : N;
  k_gather_dense<P><<<C, 256, 0, st>>>(M, N, static_cast<const P*>(dW), static_cast<const P*>(vals), asoft, slot,
                                       n_act, static_cast<P*>(g_values), g_soft);
  note_launch();
  return status_from_cuda();
}

// explicit instantiations used by capi.cu
#define DIAGMM_INST(T)                                                                                    \
  template int run_product<T>(bool, int, int, int, const void*, const void*, const double*,               \
                              const int32_t*, const int32_t*, int, const void*, void*, void*, size_t,     \
                              cudaStream_t);                                                              \
  template size_t product_workspace<T>(bool, int, int, int, int);                                         \
  template size_t dw_workspace<T>(int, int, int, int);                                                    \
  template int run_dw<T>(int, int, int, const void*, const void*, const void*, const double*,             \
                         const int32_t*, const int32_t*, const int32_t*, int, void*, double*, void*,      \
                         void*, size_t, cudaStream_t);                                                    \
  template int run_materialize<T>(int, int, const void*, const double*, const int32_t*, const int32_t*,   \
                                  int, void*, cudaStream_t);
DIAGMM_INST(double)
DIAGMM_INST(float)
DIAGMM_INST(__nv_bfloat16)
template int run_gather_dense<double>(int, int, const void*, const void*, const double*, const int32_t*,
                                      const int32_t*, void*, double*, cudaStream_t);
template int run_gather_dense<float>(int, int, const void*, const void*, const double*, const int32_t*,
                                     const int32_t*, void*, double*, cudaStream_t);

}  // namespace diagmm

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
// B200 design (measurements in profiles/):
//  * Staging: the gathered operand's rows are copied global->shared by the TMA
//    engine (cp.async.bulk, one instruction per row segment, completion on an
//    mbarrier); a circular halo of 128 columns after each row removes the
//    per-element `mod`.  Every output tile of a 10%-dense wrap-around matrix
//    touches almost every input column, so whole rows are staged once per CTA
//    and reused by every diagonal.
//  * Lanes take positions p0 + lane + 32u (u < 4): every diagonal-value load is a
//    coalesced 128-byte warp access and every shared-memory read is
//    bank-conflict free for any offset, wrap or alignment.
//  * Offsets/scales of the next 32 diagonals live in a per-lane cache (shuffled
//    out) and the values of diagonal q+1 are loaded while diagonal q is being
//    multiplied, hiding the dependent global-load latency.
//  * Two tilings: WIDE (large batch) — each warp owns 128 positions of a
//    1024-position tile and walks every diagonal that can touch them, BT rows
//    in registers, no cross-warp reduction; SPLIT (small batch) — the 8 warps
//    (and, via grid.z, several CTAs) split the diagonal list of one 128-position
//    tile and reduce in a fixed order (deterministic), so B = 1 fills 148 SMs.
//  * dW: a CTA owns 256 positions x 64 consecutive diagonals; because offsets
//    ascend, the tile reads one short circular window of each Aop row.  Row
//    chunks stream through a two-stage TMA/mbarrier pipeline.
//  Shared-memory delivery (128 B/clk/SM, profiles/r01_microbench_fma_lds.txt)
//  bounds every FMA that needs a fresh gathered operand at 32 fp32 FMA/clk/SM.
#include "common.cuh"

namespace diagmm {

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / kWarp;
constexpr int kWarpPos = 128;              // positions per warp
constexpr int kU = kWarpPos / kWarp;       // positions per lane
constexpr int kHalo = 128;                 // circular halo after each staged row
constexpr int kWideTile = kWarps * kWarpPos;  // 1024 positions per WIDE CTA
constexpr int kSplitTile = kWarpPos;          // 128 positions per SPLIT CTA

// Row stride (elements) of a staged tile holding `cols` columns: 16-byte multiple.
template <typename T>
__host__ __device__ inline int row_stride(int cols) {
  constexpr int v = 16 / sizeof(T);
  return (cols + v - 1) / v * v;
}

// Stage rows [b0, b0+nb) of a row-major (B, W) matrix into dst (row stride rs):
// columns [0, W) followed by `halo` columns taken circularly from column 0.
// TMA bulk copies when aligned (one elected thread), else a coalesced loop.
template <typename T>
__device__ __forceinline__ void stage_rows(T* __restrict__ dst, int rs, const T* __restrict__ src, int b0,
                                           int nb, int B, int W, int halo, bool bulk, uint64_t* bar) {
  if (bulk) {
    if (threadIdx.x == 0) {
      uint32_t bytes = 0;
      const int hv = halo < W ? halo : 0;
      for (int b = 0; b < nb && b0 + b < B; ++b) bytes += (uint32_t)((W + hv) * sizeof(T));
      mbar_expect_tx(bar, bytes);
      for (int b = 0; b < nb && b0 + b < B; ++b) {
        const T* row = src + (size_t)(b0 + b) * W;
        bulk_g2s(dst + (size_t)b * rs, row, (uint32_t)(W * sizeof(T)), bar);
        if (hv) bulk_g2s(dst + (size_t)b * rs + W, row, (uint32_t)(hv * sizeof(T)), bar);
      }
    }
    for (int b = B - b0; b < nb; ++b)  // rows past the batch: zeros
      for (int c = threadIdx.x; c < W + halo; c += blockDim.x) dst[(size_t)b * rs + c] = T(0);
  } else {
    for (int b = 0; b < nb; ++b) {
      const bool in = b0 + b < B;
      const T* row = src + (size_t)(b0 + b) * W;
      for (int c = threadIdx.x; c < W + halo; c += blockDim.x) {
        int cc = c;
        while (cc >= W) cc -= W;
        dst[(size_t)b * rs + c] = in ? row[cc] : T(0);
      }
    }
  }
}

// Diagonal range touching positions [p0, p0+n) in the S form: o in cyclic
// [p0 - L + 1, p0 + n - 1] -> up to two ranges of the ascending active list.
__device__ __forceinline__ void scatter_ranges(const int32_t* active, int n_act, int C, int L, int p0, int n,
                                               int& lo1, int& hi1, int& lo2, int& hi2) {
  lo1 = 0; hi1 = n_act; lo2 = 0; hi2 = 0;
  if (L + n - 1 >= C) return;
  const int lo = p0 - L + 1, hi = p0 + n - 1;
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

// --------------------------------------------------------------------------- K1/K2
// GATHER: out width L (positions t), in width C, staged columns C + halo.
// !GATHER: out width C (positions r), in width L, staged columns L.
template <typename T, int BT, bool GATHER, bool WIDE>
__global__ void __launch_bounds__(kThreads, 2)
k_product(int B, int C, int L, const T* __restrict__ in, const typename Traits<T>::P* __restrict__ vals,
          const double* __restrict__ asoft, const int32_t* __restrict__ active,
          const int32_t* __restrict__ n_act_p, int max_act, const typename Traits<T>::P* __restrict__ bias,
          T* __restrict__ out, typename Traits<T>::A* __restrict__ part, int nsplit, int bulk) {
  using A = typename Traits<T>::A;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  T* xs = reinterpret_cast<T*>(smem + 128);
  A* red = reinterpret_cast<A*>(smem + 128);  // SPLIT: reused after the main loop
  const int n_act = min(*n_act_p, max_act);
  const int in_w = GATHER ? C : L;
  const int out_w = GATHER ? L : C;
  const int halo = GATHER ? kHalo : 0;
  const int rs = row_stride<T>(in_w + halo);
  constexpr int TT = WIDE ? kWideTile : kSplitTile;
  const int t0 = blockIdx.x * TT;
  const int b0 = blockIdx.y * BT;
  const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;
  const int p0 = WIDE ? t0 + warp * kWarpPos : t0;  // this warp's first position

  if (bulk && threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  stage_rows<T>(xs, rs, in, b0, BT, B, in_w, halo, bulk != 0, bar);

  int lo1, hi1, lo2, hi2;
  if (GATHER) { lo1 = 0; hi1 = n_act; lo2 = 0; hi2 = 0; }
  else scatter_ranges(active, n_act, C, L, p0, kWarpPos, lo1, hi1, lo2, hi2);
  const int len1 = hi1 - lo1, total = len1 + (hi2 - lo2);
  int vb, stride, nq;
  if (WIDE) {
    vb = 0; stride = 1;
    nq = p0 < out_w ? total : 0;
  } else {
    const int per = (total + nsplit - 1) / nsplit;
    const int cb = min(total, (int)blockIdx.z * per), ce = min(total, cb + per);
    vb = cb + warp; stride = kWarps;
    nq = ce - vb > 0 ? (ce - vb + kWarps - 1) / kWarps : 0;
  }
  __syncthreads();
  if (bulk) mbar_wait(bar, 0);

  A acc[BT][kU];
#pragma unroll
  for (int b = 0; b < BT; ++b)
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[b][u] = A(0);

  int o_cache = 0;
  A s_cache = A(0);
  auto fill = [&](int q0) {
    if (q0 + lane < nq) {
      const int v = vb + stride * (q0 + lane);
      const int j = v < len1 ? lo1 + v : lo2 + (v - len1);
      o_cache = active[j];
      s_cache = asoft ? (A)asoft[o_cache] : A(1);
    }
  };
  auto fetch = [&](int o, A s, A (&vv)[kU], int (&ci)[kU]) {
    int base = o + p0;
    base = base >= C ? base - C : base;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = p0 + lane + kWarp * u;
      if (GATHER) {
        const bool ok = p < L;
        vv[u] = ok ? s * (A)__ldg(vals + (size_t)o * L + p) : A(0);
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
    fetch(__shfl_sync(0xffffffffu, o_cache, 0), __shfl_sync(0xffffffffu, s_cache, 0), vcur, ccur);
  }
  for (int q = 0; q < nq; ++q) {
    if (q + 1 < nq) {
      const int qn = q + 1;
      if ((qn & (kWarp - 1)) == 0) fill(qn);
      fetch(__shfl_sync(0xffffffffu, o_cache, qn & (kWarp - 1)),
            __shfl_sync(0xffffffffu, s_cache, qn & (kWarp - 1)), vnxt, cnxt);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const T* xp = xs + ccur[u];
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b][u] = fma(vcur[u], to_acc<A>(xp[(size_t)b * rs]), acc[b][u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) { vcur[u] = vnxt[u]; ccur[u] = cnxt[u]; }
  }

  if (WIDE) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = p0 + lane + kWarp * u;
      if (p >= out_w) continue;
      const A bb = bias ? (A)bias[p] : A(0);
#pragma unroll
      for (int b = 0; b < BT; ++b)
        if (b0 + b < B) out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(acc[b][u] + bb);
    }
    return;
  }
  // SPLIT: fixed-order cross-warp reduction through shared memory
  __syncthreads();
#pragma unroll
  for (int b = 0; b < BT; ++b)
#pragma unroll
    for (int u = 0; u < kU; ++u) red[((size_t)warp * BT + b) * kWarpPos + lane + kWarp * u] = acc[b][u];
  __syncthreads();
  for (int i = threadIdx.x; i < BT * kWarpPos; i += kThreads) {
    const int b = i / kWarpPos, tt = i - b * kWarpPos;
    const int p = t0 + tt;
    if (b0 + b >= B || p >= out_w) continue;
    A s = A(0);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[((size_t)w * BT + b) * kWarpPos + tt];
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
constexpr int kDwPosWarps = 2;                         // warps along positions
constexpr int kDwTile = kDwPosWarps * kWarpPos;        // 256 positions per CTA
constexpr int kDwGroups = kWarps / kDwPosWarps;        // 4 diagonal groups
template <typename T> struct DwRows;
template <> struct DwRows<double> { static constexpr int RB = 4; };
template <> struct DwRows<float> { static constexpr int RB = 4; };
template <> struct DwRows<__nv_bfloat16> { static constexpr int RB = 8; };
constexpr int kJW = 16;                                // diagonals per warp
constexpr int kDwJ = kDwGroups * kJW;                  // 64 diagonals per CTA

struct DwStage {  // per-stage layout offsets (bytes, from the stage base)
  int a_off, b_off, bytes;
};

template <typename T>
__host__ __device__ inline DwStage dw_stage(int win_cap) {
  constexpr int RB = DwRows<T>::RB;
  DwStage s;
  s.a_off = 0;
  s.b_off = (int)align16((size_t)RB * row_stride<T>(win_cap) * sizeof(T));
  s.bytes = s.b_off + (int)align16((size_t)RB * kDwTile * sizeof(T));
  return s;
}

// CTA: kDwTile positions x kDwJ diagonals x one batch part.  Warp w: positions
// t0 + (w % 2)*128 + lane + 32u, diagonals j0 + (w / 2)*kJW + q.
template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
k_dw(int B, int C, int L, const T* __restrict__ aop, const T* __restrict__ bop,
     const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act, int win_cap,
     int rows_per_part, typename Traits<T>::A* __restrict__ partial, int bulk) {
  using A = typename Traits<T>::A;
  constexpr int RB = DwRows<T>::RB;
  constexpr int V = 16 / sizeof(T);  // elements per 16 bytes
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // 2 stages
  unsigned char* stage_base = smem + 128;
  const DwStage L_ = dw_stage<T>(win_cap);
  const int n_act = min(*n_act_p, max_act);
  const int j0 = blockIdx.y * kDwJ;
  if (j0 >= n_act) return;
  const int nj = min(kDwJ, n_act - j0);
  const int t0 = blockIdx.x * kDwTile;
  const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;
  const int pw = warp % kDwPosWarps, grp = warp / kDwPosWarps;
  const int pbase = pw * kWarpPos;
  const int tcols = min(kDwTile, L - t0);
  const int o_first = active[j0], o_last = active[j0 + nj - 1];
  // Aop window: columns (o_first + t0) .. (o_last + t0 + kDwTile - 1), circular
  int ws = o_first + t0;
  ws = ws >= C ? ws - C : ws;
  const int aws = bulk ? ws / V * V : ws;  // 16-byte aligned start for TMA
  const int lead = ws - aws;
  // staged columns, a whole number of 16-byte units (TMA sizes are multiples of 16 B)
  const int wcols = (o_last - o_first + kDwTile + lead + V - 1) / V * V;
  const bool direct = wcols > win_cap;  // window too wide for smem: read Aop from global
  const int ars = row_stride<T>(win_cap);
  int oq[kJW];
#pragma unroll
  for (int q = 0; q < kJW; ++q) {
    const int j = j0 + grp * kJW + q;
    oq[q] = j < j0 + nj ? active[j] : -1;
  }
  A acc[kJW][kU];
#pragma unroll
  for (int q = 0; q < kJW; ++q)
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[q][u] = A(0);

  const int rb = blockIdx.z * rows_per_part, re = min(B, rb + rows_per_part);
  const int nchunks = re > rb ? (re - rb + RB - 1) / RB : 0;
  if (bulk && threadIdx.x == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); }
  __syncthreads();

  // issue chunk c into stage (c & 1)
  auto issue = [&](int c) {
    unsigned char* base = stage_base + (size_t)(c & 1) * L_.bytes;
    T* as = reinterpret_cast<T*>(base + L_.a_off);
    T* bs = reinterpret_cast<T*>(base + L_.b_off);
    const int r0 = rb + c * RB;
    const int nr = min(RB, re - r0);
    if (bulk) {
      if (threadIdx.x == 0) {
        fence_proxy_async();
        uint32_t bytes = 0;
        // window [aws, aws + wcols) circularly: at most two linear pieces, both
        // multiples of V because C, aws and wcols are (wcols <= win_cap <= C)
        const int seg1 = direct ? 0 : min(wcols, C - aws);
        const int seg2r = direct ? 0 : wcols - seg1;
        const int bcols = (tcols + V - 1) / V * V;
        bytes = (uint32_t)nr * (uint32_t)((seg1 + seg2r + bcols) * sizeof(T));
        mbar_expect_tx(&bars[c & 1], bytes);
        for (int r = 0; r < nr; ++r) {
          const T* arow = aop + (size_t)(r0 + r) * C;
          if (seg1) bulk_g2s(as + (size_t)r * ars, arow + aws, (uint32_t)(seg1 * sizeof(T)), &bars[c & 1]);
          if (seg2r) bulk_g2s(as + (size_t)r * ars + seg1, arow, (uint32_t)(seg2r * sizeof(T)), &bars[c & 1]);
          bulk_g2s(bs + (size_t)r * kDwTile, bop + (size_t)(r0 + r) * L + t0, (uint32_t)(bcols * sizeof(T)),
                   &bars[c & 1]);
        }
      }
    } else {
      for (int r = 0; r < RB; ++r) {
        const bool in = r < nr;
        if (!direct)
          for (int i = threadIdx.x; i < wcols; i += kThreads) {
            int cc = aws + i;
            while (cc >= C) cc -= C;
            as[(size_t)r * ars + i] = in ? aop[(size_t)(r0 + r) * C + cc] : T(0);
          }
        for (int i = threadIdx.x; i < kDwTile; i += kThreads)
          bs[(size_t)r * kDwTile + i] = (in && i < tcols) ? bop[(size_t)(r0 + r) * L + t0 + i] : T(0);
      }
    }
  };

  if (nchunks > 0) issue(0);
  for (int c = 0; c < nchunks; ++c) {
    __syncthreads();  // stage (c+1)&1 is free (its previous chunk was consumed)
    if (c + 1 < nchunks) issue(c + 1);
    if (bulk) mbar_wait(&bars[c & 1], (c >> 1) & 1);
    else __syncthreads();
    const unsigned char* base = stage_base + (size_t)(c & 1) * L_.bytes;
    const T* as = reinterpret_cast<const T*>(base + L_.a_off);
    const T* bs = reinterpret_cast<const T*>(base + L_.b_off);
    const int r0 = rb + c * RB;
    const int nr = min(RB, re - r0);
#pragma unroll 1
    for (int r = 0; r < nr; ++r) {
      A bm[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) bm[u] = to_acc<A>(bs[(size_t)r * kDwTile + pbase + lane + kWarp * u]);
      if (!direct) {
        const T* arow = as + (size_t)r * ars + lead + pbase + lane;
#pragma unroll
        for (int q = 0; q < kJW; ++q) {
          if (oq[q] < 0) continue;
          const T* ap = arow + (oq[q] - o_first);
#pragma unroll
          for (int u = 0; u < kU; ++u) acc[q][u] = fma(to_acc<A>(ap[kWarp * u]), bm[u], acc[q][u]);
        }
      } else {
        const T* arow = aop + (size_t)(r0 + r) * C;
#pragma unroll
        for (int q = 0; q < kJW; ++q) {
          if (oq[q] < 0) continue;
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            int col = oq[q] + t0 + pbase + lane + kWarp * u;
            col = col >= C ? col - C : col;
            col = col >= C ? col - C : col;
            acc[q][u] = fma(to_acc<A>(__ldg(arow + col)), bm[u], acc[q][u]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kJW; ++q) {
    const int j = j0 + grp * kJW + q;
    if (oq[q] < 0) continue;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = t0 + pbase + lane + kWarp * u;
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
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

struct ProductPlan {
  int bt, gx, gy, nsplit;
  bool wide;
  size_t smem;
};

template <typename T>
static size_t product_smem(bool wide, int bt, int cols) {
  using A = typename Traits<T>::A;
  const size_t tile = (size_t)bt * row_stride<T>(cols) * sizeof(T);
  const size_t red = wide ? 0 : (size_t)kWarps * bt * kWarpPos * sizeof(A);
  return 128 + align16(tile > red ? tile : red);
}

template <typename T>
static ProductPlan plan_product(int B, int out_w, int cols, int max_act) {
  const size_t kSmem2 = 113 * 1024, kSmem1 = 220 * 1024;
  const int sms = num_sms();
  // WIDE: the largest row tile whose grid still covers the SMs
  const int wide_bt[3] = {sizeof(T) == 8 ? 8 : 16, sizeof(T) == 8 ? 4 : 8, sizeof(T) == 8 ? 2 : 4};
  const int gxw = ceil_div(out_w, kWideTile);
  for (size_t cap : {kSmem2, kSmem1}) {
    for (int bt : wide_bt) {
      const size_t sm = product_smem<T>(true, bt, cols);
      if (sm > cap) continue;
      const long long ctas = (long long)gxw * ceil_div(B, bt);
      if (ctas >= sms) return {bt, gxw, ceil_div(B, bt), 1, true, sm};
    }
  }
  // SPLIT: small batches; diagonals split across warps and across CTAs
  const int split_bt[3] = {8, 4, 1};
  ProductPlan p{0, 0, 0, 1, false, 0};
  for (int bt : split_bt) {
    const size_t sm = product_smem<T>(false, bt, cols);
    if (sm > kSmem1) continue;
    p = {bt, ceil_div(out_w, kSplitTile), ceil_div(B, bt), 1, false, sm};
    if (bt <= B) break;
  }
  if (p.bt == 0) return p;
  const long long ctas = (long long)p.gx * p.gy;
  if (ctas < 2LL * sms) {
    const int ns = (int)ceil_div(2LL * sms, ctas);
    const int max_ns = max_act / 16 > 1 ? max_act / 16 : 1;
    p.nsplit = ns < max_ns ? ns : max_ns;
  }
  return p;
}

template <typename T, int BT, bool G, bool W>
static void launch_product(const ProductPlan& p, cudaStream_t st, int B, int C, int L, const T* in,
                           const typename Traits<T>::P* vals, const double* asoft, const int32_t* active,
                           const int32_t* n_act, int max_act, const typename Traits<T>::P* bias, T* out,
                           typename Traits<T>::A* part, int bulk) {
  auto k = k_product<T, BT, G, W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  k<<<dim3(p.gx, p.gy, p.nsplit), kThreads, p.smem, st>>>(B, C, L, in, vals, asoft, active, n_act, max_act,
                                                          bias, out, part, p.nsplit, bulk);
  note_launch();
}

template <typename T>
size_t product_workspace(bool gather, int B, int C, int L, int max_act) {
  using A = typename Traits<T>::A;
  const int out_w = gather ? L : C, cols = gather ? C + kHalo : L;
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
  const int out_w = gather ? L : C, in_w = gather ? C : L;
  const int cols = in_w + (gather ? kHalo : 0);
  ProductPlan p = plan_product<T>(B, out_w, cols, max_act);
  if (p.bt == 0) return DIAGMM_ETOOLARGE;
  if (p.nsplit > 1 && (ws == nullptr || ws_bytes < (size_t)p.nsplit * B * out_w * sizeof(A))) p.nsplit = 1;
  const int bulk = ((size_t)in_w * sizeof(T)) % 16 == 0 && aligned16(in) && (!gather || in_w >= kHalo);
  auto tin = static_cast<const T*>(in);
  auto tv = static_cast<const P*>(vals);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
  auto part = static_cast<A*>(ws);
#define DIAGMM_GO(BT, W)                                                                                     \
  if (p.bt == BT && p.wide == W) {                                                                           \
    if (gather)                                                                                              \
      launch_product<T, BT, true, W>(p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to, part, bulk);  \
    else                                                                                                     \
      launch_product<T, BT, false, W>(p, st, B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to, part, bulk); \
  }
  if constexpr (sizeof(T) == 8) {
    DIAGMM_GO(8, true) DIAGMM_GO(4, true) DIAGMM_GO(2, true)
  } else {
    DIAGMM_GO(16, true) DIAGMM_GO(8, true) DIAGMM_GO(4, true)
  }
  DIAGMM_GO(8, false) DIAGMM_GO(4, false) DIAGMM_GO(1, false)
#undef DIAGMM_GO
  if (p.nsplit > 1) {
    const size_t n = (size_t)B * out_w;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    k_split_reduce<T><<<blocks, 256, 0, st>>>(B, out_w, p.nsplit, part, tb, to);
    note_launch();
  }
  return status_from_cuda();
}

// ---- dW
template <typename T>
static int dw_win_cap(int C, int max_act) {
  constexpr int V = 16 / sizeof(T);
  const double span = max_act > 0 ? (double)kDwJ * C / max_act : (double)C;
  int cap = (int)(kDwTile + 2.5 * span) + 2 * V;
  cap = cap < C ? cap : C;
  // keep two stages within the shared-memory budget
  while (cap > kDwTile && 128 + 2 * (size_t)dw_stage<T>(cap).bytes > 200 * 1024) cap -= 64;
  return cap;
}

static void dw_parts(int B, int L, int max_act, int rb, int* parts, int* rows_per_part) {
  const long long tiles = (long long)ceil_div(L, kDwTile) * ceil_div(max_act > 0 ? max_act : 1, kDwJ);
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
  size_t w = dw > prod_f ? dw : prod_f;
  return w > prod_b ? w : prod_b;
}

template <typename T>
int run_dw(int M, int N, int B, const void* dy, const void* x, const void* vals, const double* asoft,
           const int32_t* active, const int32_t* slot, const int32_t* n_act, int max_act, void* g_values,
           double* g_soft, void* g_bias, void* ws, size_t ws_bytes, cudaStream_t st) {
  using P = typename Traits<T>::P;
  using A = typename Traits<T>::A;
  constexpr int RB = DwRows<T>::RB;
  constexpr int V = 16 / sizeof(T);
  const int C = M > N ? M : N, L = M < N ? M : N;
  if (ws_bytes < dw_workspace<T>(M, N, B, max_act)) return DIAGMM_EWORKSPACE;
  int parts, rpp;
  dw_parts(B > 0 ? B : 1, L, max_act, RB, &parts, &rpp);
  A* partial = static_cast<A*>(ws);
  const bool tall = M >= N;
  const T* aop = static_cast<const T*>(tall ? dy : x);
  const T* bop = static_cast<const T*>(tall ? x : dy);
  if (B > 0 && max_act > 0) {
    const int cap = dw_win_cap<T>(C, max_act);
    const size_t sm = 128 + 2 * (size_t)dw_stage<T>(cap).bytes;
    const int bulk = C % V == 0 && L % V == 0 && aligned16(aop) && aligned16(bop);
    auto k = k_dw<T>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid(ceil_div(L, kDwTile), ceil_div(max_act, kDwJ), parts);
    k<<<grid, kThreads, sm, st>>>(B, C, L, aop, bop, active, n_act, max_act, cap, rpp, partial, bulk);
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

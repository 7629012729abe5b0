// topk_kernels.cu — on-device float64 diagonal (re)selection (K4/K5).
//
// K4 restates the capped water-filling soft TopK of selection.py:100-142 and
// the active-set rule of layers.py:234; K5 restates soft_topk_grad
// (selection.py:145-173) with the l1 penalty gradient (selection.py:217-222)
// fused in.  select_hard restates selection.py:176-186.
//
// One CTA of 1024 threads per call (C <= 8192 candidates): a bitonic sort of
// (key desc, index asc) pairs reproduces numpy's stable argsort(-z) order
// exactly (ties -> smaller index; -0.0 == +0.0 compare equal, so they tie as in
// numpy).  The tail log-sum-exp that the reference accumulates sequentially
// with np.logaddexp (selection.py:112) is computed here as
//   S_i = z_i + log1p(R_i),   R_i = sum_{l>i} exp(z_l - z_i),
//   R_i = a_i (1 + R_{i+1}),  a_i = exp(z_{i+1} - z_i) in (0, 1],
// a linear recurrence evaluated by a parallel suffix scan of affine maps.
// Every quantity stays finite at arbitrarily cold temperatures (a_i -> 0), the
// same guarantee the reference gets from logaddexp.  S_i agrees with the
// reference's to a few ulp; the clamp/active decisions compare against 1.0
// and 1e-3 with margins many orders of magnitude larger (SURVEY §7 hard part
// 3), and the tests check the masks bit-for-bit.
#include "common.cuh"
#include <math_constants.h>
#include <type_traits>
#include <cstdlib>

namespace diagmm {

constexpr int kSelThreads = 1024;
constexpr int kSelMaxC = 8192;

// numpy orders -0.0 and +0.0 as equal (stable sort keeps index order); make
// that explicit so no comparison can separate them.
__device__ __forceinline__ double canon(double v) { return v == 0.0 ? 0.0 : v; }

// Written as explicit early returns: nvcc 12.9 -O3 dropped the index tie-break
// from the equivalent one-line `ka > kb || (!(ka < kb) && !(ka > kb) && ia < ib)`
// (SASS had no index compare; tools/debug_sort.cu reproduces it).
__device__ __forceinline__ bool before(double ka, int ia, double kb, int ib) {
  if (ka > kb) return true;
  if (ka < kb) return false;
  return ia < ib;
}

// Bitonic sort of NP (power of two) (key, idx) pairs so that position 0 holds
// the largest key (smallest index among equal keys).
__device__ void bitonic_sort_desc(double* key, int* idx, int NP) {
  for (int k = 2; k <= NP; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < NP; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double ka = key[i], kb = key[ixj];
          const int ia = idx[i], ib = idx[ixj];
          const bool up = (i & k) == 0;
          const bool swap = up ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
          if (swap) {
            key[i] = kb; key[ixj] = ka;
            idx[i] = ib; idx[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Same ordering, fewer instructions and barriers: every thread holds E = NP / blockDim
// consecutive positions in registers; a compare-exchange stage whose partner distance j
// is below E stays inside the thread, below 32E it is a warp shuffle, and only the
// j >= 32E stages (15 of the 78 at NP = 4096) go through shared memory with barriers.
// The result is the unique (key desc, index asc) order, identical to bitonic_sort_desc.
template <int E>
__device__ void sort_desc_regs(double* key, int* idx, int NP) {
  const int t = threadIdx.x;
  double kr[E];
  int ir[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    kr[e] = key[t * E + e];
    ir[e] = idx[t * E + e];
  }
  for (int k = 2; k <= NP; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < E) {
        // in-thread pairs (e, e ^ j); j is a power of two below E, dispatched to a
        // compile-time distance so the arrays stay in registers
        auto local = [&](auto J) {
          constexpr int JJ = decltype(J)::value;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int f = e ^ JJ;
            if (f > e) {
              const bool up = ((t * E + e) & k) == 0;
              const bool swap = up ? before(kr[f], ir[f], kr[e], ir[e]) : before(kr[e], ir[e], kr[f], ir[f]);
              if (swap) {
                const double tk = kr[e]; kr[e] = kr[f]; kr[f] = tk;
                const int ti = ir[e]; ir[e] = ir[f]; ir[f] = ti;
              }
            }
          }
        };
        if (j == 1) local(std::integral_constant<int, 1>{});
        else if (j == 2) local(std::integral_constant<int, (E > 2 ? 2 : 1)>{});
        else local(std::integral_constant<int, (E > 4 ? 4 : 1)>{});
      } else if (j < 32 * E) {
        const int lm = j / E;
        const bool lower = (t & lm) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double pk = __shfl_xor_sync(0xffffffffu, kr[e], lm);
          const int pi = __shfl_xor_sync(0xffffffffu, ir[e], lm);
          const bool up = ((t * E + e) & k) == 0;
          const bool mine_first = before(kr[e], ir[e], pk, pi);
          // the lower position of an ascending ("up") pair keeps the element that comes first
          const bool keep_mine = (lower == up) ? mine_first : !mine_first;
          if (!keep_mine) { kr[e] = pk; ir[e] = pi; }
        }
      } else {
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) { key[t * E + e] = kr[e]; idx[t * E + e] = ir[e]; }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = t * E + e, q = p ^ j;
          const double pk = key[q];
          const int pi = idx[q];
          const bool up = (p & k) == 0, lower = p < q;
          const bool mine_first = before(kr[e], ir[e], pk, pi);
          const bool keep_mine = (lower == up) ? mine_first : !mine_first;
          if (!keep_mine) { kr[e] = pk; ir[e] = pi; }
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) { key[t * E + e] = kr[e]; idx[t * E + e] = ir[e]; }
  __syncthreads();
}

// key / idx: NP (power of two) entries in shared memory, sorted in place
__device__ void sort_desc(double* key, int* idx, int NP) {
  const int nt = blockDim.x;
  if (nt == 1024 && NP == 1024) sort_desc_regs<1>(key, idx, NP);
  else if (nt == 1024 && NP == 2048) sort_desc_regs<2>(key, idx, NP);
  else if (nt == 1024 && NP == 4096) sort_desc_regs<4>(key, idx, NP);
  else if (nt == 1024 && NP == 8192) sort_desc_regs<8>(key, idx, NP);
  else bitonic_sort_desc(key, idx, NP);
}

__device__ __forceinline__ int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Exclusive prefix sum of one int per thread over the block: warp shuffles, the
// warp totals scanned by warp 0, 3 barriers (integer: exact in any order).
__device__ int block_exclusive_scan(int v, int* buf, int* total) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = (blockDim.x + 31) >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) buf[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int t = lane < nw ? buf[lane] : 0;
    int ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < nw) buf[32 + lane] = ti - t;  // exclusive warp bases
    if (lane == 31) buf[64] = ti;
  }
  __syncthreads();
  const int r = buf[32 + w] + inc - v;
  *total = buf[64];
  __syncthreads();
  return r;
}

// Compact the flagged indices (flag[i] != 0, i < C) into `out` ascending.
__device__ void compact_flags(const unsigned char* flag, int C, int32_t* out, int32_t* slot,
                              int32_t* n_out, int* scan_buf) {
  const int per = (C + blockDim.x - 1) / blockDim.x;
  const int lo = min(C, (int)threadIdx.x * per), hi = min(C, lo + per);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += flag[i] ? 1 : 0;
  int total = 0;
  int pos = block_exclusive_scan(cnt, scan_buf, &total);
  for (int i = lo; i < hi; ++i) {
    if (flag[i]) {
      if (out) out[pos] = i;
      if (slot) slot[i] = pos;
      ++pos;
    } else if (slot) {
      slot[i] = -1;
    }
  }
  if (n_out && threadIdx.x == 0) *n_out = total;
}

struct Affine { double a, b; };  // x -> a*x + b
__device__ __forceinline__ Affine compose(Affine f, Affine g) {  // f o g
  return {f.a * g.a, f.a * g.b + f.b};
}

// Deterministic block reductions over per-thread partials: a fixed shuffle
// tree inside each warp, then warp 0 folds the 32 warp results (2 barriers).
__device__ double block_reduce_sum(double v, double* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) buf[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < (int)(blockDim.x >> 5) ? buf[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0) buf[32] = r;
  }
  __syncthreads();
  r = buf[32];
  __syncthreads();
  return r;
}
__device__ double block_reduce_max(double v, double* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) buf[w] = v;
  __syncthreads();
  double r = -CUDART_INF;
  if (w == 0) {
    r = lane < (int)(blockDim.x >> 5) ? buf[lane] : -CUDART_INF;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (lane == 0) buf[32] = r;
  }
  __syncthreads();
  r = buf[32];
  __syncthreads();
  return r;
}

// ---- K4 through a radix select (k < C, k <= 1024): only the top-k need an order.
// The reference's tail log-sum-exp over sorted positions i < k splits into the
// top-k part (a suffix scan over the k sorted keys) and the rest, which enters
// only through R_k = sum_{l > k} exp(z_l - z_k) at the (k+1)-th largest key z_k
// (a fixed-order block reduction).  Soft scores of every candidate are
// (k - m) exp(z_i - S_m) or 1 (the top m), so the rest never needs sorting.
// The k-th largest key comes from 8 MSB-first 8-bit histogram passes over
// order-preserving 64-bit keys; ties at it are taken in index order (numpy's
// stable argsort).  Same decisions as the full sort (tests: masks bit-exact vs
// the golden vectors and the oracle); S differs from the full-sort path's in the
// last ulps only (different summation tree for the tail).

// larger double -> larger unsigned key (z canon'd: no -0.0)
__device__ __forceinline__ unsigned long long okey(double z) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(z);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ int block_reduce_min_int(int v, double* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  int* ib = reinterpret_cast<int*>(buf);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) ib[w] = v;
  __syncthreads();
  if (w == 0) {
    int r = lane < (int)(blockDim.x >> 5) ? ib[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r = min(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (lane == 0) ib[32] = r;
  }
  __syncthreads();
  const int r = ib[32];
  __syncthreads();
  return r;
}

// key: z in index order (C); skey / sidx: >= next_pow2(k) scratch entries;
// buf: >= 66 doubles; ibuf: blockDim ints.  Writes asoft / clamped / key (= scores).
__device__ void waterfill_radix(int C, int k, double* key, double* skey, int* sidx, Affine* maps, double* buf,
                                int* ibuf, double* __restrict__ asoft, uint8_t* __restrict__ clamped) {
  __shared__ int s_b, s_need, s_m;
  __shared__ double s_Sm;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (C + nt - 1) / nt;
  const int lo = min(C, tid * per), hi = min(C, lo + per);
  // ---- radix select of the k-th largest key
  unsigned long long prefix = 0;
  int need = k;
  // two histograms used alternately: a pass zeroes the next pass's while it counts (2 barriers a pass)
  if (tid < 256) ibuf[tid] = 0;
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    int* hist = ibuf + (pass & 1) * 256;
    if (tid < 256) ibuf[((pass + 1) & 1) * 256 + tid] = 0;
    // warp-aggregated: keys of similar magnitude share their top bytes, so most of
    // a warp hits one bin (one atomic per distinct digit per warp instead)
    for (int e = 0; e < per; ++e) {
      const int i = lo + e;
      int digit = -1;
      if (i < hi) {
        const unsigned long long u = okey(key[i]);
        if (pass == 0 || (u >> (shift + 8)) == prefix) digit = (int)((u >> shift) & 255);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, digit);
      if (digit >= 0 && (tid & 31) == __ffs(peers) - 1) atomicAdd(&hist[digit], __popc(peers));
    }
    __syncthreads();
    if (tid < 32) {  // lane l: bins 255 - 8l .. 248 - 8l, the highest first
      int c[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { c[q] = hist[255 - 8 * tid - q]; sum += c[q]; }
      int inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (tid >= o) inc += v;
      }
      const unsigned ball = __ballot_sync(0xffffffffu, inc >= need);
      if (tid == __ffs(ball) - 1) {
        int cum = inc - sum, b = 255 - 8 * tid;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (cum + c[q] >= need) { b = 255 - 8 * tid - q; break; }
          cum += c[q];
        }
        s_b = b;
        s_need = need - cum;
      }
    }
    __syncthreads();
    prefix = (prefix << 8) | (unsigned long long)s_b;
    need = s_need;
  }
  __syncthreads();  // s_b / s_need / the histograms are reused below
  const unsigned long long ustar = prefix;  // the k-th largest; `need` of its ties are taken, in index order
  // ---- compact the top-k (index order), pad, sort by (key desc, index asc)
  int nties = 0;
  for (int i = lo; i < hi; ++i) nties += okey(key[i]) == ustar ? 1 : 0;
  int tot = 0;
  int tie_rank = block_exclusive_scan(nties, ibuf, &tot);
  int nsel = 0;
  for (int i = lo; i < hi; ++i) {
    const unsigned long long u = okey(key[i]);
    if (u > ustar) ++nsel;
    else if (u == ustar) { if (tie_rank < need) ++nsel; ++tie_rank; }
  }
  tie_rank -= nties;
  int pos = block_exclusive_scan(nsel, ibuf, &tot);
  const int NPk = nt;  // k <= nt: pad to the block width for the register / shuffle sort
  for (int i = lo; i < hi; ++i) {
    const unsigned long long u = okey(key[i]);
    bool take = u > ustar;
    if (u == ustar) { take = tie_rank < need; ++tie_rank; }
    if (take) { skey[pos] = key[i]; sidx[pos] = i; ++pos; }
  }
  tie_rank -= nties;
  for (int p = k + tid; p < NPk; p += nt) { skey[p] = -CUDART_INF; sidx[p] = 0x7fffffff; }
  __syncthreads();
  sort_desc(skey, sidx, NPk);
  // ---- the rest: z_k = its largest key, R_k = sum over the rest but that element
  double zr = -CUDART_INF;
  for (int i = lo; i < hi; ++i) {
    const unsigned long long u = okey(key[i]);
    if (u < ustar || (u == ustar && tie_rank >= need)) zr = fmax(zr, key[i]);
    if (u == ustar) ++tie_rank;
  }
  tie_rank -= nties;
  const double zk = block_reduce_max(zr, buf);
  int first = 0x7fffffff;  // the rest's element at sorted position k: smallest index with key zk
  for (int i = lo; i < hi; ++i) {
    const unsigned long long u = okey(key[i]);
    const bool rest = u < ustar || (u == ustar && tie_rank >= need);
    if (u == ustar) ++tie_rank;
    if (rest && key[i] == zk && first == 0x7fffffff) first = i;
  }
  tie_rank -= nties;
  const int ik = block_reduce_min_int(first, buf);
  double sr = 0.0;
  for (int i = lo; i < hi; ++i) {
    const unsigned long long u = okey(key[i]);
    const bool rest = u < ustar || (u == ustar && tie_rank >= need);
    if (u == ustar) ++tie_rank;
    if (rest && i != ik) sr += exp(key[i] - zk);
  }
  const double Rk = block_reduce_sum(sr, buf);
  // ---- suffix scan over the k sorted positions (one per thread): R_i = a_i (1 + R_{i+1})
  const double zi = tid < k ? skey[tid] : 0.0;
  const double znext = tid + 1 < k ? skey[tid + 1] : zk;
  const double a = tid < k ? exp(znext - zi) : 0.0;
  // inclusive suffix composition F_t o F_{t+1} o ... : shuffles inside each warp, then
  // the warps' totals composed by warp 0 (2 barriers)
  Affine F = tid < k ? Affine{a, a} : Affine{1.0, 0.0};
  const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double na = __shfl_down_sync(0xffffffffu, F.a, o), nb = __shfl_down_sync(0xffffffffu, F.b, o);
    if (lane + o < 32) F = compose(F, Affine{na, nb});
  }
  if (lane == 0) maps[w] = F;  // the whole warp's map
  if (tid == 0) s_m = k;
  __syncthreads();
  if (w == 0) {
    Affine G = lane < nw ? maps[lane] : Affine{1.0, 0.0};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double na = __shfl_down_sync(0xffffffffu, G.a, o), nb = __shfl_down_sync(0xffffffffu, G.b, o);
      if (lane + o < 32) G = compose(G, Affine{na, nb});
    }
    maps[32 + lane] = G;  // composition of warps lane .. nw-1
  }
  __syncthreads();
  if (w + 1 < nw) F = compose(F, maps[32 + w + 1]);
  const double Ri = F.a * Rk + F.b;
  // ---- clamp count m = first i < k with (k - i) exp(z_i - S_i) < 1
  double Si = 0.0;
  if (tid < k) {
    Si = zi + log1p(Ri);
    if (!((double)(k - tid) * exp(zi - Si) >= 1.0)) atomicMin(&s_m, tid);
  }
  __syncthreads();
  const int m = s_m;
  if (m < k && tid == m) s_Sm = Si;
  if (m == k && tid == 0) s_Sm = zk + log1p(Rk);
  __syncthreads();
  const double Sm = s_Sm;
  // ---- scores in index order, then the top m clamped to 1
  for (int i = lo; i < hi; ++i) {
    const double v = (double)(k - m) * exp(key[i] - Sm);
    key[i] = v;
    asoft[i] = v;
    if (clamped) clamped[i] = 0;
  }
  __syncthreads();
  if (tid < m) {
    const int o = sidx[tid];
    key[o] = 1.0;
    asoft[o] = 1.0;
    if (clamped) clamped[o] = 1;
  }
  __syncthreads();
}

// Up to kMaxJobs independent selections per launch, one CTA each (all the
// DiagLinear layers of a model re-select in one launch, SURVEY §7 hard part 2).
constexpr int kMaxJobs = 64;
struct WaterfillJobs {
  diagmm_topk_job j[kMaxJobs];
  int radix;  // top-k radix-select path (DIAGMM_K4_RADIX, default on)
};

__global__ void __launch_bounds__(kSelThreads)
k_waterfill(const __grid_constant__ WaterfillJobs jobs) {
  const diagmm_topk_job& J = jobs.j[blockIdx.x];
  // device {T, k} (a CUDA-graph replay of an annealing schedule) or the launch values
  const int C = J.C, k = J.params ? (int)J.params[1] : J.k;
  const double temperature = J.params ? J.params[0] : J.temperature;
  const double* __restrict__ alpha = J.alpha;
  double* __restrict__ asoft = J.alpha_soft;
  uint8_t* __restrict__ clamped = J.clamped;
  int32_t* __restrict__ active = J.active;
  int32_t* __restrict__ slot = J.slot;
  int32_t* __restrict__ n_act = J.n_act;
  extern __shared__ __align__(16) unsigned char smem[];
  const int NP = next_pow2(C);
  const int NPs = NP > kSelThreads ? NP : kSelThreads;  // regions hold the radix path's padded top-k too
  double* key = reinterpret_cast<double*>(smem);                              // NPs
  double* R = key + NPs;                                                      // NPs
  int* idx = reinterpret_cast<int*>(R + NPs);                                 // NPs
  Affine* maps = reinterpret_cast<Affine*>(smem + ((size_t)NPs * 20 + 15) / 16 * 16);  // blockDim
  int* ibuf = reinterpret_cast<int*>(maps + blockDim.x);                      // blockDim
  __shared__ int s_m;
  __shared__ double s_Sm;
  const int tid = threadIdx.x, nt = blockDim.x;

  for (int i = tid; i < NP; i += nt) {
    key[i] = i < C ? canon(alpha[i] / temperature) : -CUDART_INF;
    idx[i] = i < C ? i : 0x7fffffff;
  }
  __syncthreads();
  // sort the top-k only — when the full sort is wider than the block (C > 1024); at
  // C <= 1024 the one-element-per-thread full sort is cheaper (C = 768: 22.6 vs 29 us)
  if (jobs.radix && k < C && k <= nt && nt == kSelThreads && NP > nt) {
    waterfill_radix(C, k, key, R, idx, maps, reinterpret_cast<double*>(maps + 64), ibuf, asoft, clamped);
    unsigned char* flag = reinterpret_cast<unsigned char*>(R);
    for (int i = tid; i < C; i += nt) flag[i] = key[i] >= 1e-3 ? 1 : 0;
    __syncthreads();
    compact_flags(flag, C, active, slot, n_act, ibuf);
    return;
  }
  sort_desc(key, idx, NP);

  // ---- suffix scan of R (positions 0..C-1, chunked per thread)
  const int per = (C + nt - 1) / nt;
  const int lo = min(C, tid * per), hi = min(C, lo + per);
  Affine F{1.0, 0.0};  // identity
  for (int i = hi - 1; i >= lo; --i) {
    Affine f = (i + 1 < C) ? Affine{exp(key[i + 1] - key[i]), 0.0} : Affine{0.0, 0.0};
    f.b = f.a;
    F = compose(f, F);
  }
  maps[tid] = F;
  __syncthreads();
  for (int d = 1; d < nt; d <<= 1) {  // inclusive suffix scan: maps[t] = F_t o F_{t+1} o ...
    Affine mine = maps[tid];
    Affine nxt = tid + d < nt ? maps[tid + d] : Affine{1.0, 0.0};
    __syncthreads();
    maps[tid] = compose(mine, nxt);
    __syncthreads();
  }
  double r = tid + 1 < nt ? maps[tid + 1].b : 0.0;  // R at position hi (0 past the end)
  for (int i = hi - 1; i >= lo; --i) {
    const double a = (i + 1 < C) ? exp(key[i + 1] - key[i]) : 0.0;
    r = a * (1.0 + r);
    R[i] = r;
  }
  if (tid == 0) s_m = min(k, C);
  __syncthreads();

  // ---- clamp count m = first i < min(k, C) with (k-i)*exp(z_i - S_i) < 1
  const int lim = min(k, C);
  for (int i = lo; i < min(hi, lim); ++i) {
    const double S = key[i] + log1p(R[i]);
    if (!((double)(k - i) * exp(key[i] - S) >= 1.0)) {
      atomicMin(&s_m, i);
      break;
    }
  }
  __syncthreads();
  const int m = s_m;
  if (m < C && m >= lo && m < hi) s_Sm = key[m] + log1p(R[m]);
  __syncthreads();
  const double Sm = m < C ? s_Sm : 0.0;

  // ---- soft scores at sorted positions, then scatter to index order
  for (int i = lo; i < hi; ++i) R[i] = i < m ? 1.0 : (double)(k - m) * exp(key[i] - Sm);
  __syncthreads();
  for (int i = lo; i < hi; ++i) {
    const int o = idx[i];
    key[o] = R[i];
    asoft[o] = R[i];
    if (clamped) clamped[o] = i < m ? 1 : 0;
  }
  __syncthreads();
  // ---- active set: flatnonzero(alpha_soft >= 1e-3)
  unsigned char* flag = reinterpret_cast<unsigned char*>(R);
  for (int i = tid; i < C; i += nt) flag[i] = key[i] >= 1e-3 ? 1 : 0;
  __syncthreads();
  compact_flags(flag, C, active, slot, n_act, ibuf);
}

__global__ void __launch_bounds__(kSelThreads)
k_select_hard(int C, int k, const double* __restrict__ alpha, int32_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int NP = next_pow2(C);
  double* key = reinterpret_cast<double*>(smem);
  int* idx = reinterpret_cast<int*>(key + NP);
  unsigned char* flag = reinterpret_cast<unsigned char*>(idx + NP);
  int* ibuf = reinterpret_cast<int*>(flag + ((NP + 15) & ~15));
  for (int i = threadIdx.x; i < NP; i += blockDim.x) {
    key[i] = i < C ? canon(alpha[i]) : -CUDART_INF;
    idx[i] = i < C ? i : 0x7fffffff;
  }
  __syncthreads();
  sort_desc(key, idx, NP);
  for (int i = threadIdx.x; i < C; i += blockDim.x) flag[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) flag[idx[i]] = 1;
  __syncthreads();
  compact_flags(flag, C, out, nullptr, nullptr, ibuf);
}

__global__ void __launch_bounds__(kSelThreads)
k_active_from_list(int C, int n, const int32_t* __restrict__ offs, int32_t* __restrict__ slot,
                   int32_t* __restrict__ n_act) {
  for (int i = threadIdx.x; i < C; i += blockDim.x) slot[i] = -1;
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) slot[offs[j]] = j;
  if (threadIdx.x == 0 && n_act) *n_act = n;
}

// Two doubles reduced at once (fixed shuffle tree, then warp 0 over the warp
// results): op 0 sums both, op 1 sums the first and takes the max of the second.
__device__ double2 block_reduce2(double a, double b, bool max_b, double* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    const double y = __shfl_xor_sync(0xffffffffu, b, o);
    b = max_b ? fmax(b, y) : b + y;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) { buf[w] = a; buf[32 + w] = b; }
  __syncthreads();
  if (w == 0) {
    double ra = lane < nw ? buf[lane] : 0.0;
    double rb = lane < nw ? buf[32 + lane] : (max_b ? -CUDART_INF : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ra += __shfl_xor_sync(0xffffffffu, ra, o);
      const double y = __shfl_xor_sync(0xffffffffu, rb, o);
      rb = max_b ? fmax(rb, y) : rb + y;
    }
    if (lane == 0) { buf[64] = ra; buf[65] = rb; }
  }
  __syncthreads();
  const double2 r = make_double2(buf[64], buf[65]);
  __syncthreads();
  return r;
}

// K5 body for one layer (one CTA); shared by the per-layer and the batched kernels.
// Two dependent block reductions: (clamped count, max free z), then (sum q, sum up*q)
// with q = exp(z - zmax) unnormalised; the candidate's alpha / clamped / up stay in
// registers between the passes (C <= 8192: <= 8 per thread).
__device__ void topk_grad_block(int C, int k_arg, double t_arg, const double* __restrict__ alpha,
                                const uint8_t* __restrict__ clamped, const double* __restrict__ up, double l1,
                                double* __restrict__ g_alpha, int accumulate, const double* __restrict__ params,
                                double* smem) {
  constexpr int kPer = kSelMaxC / kSelThreads;
  const int k = params ? (int)params[1] : k_arg;
  const double temperature = params ? params[0] : t_arg;
  double* buf = smem;  // 66 doubles
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (C + nt - 1) / nt;
  const int lo = min(C, tid * per), hi = min(C, lo + per);
  unsigned clm = 0;  // clamped flags of this thread's candidates (alpha / up re-read: L1 hits)
  double ncl = 0.0, zmax = -CUDART_INF;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int i = lo + e;
    if (e < per && i < hi) {
      if (clamped[i]) { clm |= 1u << e; ncl += 1.0; }
      else zmax = fmax(zmax, alpha[i] / temperature);
    }
  }
  const double2 r1 = block_reduce2(ncl, zmax, true, buf);
  const int n_clamped = (int)r1.x;
  zmax = r1.y;
  const int budget = k - n_clamped;
  const bool any_free = n_clamped < C;
  double v[kPer];
  double sq = 0.0, su = 0.0;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int i = lo + e;
    v[e] = 0.0;
    if (e < per && i < hi && !(clm >> e & 1u)) {
      v[e] = exp(alpha[i] / temperature - zmax);
      sq += v[e];
      su += up[i] * v[e];
    }
  }
  const double2 r2 = block_reduce2(sq, su, false, buf);
  const double sum_q = r2.x;
  const double sum_w = r2.y / sum_q;  // = sum up * q with q = v / sum_q
  const double coef = (double)budget / temperature;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int i = lo + e;
    if (!(e < per && i < hi)) continue;
    double g = 0.0;
    if (any_free && budget > 0 && !(clm >> e & 1u)) {
      const double q = v[e] / sum_q;
      g = coef * (up[i] * q - q * sum_w);
    }
    if (l1 != 0.0) {
      const double av = alpha[i];
      g += l1 * (av > 0.0 ? 1.0 : (av < 0.0 ? -1.0 : 0.0));
    }
    g_alpha[i] = accumulate ? g_alpha[i] + g : g;
  }
}

__global__ void __launch_bounds__(kSelThreads)
k_topk_grad(int C, int k_arg, double t_arg, const double* __restrict__ alpha,
            const uint8_t* __restrict__ clamped, const double* __restrict__ up, double l1,
            double* __restrict__ g_alpha, int accumulate, const double* __restrict__ params) {
  extern __shared__ __align__(16) unsigned char smem[];
  topk_grad_block(C, k_arg, t_arg, alpha, clamped, up, l1, g_alpha, accumulate, params,
                  reinterpret_cast<double*>(smem));
}

struct TopkGradJobs { diagmm_topk_grad_job j[kMaxJobs]; };
__global__ void __launch_bounds__(kSelThreads)
k_topk_grad_batched(const __grid_constant__ TopkGradJobs jobs) {
  extern __shared__ __align__(16) unsigned char smem[];
  const diagmm_topk_grad_job& J = jobs.j[blockIdx.x];
  topk_grad_block(J.C, J.k, J.temperature, J.alpha, J.clamped, J.g_soft, J.l1_coeff, J.g_alpha, J.accumulate,
                  J.params, reinterpret_cast<double*>(smem));
}

// ---------------------------------------------------------------- launchers
static size_t waterfill_smem(int C) {
  int NP = kSelThreads;  // at least the radix path's padded top-k (k_waterfill: NPs)
  while (NP < C) NP <<= 1;
  return ((size_t)NP * 20 + 15) / 16 * 16 + kSelThreads * (sizeof(Affine) + sizeof(int)) + 64;
}

static int check_job(const diagmm_topk_job& j) {
  if (j.C < 1) return DIAGMM_ESHAPE;
  if (!(j.temperature > 0.0)) return DIAGMM_ETEMPERATURE;
  if (j.k < 1 || j.k > j.C) return DIAGMM_EK;
  if (j.C > kSelMaxC) return DIAGMM_ETOOLARGE;
  return DIAGMM_OK;
}

int run_waterfill_batched(int n, const diagmm_topk_job* jobs, cudaStream_t st) {
  if (n < 0 || (n > 0 && jobs == nullptr)) return DIAGMM_ESHAPE;
  for (int i = 0; i < n; ++i)
    if (int e = check_job(jobs[i])) return e;
  for (int b = 0; b < n; b += kMaxJobs) {
    const int cnt = n - b < kMaxJobs ? n - b : kMaxJobs;
    WaterfillJobs P{};
    const char* re = getenv("DIAGMM_K4_RADIX");  // read per call (A/B tests flip it)
    P.radix = re ? atoi(re) : 1;
    int cmax = 1;
    for (int i = 0; i < cnt; ++i) {
      P.j[i] = jobs[b + i];
      cmax = P.j[i].C > cmax ? P.j[i].C : cmax;
    }
    const size_t sm = waterfill_smem(cmax);
    cudaFuncSetAttribute(k_waterfill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_waterfill<<<cnt, kSelThreads, sm, st>>>(P);
    note_launch();
  }
  return status_from_cuda();
}

int run_waterfill(int C, int k, double T, const double* alpha, double* asoft, uint8_t* clamped,
                  int32_t* active, int32_t* slot, int32_t* n_act, cudaStream_t st) {
  diagmm_topk_job j{C, k, T, alpha, asoft, clamped, active, slot, n_act, nullptr};
  return run_waterfill_batched(1, &j, st);
}

int run_select_hard(int C, int k, const double* alpha, int32_t* idx, cudaStream_t st) {
  if (C < 1) return DIAGMM_ESHAPE;
  if (k < 1 || k > C) return DIAGMM_EK;
  if (C > kSelMaxC) return DIAGMM_ETOOLARGE;
  int NP = 1;
  while (NP < C) NP <<= 1;
  size_t sm = (size_t)NP * 12 + ((NP + 15) & ~15) + kSelThreads * sizeof(int) + 64;
  cudaFuncSetAttribute(k_select_hard, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_select_hard<<<1, kSelThreads, sm, st>>>(C, k, alpha, idx);
  note_launch();
  return status_from_cuda();
}

int run_active_from_list(int C, int n, const int32_t* offs, int32_t* slot, int32_t* n_act,
                         cudaStream_t st) {
  if (C < 1 || n < 0 || n > C) return DIAGMM_ESHAPE;
  k_active_from_list<<<1, kSelThreads, 0, st>>>(C, n, offs, slot, n_act);
  note_launch();
  return status_from_cuda();
}

int run_topk_grad_batched(int n, const diagmm_topk_grad_job* jobs, cudaStream_t st) {
  if (n < 0) return DIAGMM_ESHAPE;
  for (int i = 0; i < n; ++i) {
    const diagmm_topk_grad_job& j = jobs[i];
    if (j.C < 1) return DIAGMM_ESHAPE;
    if (!(j.temperature > 0.0)) return DIAGMM_ETEMPERATURE;
    if (j.k < 1 || j.k > j.C) return DIAGMM_EK;
    if (j.C > kSelMaxC) return DIAGMM_ETOOLARGE;
  }
  for (int b = 0; b < n; b += kMaxJobs) {
    const int cnt = n - b < kMaxJobs ? n - b : kMaxJobs;
    TopkGradJobs P{};
    int cmax = 1;
    for (int i = 0; i < cnt; ++i) {
      P.j[i] = jobs[b + i];
      cmax = P.j[i].C > cmax ? P.j[i].C : cmax;
    }
    const size_t sm = 66 * sizeof(double);  // block_reduce2 scratch (the values stay in registers)
    cudaFuncSetAttribute(k_topk_grad_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_topk_grad_batched<<<cnt, kSelThreads, sm, st>>>(P);
    note_launch();
  }
  return status_from_cuda();
}

int run_topk_grad(int C, int k, double T, const double* alpha, const uint8_t* clamped,
                  const double* up, double l1, double* g_alpha, int accumulate, const double* params,
                  cudaStream_t st) {
  if (C < 1) return DIAGMM_ESHAPE;
  if (!(T > 0.0)) return DIAGMM_ETEMPERATURE;
  if (k < 1 || k > C) return DIAGMM_EK;
  if (C > kSelMaxC) return DIAGMM_ETOOLARGE;
  const size_t sm = 66 * sizeof(double);
  cudaFuncSetAttribute(k_topk_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_topk_grad<<<1, kSelThreads, sm, st>>>(C, k, T, alpha, clamped, up, l1, g_alpha, accumulate, params);
  note_launch();
  return status_from_cuda();
}

// DiagHeur prune / regrow (layers.py:381-413) on the device, one CTA:
// L2 norms of the k active rows (float64), a stable ascending sort by
// (norm, offset) (np.lexsort((active, norms)), ties -> smaller offset), the
// first n_prune are pruned; the regrown offsets are grow_idx[i]-th entries of
// the ascending list of the offsets inactive BEFORE the swap (numpy's
// rng.choice(pool, n) is pool[rng.choice(len(pool), n)], so the host draws only
// the indices from the reference's RNG stream); their value rows are zeroed,
// and the new active set (sorted survivors + grown) is compacted in place.
template <typename P>
__global__ void __launch_bounds__(kSelThreads)
k_diagheur_update(int C, int L, int k, int32_t* __restrict__ active, int32_t* __restrict__ slot,
                  int32_t* __restrict__ n_act, P* __restrict__ values, int n_prune,
                  const int32_t* __restrict__ grow_idx) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int NP = next_pow2(k);
  double* key = reinterpret_cast<double*>(smem);                          // NP
  int* idx = reinterpret_cast<int*>(key + NP);                            // NP
  int* inact = idx + NP;                                                  // C
  int* ibuf = inact + C;                                                  // blockDim
  unsigned char* flag = reinterpret_cast<unsigned char*>(ibuf + blockDim.x);  // C
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < C; i += blockDim.x) flag[i] = 0;
  for (int i = tid; i < NP; i += blockDim.x) {
    key[i] = -CUDART_INF;
    idx[i] = 0x7fffffff;
  }
  __syncthreads();
  for (int j = tid; j < k; j += blockDim.x) flag[active[j]] = 1;
  // ---- norms of the active rows: one warp per row, fixed lane order + shuffle tree
  for (int j = warp; j < k; j += nw) {
    const int o = active[j];
    const P* row = values + (size_t)o * L;
    double acc = 0.0;
    for (int t = lane; t < L; t += 32) {
      const double v = (double)row[t];
      acc = fma(v, v, acc);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) {
      key[j] = -sqrt(acc);  // descending sort of -norm = ascending norm; ties -> smaller offset
      idx[j] = o;
    }
  }
  __syncthreads();
  sort_desc(key, idx, NP);
  // ---- the pool: offsets inactive before the swap, ascending
  {
    const int per = (C + blockDim.x - 1) / blockDim.x;
    const int lo = min(C, tid * per), hi = min(C, lo + per);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += flag[i] ? 0 : 1;
    int total = 0;
    int pos = block_exclusive_scan(cnt, ibuf, &total);
    for (int i = lo; i < hi; ++i)
      if (!flag[i]) inact[pos++] = i;
  }
  __syncthreads();
  for (int i = tid; i < n_prune; i += blockDim.x) flag[idx[i]] = 0;
  __syncthreads();
  for (int i = tid; i < n_prune; i += blockDim.x) flag[inact[grow_idx[i]]] = 1;
  // regrown rows start from zero (the reference's values[grown] = 0)
  for (int i = warp; i < n_prune; i += nw) {
    P* row = values + (size_t)inact[grow_idx[i]] * L;
    for (int t = lane; t < L; t += 32) row[t] = P(0);
  }
  __syncthreads();
  compact_flags(flag, C, active, slot, n_act, ibuf);
}

template <typename P>
int run_diagheur_update(int C, int L, int k, int32_t* active, int32_t* slot, int32_t* n_act, void* values,
                        int n_prune, const int32_t* grow_idx, cudaStream_t st) {
  if (C < 1 || L < 1 || k < 1 || k > C || n_prune < 0 || n_prune > k || n_prune > C - k) return DIAGMM_ESHAPE;
  if (C > kSelMaxC) return DIAGMM_ETOOLARGE;
  if (n_prune == 0) return DIAGMM_OK;
  int NP = 1;
  while (NP < k) NP <<= 1;
  const size_t sm = (size_t)NP * 12 + (size_t)C * 4 + kSelThreads * 4 + C + 16;
  cudaFuncSetAttribute(k_diagheur_update<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_diagheur_update<P><<<1, kSelThreads, sm, st>>>(C, L, k, active, slot, n_act, static_cast<P*>(values), n_prune,
                                                   grow_idx);
  note_launch();
  return status_from_cuda();
}
template int run_diagheur_update<double>(int, int, int, int32_t*, int32_t*, int32_t*, void*, int, const int32_t*,
                                         cudaStream_t);
template int run_diagheur_update<float>(int, int, int, int32_t*, int32_t*, int32_t*, void*, int, const int32_t*,
                                        cudaStream_t);

}  // namespace diagmm

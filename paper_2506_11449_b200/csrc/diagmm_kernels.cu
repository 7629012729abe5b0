// diagmm_kernels.cu — sm_100a kernels for the DiagLinear products (K1 forward,
// K2 input gradient, K3 per-diagonal weight gradient) and the dense-equivalent
// helpers (materialize / gather of a dense dW).
//
// Exact math (verified against the reference):
//   W is M x N, C = max(M,N), L = min(M,N), active offsets o_j ascending,
//   V[j,t] = s_j * values[o_j, t]  with s_j = alpha_soft[o_j]   (layers.py:235).
//   "gather" form  (G): out[b,t] = sum_j V[j,t] * in[b, (o_j + t) mod C],  t < L
//        = wide forward (diagcore.py:234-237) and tall/square dX (the transpose
//          of diagcore.py:162-191 read "by own index, +o").
//   "scatter" form (S): out[b,r] = sum_j [c=(r-o_j) mod C < L] V[j,c]*in[b,c], r < C
//        = tall/square forward (diagcore.py:230-233) and wide dX.
//   dW: gw[j,t] = sum_b Aop[b,(o_j+t) mod C] * Bop[b,t]   (layers.py:149-158)
//        tall: Aop = dy, Bop = x;   wide: Aop = x, Bop = dy.
//
// Which kernel runs (run_product / run_dw):
//   products  B <= 4: k_product_rows; bf16 B 5..8: k_product_pk (>= 128 diagonals) or
//             k_product_rows; bf16 B >= 32: k_product6 (v6); otherwise k_product (v4)
//   dW        B <= 8: k_dw_narrow; bf16 / fp32 B > 8: k_dw6 (v6); fp64: k_dw (v4)
//
// B200 design (v4):
//  * Every multiply needs a gathered operand at a data-dependent shift, so
//    there is no register reuse of it: each FMA consumes one value read from
//    shared memory, and the 128 B/clk/SM shared-memory crossbar bounds the
//    kernels (profiles/r01_microbench_fhfma_lds.txt).  The kernels are built
//    to sit on that bound with the fewest bytes per FMA:
//  * Activations are staged TRANSPOSED and packed: smem column c of a row group
//    holds VEC = 16/sizeof(T) consecutive batch rows in 16 bytes ([g][col][VEC]).
//    One conflict-free LDS.128 then feeds VEC FMAs that share one weight, for
//    any offset, wrap or alignment.  bf16: 8 rows per LDS.128, fp32: 4, fp64: 2.
//  * bf16 multiplies use FHFMA.BF16 (PTX fma.rn.f32.bf16: bf16 x bf16 + fp32
//    accumulate, halves taken straight from the packed registers — no unpack
//    instructions); weights are pre-scaled once per call into a compact bf16
//    store V (k_prescale, the reference's `weights = alpha_soft * values`).
//  * Lanes own output positions p0 + lane + 32u (u < 4): weight loads are
//    coalesced, the per-diagonal offset list is cached per lane and shuffled
//    out, and the next diagonal's weights are prefetched.
//  * Tilings: WIDE (many rows) — a warp owns 128 positions x (G*VEC) rows and
//    walks every diagonal touching them; SPLIT (few rows) — the warps of a CTA
//    (and several CTAs, grid.z) split the diagonal list of one 128-position
//    tile and reduce in a fixed order (deterministic), so B = 1 fills the GPU.
//  * dW: a CTA owns 256 positions x 64 consecutive diagonals; offsets ascend,
//    so the tile reads one short circular window of each Aop row.  Row chunks
//    are staged (transposed) by 8x8 register transposes; 2+ CTAs per SM
//    overlap one CTA's staging with another's FMAs.
#include "common.cuh"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

namespace diagmm {

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Weight type of the compact pre-scaled store: bf16 activations multiply with
// bf16 weights (FHFMA.BF16, fp32 accumulate); fp32 / fp64 keep their type.
template <typename T> struct WType { using type = T; };

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / kWarp;
constexpr int kWarpPos = 128;              // positions per warp
constexpr int kU = kWarpPos / kWarp;       // positions per lane
constexpr int kHalo = 128;                 // circular halo after each staged gather row

template <typename T> __host__ __device__ constexpr int vec_rows() { return 16 / (int)sizeof(T); }

// ------------------------------------------------------------------ FMA atoms
// acc[r] += x[r] * w for the VEC rows packed in one 16-byte smem unit.
__device__ __forceinline__ void fma_bf16_pair(float& a0, float& a1, uint32_t x, uint32_t w) {
  asm("{\n.reg .b16 x0, x1, w0, w1;\n"
      "mov.b32 {x0, x1}, %2;\n"
      "mov.b32 {w0, w1}, %3;\n"
      "fma.rn.f32.bf16 %0, x0, w0, %0;\n"
      "fma.rn.f32.bf16 %1, x1, w0, %1;\n}"
      : "+f"(a0), "+f"(a1)
      : "r"(x), "r"(w));
}
__device__ __forceinline__ void fma_vec(float (&a)[8], uint4 x, uint32_t w /* bf16 in low half */) {
  fma_bf16_pair(a[0], a[1], x.x, w);
  fma_bf16_pair(a[2], a[3], x.y, w);
  fma_bf16_pair(a[4], a[5], x.z, w);
  fma_bf16_pair(a[6], a[7], x.w, w);
}
__device__ __forceinline__ void fma_vec(float (&a)[4], float4 x, float w) {
  a[0] = fmaf(x.x, w, a[0]);
  a[1] = fmaf(x.y, w, a[1]);
  a[2] = fmaf(x.z, w, a[2]);
  a[3] = fmaf(x.w, w, a[3]);
}
__device__ __forceinline__ void fma_vec(double (&a)[2], double2 x, double w) {
  a[0] = fma(x.x, w, a[0]);
  a[1] = fma(x.y, w, a[1]);
}
// dot-style: acc += sum_r a[r] * b[r] (dW: contraction over the VEC rows)
__device__ __forceinline__ void dot_bf16_pair(float& acc, uint32_t a, uint32_t b) {
  asm("{\n.reg .b16 a0, a1, b0, b1;\n"
      "mov.b32 {a0, a1}, %1;\n"
      "mov.b32 {b0, b1}, %2;\n"
      "fma.rn.f32.bf16 %0, a0, b0, %0;\n"
      "fma.rn.f32.bf16 %0, a1, b1, %0;\n}"
      : "+f"(acc)
      : "r"(a), "r"(b));
}

template <typename T> struct Vec;  // 16-byte smem unit and accumulator shape
template <> struct Vec<__nv_bfloat16> {
  using U = uint4; using A = float; using W = uint32_t; static constexpr int R = 8;
  static __device__ __forceinline__ W load_w(const __nv_bfloat16* p) {
    return (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p));
  }
  static __device__ __forceinline__ void dot(A& acc, U a, U b) {
    dot_bf16_pair(acc, a.x, b.x); dot_bf16_pair(acc, a.y, b.y);
    dot_bf16_pair(acc, a.z, b.z); dot_bf16_pair(acc, a.w, b.w);
  }
};
template <> struct Vec<float> {
  using U = float4; using A = float; using W = float; static constexpr int R = 4;
  static __device__ __forceinline__ W load_w(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ void dot(A& acc, U a, U b) {
    acc = fmaf(a.x, b.x, acc); acc = fmaf(a.y, b.y, acc); acc = fmaf(a.z, b.z, acc); acc = fmaf(a.w, b.w, acc);
  }
};
template <> struct Vec<double> {
  using U = double2; using A = double; using W = double; static constexpr int R = 2;
  static __device__ __forceinline__ W load_w(const double* p) { return __ldg(p); }
  static __device__ __forceinline__ void dot(A& acc, U a, U b) {
    acc = fma(a.x, b.x, acc); acc = fma(a.y, b.y, acc);
  }
};

// ------------------------------------------------------------------ staging
// Transposed, packed staging: dst unit (g, col) <- rows b0 + g*VEC + r (r < VEC)
// of column src_col(col) of a row-major (B, W) source; rows >= B and columns
// mapped to -1 are zero.  Column chunks of VEC consecutive columns are moved by
// one VEC x VEC register transpose: VEC 16-byte loads, VEC 16-byte stores.
template <typename T>
__device__ __forceinline__ void transpose_store(typename Vec<T>::U (&r)[vec_rows<T>()], typename Vec<T>::U* dst,
                                                int stride_units);
template <>
__device__ __forceinline__ void transpose_store<__nv_bfloat16>(uint4 (&r)[8], uint4* dst, int su) {
  // r[i] = row i, 8 columns (4 u32 pairs).  Column j of rows (2i, 2i+1) is
  // byte_perm of the j-th halves of r[2i] and r[2i+1].
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t* ra = reinterpret_cast<const uint32_t*>(&r[2 * i]);
      const uint32_t* rb = reinterpret_cast<const uint32_t*>(&r[2 * i + 1]);
      w[i] = __byte_perm(ra[j >> 1], rb[j >> 1], (j & 1) ? 0x7632 : 0x5410);
    }
    dst[(size_t)j * su] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
template <>
__device__ __forceinline__ void transpose_store<float>(float4 (&r)[4], float4* dst, int su) {
  dst[0] = make_float4(r[0].x, r[1].x, r[2].x, r[3].x);
  dst[(size_t)su] = make_float4(r[0].y, r[1].y, r[2].y, r[3].y);
  dst[(size_t)2 * su] = make_float4(r[0].z, r[1].z, r[2].z, r[3].z);
  dst[(size_t)3 * su] = make_float4(r[0].w, r[1].w, r[2].w, r[3].w);
}
template <>
__device__ __forceinline__ void transpose_store<double>(double2 (&r)[2], double2* dst, int su) {
  dst[0] = make_double2(r[0].x, r[1].x);
  dst[(size_t)su] = make_double2(r[0].y, r[1].y);
}

// Stage NG row groups x ncols columns (group stride ld units).  Column col
// takes source column sc = (c0 + col) mod `mod` if sc < `limit`, else zero;
// rows >= B are zero.  `vec_ok`: mod, limit, c0 multiples of VEC and src
// 16-byte aligned (then every VEC-chunk is one aligned load).
template <typename T, int UNR = 1>
__device__ void stage_t(typename Vec<T>::U* __restrict__ dst, int ld, int ncols, const T* __restrict__ src, int B,
                        int W, int b0, int NG, int c0, int mod, int limit, bool vec_ok) {
  using U = typename Vec<T>::U;
  constexpr int VEC = vec_rows<T>();
  if (vec_ok) {
    // UNR items per thread per pass: all their loads are issued before the
    // first transpose, so a pass costs one memory latency, not UNR of them
    const int chunks = (ncols + VEC - 1) / VEC;
    const int total = NG * chunks;
    for (int base = threadIdx.x; base < total; base += blockDim.x * UNR) {
      U r[UNR][VEC];
#pragma unroll
      for (int k = 0; k < UNR; ++k) {
        const int it = base + k * blockDim.x;
        const int g = it / chunks, ch = it - g * chunks;
        const int sc = (c0 + ch * VEC) % mod;
        const bool valid = it < total && sc < limit;
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          const int b = b0 + g * VEC + i;
          if (valid && b < B) r[k][i] = *reinterpret_cast<const U*>(src + (size_t)b * W + sc);
          else r[k][i] = U{};
        }
      }
#pragma unroll
      for (int k = 0; k < UNR; ++k) {
        const int it = base + k * blockDim.x;
        if (it >= total) break;
        const int g = it / chunks, ch = it - g * chunks;
        U* d = dst + (size_t)g * ld + ch * VEC;
        if (ch * VEC + VEC <= ncols) {
          transpose_store<T>(r[k], d, 1);
        } else {  // ragged last chunk: store the columns that fit
          U tmp[VEC];
          transpose_store<T>(r[k], tmp, 1);
#pragma unroll
          for (int j = 0; j < VEC; ++j)
            if (ch * VEC + j < ncols) d[j] = tmp[j];
        }
      }
    }
  } else {
    T* dd = reinterpret_cast<T*>(dst);
    for (int it = threadIdx.x; it < NG * ncols * VEC; it += blockDim.x) {
      const int r = it % VEC, rest = it / VEC;
      const int col = rest % ncols, g = rest / ncols;
      const int b = b0 + g * VEC + r;
      const int sc = (int)(((long long)c0 + col) % mod);
      const bool valid = b < B && sc < limit;
      dd[((size_t)g * ld + col) * VEC + r] = valid ? src[(size_t)b * W + sc] : T(0);
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

// scatter-form staged width: the L real columns + zero column(s), VEC-aligned
template <typename T>
__host__ __device__ inline int scatter_cols(int L) {
  constexpr int VEC = vec_rows<T>();
  return (L + 1 + VEC - 1) / VEC * VEC;
}

// ------------------------------------------------------------------ prescale
// The compact weight store, indexed by OUTPUT position p (< out_w) so that the
// product kernels read it with one aligned base + immediate offsets:
//   gather  form: w[j, p] = s_j * values[o_j, p]                       (p < L)
//   scatter form: w[j, p] = s_j * values[o_j, c], c = (p - o_j) mod C,  0 if c >= L
// s_j = alpha_soft[o_j] (the reference's `weights`, layers.py:235); one
// rounding from the float64 product.  Columns [out_w, ldw) are zero.
// Each thread writes 4 consecutive positions of one diagonal row (one 16-byte
// load in the aligned gather form, 4 independent loads otherwise), so the
// HBM-bound pass keeps enough bytes in flight.
constexpr int kPreVec = 4;
template <typename T>
__global__ void __launch_bounds__(256)
k_prescale(int C, int L, int out_w, int ldw, int gather, const typename Traits<T>::P* __restrict__ vals,
           const double* __restrict__ asoft, const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p,
           int max_act, typename WType<T>::type* __restrict__ w) {
  using P = typename Traits<T>::P;
  using WT = typename WType<T>::type;
  const int n_act = min(*n_act_p, max_act);
  const int p0 = (blockIdx.x * blockDim.x + threadIdx.x) * kPreVec;
  if (p0 >= ldw) return;
  const bool vec = gather && (L % 4 == 0) && p0 + kPreVec <= L && (reinterpret_cast<uintptr_t>(vals) & 15) == 0;
  for (int j = blockIdx.y; j < n_act; j += gridDim.y) {
    const int o = active[j];
    const double s = asoft ? asoft[o] : 1.0;
    const P* vr = vals + (size_t)o * L;
    P v[kPreVec];
    if (vec && sizeof(P) == 4) {
      const float4 f = *reinterpret_cast<const float4*>(vr + p0);
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    } else {
#pragma unroll
      for (int e = 0; e < kPreVec; ++e) {
        const int p = p0 + e;
        int c = p;
        if (!gather) { c = p - o; c = c < 0 ? c + C : c; }
        v[e] = (p < out_w && c < L) ? vr[c] : P(0);
      }
    }
    WT* wr = w + (size_t)j * ldw + p0;
#pragma unroll
    for (int e = 0; e < kPreVec; ++e) {
      const double x = s * (double)v[e];
      if constexpr (sizeof(WT) == 2) wr[e] = __double2bfloat16(x);
      else wr[e] = (WT)x;
    }
  }
}

// --------------------------------------------------------------------------- K1/K2
// Both forms as one gather over output positions p (< out_w):
//   out[b, p] = sum_j w[j, p] * in[b, (p + shift_j) mod C]
// shift_j = o_j (gather form) or C - o_j (scatter form); weights are zero
// wherever the reference has no entry.  Gather form: the staged row is C +
// halo columns, so the inner loop has no mask or modulo at all.  Scatter form:
// the staged row is the L real columns plus zero columns; an index c >= L
// (no entry) is clamped onto a zero column (one IMNMX per position).
// A CTA is PW position-warps x DW = 8/PW diagonal-warps: it covers 128*PW
// positions x G*VEC rows; the DW warps of a position block (and nsplit CTAs,
// grid.z) take interleaved slices of its diagonal list and are folded in a
// fixed order (deterministic).  PW = 8 is the pure position tiling (large
// batches), PW = 1 with nsplit > 1 the pure diagonal split (B = 1).
// bytes of the staged tile / fold buffer of k_product (the active list follows)
template <typename T>
__host__ __device__ inline size_t product_tile_bytes(int g, int cols, bool cluster = false) {
  const size_t tile = (size_t)g * cols * 16;
  const size_t row = (size_t)g * vec_rows<T>() * kWarpPos * sizeof(typename Vec<T>::A);
  const size_t red = kWarps * row + (cluster ? row : 0);  // + the folded tile (cluster fold, PW = 1)
  return align16(tile > red ? tile : red);
}

// Weight of the compute type formed in the kernel (FW): s_j * values in fp32
// for bf16 / fp32 (a float64 product plus its F2F conversions costs more than
// the FMAs it feeds at these batch sizes; the fp32 product is within 2 ulp of
// k_prescale's single rounding), in fp64 for fp64.
template <typename T> struct FwScale { using S = float; };
template <> struct FwScale<double> { using S = double; };
template <typename T> __device__ __forceinline__ typename Vec<T>::W weight_from(typename FwScale<T>::S s,
                                                                               typename Traits<T>::P v);
template <> __device__ __forceinline__ uint32_t weight_from<__nv_bfloat16>(float s, float v) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(s * v));
}
template <> __device__ __forceinline__ float weight_from<float>(float s, float v) { return s * v; }
template <> __device__ __forceinline__ double weight_from<double>(double s, double v) { return s * v; }

// FW (fused weights, small batches): the ring fetches the stored values and
// alpha_soft and forms the weight at use time — no k_prescale pass.  With
// nsplit > 1 the grid.z CTAs of a tile form one thread-block cluster and fold
// their partial tiles through distributed shared memory (fixed rank order),
// so there is no partial buffer and no second kernel either.
template <typename T, int G, bool GATHER, bool FW>
__global__ void __launch_bounds__(kThreads, 2)
k_product(int B, int C, int L, const T* __restrict__ in, const typename WType<T>::type* __restrict__ wts, int ldw,
          const typename Traits<T>::P* __restrict__ vals, const double* __restrict__ asoft,
          const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act,
          const typename Traits<T>::P* __restrict__ bias, T* __restrict__ out, typename Vec<T>::A* __restrict__ part,
          int PW, int nsplit, int vec_ok) {
  using U = typename Vec<T>::U;
  using A = typename Vec<T>::A;
  using Wt = typename Vec<T>::W;
  using P = typename Traits<T>::P;
  using RW = typename std::conditional<FW, P, Wt>::type;  // what the ring holds
  constexpr int VEC = vec_rows<T>();
  constexpr int RT = G * VEC;  // rows per CTA
  extern __shared__ __align__(128) unsigned char smem[];
  U* xs = reinterpret_cast<U*>(smem);
  A* red = reinterpret_cast<A*>(smem);  // reused after the main loop
  const int n_act = min(*n_act_p, max_act);
  const int in_w = GATHER ? C : L;
  const int out_w = GATHER ? L : C;
  const int cols = GATHER ? C + kHalo : scatter_cols<T>(L);
  const int DW = kWarps / PW;
  const int t0 = blockIdx.x * PW * kWarpPos;
  const int b0 = blockIdx.y * RT;
  const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;
  const int pw = warp % PW, dw = warp / PW;
  const int p0 = t0 + pw * kWarpPos;  // this warp's first position

  // the active offsets live in shared memory behind the tile: the scatter-form
  // range search and the per-diagonal offset reads then cost no L2 round trips
  int32_t* s_act = reinterpret_cast<int32_t*>(smem + product_tile_bytes<T>(G, cols, FW && nsplit > 1));
  for (int i = threadIdx.x; i < n_act; i += kThreads) s_act[i] = __ldg(active + i);
  stage_t<T, 16 / vec_rows<T>()>(xs, cols, cols, in, B, in_w, b0, G, 0, GATHER ? C : 0x7fffffff, in_w, vec_ok != 0);
  __syncthreads();

  int lo1, hi1, lo2, hi2;
  if (GATHER) { lo1 = 0; hi1 = n_act; lo2 = 0; hi2 = 0; }
  else scatter_ranges(s_act, n_act, C, L, p0, kWarpPos, lo1, hi1, lo2, hi2);
  const int len1 = hi1 - lo1;
  const int total = p0 < out_w ? len1 + (hi2 - lo2) : 0;
  const int per = (total + nsplit - 1) / nsplit;
  const int cb = min(total, (int)blockIdx.z * per), ce = min(total, cb + per);
  const int vb = cb + dw;
  const int nq = ce - vb > 0 ? (ce - vb + DW - 1) / DW : 0;
  bool pok[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) pok[u] = p0 + lane + kWarp * u < out_w;
  __syncthreads();

  A acc[G][kU][VEC];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int r = 0; r < VEC; ++r) acc[g][u][r] = A(0);

  // Diagonal q+D is fetched (weights + staged-row index) while diagonal q is
  // multiplied: a D-deep register ring hides the L2 latency of the weights.
  using SC = typename FwScale<T>::S;
  auto fetch = [&](int q, RW (&wv)[kU], SC& sc, int& ci) {
    if (q < nq) {
      const int v = vb + DW * q;
      const int j = v < len1 ? lo1 + v : lo2 + (v - len1);
      const int o = s_act[j];
      const int base = p0 + lane + (GATHER ? o : C - o);
      ci = base >= C ? base - C : base;  // < C
      if constexpr (FW) {
        sc = asoft ? (SC)__ldg(asoft + o) : SC(1);
        const P* vr = vals + (size_t)o * L;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          int c = GATHER ? p0 + lane + kWarp * u : ci + kWarp * u;
          if (!GATHER) c = c >= C ? c - C : c;
          wv[u] = (pok[u] && c < L) ? __ldg(vr + c) : P(0);
        }
      } else {
        const typename WType<T>::type* wr = wts + (size_t)j * ldw + p0 + lane;
#pragma unroll
        for (int u = 0; u < kU; ++u) wv[u] = pok[u] ? Vec<T>::load_w(wr + kWarp * u) : Wt(0);
      }
    }
  };
  constexpr int D = (sizeof(Wt) == 8 || RT > 8) ? 4 : 8;
  RW wb[D][kU];
  SC sb[D];
  int cb_[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
#pragma unroll
    for (int u = 0; u < kU; ++u) wb[d][u] = RW(0);
    sb[d] = SC(0);
    cb_[d] = 0;
    fetch(d, wb[d], sb[d], cb_[d]);
  }
  for (int q0 = 0; q0 < nq; q0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (q0 + d < nq) {  // warp-uniform
        Wt w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if constexpr (FW) w[u] = weight_from<T>(sb[d], wb[d][u]);
          else w[u] = wb[d][u];
        }
        if (GATHER) {
          const U* xr = xs + cb_[d];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
#pragma unroll
            for (int g = 0; g < G; ++g) fma_vec(acc[g][u], xr[(size_t)g * cols + kWarp * u], w[u]);
          }
        } else {
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            int c = cb_[d] + kWarp * u;
            c = c >= C ? c - C : c;
            c = c < L ? c : L;  // column L is zero
#pragma unroll
            for (int g = 0; g < G; ++g) fma_vec(acc[g][u], xs[(size_t)g * cols + c], w[u]);
          }
        }
      }
      fetch(q0 + d + D, wb[d], sb[d], cb_[d]);
    }
  }

  if (DW == 1 && nsplit == 1) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = p0 + lane + kWarp * u;
      if (p >= out_w) continue;
      const A bb = bias ? (A)bias[p] : A(0);
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int r = 0; r < VEC; ++r) {
          const int b = b0 + g * VEC + r;
          if (b < B) out[(size_t)b * out_w + p] = from_acc<T>(acc[g][u][r] + bb);
        }
    }
    return;
  }
  // fixed-order fold of the DW diagonal slices through shared memory:
  // red[dw][row][pos] with pos over the CTA's PW*128 positions
  const int TT = PW * kWarpPos;
  const int tt_shift = 31 - __clz(TT);  // TT is 128 * a power of two
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int r = 0; r < VEC; ++r)
#pragma unroll
      for (int u = 0; u < kU; ++u)
        red[((size_t)dw * RT + g * VEC + r) * TT + pw * kWarpPos + lane + kWarp * u] = acc[g][u][r];
  __syncthreads();
  const bool cluster_fold = FW && nsplit > 1;
  A* fin = red + (size_t)DW * RT * TT;  // this CTA's folded tile (cluster fold only)
  for (int i = threadIdx.x; i < RT * TT; i += kThreads) {
    const int b = i >> tt_shift, tt = i & (TT - 1);
    const int p = t0 + tt;
    A s = A(0);
    for (int w = 0; w < DW; ++w) s += red[((size_t)w * RT + b) * TT + tt];
    if (cluster_fold) {
      fin[i] = s;
    } else if (b0 + b < B && p < out_w) {
      if (nsplit == 1) {
        if (bias) s += (A)bias[p];
        out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(s);
      } else {
        part[((size_t)blockIdx.z * B + b0 + b) * out_w + p] = s;
      }
    }
  }
  if constexpr (FW) {
    if (cluster_fold) {
      // every rank folds one slice of the tile, reading the partial tiles of all
      // ranks in rank order (deterministic), then the cluster waits so no CTA
      // leaves while its shared memory is still being read
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      cl.sync();
      const int rank = (int)cl.block_rank(), nr = (int)cl.num_blocks();
      const int per_r = (RT * TT + nr - 1) / nr;
      const int i0 = rank * per_r, i1 = min(RT * TT, i0 + per_r);
      for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
        const int b = i >> tt_shift, tt = i & (TT - 1);
        const int p = t0 + tt;
        if (b0 + b >= B || p >= out_w) continue;
        A s = A(0);
        for (int r = 0; r < nr; ++r) s += cl.map_shared_rank(fin, r)[i];
        if (bias) s += (A)bias[p];
        out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(s);
      }
      cl.sync();
    }
  }
}

// --------------------------------------------------------------------------- narrow batches
// B <= kNarrowB: the weights dominate the traffic (HBM-bound regime), so they
// are streamed ONCE in their stored fp32/fp64 form and scaled on the fly (no
// prescale pass, no staging); the few input rows come through L1.  A CTA is
// 128 positions (lane + 32u) x one chunk of the diagonal list; its 8 warps
// interleave over the chunk and are folded in a fixed order; chunks (grid.y)
// are folded by k_split_reduce in a fixed order.
constexpr int kNarrowB = 8;  // rows per CTA (grid.z walks row blocks)
template <typename T, int BT, bool GATHER>
__global__ void __launch_bounds__(kThreads)
k_product_narrow(int B, int C, int L, const T* __restrict__ in, const typename Traits<T>::P* __restrict__ vals,
                 const double* __restrict__ asoft, const int32_t* __restrict__ active,
                 const int32_t* __restrict__ n_act_p, int max_act, const typename Traits<T>::P* __restrict__ bias,
                 T* __restrict__ out, typename Vec<T>::A* __restrict__ part, int nchunk) {
  using A = typename Vec<T>::A;
  __shared__ A red[kWarps][kWarpPos];
  const int n_act = min(*n_act_p, max_act);
  const int in_w = GATHER ? C : L, out_w = GATHER ? L : C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p0 = blockIdx.x * kWarpPos;
  const int b0 = blockIdx.z * BT;
  const int Bt = B;  // total rows (partials are indexed by global row)
  B = min(BT, Bt - b0);  // rows of this block
  in += (size_t)b0 * in_w;
  out += (size_t)b0 * out_w;
  const int per = (n_act + nchunk - 1) / nchunk;
  const int jb = min(n_act, (int)blockIdx.y * per), je = min(n_act, jb + per);
  A acc[BT][kU];
#pragma unroll
  for (int b = 0; b < BT; ++b)
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[b][u] = A(0);
  // this warp's diagonals: j = jb + warp + 8q.  Offsets/scales of 32 of them
  // are fetched lane-parallel, then 4 diagonals' weights are loaded together
  // (16 independent loads per lane in flight) before they are used.
  const int nq = je - jb - warp > 0 ? (je - jb - warp + kWarps - 1) / kWarps : 0;
  constexpr int UNR = 4;
  for (int q0 = 0; q0 < nq; q0 += 32) {
    int o_l = 0;
    double s_l = 0.0;
    if (q0 + lane < nq) {
      o_l = __ldg(active + jb + warp + kWarps * (q0 + lane));
      s_l = asoft ? asoft[o_l] : 1.0;
    }
    const int cnt = min(32, nq - q0);
    for (int qq = 0; qq < cnt; qq += UNR) {
      A wv[UNR][kU];
      typename Traits<T>::P wraw[UNR][kU];
      int xi[UNR][kU];
      // raw weights first (they depend only on the offset), the scale after
#pragma unroll
      for (int r = 0; r < UNR; ++r) {
        const int o = __shfl_sync(0xffffffffu, o_l, (qq + r) & 31);
        const bool live = qq + r < cnt;
        const typename Traits<T>::P* vr = vals + (size_t)o * L;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int p = p0 + lane + kWarp * u;
          int c, xx;
          bool ok;
          if (GATHER) {
            c = p; ok = p < L;
            xx = p + o; xx = xx >= C ? xx - C : xx;
          } else {
            c = p - o; c = c < 0 ? c + C : c;
            ok = p < C && c < L;
            xx = c;
          }
          ok = ok && live;
          wraw[r][u] = ok ? __ldg(vr + c) : typename Traits<T>::P(0);
          xi[r][u] = ok ? xx : 0;
        }
      }
#pragma unroll
      for (int r = 0; r < UNR; ++r) {
        const double sc = __shfl_sync(0xffffffffu, s_l, (qq + r) & 31);
#pragma unroll
        for (int u = 0; u < kU; ++u) wv[r][u] = (A)(sc * (double)wraw[r][u]);
      }
#pragma unroll
      for (int r = 0; r < UNR; ++r)
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int b = 0; b < BT; ++b)
            if (b < B) acc[b][u] = fma(wv[r][u], to_acc<A>(__ldg(in + (size_t)b * in_w + xi[r][u])), acc[b][u]);
    }
  }
  // fixed-order fold of the 8 warps, one batch row at a time
#pragma unroll
  for (int b = 0; b < BT; ++b) {
    if (b >= B) break;
#pragma unroll
    for (int u = 0; u < kU; ++u) red[warp][lane + kWarp * u] = acc[b][u];
    __syncthreads();
    for (int tt = threadIdx.x; tt < kWarpPos; tt += kThreads) {
      const int p = p0 + tt;
      if (p >= out_w) continue;
      A s_ = A(0);
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s_ += red[w][tt];
      if (nchunk == 1) {
        if (bias) s_ += (A)bias[p];
        out[(size_t)b * out_w + p] = from_acc<T>(s_);
      } else {
        part[((size_t)blockIdx.y * Bt + b0 + b) * out_w + p] = s_;
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------------- few rows, one launch
// B <= kRowsMax (weights dominate the traffic): ONE kernel, no pre-scale pass, no
// partial buffer, no reduce launch.  A CTA owns 32 output positions (one per
// lane) x BT rows; its 16 warps take interleaved slices of the active list and
// are folded in a fixed order in shared memory; with NS > 1 the diagonal list is
// also split over the NS CTAs of a thread-block cluster, folded through
// distributed shared memory in rank order (deterministic).  Weights are formed
// at use time (alpha_soft x the stored fp32 / fp64 value, the reference's
// `weights`, layers.py:235); a lane loads its weight and its input elements
// with coalesced warp-wide loads (32 consecutive positions), U diagonals ahead.
constexpr int kRowsMax = 8;
constexpr int kRowsWarps = 16;
template <typename T, int BT, bool GATHER, int NS>
__global__ void __launch_bounds__(kRowsWarps * 32)
k_product_rows(int B, int C, int L, const T* __restrict__ in, const typename Traits<T>::P* __restrict__ vals,
               const double* __restrict__ asoft, const int32_t* __restrict__ active,
               const int32_t* __restrict__ n_act_p, int max_act, const typename Traits<T>::P* __restrict__ bias,
               T* __restrict__ out) {
  using A = typename Vec<T>::A;
  using P = typename Traits<T>::P;
  __shared__ A red[kRowsWarps][BT][32];
  const int n_act = min(*n_act_p, max_act);
  const int in_w = GATHER ? C : L, out_w = GATHER ? L : C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + lane;
  const int b0 = blockIdx.y * BT;
  const int nb = min(BT, B - b0);
  const int rank = NS > 1 ? (int)blockIdx.z : 0;
  in += (size_t)b0 * in_w;
  A acc[BT];
#pragma unroll
  for (int b = 0; b < BT; ++b) acc[b] = A(0);
  // diagonals of this warp: j = rank * kRowsWarps + warp + (NS * kRowsWarps) * q
  constexpr int STRIDE = NS * kRowsWarps;
  const int jfirst = rank * kRowsWarps + warp;
  const int nq = n_act > jfirst ? (n_act - jfirst + STRIDE - 1) / STRIDE : 0;
  constexpr int U = BT <= 2 ? 8 : 4;
  for (int q0 = 0; q0 < nq; q0 += 32) {
    // 32 diagonals' offsets and scales fetched lane-parallel, then shuffled out
    int o_l = 0;
    double s_l = 0.0;
    if (q0 + lane < nq) {
      o_l = __ldg(active + jfirst + STRIDE * (q0 + lane));
      s_l = asoft ? __ldg(asoft + o_l) : 1.0;
    }
    const int cnt = min(32, nq - q0);
    for (int qq = 0; qq < cnt; qq += U) {
      P wr[U];
      int xi[U];
      double sc[U];
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const int o = __shfl_sync(0xffffffffu, o_l, (qq + r) & 31);
        sc[r] = __shfl_sync(0xffffffffu, s_l, (qq + r) & 31);
        int c, xx;
        bool ok;
        if (GATHER) {
          c = p;
          ok = p < L;
          xx = p + o;
          xx = xx >= C ? xx - C : xx;
        } else {
          c = p - o;
          c = c < 0 ? c + C : c;
          ok = p < C && c < L;
          xx = c;
        }
        ok = ok && (qq + r < cnt);
        wr[r] = ok ? __ldg(vals + (size_t)o * L + c) : P(0);
        xi[r] = ok ? xx : 0;
      }
      A xv[U][BT];
#pragma unroll
      for (int r = 0; r < U; ++r)
#pragma unroll
        for (int b = 0; b < BT; ++b) xv[r][b] = b < nb ? to_acc<A>(__ldg(in + (size_t)b * in_w + xi[r])) : A(0);
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const A w = (A)(sc[r] * (double)wr[r]);
#pragma unroll
        for (int b = 0; b < BT; ++b) acc[b] = fma(w, xv[r][b], acc[b]);
      }
    }
  }
  // fixed-order fold: the 16 warps, then (NS > 1) the cluster ranks
#pragma unroll
  for (int b = 0; b < BT; ++b) red[warp][b][lane] = acc[b];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      A sum = A(0);
#pragma unroll
      for (int w = 0; w < kRowsWarps; ++w) sum += red[w][b][lane];
      red[0][b][lane] = sum;
    }
  }
  if constexpr (NS > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (rank == 0 && warp == 0) {
      for (int r = 1; r < NS; ++r) {
        const A* peer = cluster.map_shared_rank(&red[0][0][0], r);
#pragma unroll
        for (int b = 0; b < BT; ++b) red[0][b][lane] += peer[b * 32 + lane];
      }
    }
    cluster.sync();  // peers keep their shared memory alive until rank 0 has read it
    if (rank != 0) return;
  }
  if (warp == 0 && p < out_w) {
    const A bz = bias ? (A)bias[p] : A(0);
    for (int b = 0; b < nb; ++b) out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(red[0][b][lane] + bz);
  }
}

template <typename T>
static int run_product_rows(bool gather, int B, int C, int L, const void* in, const void* vals, const double* asoft,
                            const int32_t* active, const int32_t* n_act, int max_act, const void* bias, void* out,
                            cudaStream_t st) {
  using P = typename Traits<T>::P;
  const int out_w = gather ? L : C;
  const int tiles = ceil_div(out_w, 32) * ceil_div(B, kRowsMax);
  // split the diagonal list over a cluster when the tiles leave SMs idle
  int ns = 1;
  while (ns < 8 && (long long)tiles * ns * 2 <= num_sms() && max_act >= ns * 2 * kRowsWarps * 4) ns *= 2;
  const int bt = B <= 1 ? 1 : (B <= 2 ? 2 : (B <= 4 ? 4 : 8));
  auto tin = static_cast<const T*>(in);
  auto tv = static_cast<const P*>(vals);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ceil_div(out_w, 32), ceil_div(B, bt), ns);
  cfg.blockDim = dim3(kRowsWarps * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = ns;
  cfg.attrs = attr;
  cfg.numAttrs = ns > 1 ? 1 : 0;
#define DIAGMM_ROWS(BT, NS)                                                                                    \
  if (bt == BT && ns == NS) {                                                                                  \
    if (gather)                                                                                                \
      cudaLaunchKernelEx(&cfg, k_product_rows<T, BT, true, NS>, B, C, L, tin, tv, asoft, active, n_act,        \
                         max_act, tb, to);                                                                     \
    else                                                                                                       \
      cudaLaunchKernelEx(&cfg, k_product_rows<T, BT, false, NS>, B, C, L, tin, tv, asoft, active, n_act,       \
                         max_act, tb, to);                                                                     \
  }
#define DIAGMM_ROWS_NS(BT) DIAGMM_ROWS(BT, 1) DIAGMM_ROWS(BT, 2) DIAGMM_ROWS(BT, 4) DIAGMM_ROWS(BT, 8)
  DIAGMM_ROWS_NS(1) DIAGMM_ROWS_NS(2) DIAGMM_ROWS_NS(4) DIAGMM_ROWS_NS(8)
#undef DIAGMM_ROWS_NS
#undef DIAGMM_ROWS
  note_launch();
  return status_from_cuda();
}

// dW for narrow batches: one warp per diagonal, lanes over 128 positions, the
// B-row contraction in registers; unscaled gw -> partial (finalized by
// k_dw_finalize exactly like the wide path).
template <typename T, int BT>
__global__ void __launch_bounds__(kThreads)
k_dw_narrow(int B, int C, int L, const T* __restrict__ aop, const T* __restrict__ bop,
            const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act,
            typename Vec<T>::A* __restrict__ gw) {
  using A = typename Vec<T>::A;
  const int n_act = min(*n_act_p, max_act);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.y * kWarps + warp;
  if (j >= n_act) return;
  const int o = __ldg(active + j);
  const int t0 = blockIdx.x * kWarpPos;
  int ca[kU];
  bool ok[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int t = t0 + lane + kWarp * u;
    ok[u] = t < L;
    int c = o + t;
    c = c >= C ? c - C : c;
    ca[u] = ok[u] ? c : 0;
  }
  A acc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) acc[u] = A(0);
  // the B-row contraction: BT rows unrolled per step (fixed order, deterministic)
  for (int b0 = 0; b0 < B; b0 += BT) {
#pragma unroll
    for (int bb = 0; bb < BT; ++bb) {
      const int b = b0 + bb;
      if (b >= B) break;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = t0 + lane + kWarp * u;
        if (ok[u])
          acc[u] = fma(to_acc<A>(__ldg(aop + (size_t)b * C + ca[u])), to_acc<A>(__ldg(bop + (size_t)b * L + t)), acc[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kU; ++u)
    if (ok[u]) gw[(size_t)j * L + t0 + lane + kWarp * u] = acc[u];
}

// Fixed-order sum of the split partials (+ bias).
template <typename T>
__global__ void __launch_bounds__(256)
k_split_reduce(int B, int out_w, int nsplit, const typename Vec<T>::A* __restrict__ part,
               const typename Traits<T>::P* __restrict__ bias, T* __restrict__ out) {
  using A = typename Vec<T>::A;
  const size_t n = (size_t)B * out_w;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    A s = A(0);
    for (int z0 = 0; z0 < nsplit; z0 += 8) {  // 8 loads in flight, summed in split order
      A v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = z0 + k < nsplit ? __ldcg(part + (size_t)(z0 + k) * n + i) : A(0);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (z0 + k < nsplit) s += v[k];
    }
    if (bias) s += (A)bias[i % out_w];
    out[i] = from_acc<T>(s);
  }
}

// small outputs use 64-thread blocks so the fold spreads over more SMs
template <typename T>
static void launch_split_reduce(int B, int out_w, int nsplit, const typename Vec<T>::A* part,
                                const typename Traits<T>::P* bias, T* out, cudaStream_t st) {
  const size_t n = (size_t)B * out_w;
  const int threads = n < (size_t)256 * num_sms() ? 64 : 256;
  long long blocks = (long long)((n + threads - 1) / threads);
  if (blocks > 4LL * num_sms()) blocks = 4LL * num_sms();
  k_split_reduce<T><<<(int)blocks, threads, 0, st>>>(B, out_w, nsplit, part, bias, out);
}

// --------------------------------------------------------------------------- K3
constexpr int kDwPosWarps = 2;                         // warps along positions
constexpr int kDwTile = kDwPosWarps * kWarpPos;        // 256 positions per CTA
constexpr int kDwGroups = kWarps / kDwPosWarps;        // 4 diagonal groups
constexpr int kDwNG = 2;                               // row groups per staged chunk
template <typename T> __host__ __device__ constexpr int kDwUnr() { return 8 / vec_rows<T>() > 1 ? 8 / vec_rows<T>() : 1; }

template <typename T>
__host__ __device__ inline size_t dw_smem(int win_cap) {
  return (size_t)kDwNG * (win_cap + kDwTile) * 16;
}

// CTA: kDwTile positions x 4*JW diagonals x one row part.  Warp w: positions
// t0 + (w % 2)*128 + lane + 32u, diagonals j0 + (w / 2)*JW + q.
template <typename T, int JW>
__global__ void __launch_bounds__(kThreads, 2)
k_dw(int B, int C, int L, const T* __restrict__ aop, const T* __restrict__ bop,
     const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act, int win_cap,
     int rows_per_part, typename Vec<T>::A* __restrict__ partial, int vec_ok) {
  using U = typename Vec<T>::U;
  using A = typename Vec<T>::A;
  constexpr int VEC = vec_rows<T>();
  constexpr int RB = kDwNG * VEC;  // rows per staged chunk
  extern __shared__ __align__(128) unsigned char smem[];
  const int n_act = min(*n_act_p, max_act);
  const int j0 = blockIdx.y * (kDwGroups * JW);
  if (j0 >= n_act) return;
  const int nj = min((kDwGroups * JW), n_act - j0);
  const int t0 = blockIdx.x * kDwTile;
  const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;
  const int pw = warp % kDwPosWarps, grp = warp / kDwPosWarps;
  const int pbase = pw * kWarpPos;
  const int o_first = active[j0], o_last = active[j0 + nj - 1];
  // Aop window: columns (o_first + t0) .. (o_last + t0 + kDwTile - 1), circular
  int ws = o_first + t0;
  ws = ws >= C ? ws - C : ws;
  const int aws = vec_ok ? ws / VEC * VEC : ws;  // VEC-aligned start for 16-byte loads
  const int lead = ws - aws;
  const int wcols = o_last - o_first + kDwTile + lead;
  const bool direct = wcols > win_cap;  // window too wide for smem: read Aop from global
  U* as = reinterpret_cast<U*>(smem);
  U* bs = as + (size_t)kDwNG * win_cap;
  int oq[JW];
#pragma unroll
  for (int q = 0; q < JW; ++q) {
    const int j = j0 + grp * JW + q;
    oq[q] = j < j0 + nj ? active[j] - o_first : -1;
  }
  A acc[JW][kU];
#pragma unroll
  for (int q = 0; q < JW; ++q)
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[q][u] = A(0);

  const int rb = blockIdx.z * rows_per_part, re = min(B, rb + rows_per_part);
  for (int r0 = rb; r0 < re; r0 += RB) {
    __syncthreads();  // previous chunk consumed
    if (!direct) stage_t<T, kDwUnr<T>()>(as, win_cap, wcols, aop, re, C, r0, kDwNG, aws, C, C, vec_ok != 0);
    stage_t<T, kDwUnr<T>()>(bs, kDwTile, kDwTile, bop, re, L, r0, kDwNG, t0, 0x7fffffff, L, vec_ok != 0);
    __syncthreads();
#pragma unroll
    for (int g = 0; g < kDwNG; ++g) {
      U bm[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) bm[u] = bs[(size_t)g * kDwTile + pbase + lane + kWarp * u];
      if (!direct) {
        const U* arow = as + (size_t)g * win_cap + lead + pbase + lane;
#pragma unroll
        for (int q = 0; q < JW; ++q) {
          if (oq[q] < 0) continue;
#pragma unroll
          for (int u = 0; u < kU; ++u) Vec<T>::dot(acc[q][u], arow[oq[q] + kWarp * u], bm[u]);
        }
      } else {
        // gather the Aop units straight from global (rare: very spread offsets)
#pragma unroll 1
        for (int q = 0; q < JW; ++q) {
          if (oq[q] < 0) continue;
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            int col = oq[q] + o_first + t0 + pbase + lane + kWarp * u;
            col = col >= C ? col - C : col;
            col = col >= C ? col - C : col;
            U a;
            T* ae = reinterpret_cast<T*>(&a);
#pragma unroll
            for (int r = 0; r < VEC; ++r) {
              const int b = r0 + g * VEC + r;
              ae[r] = b < re ? aop[(size_t)b * C + col] : T(0);
            }
            Vec<T>::dot(acc[q][u], a, bm[u]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < JW; ++q) {
    const int j = j0 + grp * JW + q;
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
// zero inactive rows, and form g_soft.  One CTA per candidate row.  The row is
// walked in 16-byte vectors with every load of the (usually single) pass
// issued before its first use, so an active row costs ~one memory latency and
// the ~90 % inactive rows are a vectorised zero fill.  g_soft: per-thread sums
// in a fixed order, then a fixed shuffle/warp tree (deterministic).
// One candidate row of the finalize (shared by the per-layer and the batched kernels):
// reduce the dW partials over parts (fixed order), scale into g_values, zero inactive
// rows, g_soft, the data-parallel bucket row.
template <typename T, int U = 1, bool BLOCK = false>
__device__ void finalize_row(int ii, int C, int L, int nparts, const typename Vec<T>::A* __restrict__ partial,
                             int max_act, const int32_t* __restrict__ slot, int n_act,
                             const double* __restrict__ asoft, const typename Traits<T>::P* __restrict__ vals,
                             typename Traits<T>::P* __restrict__ g_values, double* __restrict__ g_soft,
                             typename Traits<T>::P* __restrict__ bucket, int bucket_rows,
                             const int32_t* __restrict__ active_rows, double* red = nullptr) {
  using P = typename Traits<T>::P;
  using A = typename Vec<T>::A;
  constexpr int VW = 16 / sizeof(P);
  using V = typename std::conditional<sizeof(P) == 8, double2, float4>::type;
  using VA = typename std::conditional<sizeof(A) == 8, double2, float4>::type;
  // one WARP per row (no barrier, rows of a CTA run concurrently), or with BLOCK the whole
  // CTA on one row (few long rows: the FMA route's 4096-wide layers at high sparsity)
  const int lane = BLOCK ? (int)threadIdx.x : (int)(threadIdx.x & 31);
  const int nth = BLOCK ? (int)blockDim.x : 32;
  do {

  // active_rows: the CTAs walk the active list only (the zero rows are filled
  // concurrently by k_zero_inactive on a side stream)
  const int i = active_rows ? active_rows[ii] : ii;
  const int s = slot[i];
  P* grow = g_values + (size_t)i * L;
  const bool vec = L % VW == 0 && (reinterpret_cast<uintptr_t>(g_values) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(vals) & 15) == 0;
  if (s < 0 || s >= n_act) {
    if (vec) {
      V* g4 = reinterpret_cast<V*>(grow);
      for (int t = lane; t < L / VW; t += nth) g4[t] = V{};
    } else {
      for (int t = lane; t < L; t += nth) grow[t] = P(0);
    }
    if (g_soft && lane == 0) g_soft[i] = 0.0;
    break;
  }
  const double sc = asoft ? asoft[i] : 1.0;
  const P* vrow = vals + (size_t)i * L;
  // data-parallel exchange: the active row also lands in its compact bucket slot
  // (bucket row s = the s-th active offset), which is what the all-reduce sends
  P* brow = (bucket && s < bucket_rows) ? bucket + (size_t)s * L : nullptr;
  const bool bvec = brow && (reinterpret_cast<uintptr_t>(bucket) & 15) == 0;
  double local = 0.0;
  if (vec) {
    // parts are summed in index order; up to 8 of their loads are in flight
    const int nv = L / VW;
    const size_t zs = (size_t)max_act * L / VW;
    const VA* pbase = reinterpret_cast<const VA*>(partial + (size_t)s * L);
    // U of the lane's positions per pass, their first loads all in flight (U = 4 in the
    // per-layer kernel, whose rows can be 4096 wide; 1 in the batched one, where registers
    // bound the occupancy); the lane still walks c = lane, lane + 32, ... in order, so
    // g_soft's per-lane sum keeps its order and both kernels give the same bits
    for (int c0 = lane; c0 < nv; c0 += nth * U) {
      V v[U];
      VA gw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + nth * u;
        if (c < nv) {
          v[u] = reinterpret_cast<const V*>(vrow)[c];
          gw[u] = nparts > 0 ? pbase[c] : VA{};
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + nth * u;
        if (c >= nv) break;
        A* ge = reinterpret_cast<A*>(&gw[u]);
        for (int p0 = 1; p0 < nparts; p0 += 8) {
          VA x[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (p0 + k < nparts) x[k] = __ldcg(pbase + (size_t)(p0 + k) * zs + c);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (p0 + k >= nparts) break;
            const A* xe = reinterpret_cast<const A*>(&x[k]);
#pragma unroll
            for (int e = 0; e < VW; ++e) ge[e] += xe[e];
          }
        }
        const P* ve = reinterpret_cast<const P*>(&v[u]);
        V o;
        P* oe = reinterpret_cast<P*>(&o);
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          oe[e] = (P)(sc * (double)ge[e]);
          local += (double)ge[e] * (double)ve[e];
        }
        reinterpret_cast<V*>(grow)[c] = o;
        if (bvec) reinterpret_cast<V*>(brow)[c] = o;
        else if (brow)
          for (int e = 0; e < VW; ++e) brow[c * VW + e] = oe[e];
      }
    }
  } else {
    for (int t = lane; t < L; t += nth) {
      A gw = A(0);
      for (int p = 0; p < nparts; ++p) gw += partial[((size_t)p * max_act + s) * L + t];
      grow[t] = (P)(sc * (double)gw);
      if (brow) brow[t] = grow[t];
      local += (double)gw * (double)vrow[t];
    }
  }
  if (g_soft) {  // per-lane sums in a fixed order, then a fixed shuffle tree (deterministic)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if constexpr (BLOCK) {  // + the warps' sums folded in warp order
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
      __syncthreads();
      if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
        g_soft[i] = tot;
      }
      __syncthreads();
    } else {
      if (lane == 0) g_soft[i] = local;
    }
  }
    } while (false);
}

template <typename T>
__global__ void __launch_bounds__(256)
k_dw_finalize(int C, int L, int nparts, const typename Vec<T>::A* __restrict__ partial, int max_act,
              const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p,
              const double* __restrict__ asoft, const typename Traits<T>::P* __restrict__ vals,
              typename Traits<T>::P* __restrict__ g_values, double* __restrict__ g_soft,
              typename Traits<T>::P* __restrict__ bucket, int bucket_rows,
              const int32_t* __restrict__ active_rows) {
  static_assert(sizeof(typename Vec<T>::A) == sizeof(typename Traits<T>::P), "partials and values share the vector width");
  const int n_act = min(*n_act_p, max_act);
  // one warp per row, grid-stride over rows: ~90 % of the rows are a zero fill
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), nw = gridDim.x * (blockDim.x >> 5);
  for (int ii = w; ii < (active_rows ? n_act : C); ii += nw)
    finalize_row<T, 4>(ii, C, L, nparts, partial, max_act, slot, n_act, asoft, vals, g_values, g_soft, bucket,
                       bucket_rows, active_rows);
}

// one CTA per candidate row: measured faster than a persistent grid-stride loop
// (4096^2, B = 1: 22.3 vs 26.6 us for the whole dW)
// The per-layer finalize for few, long rows (FMA route, L >= 1024): one CTA per active row.
template <typename T>
__global__ void __launch_bounds__(256)
k_dw_finalize_blk(int C, int L, int nparts, const typename Vec<T>::A* __restrict__ partial, int max_act,
                  const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p,
                  const double* __restrict__ asoft, const typename Traits<T>::P* __restrict__ vals,
                  typename Traits<T>::P* __restrict__ g_values, double* __restrict__ g_soft,
                  typename Traits<T>::P* __restrict__ bucket, int bucket_rows, const int32_t* __restrict__ active_rows) {
  __shared__ double red[kWarps];
  const int n_act = min(*n_act_p, max_act);
  for (int ii = blockIdx.x; ii < n_act; ii += gridDim.x)
    finalize_row<T, 2, true>(ii, C, L, nparts, partial, max_act, slot, n_act, asoft, vals, g_values, g_soft, bucket,
                             bucket_rows, active_rows, red);
}

static int finalize_grid(int C) { return C; }

// The reference's zero rows of g_values (inactive candidates, layers.py:159-163)
// and their g_soft, one CTA per candidate row; active rows are left to the finalize.
template <typename P>
__global__ void __launch_bounds__(256)
k_zero_inactive(int C, int L, const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p, int max_act,
                P* __restrict__ g_values, double* __restrict__ g_soft) {
  constexpr int VW = 16 / sizeof(P);
  using V = typename std::conditional<sizeof(P) == 8, double2, float4>::type;
  const int i = blockIdx.x;
  const int n_act = min(*n_act_p, max_act);
  const int s = slot[i];
  if (s >= 0 && s < n_act) return;
  P* grow = g_values + (size_t)i * L;
  if (L % VW == 0 && (reinterpret_cast<uintptr_t>(g_values) & 15) == 0) {
    V* g4 = reinterpret_cast<V*>(grow);
    for (int t = threadIdx.x; t < L / VW; t += blockDim.x) g4[t] = V{};
  } else {
    for (int t = threadIdx.x; t < L; t += blockDim.x) grow[t] = P(0);
  }
  if (g_soft && threadIdx.x == 0) g_soft[i] = 0.0;
}

// A side stream per device for work that overlaps the main stream's kernels
// inside one C-ABI call (fork / join through events: legal under CUDA-graph
// capture, where it becomes two parallel branches).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream& side_stream() {
  static SideStream ss[16];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& r = ss[dev & 15];
  if (!r.s) {
    cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming);
  }
  return r;
}

// Column sums of dy (bias gradient): 32-row partials, then a fixed-order fold.
constexpr int kColRows = 32;
template <typename T>
__global__ void __launch_bounds__(256)
k_colsum_partial(int B, int M, const T* __restrict__ dy, typename Vec<T>::A* __restrict__ part) {
  using A = typename Vec<T>::A;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  const int bb = blockIdx.y * kColRows, be = min(B, bb + kColRows);
  A acc = A(0);
  for (int b = bb; b < be; ++b) acc += to_acc<A>(dy[(size_t)b * M + r]);
  part[(size_t)blockIdx.y * M + r] = acc;
}
template <typename T>
__device__ void colsum_final_block(int M, int nparts, const typename Vec<T>::A* __restrict__ part,
                                   typename Traits<T>::P* __restrict__ g_bias, int blk) {
  using A = typename Vec<T>::A;
  __shared__ A red[8][33];
  // 32 columns per CTA, the 8 warps split the parts, fixed-order fold
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blk * 32 + lane;
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
template <typename T>
__global__ void __launch_bounds__(256)
k_colsum_final(int M, int nparts, const typename Vec<T>::A* __restrict__ part,
               typename Traits<T>::P* __restrict__ g_bias) {
  colsum_final_block<T>(M, nparts, part, g_bias, blockIdx.x);
}

// Every layer's finalize (+ bias column fold) in ONE launch: per job C / kFinRows row CTAs, then
// ceil(M / 32) bias CTAs; a CTA finds its job by binary search on the prefix.
constexpr int kFinJobs = 64;
constexpr int kFinRows = 8;  // a CTA per row made the batched launch CTA-launch bound (0.31 ms for ViT-B)
struct FinJobs {
  diagmm_dw_finalize_job j[kFinJobs];
  int start[kFinJobs + 1];
  int rows[kFinJobs];
  int n;
};
__global__ void __launch_bounds__(256)
k_dw_finalize_batched(const __grid_constant__ FinJobs P) {
  using T = __nv_bfloat16;
  int lo = 0, hi = P.n - 1;
  const int t = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const diagmm_dw_finalize_job& J = P.j[lo];
  const int local = t - P.start[lo];
  const int C = J.M > J.N ? J.M : J.N, L = J.M < J.N ? J.M : J.N;
  if (local < P.rows[lo]) {  // kFinRows = 8 candidate rows per CTA, one per warp (most are zero fills)
    const int n_act = min(*J.n_act, J.max_act);
    const int r = local * kFinRows + (threadIdx.x >> 5);
    if (r < C)
      finalize_row<T>(r, C, L, J.parts, J.partial, J.max_act, J.slot, n_act, J.alpha_soft, J.values, J.g_values,
                      J.g_soft, J.bucket, J.bucket_rows, nullptr);
  } else {
    colsum_final_block<T>(J.M, J.parts, J.colsum, J.g_bias, local - P.rows[lo]);
  }
}

int run_dw_finalize_batched(int n, const diagmm_dw_finalize_job* jobs, cudaStream_t st) {
  for (int b = 0; b < n; b += kFinJobs) {
    FinJobs P{};
    P.n = n - b < kFinJobs ? n - b : kFinJobs;
    int total = 0;
    for (int i = 0; i < P.n; ++i) {
      const diagmm_dw_finalize_job& j = jobs[b + i];
      if (j.M < 1 || j.N < 1 || j.parts < 0 || j.max_act < 0) return DIAGMM_ESHAPE;
      P.j[i] = j;
      P.start[i] = total;
      P.rows[i] = ceil_div(j.M > j.N ? j.M : j.N, kFinRows);
      total += P.rows[i] + (j.g_bias && j.colsum ? ceil_div(j.M, 32) : 0);
    }
    P.start[P.n] = total;
    k_dw_finalize_batched<<<total, 256, 0, st>>>(P);
    note_launch();
  }
  return status_from_cuda();
}

// --------------------------------------------------------------------------- dense route
// W_K (M, N) row-major in the activation type, written in ONE coalesced pass
// (no memset): entry (r, c) belongs to offset o = (r - c) mod M (tall/square,
// t = c) or (c - r) mod N (wide, t = r); a per-CTA offset -> slot table says
// whether o is active.  8 consecutive columns per thread, 16-byte stores when
// aligned.  (materialize, diagcore.py:153-159, with the weights of layers.py:235.)
constexpr int kMatRows = 2;
// TRANS: write W_K^T (N, M) instead (the B operand of the tensor-core dX).
template <typename T, bool TRANS>
__global__ void __launch_bounds__(256)
k_materialize(int M, int N, const typename Traits<T>::P* __restrict__ vals, const double* __restrict__ asoft,
              const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p, int max_act,
              T* __restrict__ w, int vec) {
  using P = typename Traits<T>::P;
  const int L = min(M, N);
  const int n_act = min(*n_act_p, max_act);
  const bool tall = M >= N;
  const int mod = tall ? M : N;
  const int R = TRANS ? N : M, Cc = TRANS ? M : N;  // output rows / cols
  const int r0 = blockIdx.x * kMatRows;
  const int chunks = (Cc + 7) / 8;
  for (int it = threadIdx.x; it < kMatRows * chunks; it += blockDim.x) {
    const int rr = it / chunks, ch = it - rr * chunks;
    const int orow = r0 + rr;
    if (orow >= R) continue;
    // branch-free: the 8 slot lookups, then the 8 value loads, all in flight
    int oo[8], tt[8];
    bool on[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ocol = ch * 8 + e;
      const int r = TRANS ? ocol : orow, c = TRANS ? orow : ocol;  // entry (r, c) of W_K
      int o = tall ? r - c : c - r;
      o = o < 0 ? o + mod : o;
      oo[e] = ocol < Cc ? o : 0;
      tt[e] = tall ? c : r;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int sl = __ldg(slot + oo[e]);
      on[e] = ch * 8 + e < Cc && sl >= 0 && sl < n_act;
    }
    P raw[8];
    double sc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      raw[e] = on[e] ? __ldg(vals + (size_t)oo[e] * L + tt[e]) : P(0);
      sc[e] = on[e] ? (asoft ? __ldg(asoft + oo[e]) : 1.0) : 0.0;
    }
    T outv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double vd = sc[e] * (double)raw[e];
      if constexpr (sizeof(T) == 8) outv[e] = (T)vd;
      else outv[e] = from_acc<T>((float)vd);
    }
    T* dst = w + (size_t)orow * Cc + ch * 8;
    if (vec && ch * 8 + 8 <= Cc) {
#pragma unroll
      for (int e = 0; e < 8; e += 16 / (int)sizeof(T))
        *reinterpret_cast<uint4*>(dst + e) = *reinterpret_cast<const uint4*>(outv + e);
    } else {
      for (int e = 0; e < 8 && ch * 8 + e < Cc; ++e) dst[e] = outv[e];
    }
  }
}

// Tiled materialize (W_K, bf16 / fp32): a CTA owns a 32 x 256 output tile,
// finds the active offsets crossing it (287 candidates, slot lookups, compacted
// in shared memory), writes their entries into a zeroed shared tile — for one
// diagonal consecutive threads read consecutive stored values — and stores the
// tile with 16-byte writes.  The per-element kernel above does a slot lookup
// and a scattered value load for every output element.
constexpr int kMTR = 32, kMTC = 256;
template <typename T>
__device__ void materialize_tile(int M, int N, const typename Traits<T>::P* __restrict__ vals, const double* __restrict__ asoft,
                    const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p, int max_act,
                    T* __restrict__ w, int vec, int tx, int ty) {
  static_assert(sizeof(T) <= 4, "tile kernel for bf16 / fp32");
  __shared__ __align__(16) T tile[kMTR][kMTC];
  __shared__ int s_list[kMTR + kMTC];
  __shared__ double s_sc[kMTR + kMTC];
  __shared__ int s_cnt;
  const int n_act = min(*n_act_p, max_act);
  const bool tall = M >= N;
  const int mod = tall ? M : N, L = tall ? N : M;
  const int r0 = ty * kMTR, c0 = tx * kMTC;
  constexpr int VW = 16 / sizeof(T);
  for (int i = threadIdx.x; i < kMTR * kMTC / VW; i += blockDim.x)
    reinterpret_cast<uint4*>(&tile[0][0])[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int lo = tall ? r0 - c0 - kMTC + 1 : c0 - r0 - kMTR + 1;
  int width = kMTR + kMTC - 1;
  if (width >= mod) { lo = 0; width = mod; }
  lo %= mod;
  lo = lo < 0 ? lo + mod : lo;
  for (int k = threadIdx.x; k < width; k += blockDim.x) {
    int o = lo + k;
    o = o >= mod ? o - mod : o;
    const int sl = __ldg(slot + o);
    if (sl >= 0 && sl < n_act) {  // order of the list is irrelevant: every entry has one writer
      const int idx = atomicAdd(&s_cnt, 1);
      s_list[idx] = o;
      s_sc[idx] = asoft ? __ldg(asoft + o) : 1.0;
    }
  }
  __syncthreads();
  const int nd = s_cnt;
  for (int it = threadIdx.x; it < nd * kMTR; it += blockDim.x) {
    const int di = it / kMTR, i = it - di * kMTR;
    const int o = s_list[di], r = r0 + i;
    if (r >= M) continue;
    int c, t;
    if (tall) { c = r - o; c = c < 0 ? c + mod : c; t = c; }
    else { c = r + o; c = c >= mod ? c - mod : c; t = r; }
    if (c < c0 || c >= c0 + kMTC || c >= N) continue;
    const double v = s_sc[di] * (double)__ldg(vals + (size_t)o * L + t);
    tile[i][c - c0] = from_acc<T>((float)v);
  }
  __syncthreads();
  const int chunks = kMTC / VW;
  for (int it = threadIdx.x; it < kMTR * chunks; it += blockDim.x) {
    const int i = it / chunks, ch = it - i * chunks;
    const int r = r0 + i, cb = c0 + ch * VW;
    if (r >= M || cb >= N) continue;
    T* dst = w + (size_t)r * N + cb;
    if (vec && cb + VW <= N) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&tile[i][ch * VW]);
    } else {
      for (int e = 0; e < VW && cb + e < N; ++e) dst[e] = tile[i][ch * VW + e];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_materialize_tiles(int M, int N, const typename Traits<T>::P* __restrict__ vals, const double* __restrict__ asoft,
                    const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p, int max_act,
                    T* __restrict__ w, int vec) {
  materialize_tile<T>(M, N, vals, asoft, slot, n_act_p, max_act, w, vec, blockIdx.x, blockIdx.y);
}

// every layer's W_K in ONE launch (the model-level pre-pass after the batched K4):
// the flat grid walks the layers' tiles; a CTA finds its layer in the tile prefix
constexpr int kMatJobs = 64;
struct MatJobs {
  diagmm_materialize_job j[kMatJobs];
  int start[kMatJobs + 1];  // first flat tile of each job
  int tiles_x[kMatJobs];
  int vec[kMatJobs];
  int n;
};
template <typename T>
__global__ void __launch_bounds__(256)
k_materialize_batched(const __grid_constant__ MatJobs P) {
  int lo = 0, hi = P.n - 1;  // the job whose [start, next start) holds this tile
  const int t = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const diagmm_materialize_job& J = P.j[lo];
  const int local = t - P.start[lo];
  materialize_tile<T>(J.M, J.N, static_cast<const typename Traits<T>::P*>(J.values), J.alpha_soft, J.slot,
                      J.n_act, J.max_act, static_cast<T*>(J.w), P.vec[lo], local % P.tiles_x[lo],
                      local / P.tiles_x[lo]);
}

// Dense dW -> per-diagonal rows, pass 1: a CTA stages a tile of dW (coalesced)
// and writes, for every ACTIVE offset crossing the tile, the unscaled entries
// gw[o, t] into row o of g_values (runs of consecutive t: coalesced).
constexpr int kGTr = 32, kGTc = 128;  // tile along the "other" axis x along t
template <typename P>
__global__ void __launch_bounds__(256)
k_gather_tiles(int M, int N, const P* __restrict__ dW, const int32_t* __restrict__ slot,
               const int32_t* __restrict__ n_act_p, P* __restrict__ g_values) {
  __shared__ P tile[kGTr][kGTc + 1];
  const bool tall = M >= N;
  const int L = min(M, N);
  // t axis = columns (tall) or rows (wide); "u" axis = the other one
  const int t0 = blockIdx.x * kGTc, u0 = blockIdx.y * kGTr;
  const int Tn = tall ? N : M, Un = tall ? M : N;
  constexpr int kPer = kGTr * kGTc / 256;  // elements per thread; all loads in flight first
  P v[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = threadIdx.x + k * 256;
    int uu, tt;
    if (tall) { uu = i / kGTc; tt = i - uu * kGTc; }   // rows = u, contiguous along t (cols)
    else { tt = i / kGTr; uu = i - tt * kGTr; }        // rows = t, contiguous along u (cols)
    const int u = u0 + uu, t = t0 + tt;
    v[k] = (u < Un && t < Tn) ? (tall ? __ldg(dW + (size_t)u * N + t) : __ldg(dW + (size_t)t * N + u)) : P(0);
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = threadIdx.x + k * 256;
    int uu, tt;
    if (tall) { uu = i / kGTc; tt = i - uu * kGTc; }
    else { tt = i / kGTr; uu = i - tt * kGTr; }
    tile[uu][tt] = v[k];
  }
  // diagonals crossing the tile: delta = uu - tt in (-(kGTc-1), kGTr-1]; offset o = (u - t) mod C
  __shared__ int s_act[kGTr + kGTc];
  const int C = max(M, N);
  const int n_act = *n_act_p;
  for (int dl = threadIdx.x; dl < kGTr + kGTc - 1; dl += blockDim.x) {
    int o = (u0 - t0 + dl - (kGTc - 1)) % C;
    o = o < 0 ? o + C : o;
    const int sl = slot[o];
    s_act[dl] = (sl >= 0 && sl < n_act) ? o : -1;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int dl = warp; dl < kGTr + kGTc - 1; dl += blockDim.x >> 5) {
    const int delta = dl - (kGTc - 1);
    const int o = s_act[dl];
    if (o < 0) continue;
    const int tt_lo = delta < 0 ? -delta : 0;
    const int tt_hi = min(kGTc, kGTr - delta);
    for (int tt = tt_lo + lane; tt < tt_hi; tt += 32) {
      const int t = t0 + tt, u = u0 + tt + delta;
      if (t < L && u < Un) g_values[(size_t)o * L + t] = tile[tt + delta][tt];
    }
  }
}

// pass 2 (per candidate row): inactive rows -> 0; active rows -> g_soft from the
// unscaled gw, then scale by alpha_soft in place (layers.py:159-165).
template <typename P>
__global__ void __launch_bounds__(256)
k_gather_finish(int C, int L, const P* __restrict__ vals, const double* __restrict__ asoft,
                const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p, P* __restrict__ g_values,
                double* __restrict__ g_soft) {
  __shared__ double red[32];
  const int i = blockIdx.x;
  const int s = slot[i];
  P* grow = g_values + (size_t)i * L;
  constexpr int W = 16 / sizeof(P);
  if (s < 0 || s >= *n_act_p) {
    if (L % W == 0 && (reinterpret_cast<uintptr_t>(g_values) & 15) == 0) {
      for (int t = threadIdx.x; t < L / W; t += blockDim.x) reinterpret_cast<uint4*>(grow)[t] = make_uint4(0, 0, 0, 0);
    } else {
      for (int t = threadIdx.x; t < L; t += blockDim.x) grow[t] = P(0);
    }
    if (g_soft && threadIdx.x == 0) g_soft[i] = 0.0;
    return;
  }
  const double sc = asoft ? asoft[i] : 1.0;
  double local = 0.0;
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    const double gw = (double)grow[t];
    local += gw * (double)vals[(size_t)i * L + t];
    grow[t] = (P)(sc * gw);
  }
  if (g_soft) {
    double tot = block_sum(local, red);
    if (threadIdx.x == 0) g_soft[i] = tot;
  }
}

// --------------------------------------------------------------------------- K1/K2 v6
// Row-tiled products, v6 (bf16, B >= 32; fp32 stays on v4).  ncu of
// the v4 kernel (profiles/r02_ncu_fma_*.txt) showed every diagonal waiting a
// full memory latency on its weights: the register ring's loads sit behind
// per-diagonal branches, so ptxas cannot count them on a scoreboard and waits
// for all of them.  v6 moves the ring into shared memory:
//  * weights are pre-scaled into a LANE-INTERLEAVED store — per 128-position
//    tile, lane l's four positions (l + 32u) are adjacent — so one diagonal of
//    one warp is 256 B (bf16) / 512 B (fp32) of contiguous memory, fetched by
//    cp.async into a per-warp D-deep ring (explicit wait_group counts: the
//    fetch of diagonal q + D - 1 overlaps the FMAs of diagonal q), and read back
//    with ONE LDS.64 / LDS.128 per lane;
//  * the staged input row is laid out so that every diagonal of a warp is a
//    single warp-uniform base column: circular rows (C + 128-column halo) for
//    the gather form and near-square scatter form, zero guard bands around the
//    L real columns for tall scatter forms (C >= L + 128) — no per-position
//    wrap or clamp in the inner loop;
//  * per diagonal a lane issues G*4 LDS.128 and G*4*VEC FMAs plus ~10 other
//    instructions: the shared-memory crossbar (one 16-byte unit per VEC FMAs)
//    stays the only bound.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// acc[r] += x[r] * w  with the bf16 weight in the low (HI = 0) or high half of w2
template <int HI>
__device__ __forceinline__ void fma_vec_h(float (&a)[8], uint4 x, uint32_t w2) {
  const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (HI == 0)
      asm("{\n.reg .b16 x0, x1, w0, w1;\n"
          "mov.b32 {x0, x1}, %2;\n"
          "mov.b32 {w0, w1}, %3;\n"
          "fma.rn.f32.bf16 %0, x0, w0, %0;\n"
          "fma.rn.f32.bf16 %1, x1, w0, %1;\n}"
          : "+f"(a[2 * i]), "+f"(a[2 * i + 1])
          : "r"(xs[i]), "r"(w2));
    else
      asm("{\n.reg .b16 x0, x1, w0, w1;\n"
          "mov.b32 {x0, x1}, %2;\n"
          "mov.b32 {w0, w1}, %3;\n"
          "fma.rn.f32.bf16 %0, x0, w1, %0;\n"
          "fma.rn.f32.bf16 %1, x1, w1, %1;\n}"
          : "+f"(a[2 * i]), "+f"(a[2 * i + 1])
          : "r"(xs[i]), "r"(w2));
  }
}

// Lane-interleaved pre-scaled weights: wil[(j * ntile + tile) * 128 + lane * 4 + u]
// = s_j * values[o_j, c(p)] at position p = tile * 128 + lane + 32u (0 where the
// reference has no entry or p >= out_w).  One thread = one lane's four weights
// (reads coalesced per u, one vector store).
constexpr int kIlJ = 4;  // diagonals per thread per pass (all their loads in flight together)
template <typename T>
__global__ void __launch_bounds__(256)
k_prescale_il(int C, int L, int out_w, int ntile, int gather, const typename Traits<T>::P* __restrict__ vals,
              const double* __restrict__ asoft, const int32_t* __restrict__ active,
              const int32_t* __restrict__ n_act_p, int max_act, typename WType<T>::type* __restrict__ wil) {
  using P = typename Traits<T>::P;
  using WT = typename WType<T>::type;
  const int n_act = min(*n_act_p, max_act);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // (tile, lane)
  if (e >= ntile * kWarp) return;
  const int tile = e >> 5, lane = e & 31;
  for (int j0 = blockIdx.y * kIlJ; j0 < n_act; j0 += gridDim.y * kIlJ) {
    int o[kIlJ];
    double sc[kIlJ];
    P v[kIlJ][4];
#pragma unroll
    for (int i = 0; i < kIlJ; ++i) o[i] = j0 + i < n_act ? __ldg(active + j0 + i) : -1;
#pragma unroll
    for (int i = 0; i < kIlJ; ++i) {
      sc[i] = (o[i] >= 0 && asoft) ? __ldg(asoft + o[i]) : 1.0;
      const P* vr = vals + (size_t)(o[i] >= 0 ? o[i] : 0) * L;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = tile * kWarpPos + lane + kWarp * u;
        int c = p;
        if (!gather) { c = p - o[i]; c = c < 0 ? c + C : c; }
        v[i][u] = (o[i] >= 0 && p < out_w && c < L) ? __ldg(vr + c) : P(0);
      }
    }
#pragma unroll
    for (int i = 0; i < kIlJ; ++i) {
      if (o[i] < 0) break;
      WT w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double x = sc[i] * (double)v[i][u];
        if constexpr (sizeof(WT) == 2) w[u] = __double2bfloat16(x);
        else w[u] = (WT)x;
      }
      WT* dst = wil + ((size_t)(j0 + i) * ntile + tile) * kWarpPos + lane * 4;
      if constexpr (sizeof(WT) == 2) {
        uint2 pk;
        pk.x = (uint32_t)__bfloat16_as_ushort(w[0]) | ((uint32_t)__bfloat16_as_ushort(w[1]) << 16);
        pk.y = (uint32_t)__bfloat16_as_ushort(w[2]) | ((uint32_t)__bfloat16_as_ushort(w[3]) << 16);
        *reinterpret_cast<uint2*>(dst) = pk;
      } else {
        *reinterpret_cast<float4*>(dst) = make_float4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

template <typename T> struct V6Ring { static constexpr int D = 8; };   // bf16: 8 x 256 B per warp
template <> struct V6Ring<float> { static constexpr int D = 8; };      // fp32: 8 x 512 B per warp
template <typename T>
__host__ __device__ constexpr int v6_wbytes() { return kWarpPos * (int)sizeof(typename WType<T>::type); }

// staged tile | fold buffer (max) ; then the per-warp weight rings ; then the active list
template <typename T>
__host__ __device__ inline size_t v6_tile_bytes(int g, int stage_w, int pw, int nw, bool cluster) {
  const size_t tile = (size_t)g * stage_w * 16;
  const size_t row = (size_t)g * vec_rows<T>() * pw * kWarpPos * sizeof(typename Vec<T>::A);
  const int dw = nw / pw;
  const size_t red = (dw > 1 || cluster) ? (size_t)dw * row + (cluster ? row : 0) : 0;
  return align16(tile > red ? tile : red);
}
template <typename T>
__host__ __device__ inline size_t v6_smem(int g, int stage_w, int pw, int nw, bool cluster, int max_act) {
  return v6_tile_bytes<T>(g, stage_w, pw, nw, cluster) + (size_t)nw * V6Ring<T>::D * v6_wbytes<T>() +
         align16((size_t)(max_act > 0 ? max_act : 1) * sizeof(int32_t));
}

// MODE: 0 gather (circular row), 1 scatter circular (zeros beyond L), 2 scatter
// with zero guard bands (C >= L + 128).  256 or 512 threads (blockDim.x);
// PW position warps x DW = warps / PW diagonal warps.
template <typename T, int G, int MODE>
__global__ void __launch_bounds__(512, 1)
k_product6(int B, int C, int L, const T* __restrict__ in, const typename WType<T>::type* __restrict__ wil,
           int ntile, const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act,
           const typename Traits<T>::P* __restrict__ bias, T* __restrict__ out, int PW, int nsplit, int stage_w,
           int vec_ok) {
  using U = typename Vec<T>::U;
  using A = typename Vec<T>::A;
  constexpr int VEC = vec_rows<T>();
  constexpr int RT = G * VEC;
  constexpr int D = V6Ring<T>::D;
  constexpr int WB = v6_wbytes<T>();
  constexpr bool kBf16 = sizeof(typename WType<T>::type) == 2;
  using WV = typename std::conditional<kBf16, uint2, float4>::type;  // one lane's four weights
  extern __shared__ __align__(128) unsigned char smem[];
  U* xs = reinterpret_cast<U*>(smem);
  A* red = reinterpret_cast<A*>(smem);  // reused after the main loop
  const bool cluster_fold = nsplit > 1;
  const int nthr = blockDim.x, nw = nthr >> 5;
  unsigned char* rings = smem + v6_tile_bytes<T>(G, stage_w, PW, nw, cluster_fold);
  int32_t* s_act = reinterpret_cast<int32_t*>(rings + nw * D * WB);
  const int n_act = min(*n_act_p, max_act);
  const int in_w = MODE == 0 ? C : L;
  const int out_w = MODE == 0 ? L : C;
  const int DW = nw / PW;
  const int t0 = blockIdx.x * PW * kWarpPos;
  const int b0 = blockIdx.y * RT;
  const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;
  const int pw = warp % PW, dw = warp / PW;
  const int p0 = t0 + pw * kWarpPos;
  const int tl = p0 / kWarpPos;

  for (int i = threadIdx.x; i < n_act; i += nthr) s_act[i] = __ldg(active + i);
  __syncthreads();
  int lo1, hi1, lo2, hi2;
  if (MODE == 0) { lo1 = 0; hi1 = n_act; lo2 = 0; hi2 = 0; }
  else scatter_ranges(s_act, n_act, C, L, p0, kWarpPos, lo1, hi1, lo2, hi2);
  const int len1 = hi1 - lo1;
  const int total = p0 < out_w ? len1 + (hi2 - lo2) : 0;
  const int per = (total + nsplit - 1) / nsplit;
  const int cb = min(total, (int)blockIdx.z * per), ce = min(total, cb + per);
  const int vb = cb + dw;
  const int nq = ce - vb > 0 ? (ce - vb + DW - 1) / DW : 0;
  unsigned char* ring = rings + warp * D * WB;
  const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(wil) + (size_t)tl * WB + lane * 16;
  const size_t jstride = (size_t)ntile * WB;
  auto jof = [&](int q) {
    const int v = vb + DW * q;
    return v < len1 ? lo1 + v : lo2 + (v - len1);
  };
  auto issue = [&](int q) {
    if (q < nq && lane * 16 < WB) cp_async16(ring + (q % D) * WB + lane * 16, wsrc + (size_t)jof(q) * jstride);
    cp_async_commit();
  };
  // warp-uniform base column of diagonal q (see the staged-row modes above)
  auto base_of = [&](int q) {
    const int o = s_act[jof(q)];
    int base;
    if (MODE == 0) {
      base = p0 + o;
      base = base >= C ? base - C : base;
    } else if (MODE == 1) {
      base = p0 + C - o;
      base = base >= C ? base - C : base;
    } else {
      int d = p0 - o;
      d = d < -(kWarpPos - 1) ? d + C : (d > L - 1 ? d - C : d);
      base = d + kWarpPos;
    }
    return base;
  };
  // the first D - 2 diagonals' weights are in flight while the rows are staged
#pragma unroll
  for (int q = 0; q < D - 2; ++q) issue(q);
  const int c0 = MODE == 2 ? C - kWarpPos : 0;
  stage_t<T, 16 / vec_rows<T>()>(xs, stage_w, stage_w, in, B, in_w, b0, G, c0, C, MODE == 0 ? C : L, vec_ok != 0);
  __syncthreads();

  A acc[G][kU][VEC];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int r = 0; r < VEC; ++r) acc[g][u][r] = A(0);

  auto fmas = [&](const U (&xv)[G][kU], const WV& w) {
    if constexpr (kBf16) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        fma_vec_h<0>(acc[g][0], xv[g][0], w.x);
        fma_vec_h<1>(acc[g][1], xv[g][1], w.x);
        fma_vec_h<0>(acc[g][2], xv[g][2], w.y);
        fma_vec_h<1>(acc[g][3], xv[g][3], w.y);
      }
    } else {
      const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int u = 0; u < kU; ++u) fma_vec(acc[g][u], xv[g][u], wv[u]);
    }
  };
  auto load_x = [&](U (&xv)[G][kU], int base) {
    const U* xr = xs + base + lane;
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int u = 0; u < kU; ++u) xv[g][u] = xr[(size_t)g * stage_w + kWarp * u];
  };
  // Two diagonals per step: both weights and all 2*G*4 input units are requested
  // before the first FMA.  The base columns of 32 diagonals are computed
  // lane-parallel once and shuffled out.
  int base_l = 0;
  int q = 0;
  for (; q + 1 < nq; q += 2) {
    if ((q & 31) == 0) base_l = q + lane < nq ? base_of(q + lane) : 0;
    __syncwarp();      // slots (q - 2) % D and (q - 1) % D were read by every lane ...
    issue(q + D - 2);  // ... before they are refilled
    issue(q + D - 1);
    cp_async_wait<D - 2>();
    __syncwarp();      // the other lanes' copies of slots q % D, (q + 1) % D are visible
    const WV w0 = *reinterpret_cast<const WV*>(ring + (q % D) * WB + lane * sizeof(WV));
    const WV w1 = *reinterpret_cast<const WV*>(ring + ((q + 1) % D) * WB + lane * sizeof(WV));
    U x0[G][kU], x1[G][kU];
    load_x(x0, __shfl_sync(0xffffffffu, base_l, q & 31));
    load_x(x1, __shfl_sync(0xffffffffu, base_l, (q + 1) & 31));
    fmas(x0, w0);
    fmas(x1, w1);
  }
  if (q < nq) {  // odd tail
    if ((q & 31) == 0) base_l = q + lane < nq ? base_of(q + lane) : 0;
    __syncwarp();
    issue(q + D - 2);
    cp_async_wait<D - 2>();
    __syncwarp();
    const WV w0 = *reinterpret_cast<const WV*>(ring + (q % D) * WB + lane * sizeof(WV));
    U x0[G][kU];
    load_x(x0, __shfl_sync(0xffffffffu, base_l, q & 31));
    fmas(x0, w0);
  }
  cp_async_wait<0>();

  if (DW == 1 && !cluster_fold) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = p0 + lane + kWarp * u;
      if (p >= out_w) continue;
      const A bb = bias ? (A)bias[p] : A(0);
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int r = 0; r < VEC; ++r) {
          const int b = b0 + g * VEC + r;
          if (b < B) out[(size_t)b * out_w + p] = from_acc<T>(acc[g][u][r] + bb);
        }
    }
    return;
  }
  // fixed-order fold of the DW diagonal slices (then the cluster ranks)
  const int TT = PW * kWarpPos;
  const int tt_shift = 31 - __clz(TT);
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int r = 0; r < VEC; ++r)
#pragma unroll
      for (int u = 0; u < kU; ++u)
        red[((size_t)dw * RT + g * VEC + r) * TT + pw * kWarpPos + lane + kWarp * u] = acc[g][u][r];
  __syncthreads();
  A* fin = red + (size_t)DW * RT * TT;
  for (int i = threadIdx.x; i < RT * TT; i += nthr) {
    const int b = i >> tt_shift, tt = i & (TT - 1);
    const int p = t0 + tt;
    A s = A(0);
    for (int w = 0; w < DW; ++w) s += red[((size_t)w * RT + b) * TT + tt];
    if (cluster_fold) {
      fin[i] = s;
    } else if (b0 + b < B && p < out_w) {
      if (bias) s += (A)bias[p];
      out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(s);
    }
  }
  if (cluster_fold) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int rank = (int)cl.block_rank(), nr = (int)cl.num_blocks();
    const int per_r = (RT * TT + nr - 1) / nr;
    const int i0 = rank * per_r, i1 = min(RT * TT, i0 + per_r);
    for (int i = i0 + threadIdx.x; i < i1; i += nthr) {
      const int b = i >> tt_shift, tt = i & (TT - 1);
      const int p = t0 + tt;
      if (b0 + b >= B || p >= out_w) continue;
      A s = A(0);
      for (int r = 0; r < nr; ++r) s += cl.map_shared_rank(fin, r)[i];
      if (bias) s += (A)bias[p];
      out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(s);
    }
    cl.sync();
  }
}

// --------------------------------------------------------------------------- K3 v6
// dW with the row loop fed by asynchronous bulk copies.  k_pack writes each
// operand once in the transposed-packed layout the FMA loop reads
// ([row group][column][VEC rows], one 16-byte unit = VEC rows of a column), so a
// CTA's share of a row group is a CONTIGUOUS run of units: the A window of its
// diagonals (circular: at most two runs) and the B tile of its positions.  One
// thread issues them as cp.async.bulk copies completing on an mbarrier, two row
// groups ahead; the FMA warps never wait on a synchronous stage.  The window
// buffer is sized for the whole circular row, so any offset spread fits (no
// direct-gather fallback).
template <typename T>
__global__ void __launch_bounds__(256)
k_pack(int B, int W, const T* __restrict__ src, typename Vec<T>::U* __restrict__ dst, int stage_w, int c0,
       int mod, int limit, int vec_ok) {
  // dst[g][col] (col < stage_w) = VEC rows of source column sc = (c0 + col) mod `mod`, zero
  // where sc >= limit or the row >= B: the packed rows of k_dw6 (stage_w = W, c0 = 0) and the
  // staged-row layouts of the product kernels (circular halo / guard bands) in global memory
  using U = typename Vec<T>::U;
  constexpr int VEC = vec_rows<T>();
  const int G = (B + VEC - 1) / VEC;
  const int chunks = (stage_w + VEC - 1) / VEC;
  const long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= (long long)G * chunks) return;
  const int g = (int)(it / chunks), ch = (int)(it - (long long)g * chunks);
  U* d = dst + (size_t)g * stage_w + (size_t)ch * VEC;
  if (vec_ok && ch * VEC + VEC <= stage_w) {
    const int sc = (int)(((long long)c0 + ch * VEC) % mod);
    const bool valid = sc < limit;
    U r[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const int b = g * VEC + i;
      r[i] = (valid && b < B) ? *reinterpret_cast<const U*>(src + (size_t)b * W + sc) : U{};
    }
    transpose_store<T>(r, d, 1);
  } else {
    T* dd = reinterpret_cast<T*>(d);
    for (int c = 0; c < VEC && ch * VEC + c < stage_w; ++c) {
      const int sc = (int)(((long long)c0 + ch * VEC + c) % mod);
      for (int i = 0; i < VEC; ++i) {
        const int b = g * VEC + i;
        dd[c * VEC + i] = (sc < limit && b < B) ? src[(size_t)b * W + sc] : T(0);
      }
    }
  }
}

constexpr int kDw6Stages = 2;
template <typename T>
__host__ __device__ inline size_t dw6_stage_units(int C, int P) { return (size_t)(C + P) + P; }
template <typename T>
__host__ __device__ inline size_t dw6_smem(int C, int P) {
  return 128 + (size_t)kDw6Stages * dw6_stage_units<T>(C, P) * 16;
}

// CTA: P = PW * 128 positions x (DW * JW) consecutive active diagonals x one
// part of the row groups.  Warp (pw, dw): positions t0 + pw*128 + lane + 32u,
// diagonals j0 + dw*JW + q.  Unscaled gw -> partial[part][j][t] (k_dw_finalize).
template <typename T, int JW>
__global__ void __launch_bounds__(512, 1)
k_dw6(int C, int L, int G, const typename Vec<T>::U* __restrict__ Ap, const typename Vec<T>::U* __restrict__ Bp,
      const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act, int PW,
      int groups_per_part, typename Vec<T>::A* __restrict__ partial) {
  using U = typename Vec<T>::U;
  using A = typename Vec<T>::A;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  U* stage0 = reinterpret_cast<U*>(smem + 128);
  const int P = PW * kWarpPos;
  const size_t su = dw6_stage_units<T>(C, P);
  const int n_act = min(*n_act_p, max_act);
  const int nw = blockDim.x >> 5, DW = nw / PW;
  const int j0 = blockIdx.y * (DW * JW);
  if (j0 >= n_act) return;
  const int nj = min(DW * JW, n_act - j0);
  const int t0 = blockIdx.x * P;
  const int nb = min(P, L - t0);  // B units of this tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pw = warp % PW, dw = warp / PW;
  const int o_first = __ldg(active + j0), o_last = __ldg(active + j0 + nj - 1);
  int ws = o_first + t0;
  ws = ws >= C ? ws - C : ws;
  const int wcols = o_last - o_first + P;  // <= C - 1 + P
  const int run1 = min(wcols, C - ws);
  const uint32_t stage_bytes = (uint32_t)(wcols + nb) * 16;
  const int g0 = blockIdx.z * groups_per_part, g1 = min(G, g0 + groups_per_part);
  auto issue = [&](int g) {  // one thread: row group g into its stage
    const int s = (g - g0) % kDw6Stages;
    U* sa = stage0 + (size_t)s * su;
    U* sb = sa + (C + P);
    mbar_expect_tx(&full[s], stage_bytes);
    const U* arow = Ap + (size_t)g * C;
    bulk_g2s(sa, arow + ws, (uint32_t)run1 * 16, &full[s]);
    if (wcols > run1) bulk_g2s(sa + run1, arow, (uint32_t)(wcols - run1) * 16, &full[s]);
    bulk_g2s(sb, Bp + (size_t)g * L + t0, (uint32_t)nb * 16, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDw6Stages; ++s) mbar_init(&full[s], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int g = g0; g < min(g1, g0 + kDw6Stages); ++g) issue(g);
  int oq[JW];
#pragma unroll
  for (int q = 0; q < JW; ++q) {
    const int jl = dw * JW + q;
    oq[q] = jl < nj ? __ldg(active + j0 + jl) - o_first : -1;
  }
  A acc[JW][kU];
#pragma unroll
  for (int q = 0; q < JW; ++q)
#pragma unroll
    for (int u = 0; u < kU; ++u) acc[q][u] = A(0);
  const int pbase = pw * kWarpPos + lane;
  for (int g = g0; g < g1; ++g) {
    const int s = (g - g0) % kDw6Stages;
    mbar_wait(&full[s], (uint32_t)(((g - g0) / kDw6Stages) & 1));
    const U* sa = stage0 + (size_t)s * su;
    const U* sb = sa + (C + P);
    U bm[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) bm[u] = sb[pbase + kWarp * u];
    const U* arow = sa + pbase;
#pragma unroll
    for (int q = 0; q < JW; ++q) {
      if (oq[q] < 0) continue;
#pragma unroll
      for (int u = 0; u < kU; ++u) Vec<T>::dot(acc[q][u], arow[oq[q] + kWarp * u], bm[u]);
    }
    __syncthreads();  // every warp is done with stage s ...
    if (threadIdx.x == 0 && g + kDw6Stages < g1) {
      fence_proxy_async();  // ... before the async proxy refills it
      issue(g + kDw6Stages);
    }
  }
#pragma unroll
  for (int q = 0; q < JW; ++q) {
    if (oq[q] < 0) continue;
    const int j = j0 + dw * JW + q;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = t0 + pbase + kWarp * u;
      if (t < L) partial[((size_t)blockIdx.z * max_act + j) * L + t] = acc[q][u];
    }
  }
}

// --------------------------------------------------------------------------- packed-direct (small B)
// bf16, B = 5..8 (use_pk): the activations of the call are packed ONCE into the
// staged-row layout of the v6 kernels (k_pack: VEC rows per 16-byte unit, circular
// halo or guard bands) in global memory; at this size the packed rows (one 8-row
// group x (C + 128) units) stay resident in each SM's L1, so the FMA loop reads its
// input units with LDG.128 straight from L1 and no CTA stages anything.  Weights are
// formed in the kernel from the stored values (a per-warp cp.async ring of the
// diagonal's 128 raw values, 4-byte copies placed lane-interleaved, zero-filled where
// the reference has no entry) and alpha_soft: no pre-scale launch.
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
constexpr int kPkRing = 8;                      // diagonals in flight per warp
constexpr int kPkSlot = kWarpPos * 4;           // 128 fp32 values
template <typename T>
__host__ __device__ inline size_t pk_smem(int g, bool cluster, int max_act) {
  const size_t rings = (size_t)kWarps * kPkRing * kPkSlot;
  const size_t row = (size_t)g * vec_rows<T>() * kWarpPos * sizeof(typename Vec<T>::A);
  const size_t red = (size_t)kWarps * row + (cluster ? row : 0);
  return rings + align16(red) + align16((size_t)(max_act > 0 ? max_act : 1) * sizeof(int32_t));
}

template <typename T, int G, int MODE>
__global__ void __launch_bounds__(kThreads)
k_product_pk(int B, int C, int L, const typename Vec<T>::U* __restrict__ xp, int stage_w,
             const typename Traits<T>::P* __restrict__ vals, const double* __restrict__ asoft,
             const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act,
             const typename Traits<T>::P* __restrict__ bias, T* __restrict__ out, int nsplit) {
  using U = typename Vec<T>::U;
  using A = typename Vec<T>::A;
  using P = typename Traits<T>::P;
  constexpr int VEC = vec_rows<T>();
  constexpr int RT = G * VEC;
  constexpr int D = kPkRing;
  static_assert(sizeof(P) == 4, "packed-direct kernels take fp32 parameters");
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* rings = smem;
  A* red = reinterpret_cast<A*>(smem + (size_t)kWarps * D * kPkSlot);
  const bool cluster_fold = nsplit > 1;
  int32_t* s_act = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(red) +
                                              align16((size_t)(kWarps + (cluster_fold ? 1 : 0)) * RT * kWarpPos *
                                                      sizeof(A)));
  const int n_act = min(*n_act_p, max_act);
  const int out_w = MODE == 0 ? L : C;
  const int p0 = blockIdx.x * kWarpPos;
  const int b0 = blockIdx.y * RT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const U* xg = xp + (size_t)blockIdx.y * G * stage_w;
  for (int i = threadIdx.x; i < n_act; i += kThreads) s_act[i] = __ldg(active + i);
  __syncthreads();
  int lo1, hi1, lo2, hi2;
  if (MODE == 0) { lo1 = 0; hi1 = n_act; lo2 = 0; hi2 = 0; }
  else scatter_ranges(s_act, n_act, C, L, p0, kWarpPos, lo1, hi1, lo2, hi2);
  const int len1 = hi1 - lo1;
  const int total = len1 + (hi2 - lo2);
  const int per = (total + nsplit - 1) / nsplit;
  const int cb = min(total, (int)blockIdx.z * per), ce = min(total, cb + per);
  const int vb = cb + warp;
  const int nq = ce - vb > 0 ? (ce - vb + kWarps - 1) / kWarps : 0;
  unsigned char* ring = rings + warp * D * kPkSlot;
  auto jof = [&](int q) {
    const int v = vb + kWarps * q;
    return v < len1 ? lo1 + v : lo2 + (v - len1);
  };
  auto issue = [&](int q) {  // the diagonal's values at this lane's 4 positions -> slot[lane][u]
    if (q < nq) {
      const int o = s_act[jof(q)];
      const P* vr = vals + (size_t)o * L;
      unsigned char* dst = ring + (q % D) * kPkSlot + lane * 16;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = p0 + lane + kWarp * u;
        int c = p;
        if (MODE != 0) { c = p - o; c = c < 0 ? c + C : c; }
        const bool ok = p < out_w && c < L;
        cp_async4(dst + u * 4, ok ? vr + c : vals, ok);
      }
    }
    cp_async_commit();
  };
  auto base_of = [&](int q, float& sc) {
    const int o = s_act[jof(q)];
    sc = asoft ? (float)__ldg(asoft + o) : 1.f;
    int base;
    if (MODE == 0) {
      base = p0 + o;
      base = base >= C ? base - C : base;
    } else if (MODE == 1) {
      base = p0 + C - o;
      base = base >= C ? base - C : base;
    } else {
      int d = p0 - o;
      d = d < -(kWarpPos - 1) ? d + C : (d > L - 1 ? d - C : d);
      base = d + kWarpPos;
    }
    return base;
  };
#pragma unroll
  for (int q = 0; q < D - 2; ++q) issue(q);
  A acc[G][kU][VEC];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int r = 0; r < VEC; ++r) acc[g][u][r] = A(0);
  auto load_x = [&](U (&xv)[G][kU], int base) {
    const U* xr = xg + base + lane;
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int u = 0; u < kU; ++u) xv[g][u] = __ldg(xr + (size_t)g * stage_w + kWarp * u);
  };
  auto fmas = [&](const U (&xv)[G][kU], float4 v, float sc) {
    if constexpr (sizeof(T) == 2) {
      const __nv_bfloat162 w01 = __floats2bfloat162_rn(sc * v.x, sc * v.y);
      const __nv_bfloat162 w23 = __floats2bfloat162_rn(sc * v.z, sc * v.w);
      const uint32_t a = *reinterpret_cast<const uint32_t*>(&w01), b = *reinterpret_cast<const uint32_t*>(&w23);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        fma_vec_h<0>(acc[g][0], xv[g][0], a);
        fma_vec_h<1>(acc[g][1], xv[g][1], a);
        fma_vec_h<0>(acc[g][2], xv[g][2], b);
        fma_vec_h<1>(acc[g][3], xv[g][3], b);
      }
    } else {
      const float wv[4] = {sc * v.x, sc * v.y, sc * v.z, sc * v.w};
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int u = 0; u < kU; ++u) fma_vec(acc[g][u], xv[g][u], wv[u]);
    }
  };
  int base_l = 0;
  float sc_l = 0.f;
  int q = 0;
  for (; q + 1 < nq; q += 2) {
    if ((q & 31) == 0 && q + lane < nq) base_l = base_of(q + lane, sc_l);
    U x0[G][kU], x1[G][kU];
    load_x(x0, __shfl_sync(0xffffffffu, base_l, q & 31));
    load_x(x1, __shfl_sync(0xffffffffu, base_l, (q + 1) & 31));
    const float s0 = __shfl_sync(0xffffffffu, sc_l, q & 31), s1 = __shfl_sync(0xffffffffu, sc_l, (q + 1) & 31);
    __syncwarp();
    issue(q + D - 2);
    issue(q + D - 1);
    cp_async_wait<D - 2>();
    __syncwarp();
    const float4 v0 = *reinterpret_cast<const float4*>(ring + (q % D) * kPkSlot + lane * 16);
    const float4 v1 = *reinterpret_cast<const float4*>(ring + ((q + 1) % D) * kPkSlot + lane * 16);
    fmas(x0, v0, s0);
    fmas(x1, v1, s1);
  }
  if (q < nq) {
    if ((q & 31) == 0 && q + lane < nq) base_l = base_of(q + lane, sc_l);
    U x0[G][kU];
    load_x(x0, __shfl_sync(0xffffffffu, base_l, q & 31));
    const float s0 = __shfl_sync(0xffffffffu, sc_l, q & 31);
    __syncwarp();
    issue(q + D - 2);
    cp_async_wait<D - 2>();
    __syncwarp();
    const float4 v0 = *reinterpret_cast<const float4*>(ring + (q % D) * kPkSlot + lane * 16);
    fmas(x0, v0, s0);
  }
  cp_async_wait<0>();
  // fixed-order fold of the 8 diagonal warps, then (nsplit > 1) the cluster ranks
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int r = 0; r < VEC; ++r)
#pragma unroll
      for (int u = 0; u < kU; ++u)
        red[((size_t)warp * RT + g * VEC + r) * kWarpPos + lane + kWarp * u] = acc[g][u][r];
  __syncthreads();
  A* fin = red + (size_t)kWarps * RT * kWarpPos;
  for (int i = threadIdx.x; i < RT * kWarpPos; i += kThreads) {
    const int b = i >> 7, tt = i & (kWarpPos - 1);
    const int p = p0 + tt;
    A s = A(0);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[((size_t)w * RT + b) * kWarpPos + tt];
    if (cluster_fold) {
      fin[i] = s;
    } else if (b0 + b < B && p < out_w) {
      if (bias) s += (A)bias[p];
      out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(s);
    }
  }
  if (cluster_fold) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int rank = (int)cl.block_rank(), nr = (int)cl.num_blocks();
    const int per_r = (RT * kWarpPos + nr - 1) / nr;
    const int i0 = rank * per_r, i1 = min(RT * kWarpPos, i0 + per_r);
    for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
      const int b = i >> 7, tt = i & (kWarpPos - 1);
      const int p = p0 + tt;
      if (b0 + b >= B || p >= out_w) continue;
      A s = A(0);
      for (int r = 0; r < nr; ++r) s += cl.map_shared_rank(fin, r)[i];
      if (bias) s += (A)bias[p];
      out[(size_t)(b0 + b) * out_w + p] = from_acc<T>(s);
    }
    cl.sync();
  }
}

// ================================================================ host side
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

struct ProductPlan {
  int g, pw, gx, gy, nsplit;
  size_t smem;
  bool fw;  // fused weights (no k_prescale); nsplit > 1 then means a cluster fold
};
template <typename T>
static size_t product_smem(int g, int cols, int max_act, bool cluster = false) {
  return product_tile_bytes<T>(g, cols, cluster) + align16((size_t)(max_act > 0 ? max_act : 1) * sizeof(int32_t));
}

template <typename T>
static int w_ld(int out_w) {  // leading dimension of the compact weight store (16-byte rows)
  constexpr int e = 16 / (int)sizeof(typename WType<T>::type);
  return (out_w + e - 1) / e * e;
}

// Tile choice: among (G row groups, PW position warps) whose grid gives at
// least one CTA per SM, take the one with the best wave quantisation at two
// resident CTAs per SM (ties: more rows, then more positions per CTA — less
// staging and fewer folds).  Tiny batches split the diagonal list across CTAs.
template <typename T>
static ProductPlan plan_product(int B, int out_w, int cols, int max_act) {
  constexpr int VEC = vec_rows<T>();
  const size_t kSmemMax = 113 * 1024;  // two CTAs per SM
  const int sms = num_sms();
  const double slots = 2.0 * sms;
  const int pw_max = ceil_div(out_w, kWarpPos);
  ProductPlan best{0, 0, 0, 0, 1, 0, false};
  double best_eff = -1.0;
  for (int g : {2, 1}) {
    const size_t sm = product_smem<T>(g, cols, max_act);
    if (sm > (g == 2 ? kSmemMax : 220 * 1024)) continue;
    for (int pw : {8, 4, 2, 1}) {
      if (pw > pw_max && pw > 1) continue;
      const long long ctas = (long long)ceil_div(out_w, pw * kWarpPos) * ceil_div(B, g * VEC);
      if (ctas < sms) continue;
      const double waves = ctas / slots;
      const double eff = waves / std::ceil(waves) - 0.02 * (g == 1) - 0.01 * (pw < 4);
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        best = {g, pw, ceil_div(out_w, pw * kWarpPos), ceil_div(B, g * VEC), 1, sm, false};
      }
    }
  }
  // row-tiled: pre-scaled weights (FW measured slower here: cfg 1 fp32 fwd
  // 35.2 vs 33.2 us, 4096^2 B=1024 bf16 fwd 415 vs 276 us)
  if (best.g) return best;
  // few rows: PW = 1, the diagonal list split over a cluster of at most 8 CTAs
  // that fold through distributed shared memory, weights formed in the kernel
  // (FW): one launch, no prescale pass, no partial buffer (B = 8 at 4096^2:
  // 15 us vs 28 us with prescale + split partials + k_split_reduce)
  const bool fw = true;
  ProductPlan p{1, 1, ceil_div(out_w, kWarpPos), ceil_div(B, VEC), 1, 0, fw};
  const long long ctas = (long long)p.gx * p.gy;
  // as many splits as fit ONE wave (a second, nearly empty wave doubles the time)
  const int ns = ctas >= (long long)slots ? 1 : (int)((long long)slots / ctas);
  int max_ns = max_act / 16 > 1 ? max_act / 16 : 1;
  if (fw && max_ns > 8) max_ns = 8;
  p.nsplit = ns < max_ns ? ns : max_ns;
  p.smem = product_smem<T>(1, cols, max_act, fw && p.nsplit > 1);
  if (p.smem > 220 * 1024) return best;
  return p;
}

template <typename T, int G, bool GA, bool FW>
static void launch_product(const ProductPlan& p, cudaStream_t st, int B, int C, int L, const T* in,
                           const typename WType<T>::type* w, int ldw, const typename Traits<T>::P* vals,
                           const double* asoft, const int32_t* active, const int32_t* n_act, int max_act,
                           const typename Traits<T>::P* bias, T* out, typename Vec<T>::A* part, int vec_ok) {
  auto k = k_product<T, G, GA, FW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.gx, p.gy, p.nsplit);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (FW && p.nsplit > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = p.nsplit;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaLaunchKernelEx(&cfg, k, B, C, L, in, w, ldw, vals, asoft, active, n_act, max_act, bias, out, part, p.pw,
                     p.nsplit, vec_ok);
  note_launch();
}

// largest batch the one-launch few-rows kernel (k_product_rows) takes
static int rows_max_b() {
  static int v = -1;
  if (v < 0) {
    // measured (4096^2, 90 %, bf16): B = 1 fwd 6.0 vs 12.9 us (narrow kernel + reduce),
    // B = 8 15.7 vs 13.4 us (the cluster-split staged kernel keeps B > 4)
    const char* e = getenv("DIAGMM_ROWS_MAX_B");
    v = e ? atoi(e) : 4;
  }
  return v;
}

// largest batch the narrow (staging-free) product kernels take (row blocks of 8)
static int narrow_max_b() {
  static int v = -1;
  if (v < 0) {
    // measured (4096^2, 90 %): the staging-free kernel wins at B <= 4, the
    // staged k_product from B = 8 (28 vs 52 us)
    const char* e = getenv("DIAGMM_NARROW_MAX_B");
    v = e ? atoi(e) : 4;
  }
  return v;
}

static int narrow_chunks(int out_w, int max_act, int B = 1) {
  const int blocks = ceil_div(out_w, kWarpPos) * ceil_div(B > 0 ? B : 1, kNarrowB);
  int nc = ceil_div(2 * num_sms(), blocks);
  const int max_nc = max_act / 32 > 1 ? max_act / 32 : 1;  // >= 4 diagonals per warp
  return nc < max_nc ? nc : max_nc;
}

template <typename T>
static int run_product_narrow(bool gather, int B, int C, int L, const void* in, const void* vals, const double* asoft,
                              const int32_t* active, const int32_t* n_act, int max_act, const void* bias, void* out,
                              typename Vec<T>::A* part, cudaStream_t st) {
  using P = typename Traits<T>::P;
  const int out_w = gather ? L : C;
  const int nc = narrow_chunks(out_w, max_act, B);
  dim3 grid(ceil_div(out_w, kWarpPos), nc, ceil_div(B, kNarrowB));
  auto tin = static_cast<const T*>(in);
  auto tv = static_cast<const P*>(vals);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
#define DIAGMM_NARROW(BT)                                                                                       \
  if (gather)                                                                                                   \
    k_product_narrow<T, BT, true><<<grid, kThreads, 0, st>>>(B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to, part, nc);  \
  else                                                                                                          \
    k_product_narrow<T, BT, false><<<grid, kThreads, 0, st>>>(B, C, L, tin, tv, asoft, active, n_act, max_act, tb, to, part, nc);
  if (B <= 1) { DIAGMM_NARROW(1) }
  else if (B <= 2) { DIAGMM_NARROW(2) }
  else if (B <= 4) { DIAGMM_NARROW(4) }
  else { DIAGMM_NARROW(8) }  // B > 8: row blocks of 8 along grid.z
#undef DIAGMM_NARROW
  note_launch();
  if (nc > 1) {
    launch_split_reduce<T>(B, out_w, nc, part, tb, to, st);
    note_launch();
  }
  return status_from_cuda();
}

// ---- v6 planner: staged-row mode and (G, warps, PW, nsplit) by a per-SM cost model
struct Plan6 {
  int g = 0, nw = 0, pw = 0, ns = 1, gx = 0, gy = 0, stage_w = 0, mode = 0;
  size_t smem = 0;
};
// smallest batch routed to v6 (0 = never): below it the cluster-split FW kernel,
// which needs no pre-scale pass, is faster (4096^2 90 % bf16, B = 8: 16 vs 19.5 us)
static int product_v6_min_b() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DIAGMM_PRODUCT_V6");
    const char* m = getenv("DIAGMM_V6_MIN_B");
    v = (e && atoi(e) == 0) ? 0 : (m ? atoi(m) : 32);
  }
  return v;
}
template <typename T>
static Plan6 plan_product6(bool gather, int B, int C, int L, int max_act) {
  constexpr int VEC = vec_rows<T>();
  const int out_w = gather ? L : C;
  Plan6 best;
  const int mode = gather ? 0 : (C >= L + kWarpPos ? 2 : 1);
  const int stage_w = mode == 2 ? (L + 2 * kWarpPos + VEC - 1) / VEC * VEC : C + kWarpPos;
  const double n = max_act > 0 ? max_act : 1;
  // diagonals touching one 128-position tile
  const double ndiag = gather ? n : n * std::min(1.0, (L + kWarpPos - 1.0) / C);
  const double fma_rate = sizeof(T) == 2 ? 64.0 : 32.0;  // FMA / clk / SM at the shared-memory bound
  const int sms = num_sms();
  const size_t smem_sm = 228 * 1024;
  double best_t = 1e30;
  const int gs[2] = {2, 1};  // fp32 G = 4 spills with two diagonals' units in flight
  const int ngs = 2;
  for (int gi = 0; gi < ngs; ++gi) {
    const int g = gs[gi];
    const int rt = g * VEC;
    for (int nw : {8, 16}) {
      for (int pw : {16, 8, 4, 2, 1}) {
        if (pw > nw || (pw > 1 && (pw / 2) * kWarpPos >= out_w)) continue;
        const int dw = nw / pw;
        for (int ns : {1, 2, 4, 8}) {
          if (ns > 1 && ndiag / ns < 4.0 * dw) break;
          const size_t sm = v6_smem<T>(g, stage_w, pw, nw, ns > 1, max_act);
          if (sm > 227 * 1024) continue;
          int res = (int)(smem_sm / (sm + 1024));
          res = std::min(res, 2048 / (nw * 32));
          res = std::min(res, 65536 / (nw * 32 * 128));  // 128 registers per thread
          if (res < 1) continue;
          const long long gx = ceil_div(out_w, pw * kWarpPos), gy = ceil_div(B, rt);
          const long long ctas = gx * gy * ns;
          // resident warps per SM hide the LDS -> FMA latency: below 16 the rate drops
          const double per_sm = std::min<double>(res, std::ceil((double)ctas / sms));
          const double warps = per_sm * nw;
          const double rate = fma_rate * std::min(1.0, warps / 16.0);
          const double work = pw * kWarpPos * (double)rt * ndiag / ns;  // FMAs per CTA
          const double stage = (double)g * stage_w * 16 / 64.0;
          const double fold = (dw > 1 || ns > 1) ? dw * (double)rt * pw * kWarpPos * 4 * 2 / 128.0 +
                                                       (ns > 1 ? (double)rt * pw * kWarpPos * 4 * ns / 64.0 : 0)
                                                 : 0.0;
          const double waves = std::ceil((double)ctas / (res * (double)sms));
          const double t = waves * (per_sm * work / rate + stage + fold + 1500.0);
          if (t < best_t * 0.999) {
            best_t = t;
            best.g = g; best.nw = nw; best.pw = pw; best.ns = ns; best.gx = (int)gx; best.gy = (int)gy;
            best.stage_w = stage_w; best.mode = mode; best.smem = sm;
          }
        }
      }
    }
  }
  return best;
}
template <typename T>
static size_t v6_wil_bytes(bool gather, int C, int L, int max_act) {
  const int out_w = gather ? L : C;
  return align16((size_t)(max_act > 0 ? max_act : 1) * ceil_div(out_w, kWarpPos) * kWarpPos *
                 sizeof(typename WType<T>::type));
}

template <typename T, int G, int MODE>
static void launch_product6(const Plan6& p, cudaStream_t st, int B, int C, int L, const T* in,
                            const typename WType<T>::type* wil, int ntile, const int32_t* active,
                            const int32_t* n_act, int max_act, const typename Traits<T>::P* bias, T* out,
                            int vec_ok) {
  auto k = k_product6<T, G, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.gx, p.gy, p.ns);
  cfg.blockDim = dim3(p.nw * kWarp);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (p.ns > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = p.ns;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaLaunchKernelEx(&cfg, k, B, C, L, in, wil, ntile, active, n_act, max_act, bias, out, p.pw, p.ns, p.stage_w,
                     vec_ok);
  note_launch();
}

template <typename T, int G>
static void launch_product6_m(const Plan6& p, cudaStream_t st, int B, int C, int L, const T* in,
                              const typename WType<T>::type* wil, int ntile, const int32_t* active,
                              const int32_t* n_act, int max_act, const typename Traits<T>::P* bias, T* out,
                              int vec_ok) {
  if (p.mode == 0) launch_product6<T, G, 0>(p, st, B, C, L, in, wil, ntile, active, n_act, max_act, bias, out, vec_ok);
  else if (p.mode == 1) launch_product6<T, G, 1>(p, st, B, C, L, in, wil, ntile, active, n_act, max_act, bias, out, vec_ok);
  else launch_product6<T, G, 2>(p, st, B, C, L, in, wil, ntile, active, n_act, max_act, bias, out, vec_ok);
}

template <typename T>
static int run_product6(bool gather, int B, int C, int L, const void* in, const void* vals, const double* asoft,
                        const int32_t* active, const int32_t* n_act, int max_act, const void* bias, void* out,
                        void* ws, cudaStream_t st) {
  using P = typename Traits<T>::P;
  using WT = typename WType<T>::type;
  constexpr int VEC = vec_rows<T>();
  const int out_w = gather ? L : C, in_w = gather ? C : L;
  Plan6 p = plan_product6<T>(gather, B, C, L, max_act);
  if (const char* f = getenv("DIAGMM_V6_FORCE")) {  // "G,warps,PW,nsplit" (tuning experiments)
    int g, nw, pw, ns;
    if (sscanf(f, "%d,%d,%d,%d", &g, &nw, &pw, &ns) == 4) {
      p.g = g; p.nw = nw; p.pw = pw; p.ns = ns;
      p.gx = ceil_div(out_w, pw * kWarpPos);
      p.gy = ceil_div(B, g * VEC);
      p.smem = v6_smem<T>(g, p.stage_w, pw, nw, ns > 1, max_act);
    }
  }
  if (p.g == 0) return DIAGMM_ETOOLARGE;
  if (getenv("DIAGMM_V6_DEBUG"))
    fprintf(stderr, "[v6] %s B=%d C=%d L=%d k=%d: G=%d warps=%d PW=%d ns=%d grid=%dx%dx%d mode=%d smem=%zu\n",
            gather ? "gather" : "scatter", B, C, L, max_act, p.g, p.nw, p.pw, p.ns, p.gx, p.gy, p.ns, p.mode, p.smem);
  const int ntile = ceil_div(out_w, kWarpPos);
  WT* wil = static_cast<WT*>(ws);
  if (max_act > 0) {
    const int jb = ceil_div(max_act, kIlJ);
    dim3 grid(ceil_div(ntile * kWarp, 256), jb < 65535 ? jb : 65535);
    k_prescale_il<T><<<grid, 256, 0, st>>>(C, L, out_w, ntile, gather ? 1 : 0, static_cast<const P*>(vals), asoft,
                                           active, n_act, max_act, wil);
    note_launch();
  }
  const int vec_ok = in_w % VEC == 0 && C % VEC == 0 && aligned16(in);
  auto tin = static_cast<const T*>(in);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
  if (p.g == 1) launch_product6_m<T, 1>(p, st, B, C, L, tin, wil, ntile, active, n_act, max_act, tb, to, vec_ok);
  else launch_product6_m<T, 2>(p, st, B, C, L, tin, wil, ntile, active, n_act, max_act, tb, to, vec_ok);
  return status_from_cuda();
}

// ---- packed-direct small-batch products (k_pack + k_product_pk)
// Batches the packed-direct products take: bf16 5..8 (one 8-row unit) with >= 128
// diagonals.  Warm 4096^2 90 %: B = 8 fwd 10.3 vs 13.7 us (cluster-split staged kernel)
// and 15.9 us (k_product_rows); B = 1..4 stay on k_product_rows (6.3 vs 10.1 us at
// B = 1), B >= 12 on the staged kernels (16.6 vs 22.8 us at B = 16: two 8-row units of
// packed input no longer fit beside the rings in L1).  DIAGMM_PK_MIN_B /
// DIAGMM_PK_MAX_B override (0 disables).
template <typename T>
static bool use_pk(int B) {
  if constexpr (sizeof(T) != 2) {
    return false;
  } else {
    static int lo = -1, hi = -1;
    if (lo < 0) {
      const char* a = getenv("DIAGMM_PK_MIN_B");
      const char* b = getenv("DIAGMM_PK_MAX_B");
      lo = a ? atoi(a) : 5;
      hi = b ? atoi(b) : 8;
      if (hi > 2 * vec_rows<T>()) hi = 2 * vec_rows<T>();
    }
    return B > 0 && B >= lo && B <= hi;
  }
}
struct PkRows {
  int mode, stage_w, c0, mod, limit;
};
static PkRows pk_rows(bool gather, int C, int L, int vec) {
  PkRows r;
  r.mode = gather ? 0 : (C >= L + kWarpPos ? 2 : 1);
  if (r.mode == 2) {
    r.stage_w = (L + 2 * kWarpPos + vec - 1) / vec * vec;
    r.c0 = C - kWarpPos; r.mod = C; r.limit = L;
  } else {
    r.stage_w = C + kWarpPos;
    r.c0 = 0; r.mod = C; r.limit = gather ? C : L;
  }
  return r;
}
template <typename T>
static size_t pk_product_workspace(bool gather, int B, int C, int L) {
  constexpr int VEC = vec_rows<T>();
  const PkRows r = pk_rows(gather, C, L, VEC);
  return align16((size_t)ceil_div(B > 0 ? B : 1, VEC) * r.stage_w * 16);
}
template <typename T, int G, int MODE>
static void launch_product_pk(int ns, size_t sm, cudaStream_t st, int B, int C, int L, const typename Vec<T>::U* xp,
                              int stage_w, const typename Traits<T>::P* vals, const double* asoft,
                              const int32_t* active, const int32_t* n_act, int max_act,
                              const typename Traits<T>::P* bias, T* out, int ntile) {
  auto k = k_product_pk<T, G, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ntile, 1, ns);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (ns > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = ns;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaLaunchKernelEx(&cfg, k, B, C, L, xp, stage_w, vals, asoft, active, n_act, max_act, bias, out, ns);
  note_launch();
}

template <typename T>
static int run_product_pk(bool gather, int B, int C, int L, const void* in, const void* vals, const double* asoft,
                          const int32_t* active, const int32_t* n_act, int max_act, const void* bias, void* out,
                          void* ws, cudaStream_t st) {
  using P = typename Traits<T>::P;
  using U = typename Vec<T>::U;
  constexpr int VEC = vec_rows<T>();
  const int in_w = gather ? C : L, out_w = gather ? L : C;
  const PkRows r = pk_rows(gather, C, L, VEC);
  const int G = ceil_div(B, VEC);
  U* xp = static_cast<U*>(ws);
  const int vec_ok = in_w % VEC == 0 && C % VEC == 0 && r.c0 % VEC == 0 && r.limit % VEC == 0 && aligned16(in);
  k_pack<T><<<ceil_div((long long)G * ceil_div(r.stage_w, VEC), 256), 256, 0, st>>>(
      B, in_w, static_cast<const T*>(in), xp, r.stage_w, r.c0, r.mod, r.limit, vec_ok);
  note_launch();
  const int ntile = ceil_div(out_w, kWarpPos);
  const double ndiag = gather ? (double)max_act : max_act * std::min(1.0, (L + kWarpPos - 1.0) / C);
  int ns = 1;
  while (ns < 8 && (long long)ntile * ns * 2 <= 2LL * num_sms() && ndiag / (2.0 * ns * kWarps) >= 4.0) ns *= 2;
  const size_t sm = pk_smem<T>(G, ns > 1, max_act);
  if (sm > 227 * 1024) return DIAGMM_ETOOLARGE;
  auto tv = static_cast<const P*>(vals);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
#define DIAGMM_PK(GG, MM)                                                                                      \
  if (G == GG && r.mode == MM)                                                                                 \
    launch_product_pk<T, GG, MM>(ns, sm, st, B, C, L, xp, r.stage_w, tv, asoft, active, n_act, max_act, tb, to, \
                                 ntile);
  DIAGMM_PK(1, 0) DIAGMM_PK(1, 1) DIAGMM_PK(1, 2) DIAGMM_PK(2, 0) DIAGMM_PK(2, 1) DIAGMM_PK(2, 2)
#undef DIAGMM_PK
  return status_from_cuda();
}

// workspace = [compact weights (max_act x ldw) | split partials]
// the fp32 tensor-core route (3xTF32, tf32_kernels.cu)
int tf32x3_min_b();
size_t tf32_product_workspace(bool gather, int B, int C, int L);
int run_product_tf32(bool gather, int B, int C, int L, const float* in, const float* vals, const double* asoft,
                     const int32_t* active, const int32_t* n_act, int max_act, const float* bias, float* out,
                     void* ws, cudaStream_t st);
size_t tf32_dw_workspace(int M, int N, int B);
int run_dw_tf32(int M, int N, int B, const float* dy, const float* x, const int32_t* active, const int32_t* n_act,
                int max_act, float* partial, void* ws, cudaStream_t st);
// fp32 on the tensor cores (3xTF32) when it beats the FMA kernels (B200,
// tools/tf32_time.py warm and bench.py's cold-L2 per-op timing, profiles/r02_tf32x3.txt):
// products from B = 512, and from B = 256 when the output is at least as wide as the
// input (scatter orientation or square: config 1 fwd 30.2 -> 23.0 us warm, 34.7 -> 32.0
// cold; the narrow-output gather product needs a 12-way split-K there and loses cold,
// 27.8 vs 32.6 us); dW from B = 512, or from B = 256 on layers of >= 8 M candidates.
// DIAGMM_TF32X3_MIN_B=n replaces the rules by B >= n (0: never).
template <typename T>
static bool use_tf32(int B, int C, int L, bool dw, bool gather = false) {
  if (!std::is_same<T, float>::value || B < 1) return false;
  const int m = tf32x3_min_b();
  if (m >= 0) return m > 0 && B >= m;
  if (!dw) return B >= 512 || (B >= 256 && (!gather || C == L));
  return B >= 512 || (B >= 256 && (long long)C * L >= (8LL << 20));
}

template <typename T>
size_t product_workspace(bool gather, int B, int C, int L, int max_act) {
  using A = typename Vec<T>::A;
  const int out_w = gather ? L : C, cols = gather ? C + kHalo : scatter_cols<T>(L);
  ProductPlan p = plan_product<T>(B > 0 ? B : 1, out_w, cols, max_act);
  const size_t wbytes = align16((size_t)(max_act > 0 ? max_act : 1) * w_ld<T>(out_w) * sizeof(typename WType<T>::type));
  const size_t narrow = B <= narrow_max_b()
                            ? (size_t)narrow_chunks(out_w, max_act, B) * B * out_w * sizeof(A) : 0;
  size_t wide = wbytes + (p.nsplit > 1 ? (size_t)p.nsplit * B * out_w * sizeof(A) : 0);
  if constexpr (sizeof(T) <= 4) {
    const size_t v6 = v6_wil_bytes<T>(gather, C, L, max_act);
    wide = wide > v6 ? wide : v6;
    if (sizeof(T) == 2 && use_pk<T>(B)) {
      const size_t pk = pk_product_workspace<T>(gather, B, C, L);
      wide = wide > pk ? wide : pk;
    }
  }
  if (use_tf32<T>(B, C, L, false, gather)) {
    const size_t tf = tf32_product_workspace(gather, B, C, L);
    wide = wide > tf ? wide : tf;
  }
  return wide > narrow ? wide : narrow;
}

template <typename T>
int run_product(bool gather, int B, int C, int L, const void* in, const void* vals, const double* asoft,
                const int32_t* active, const int32_t* n_act, int max_act, const void* bias, void* out,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  using P = typename Traits<T>::P;
  using A = typename Vec<T>::A;
  using WT = typename WType<T>::type;
  constexpr int VEC = vec_rows<T>();
  if (B == 0) return DIAGMM_OK;
  if (ws == nullptr || ws_bytes < product_workspace<T>(gather, B, C, L, max_act)) return DIAGMM_EWORKSPACE;
  if constexpr (sizeof(T) == 2) {
    // bf16, B = 5..8: the packed-direct kernel when the diagonal list is long (warm
    // 4096^2: 90 %, k = 410: 10.3 vs 15.9 us for k_product_rows), the few-rows kernel when
    // it is short (99 %, k = 41: 4.5 vs 7.6 us) — max_act is the layer's known count
    if (use_pk<T>(B) && max_act > 0) {
      if (max_act >= 128)
        return run_product_pk<T>(gather, B, C, L, in, vals, asoft, active, n_act, max_act, bias, out, ws, st);
      return run_product_rows<T>(gather, B, C, L, in, vals, asoft, active, n_act, max_act, bias, out, st);
    }
  }
  if constexpr (std::is_same<T, float>::value) {
    // fp32 with a batch the FMA pipe cannot keep up with: 3xTF32 on the tensor cores
    if (use_tf32<T>(B, C, L, false, gather))
      return run_product_tf32(gather, B, C, L, static_cast<const float*>(in), static_cast<const float*>(vals), asoft,
                              active, n_act, max_act, static_cast<const float*>(bias), static_cast<float*>(out), ws,
                              st);
  }
  if (B <= rows_max_b())
    return run_product_rows<T>(gather, B, C, L, in, vals, asoft, active, n_act, max_act, bias, out, st);
  if (B <= narrow_max_b())
    return run_product_narrow<T>(gather, B, C, L, in, vals, asoft, active, n_act, max_act, bias, out,
                                 static_cast<A*>(ws), st);
  // v6 for bf16 only: at config 1 (fp32, B = 256) the v4 kernel stays ahead
  // (fwd 33.2 vs 36.9 us, dX 27.5 vs 29.2 us; profiles/r02_fma_v6.txt)
  if constexpr (sizeof(T) == 2) {
    if (product_v6_min_b() > 0 && B >= product_v6_min_b())
      return run_product6<T>(gather, B, C, L, in, vals, asoft, active, n_act, max_act, bias, out, ws, st);
  }
  const int out_w = gather ? L : C, in_w = gather ? C : L;
  const int cols = gather ? C + kHalo : scatter_cols<T>(L);
  ProductPlan p = plan_product<T>(B, out_w, cols, max_act);
  if (p.g == 0) return DIAGMM_ETOOLARGE;
  const int ldw = w_ld<T>(out_w);
  WT* w = static_cast<WT*>(ws);
  A* part = reinterpret_cast<A*>(static_cast<char*>(ws) + align16((size_t)(max_act > 0 ? max_act : 1) * ldw * sizeof(WT)));
  if (max_act > 0 && !p.fw) {
    dim3 grid(ceil_div(ldw, 256 * kPreVec), max_act < 65535 ? max_act : 65535);
    k_prescale<T><<<grid, 256, 0, st>>>(C, L, out_w, ldw, gather ? 1 : 0, static_cast<const P*>(vals), asoft, active,
                                        n_act, max_act, w);
    note_launch();
  }
  const int vec_ok = in_w % VEC == 0 && C % VEC == 0 && aligned16(in);
  auto tin = static_cast<const T*>(in);
  auto tv = static_cast<const P*>(vals);
  auto tb = static_cast<const P*>(bias);
  auto to = static_cast<T*>(out);
#define DIAGMM_GO(G, FW)                                                                                          \
  if (p.g == G && p.fw == FW) {                                                                                   \
    if (gather)                                                                                                   \
      launch_product<T, G, true, FW>(p, st, B, C, L, tin, w, ldw, tv, asoft, active, n_act, max_act, tb, to, part, \
                                     vec_ok);                                                                     \
    else                                                                                                          \
      launch_product<T, G, false, FW>(p, st, B, C, L, tin, w, ldw, tv, asoft, active, n_act, max_act, tb, to, part,\
                                      vec_ok);                                                                    \
  }
  DIAGMM_GO(2, false) DIAGMM_GO(1, false) DIAGMM_GO(2, true) DIAGMM_GO(1, true)
#undef DIAGMM_GO
  if (p.nsplit > 1 && !p.fw) {
    launch_split_reduce<T>(B, out_w, p.nsplit, part, tb, to, st);
    note_launch();
  }
  return status_from_cuda();
}

// ---- dW
static int narrow_dw_max_b() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DIAGMM_NARROW_DW_MAX_B");
    v = e ? atoi(e) : 8;
  }
  return v;
}

template <typename T>
static int dw_win_cap(int C, int max_act, int dwj) {
  constexpr int V = vec_rows<T>();
  const double span = max_act > 0 ? (double)dwj * C / max_act : (double)C;
  int cap = (int)(kDwTile + 2.5 * span) + 2 * V;
  cap = cap < C + kDwTile ? cap : C + kDwTile;
  cap = (cap + V - 1) / V * V;
  // keep two CTAs per SM within the shared-memory budget
  while (cap > kDwTile && dw_smem<T>(cap) > 110 * 1024) cap -= 64;
  return cap;
}

// diagonals per dW CTA: 64, or 32 when 64-diagonal tiles would not cover the SMs
static int dw_diags(int C, int L, int max_act) {
  const int n = max_act > 0 ? max_act : 1;
  const long long t64 = (long long)ceil_div(L, kDwTile) * ceil_div(n, kDwGroups * 16);
  int jw = t64 < num_sms() ? 8 : 16;
  // a CTA stages the circular window spanned by its diagonals: spread offsets
  // (high sparsity) take fewer diagonals per CTA so the window stays in shared
  // memory (2 CTAs / SM) instead of falling back to the direct global gather
  while (jw > 2 && kDwTile + 1.5 * kDwGroups * jw * (double)C / n > 3200.0) jw /= 2;
  return kDwGroups * jw;
}
static void dw_parts(int B, int C, int L, int max_act, int rb, int* parts, int* rows_per_part) {
  // as many row parts as keep the grid within ONE wave at two resident CTAs
  // per SM (a second, partial wave would double the kernel time)
  const long long tiles = (long long)ceil_div(L, kDwTile) * ceil_div(max_act > 0 ? max_act : 1, dw_diags(C, L, max_act));
  long long p = 2LL * num_sms() / tiles;
  if (p < 1) p = 1;
  const long long max_p = ceil_div(B, rb);
  if (p > max_p) p = max_p;
  if (p < 1) p = 1;
  int rpp = ceil_div(B, p);
  rpp = ceil_div(rpp, rb) * rb;
  *rows_per_part = rpp;
  *parts = ceil_div(B, rpp);
}

// ---- dW v6 planner (bf16 / fp32, B above the narrow kernel)
struct Dw6Plan {
  int pw = 0, nw = 0, jw = 0, jgroups = 0, parts = 0, gpp = 0, G = 0;
  size_t smem = 0;
};
static bool dw_v6_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DIAGMM_DW_V6");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}
template <typename T>
static Dw6Plan plan_dw6(int B, int C, int L, int max_act) {
  constexpr int VEC = vec_rows<T>();
  Dw6Plan best;
  const int sms = num_sms();
  const int n = max_act > 0 ? max_act : 1;
  int best_res = 0;
  for (int pw : {2, 1}) {
    if (pw == 2 && L <= kWarpPos) continue;
    const size_t sm = dw6_smem<T>(C, pw * kWarpPos);
    if (sm > 227 * 1024) continue;
    const int res = 2 * (sm + 1024) <= 228 * 1024 ? 2 : 1;
    if (res > best_res) {
      best_res = res;
      best.pw = pw;
      best.smem = sm;
    }
  }
  if (!best_res) return Dw6Plan{};
  Dw6Plan& p = best;
  p.G = ceil_div(B, VEC);
  p.nw = best_res == 2 ? 8 : 16;
  const int dw = p.nw / p.pw;
  const int ptiles = ceil_div(L, p.pw * kWarpPos);
  p.jw = 16;
  while (p.jw > 4 && (long long)ptiles * ceil_div(n, dw * p.jw) < (long long)best_res * sms) p.jw /= 2;
  p.jgroups = ceil_div(n, dw * p.jw);
  const long long tiles = (long long)ptiles * p.jgroups;
  long long parts = (long long)best_res * sms / tiles;  // about one wave
  const long long max_parts = p.G / 4 > 1 ? p.G / 4 : 1;  // >= 4 row groups per part (pipeline depth)
  parts = parts < 1 ? 1 : (parts > max_parts ? max_parts : parts);
  p.gpp = ceil_div(p.G, parts);
  p.parts = ceil_div(p.G, p.gpp);
  return p;
}
template <typename T>
static size_t dw6_workspace(int M, int N, int B, int max_act) {
  using A = typename Vec<T>::A;
  const int L = M < N ? M : N, C = M > N ? M : N;
  const Dw6Plan p = plan_dw6<T>(B > 0 ? B : 1, C, L, max_act);
  if (!p.G) return 0;
  const int cparts = ceil_div(B > 0 ? B : 1, kColRows);
  return align16((size_t)p.parts * (max_act > 0 ? max_act : 1) * L * sizeof(A)) +
         align16((size_t)cparts * M * sizeof(A)) + (size_t)p.G * (C + L) * 16;
}

template <typename T>
size_t dw_workspace(int M, int N, int B, int max_act) {
  using A = typename Vec<T>::A;
  const int L = M < N ? M : N;
  const int C = M > N ? M : N;
  int parts, rpp;
  dw_parts(B > 0 ? B : 1, C, L, max_act, kDwNG * vec_rows<T>(), &parts, &rpp);
  const int cparts = ceil_div(B > 0 ? B : 1, kColRows);
  const size_t prod_f = product_workspace<T>(M < N, B, C, L, max_act);
  const size_t prod_b = product_workspace<T>(M >= N, B, C, L, max_act);
  size_t dw = align16((size_t)parts * max_act * L * sizeof(A)) + align16((size_t)cparts * M * sizeof(A));
  if constexpr (sizeof(T) <= 4) {
    const size_t d6 = dw6_workspace<T>(M, N, B, max_act);
    dw = dw > d6 ? dw : d6;
  }
  if (use_tf32<T>(B, C, L, true)) {
    const size_t tf = align16((size_t)max_act * L * sizeof(A)) + align16((size_t)cparts * M * sizeof(A)) +
                      tf32_dw_workspace(M, N, B);
    dw = dw > tf ? dw : tf;
  }
  size_t w = dw > prod_f ? dw : prod_f;
  return w > prod_b ? w : prod_b;
}

template <typename T>
int run_dw(int M, int N, int B, const void* dy, const void* x, const void* vals, const double* asoft,
           const int32_t* active, const int32_t* slot, const int32_t* n_act, int max_act, void* g_values,
           double* g_soft, void* g_bias, void* ws, size_t ws_bytes, cudaStream_t st, void* bucket, int bucket_rows) {
  using P = typename Traits<T>::P;
  using A = typename Vec<T>::A;
  constexpr int VEC = vec_rows<T>();
  const int C = M > N ? M : N, L = M < N ? M : N;
  if (ws_bytes < dw_workspace<T>(M, N, B, max_act)) return DIAGMM_EWORKSPACE;
  const bool tall = M >= N;
  const T* aop = static_cast<const T*>(tall ? dy : x);
  const T* bop = static_cast<const T*>(tall ? x : dy);
  int parts, rpp;
  dw_parts(B > 0 ? B : 1, C, L, max_act, kDwNG * VEC, &parts, &rpp);
  A* partial = static_cast<A*>(ws);
  const int cparts = ceil_div(B > 0 ? B : 1, kColRows);
  const bool narrow = B > 0 && B <= narrow_dw_max_b() && max_act > 0;
  if (narrow) parts = 1;
  const bool tf = use_tf32<T>(B, C, L, true) && max_act > 0;  // 3xTF32 dense gw, gathered: one part
  if (tf) parts = 1;
  Dw6Plan p6;
  if constexpr (sizeof(T) <= 4) {
    if (!tf && !narrow && B > 0 && max_act > 0 && dw_v6_enabled()) p6 = plan_dw6<T>(B, C, L, max_act);
  }
  const bool v6 = p6.G > 0 && aligned16(aop) && aligned16(bop);
  if (v6) parts = p6.parts;
  // side stream, concurrently with the dW kernels and the active-row finalize on
  // `st` (disjoint outputs): the zero rows of g_values (+ g_soft) and the bias
  // gradient; joined back into `st` at the end
  SideStream& ss = side_stream();
  cudaEventRecord(ss.fork, st);
  cudaStreamWaitEvent(ss.s, ss.fork, 0);
  k_zero_inactive<P><<<C, 256, 0, ss.s>>>(C, L, slot, n_act, max_act, static_cast<P*>(g_values), g_soft);
  note_launch();
  if (g_bias) {
    A* cpart = reinterpret_cast<A*>(static_cast<char*>(ws) + align16((size_t)parts * max_act * L * sizeof(A)));
    if (B > 0) {
      k_colsum_partial<T><<<dim3(ceil_div(M, 256), cparts), 256, 0, ss.s>>>(B, M, static_cast<const T*>(dy), cpart);
      note_launch();
      k_colsum_final<T><<<ceil_div(M, 32), 256, 0, ss.s>>>(M, cparts, cpart, static_cast<P*>(g_bias));
      note_launch();
    } else {
      cudaMemsetAsync(g_bias, 0, (size_t)M * sizeof(P), ss.s);
    }
  }
  cudaEventRecord(ss.join, ss.s);
  if (tf) {
    if constexpr (std::is_same<T, float>::value) {
      void* tws = static_cast<char*>(ws) + align16((size_t)max_act * L * sizeof(A)) + align16((size_t)cparts * M * sizeof(A));
      if (int e = run_dw_tf32(M, N, B, static_cast<const float*>(dy), static_cast<const float*>(x), active, n_act,
                              max_act, partial, tws, st)) {
        cudaStreamWaitEvent(st, ss.join, 0);
        return e;
      }
    }
  } else if (v6) {
    if constexpr (sizeof(T) <= 4) {
      using U = typename Vec<T>::U;
      U* ap = reinterpret_cast<U*>(static_cast<char*>(ws) + align16((size_t)parts * max_act * L * sizeof(A)) +
                                   align16((size_t)cparts * M * sizeof(A)));
      U* bp = ap + (size_t)p6.G * C;
      const int vc = C % VEC == 0, vl = L % VEC == 0;
      k_pack<T><<<ceil_div((long long)p6.G * ceil_div(C, VEC), 256), 256, 0, st>>>(B, C, aop, ap, C, 0, C, C, vc);
      k_pack<T><<<ceil_div((long long)p6.G * ceil_div(L, VEC), 256), 256, 0, st>>>(B, L, bop, bp, L, 0, 0x7fffffff, L, vl);
      note_launch(2);
      auto k = p6.jw == 16 ? k_dw6<T, 16> : (p6.jw == 8 ? k_dw6<T, 8> : k_dw6<T, 4>);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p6.smem);
      dim3 grid(ceil_div(L, p6.pw * kWarpPos), p6.jgroups, p6.parts);
      k<<<grid, p6.nw * kWarp, p6.smem, st>>>(C, L, p6.G, ap, bp, active, n_act, max_act, p6.pw, p6.gpp, partial);
      note_launch();
    }
  } else if (narrow) {
    dim3 grid(ceil_div(L, kWarpPos), ceil_div(max_act, kWarps));
    if (B <= 4) k_dw_narrow<T, 4><<<grid, kThreads, 0, st>>>(B, C, L, aop, bop, active, n_act, max_act, partial);
    else k_dw_narrow<T, 8><<<grid, kThreads, 0, st>>>(B, C, L, aop, bop, active, n_act, max_act, partial);
    note_launch();
  } else if (B > 0 && max_act > 0) {
    const int dwj = dw_diags(C, L, max_act);
    const int cap = dw_win_cap<T>(C, max_act, dwj);
    const size_t sm = dw_smem<T>(cap);
    const int vec_ok = C % VEC == 0 && L % VEC == 0 && aligned16(aop) && aligned16(bop);
    auto k = dwj == kDwGroups * 16 ? k_dw<T, 16>
             : dwj == kDwGroups * 8 ? k_dw<T, 8>
             : dwj == kDwGroups * 4 ? k_dw<T, 4> : k_dw<T, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid(ceil_div(L, kDwTile), ceil_div(max_act, dwj), parts);
    k<<<grid, kThreads, sm, st>>>(B, C, L, aop, bop, active, n_act, max_act, cap, rpp, partial, vec_ok);
    note_launch();
  } else {
    parts = 0;
  }
  if (L >= 1024)  // few long rows: a CTA per row keeps enough loads in flight
    k_dw_finalize_blk<T><<<max_act > 0 ? max_act : 1, 256, 0, st>>>(C, L, parts, partial, max_act, slot, n_act, asoft,
                                       static_cast<const P*>(vals), static_cast<P*>(g_values), g_soft,
                                       static_cast<P*>(bucket), bucket_rows, active);
  else
    k_dw_finalize<T><<<ceil_div(max_act > 0 ? max_act : 1, kWarps), 256, 0, st>>>(C, L, parts, partial, max_act, slot, n_act, asoft,
                                       static_cast<const P*>(vals), static_cast<P*>(g_values), g_soft,
                                       static_cast<P*>(bucket), bucket_rows, active);
  note_launch();
  cudaStreamWaitEvent(st, ss.join, 0);
  return status_from_cuda();
}

template <typename T>
int run_materialize(int M, int N, const void* vals, const double* asoft, const int32_t* slot,
                    const int32_t* n_act, int max_act, void* w, cudaStream_t st, bool trans) {
  using P = typename Traits<T>::P;
  const int R = trans ? N : M, Cc = trans ? M : N;
  const int vec = (Cc % 8 == 0) && aligned16(w);
  if constexpr (sizeof(T) <= 4) {
    if (!trans) {
      const int vt = (N % (16 / (int)sizeof(T)) == 0) && aligned16(w);
      k_materialize_tiles<T><<<dim3(ceil_div(N, kMTC), ceil_div(M, kMTR)), 256, 0, st>>>(
          M, N, static_cast<const P*>(vals), asoft, slot, n_act, max_act, static_cast<T*>(w), vt);
      note_launch();
      return status_from_cuda();
    }
  }
  auto k = trans ? k_materialize<T, true> : k_materialize<T, false>;
  k<<<ceil_div(R, kMatRows), 256, 0, st>>>(M, N, static_cast<const P*>(vals), asoft, slot, n_act, max_act,
                                           static_cast<T*>(w), vec);
  note_launch();
  return status_from_cuda();
}

template <typename T>
int run_materialize_batched(int n, const diagmm_materialize_job* jobs, cudaStream_t st) {
  if constexpr (sizeof(T) > 4) {
    return DIAGMM_ESHAPE;
  } else {
    for (int b = 0; b < n; b += kMatJobs) {
      MatJobs P{};
      P.n = n - b < kMatJobs ? n - b : kMatJobs;
      int total = 0;
      for (int i = 0; i < P.n; ++i) {
        const diagmm_materialize_job& j = jobs[b + i];
        if (j.M < 1 || j.N < 1) return DIAGMM_ESHAPE;
        P.j[i] = j;
        P.start[i] = total;
        P.tiles_x[i] = ceil_div(j.N, kMTC);
        P.vec[i] = (j.N % (16 / (int)sizeof(T)) == 0) && aligned16(j.w);
        total += P.tiles_x[i] * ceil_div(j.M, kMTR);
      }
      P.start[P.n] = total;
      k_materialize_batched<T><<<total, 256, 0, st>>>(P);
      note_launch();
    }
    return status_from_cuda();
  }
}
template int run_materialize_batched<float>(int, const diagmm_materialize_job*, cudaStream_t);
template int run_materialize_batched<__nv_bfloat16>(int, const diagmm_materialize_job*, cudaStream_t);

template <typename P>
int run_gather_dense(int M, int N, const void* dW, const void* vals, const double* asoft, const int32_t* slot,
                     const int32_t* n_act, void* g_values, double* g_soft, cudaStream_t st) {
  const int C = M > N ? M : N, L = M < N ? M : N;
  const bool tall = M >= N;
  dim3 grid(ceil_div(L, kGTc), ceil_div(tall ? M : N, kGTr));
  k_gather_tiles<P><<<grid, 256, 0, st>>>(M, N, static_cast<const P*>(dW), slot, n_act, static_cast<P*>(g_values));
  note_launch();
  k_gather_finish<P><<<C, 256, 0, st>>>(C, L, static_cast<const P*>(vals), asoft, slot, n_act,
                                        static_cast<P*>(g_values), g_soft);
  note_launch();
  return status_from_cuda();
}

// ---- dW on the tensor cores (tc_kernels.cu) + the same finalize
int tc_dw_splits(int M, int N, int ntok);
int run_tc_dw(int M, int N, int ntok, const void* dy, const void* x, const int32_t* slot, const int32_t* n_act,
              int max_act, float* partial, size_t partial_bytes, float* colsum, cudaStream_t st, const void* dy1,
              const void* dy2, int a_ms);

size_t tc_dw_workspace(int M, int N, int B, int max_act) {
  const int L = M < N ? M : N;
  const int ks = tc_dw_splits(M, N, B > 0 ? B : 1);
  return align16((size_t)ks * (max_act > 0 ? max_act : 1) * L * sizeof(float)) + align16((size_t)ks * M * sizeof(float));
}

int run_tc_dw_full(int M, int N, int B, const void* dy, const void* x, const void* vals, const double* asoft,
                   const int32_t* slot, const int32_t* n_act, int max_act, void* g_values, double* g_soft,
                   void* g_bias, void* ws, size_t ws_bytes, cudaStream_t st, const void* dy1, const void* dy2,
                   int a_ms, void* bucket, int bucket_rows) {
  using T = __nv_bfloat16;
  using P = typename Traits<T>::P;
  const int C = M > N ? M : N, L = M < N ? M : N;
  if (ws_bytes < tc_dw_workspace(M, N, B, max_act)) return DIAGMM_EWORKSPACE;
  float* partial = static_cast<float*>(ws);
  const int ks = tc_dw_splits(M, N, B > 0 ? B : 1);
  const size_t pbytes = align16((size_t)ks * (max_act > 0 ? max_act : 1) * L * sizeof(float));
  float* colsum = reinterpret_cast<float*>(static_cast<char*>(ws) + pbytes);
  int parts = 0;
  if (B > 0 && (max_act > 0 || g_bias)) {
    if (int e = run_tc_dw(M, N, B, dy, x, slot, n_act, max_act > 0 ? max_act : 1, partial, pbytes,
                          g_bias ? colsum : nullptr, st, dy1, dy2, a_ms))
      return e;
    parts = max_act > 0 ? ks : 0;
  }
  if (g_bias) {
    if (B > 0) {
      k_colsum_final<T><<<ceil_div(M, 32), 256, 0, st>>>(M, ks, colsum, static_cast<P*>(g_bias));
      note_launch();
    } else {
      cudaMemsetAsync(g_bias, 0, (size_t)M * sizeof(P), st);
    }
  }
  k_dw_finalize<T><<<ceil_div(C, kWarps), 256, 0, st>>>(C, L, parts, partial, max_act, slot, n_act, asoft,
                                       static_cast<const P*>(vals), static_cast<P*>(g_values), g_soft,
                                       static_cast<P*>(bucket), bucket_rows, nullptr);
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
                         void*, size_t, cudaStream_t, void*, int);                                        \
  template int run_materialize<T>(int, int, const void*, const double*, const int32_t*, const int32_t*,   \
                                  int, void*, cudaStream_t, bool);
DIAGMM_INST(double)
DIAGMM_INST(float)
DIAGMM_INST(__nv_bfloat16)
template int run_gather_dense<double>(int, int, const void*, const void*, const double*, const int32_t*,
                                      const int32_t*, void*, double*, cudaStream_t);
template int run_gather_dense<float>(int, int, const void*, const void*, const double*, const int32_t*,
                                     const int32_t*, void*, double*, cudaStream_t);

}  // namespace diagmm

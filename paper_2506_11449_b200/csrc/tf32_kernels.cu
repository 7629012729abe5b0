// tf32_kernels.cu — the fp32 tensor-core route (3xTF32): products and dW of
// float32 DiagLinear layers at batch sizes where the FMA pipe cannot keep up
// (BASELINE config 1: 768 -> 3072, B = 256).
//
// Each fp32 operand v is split into two tf32 values, hi = v rounded to tf32
// and lo = v - hi (exact in fp32), and
//     sum_k A[m,k] B[n,k]  ~=  sum_k (Al Bh + Ah Bl + Ah Bh)[m,k,n]
// accumulated in fp32 in TMEM by tcgen05.mma kind::tf32 (the dropped Al Bl
// term and lo's own tf32 reading are <= 2^-22 of each product): fp32-level
// accuracy on the tensor cores, 3 MMAs per K step.  Operands are K-major raw
// fp32, staged by TMA with the 128-byte swizzle (32 fp32 per swizzle row)
// into a 2-4 stage mbarrier ring; four split warps turn each landed stage
// into its hi / lo halves in shared memory (so L2 -> SM moves 4 bytes per
// element, not 8); one elected thread issues the MMAs; the split warps drain
// TMEM afterwards.  One output tile (128 x BN) per CTA, split-K over
// gridDim.z when the tile count alone would leave SMs idle (partials summed
// in a fixed order: deterministic).
//
// Callers (diagmm_kernels.cu, use_tf32): run_product — E (out_w x in_w, the
// layer's effective matrix in the product's orientation, materialized fp32
// tile by tile) and the input rows -> out = in E^T + bias; run_dw — dy^T and
// x^T (transposed: K = tokens) -> dense G = dy^T x partials -> gathered onto
// the active diagonals -> the shared finalize (zero rows, g_soft, bias).
// Measured (profiles/r02_tf32x3.txt): 1.4-1.6x the FMA kernels from B = 512;
// latency-bound per CTA (tensor pipe ~22 % active at config 1).
// Parity: tests/test_gpu_tf32x3.py against the fp64 oracle at the fp32 bar.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "tc_gemm.cuh"

namespace diagmm {
namespace tc {

constexpr int kTfBK = 32;  // fp32 per 128-byte swizzle row

// hi: v rounded to the nearest tf32 (ties away from zero) with two integer ops;
// lo = v - hi is exact in fp32 and its own tf32 reading by the MMA drops at most
// 2^-11 |lo| <= 2^-23 |v|
__device__ __forceinline__ void split_tf32(float v, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
  lo = v - hi;
}

// kind::tf32, A = B = tf32, D = f32, both K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}

template <int BN>
struct TfSmem {
  static constexpr int a_bytes = BM * kTfBK * 4;  // one of hi / lo
  static constexpr int b_bytes = BN * kTfBK * 4;
  static constexpr int half = a_bytes + b_bytes;  // [A | B] hi, then [A | B] lo
  static constexpr int stage = 2 * half;
  static constexpr int NST = (192 * 1024) / stage;  // BN 64: 4, 128: 3, 256: 2
  static constexpr size_t total = 1024 + (size_t)NST * stage + 256;
};

// out[split][m][n] = sum over this split's K range of A[m,k] B[n,k] (3xTF32),
// + bias[n] when bias != nullptr (the single-split case).  A, B raw fp32.
// Warp 0: TMA producer (raw tiles into the hi half of a stage); warp 1: TMEM
// allocation + the MMA thread; warps 2-5: the split — hi = rna(v) in place and
// lo = rna(v - hi) at the same swizzled offset of the lo half (an elementwise
// map keeps the 128-byte swizzle valid) — then the epilogue.
constexpr int kTfThreads = 192;
template <int BN>
__global__ void __launch_bounds__(kTfThreads, 1)
k_tf32x3(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int Mo, int No, int K,
         int kb_per_split, const float* __restrict__ bias, float* __restrict__ out, int ldo, size_t split_stride) {
  using S = TfSmem<BN>;
  constexpr int NST = S::NST;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * S::stage);
  uint64_t* ready = full + NST;
  uint64_t* empty = ready + NST;
  uint64_t* done = empty + NST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KB = (K + kTfBK - 1) / kTfBK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = max(0, min(KB, kb0 + kb_per_split) - kb0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(&ready[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(done)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int it = 0; it < nkb; ++it) {
        const int s = it % NST, round = it / NST;
        mbar_wait_parity(&empty[s], (round & 1) ^ 1);
        unsigned char* st = smem + (size_t)s * S::stage;
        mbar_expect_tx(&full[s], (uint32_t)S::half);
        const int kc = (kb0 + it) * kTfBK;
        tma_load_2d(st, &ta, kc, m0, &full[s]);
        tma_load_2d(st + S::a_bytes, &tb, kc, n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = idesc_tf32(BM, BN);
      for (int it = 0; it < nkb; ++it) {
        const int s = it % NST, round = it / NST;
        mbar_wait_parity(&ready[s], round & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        unsigned char* st = smem + (size_t)s * S::stage;
        const uint64_t dah = smem_desc_sw128(st), dbh = smem_desc_sw128(st + S::a_bytes);
        const uint64_t dal = smem_desc_sw128(st + S::half), dbl = smem_desc_sw128(st + S::half + S::a_bytes);
#pragma unroll
        for (int k = 0; k < kTfBK / 8; ++k) {  // UMMA K = 8 tf32 = 32 bytes = +2 in the descriptor
          umma_tf32(tmem, dal + 2 * k, dbh + 2 * k, idesc, (it | k) != 0);  // small terms first
          umma_tf32(tmem, dah + 2 * k, dbl + 2 * k, idesc, 1);
          umma_tf32(tmem, dah + 2 * k, dbh + 2 * k, idesc, 1);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(done);  // with no MMA issued this arrives at once
    }
  } else {  // split warps
    const int tt = threadIdx.x - 64;
    for (int it = 0; it < nkb; ++it) {
      const int s = it % NST, round = it / NST;
      mbar_wait_parity(&full[s], round & 1);
      // explicit shared-space accesses (a generic pointer here compiles to LD / ST.E)
      const uint32_t sb = smem_u32(smem + (size_t)s * S::stage);
#pragma unroll 4
      for (int q = tt; q < S::half / 16; q += 128) {
        const uint32_t a = sb + (uint32_t)q * 16;
        float4 v, h, l;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
        split_tf32(v.x, h.x, l.x); split_tf32(v.y, h.y, l.y); split_tf32(v.z, h.z, l.z); split_tf32(v.w, h.w, l.w);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(h.x), "f"(h.y), "f"(h.z), "f"(h.w)
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a + (uint32_t)S::half), "f"(l.x), "f"(l.y),
                     "f"(l.z), "f"(l.w)
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ready[s])) : "memory");
    }
  }
  __syncwarp();
  if (warp >= 2) {
    mbar_wait_parity(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: warp w owns TMEM lanes 32 (w % 4) .. +31 = tile rows; 32 columns per tcgen05.ld
    const int q4 = warp & 3;
    const int row = m0 + q4 * 32 + lane;
    float* orow = out + blockIdx.z * split_stride + (size_t)row * ldo;
    const bool vec = (ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (split_stride & 3) == 0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      const int col0 = n0 + c * 32;
      if (col0 >= No) break;  // warp-uniform
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(c * 32), r);
      if (row >= Mo) continue;
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        v[j] = nkb > 0 ? __uint_as_float(r[j]) : 0.f;
        if (bias && col0 + j < No) v[j] += __ldg(bias + col0 + j);
      }
      if (vec && col0 + 32 <= No) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(orow + col0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        for (int j = 0; j < 32 && col0 + j < No; ++j) orow[col0 + j] = v[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN) : "memory");
}

}  // namespace tc

using tc::split_tf32;

// ---- operand preparation ----------------------------------------------------

// lower_bound over an ascending list, 32-ary with one warp (2-3 dependent loads
// instead of a 10-15 step binary search); every lane returns the answer
__device__ __forceinline__ int warp_lower_bound(const int32_t* __restrict__ a, int n, int key) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n;
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const int idx = lo + lane * step;
    const int cnt = __popc(__ballot_sync(0xffffffffu, idx < hi && __ldg(a + idx) < key));
    if (cnt == 0) return lo;
    const int nlo = lo + (cnt - 1) * step + 1, nhi = min(hi, lo + cnt * step);
    lo = nlo;
    hi = nhi;
  }
  const int idx = lo + lane;
  return lo + __popc(__ballot_sync(0xffffffffu, idx < hi && __ldg(a + idx) < key));
}

// The effective matrix E (out_w x in_w, row stride ldd) of a product, fp32,
// one 32 x 128 tile per CTA written with 16-byte stores (zeros included).
// gather (out_w = L, in_w = C): E[i][(i + o) mod C] = a(o) v[o][i];
// scatter (out_w = C, in_w = L): E[(j + o) mod C][j] = a(o) v[o][j] — the
// entries the FMA kernels use, weight = (float)(alpha_soft * value) as in
// materialize_tile.  The active offsets crossing the tile are a contiguous
// (cyclic) range of the ascending active list.
constexpr int kEsR = 32, kEsC = 128;
__global__ void __launch_bounds__(256)
k_materialize_e(bool gather, int C, int L, const float* __restrict__ vals, const double* __restrict__ asoft,
                const int32_t* __restrict__ active, const int32_t* __restrict__ n_act_p, int max_act,
                float* __restrict__ e, int ldd) {
  __shared__ __align__(16) float tile[kEsR][kEsC];
  __shared__ int s_rng[4];
  const int out_w = gather ? L : C, in_w = gather ? C : L;
  const int i0 = blockIdx.y * kEsR, j0 = blockIdx.x * kEsC;
  const int n_act = min(*n_act_p, max_act);
  for (int q = threadIdx.x; q < kEsR * kEsC / 4; q += 256)
    reinterpret_cast<float4*>(&tile[0][0])[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x < 32) {
    // offsets o = (j - i) mod C (gather) / (i - j) mod C (scatter) over the tile
    int olo = gather ? j0 - (i0 + kEsR - 1) : i0 - (j0 + kEsC - 1);
    const int width = kEsR + kEsC - 1;
    int a0 = 0, a1 = n_act, b1 = 0;
    if (width < C) {
      olo %= C;
      olo = olo < 0 ? olo + C : olo;
      a0 = warp_lower_bound(active, n_act, olo);
      if (olo + width <= C) a1 = warp_lower_bound(active, n_act, olo + width);
      else b1 = warp_lower_bound(active, n_act, olo + width - C);
    }
    if (threadIdx.x == 0) { s_rng[0] = a0; s_rng[1] = a1; s_rng[2] = 0; s_rng[3] = b1; }
  }
  __syncthreads();
  const int n1 = s_rng[1] - s_rng[0], nd = n1 + s_rng[3];
  // one (diagonal, tile row) pair per thread step: a diagonal crosses a row at most once
  for (int it = threadIdx.x; it < nd * kEsR; it += 256) {
    const int di = it / kEsR, ii = it - di * kEsR;
    const int o = __ldg(active + (di < n1 ? s_rng[0] + di : di - n1));
    const int i = i0 + ii;
    if (i >= out_w) continue;
    int j, t;
    if (gather) { j = i + o; j = j >= C ? j - C : j; t = i; }
    else { j = i - o; j = j < 0 ? j + C : j; t = j; }
    if (j < j0 || j >= j0 + kEsC || j >= in_w) continue;
    const double sc = asoft ? __ldg(asoft + o) : 1.0;
    tile[ii][j - j0] = (float)(sc * (double)__ldg(vals + (size_t)o * L + t));
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kEsR * kEsC / 4; q += 256) {
    const int ii = q / (kEsC / 4), c4 = (q - ii * (kEsC / 4)) * 4;
    const int i = i0 + ii, j = j0 + c4;
    if (i >= out_w || j >= ldd) continue;  // the pad columns in_w .. ldd get zeros
    *reinterpret_cast<float4*>(e + (size_t)i * ldd + j) = *reinterpret_cast<const float4*>(&tile[ii][c4]);
  }
}

// rows x cols (row stride lds) -> rows x ldd copy with zero pad columns (16-byte rows for TMA)
__global__ void __launch_bounds__(256)
k_pad_rows(int rows, int cols, const float* __restrict__ src, int lds, float* __restrict__ dst, int ldd) {
  const long long n = (long long)rows * ldd;
  for (long long q = blockIdx.x * 256LL + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
    const int r = (int)(q / ldd), c = (int)(q - (long long)r * ldd);
    dst[q] = c < cols ? __ldg(src + (size_t)r * lds + c) : 0.f;
  }
}

// rows x cols (row stride lds) -> transposed cols x rows (row stride ldd, pad zeros)
__global__ void __launch_bounds__(256)
k_transpose_pad(int rows, int cols, const float* __restrict__ src, int lds, float* __restrict__ dst, int ldd) {
  __shared__ float t[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + tx;
    t[i][tx] = (r < rows && c < cols) ? __ldg(src + (size_t)r * lds + c) : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + tx;  // output row c, column r
    if (c < cols && r < ldd) dst[(size_t)c * ldd + r] = t[tx][i];
  }
}

// out[r][c] = sum_s part[s][r][c] (+ bias[c]), s in index order; 4 columns per thread
__global__ void __launch_bounds__(256)
k_sum_splits(int rows, int cols, int ks, const float* __restrict__ part, size_t stride, const float* __restrict__ bias,
             float* __restrict__ out, int ldo) {
  const int c4n = (cols + 3) >> 2;
  const long long n = (long long)rows * c4n;
  const bool vec = (cols & 3) == 0 && (ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (long long q = blockIdx.x * 256LL + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
    const int r = (int)(q / c4n), c = (int)(q - (long long)r * c4n) * 4;
    const size_t base = (size_t)r * cols + c;
    if (vec) {
      float4 v = __ldcg(reinterpret_cast<const float4*>(part + base));
      for (int s = 1; s < ks; ++s) {
        const float4 w = __ldcg(reinterpret_cast<const float4*>(part + s * stride + base));
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      if (bias) {
        v.x += __ldg(bias + c); v.y += __ldg(bias + c + 1); v.z += __ldg(bias + c + 2); v.w += __ldg(bias + c + 3);
      }
      *reinterpret_cast<float4*>(out + (size_t)r * ldo + c) = v;
    } else {
      for (int k = 0; k < 4 && c + k < cols; ++k) {
        float v = part[base + k];
        for (int s = 1; s < ks; ++s) v += __ldcg(part + s * stride + base + k);
        if (bias) v += __ldg(bias + c + k);
        out[(size_t)r * ldo + c + k] = v;
      }
    }
  }
}

// dW: partial[s][t] = sum_split G[split][r][c] at the entry (r, c) of active
// diagonal s, position t (tall M >= N: c = t, r = (t + o) mod M; wide: r = t,
// c = (t + o) mod N — layers.py:149-165's gw, indexed as the FMA dW writes it)
__global__ void __launch_bounds__(256)
k_gather_splits(int M, int N, int ks, const float* __restrict__ G, size_t stride, const int32_t* __restrict__ active,
                const int32_t* __restrict__ n_act_p, int max_act, float* __restrict__ partial) {
  const int L = min(M, N);
  const bool tall = M >= N;
  const int n_act = min(*n_act_p, max_act);
  for (int s = blockIdx.y; s < n_act; s += gridDim.y) {
    const int o = active[s];
    for (int t = blockIdx.x * 256 + threadIdx.x; t < L; t += gridDim.x * 256) {
      int r, c;
      if (tall) { c = t; r = t + o; r = r >= M ? r - M : r; }
      else { r = t; c = t + o; c = c >= N ? c - N : c; }
      const size_t q = (size_t)r * N + c;
      float v = __ldcg(G + q);
      for (int k = 1; k < ks; ++k) v += __ldcg(G + k * stride + q);
      partial[(size_t)s * L + t] = v;
    }
  }
}

// ---- host ---------------------------------------------------------------------

// DIAGMM_TF32X3_MIN_B=n: the route for every fp32 call with B >= n (0: never);
// unset: -1, the measured rule in use_tf32 (diagmm_kernels.cu).  Read per call.
int tf32x3_min_b() {
  const char* e = getenv("DIAGMM_TF32X3_MIN_B");
  if (!e) return -1;
  const int v = atoi(e);
  return v < 0 ? 0 : v;
}

static int pad4(int x) { return (x + 3) & ~3; }
static size_t align16(size_t b) { return (b + 15) & ~size_t(15); }
static int grid_1d(long long n) { return (int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 8); }

struct TfPlan {
  int bn = 128, ks = 1;
};

// tile width and split count: the fewest waves of per-CTA operand bytes (raw fp32
// A and B rows), plus the split-K partial traffic
static TfPlan tf_plan(int Mo, int No, int K) {
  const int sms = num_sms();
  const int KB = ceil_div(K > 0 ? K : 1, tc::kTfBK);
  TfPlan best;
  double best_cost = 1e300;
  for (int bn : {64, 128, 256}) {
    if (bn > 64 && No <= bn / 2) continue;
    const int tiles = ceil_div(Mo, tc::BM) * ceil_div(No, bn);
    for (int ks = 1; ks <= 16 && ks <= KB; ++ks) {
      const int kbs = ceil_div(KB, ks);
      const double waves = std::ceil((double)tiles * ks / sms);
      const double per_cta = (double)(tc::BM + bn) * 4.0 * kbs * tc::kTfBK + 48.0 * 1024;  // + fill / drain
      const double reduce = ks > 1 ? (double)ks * Mo * No * 8.0 / sms : 0.0;
      const double cost = waves * per_cta + reduce;
      if (cost < best_cost * 0.98) {
        best_cost = cost;
        best.bn = bn;
        best.ks = ks;
      }
    }
  }
  return best;
}

// out (Mo x No, ldo) = A (Mo x K, lda) . B (No x K, ldb)^T (+ bias), fp32-accurate;
// part: ks partial tiles when the plan splits K (sum_out: summed into out here;
// otherwise left for the caller)
static int tf_gemm(int Mo, int No, int K, const float* A, int lda, const float* B, int ldb, const float* bias,
                   float* out, int ldo, float* part, bool sum_out, int* ks_out, cudaStream_t st) {
  using namespace tc;
  const TfPlan p = tf_plan(Mo, No, K);
  CUtensorMap ma, mb;
  if (!make_tmap_f32(&ma, A, (uint64_t)Mo, (uint64_t)K, BM, (uint64_t)lda) ||
      !make_tmap_f32(&mb, B, (uint64_t)No, (uint64_t)K, (uint32_t)p.bn, (uint64_t)ldb))
    return DIAGMM_ECUDA;
  const int KB = ceil_div(K > 0 ? K : 1, kTfBK);
  const int kbs = ceil_div(KB, p.ks);
  const int ks = ceil_div(KB, kbs);  // no empty split
  dim3 grid(ceil_div(No, p.bn), ceil_div(Mo, BM), ks);
  float* dst = ks > 1 ? part : out;
  const int ldd = ks > 1 ? No : ldo;
  const size_t stride = (size_t)Mo * No;
  const float* b = ks > 1 ? nullptr : bias;
#define DIAGMM_TF(BNV)                                                                                  \
  if (p.bn == BNV) {                                                                                    \
    auto k = k_tf32x3<BNV>;                                                                             \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TfSmem<BNV>::total);      \
    k<<<grid, kTfThreads, TfSmem<BNV>::total, st>>>(ma, mb, Mo, No, K, kbs, b, dst, ldd, stride);       \
  }
  DIAGMM_TF(64) DIAGMM_TF(128) DIAGMM_TF(256)
#undef DIAGMM_TF
  note_launch();
  if (ks > 1 && sum_out) {
    k_sum_splits<<<grid_1d((long long)Mo * ((No + 3) / 4)), 256, 0, st>>>(Mo, No, ks, part, stride, bias, out, ldo);
    note_launch();
  }
  if (ks_out) *ks_out = ks;
  return status_from_cuda();
}

static size_t tf_split_bytes(int Mo, int No, int K) {
  const TfPlan p = tf_plan(Mo, No, K);
  return p.ks > 1 ? align16((size_t)p.ks * Mo * No * sizeof(float)) : 0;
}

// ---- products (fp32): out (B x out_w) = in (B x in_w) E^T + bias
size_t tf32_product_workspace(bool gather, int B, int C, int L) {
  const int out_w = gather ? L : C, in_w = gather ? C : L;
  const int ld = pad4(in_w);
  const int b = B > 0 ? B : 1;
  return align16((size_t)out_w * ld * 4) + align16((size_t)b * ld * 4) + tf_split_bytes(b, out_w, in_w);
}

int run_product_tf32(bool gather, int B, int C, int L, const float* in, const float* vals, const double* asoft,
                     const int32_t* active, const int32_t* n_act, int max_act, const float* bias, float* out,
                     void* ws, cudaStream_t st) {
  const int out_w = gather ? L : C, in_w = gather ? C : L;
  const int ld = pad4(in_w);
  const size_t eb = align16((size_t)out_w * ld * 4), xb = align16((size_t)B * ld * 4);
  char* p = static_cast<char*>(ws);
  float* E = reinterpret_cast<float*>(p);
  float* xp = reinterpret_cast<float*>(p + eb);
  float* part = reinterpret_cast<float*>(p + eb + xb);
  k_materialize_e<<<dim3(ceil_div(ld, kEsC), ceil_div(out_w, kEsR)), 256, 0, st>>>(gather, C, L, vals, asoft, active,
                                                                                  n_act, max_act > 0 ? max_act : 0, E, ld);
  note_launch();
  const float* A = in;
  if (in_w != ld || (reinterpret_cast<uintptr_t>(in) & 15) != 0) {  // TMA needs 16-byte rows
    k_pad_rows<<<grid_1d((long long)B * ld), 256, 0, st>>>(B, in_w, in, in_w, xp, ld);
    note_launch();
    A = xp;
  }
  return tf_gemm(B, out_w, in_w, A, A == in ? in_w : ld, E, ld, bias, out, out_w, part, true, nullptr, st);
}

// ---- dW (fp32): partial[s][t] (max_act x L, one part) = gw of active diagonal s
size_t tf32_dw_workspace(int M, int N, int B) {
  const int bp = pad4(B > 0 ? B : 1);
  const TfPlan p = tf_plan(M, N, B > 0 ? B : 1);
  return align16((size_t)M * bp * 4) + align16((size_t)N * bp * 4) + align16((size_t)p.ks * M * N * 4);
}

int run_dw_tf32(int M, int N, int B, const float* dy, const float* x, const int32_t* active, const int32_t* n_act,
                int max_act, float* partial, void* ws, cudaStream_t st) {
  const int bp = pad4(B);
  const size_t db = align16((size_t)M * bp * 4), xb = align16((size_t)N * bp * 4);
  char* p = static_cast<char*>(ws);
  float* dT = reinterpret_cast<float*>(p);
  float* xT = reinterpret_cast<float*>(p + db);
  float* G = reinterpret_cast<float*>(p + db + xb);
  k_transpose_pad<<<dim3(ceil_div(M, 32), ceil_div(bp, 32)), 256, 0, st>>>(B, M, dy, M, dT, bp);
  k_transpose_pad<<<dim3(ceil_div(N, 32), ceil_div(bp, 32)), 256, 0, st>>>(B, N, x, N, xT, bp);
  note_launch(2);
  int ks = 1;
  if (int e = tf_gemm(M, N, B, dT, bp, xT, bp, nullptr, G, N, G, false, &ks, st)) return e;
  const int L = M < N ? M : N;
  dim3 g(ceil_div(L, 256), max_act < 65535 ? max_act : 65535);
  k_gather_splits<<<g, 256, 0, st>>>(M, N, ks, G, (size_t)M * N, active, n_act, max_act, partial);
  note_launch();
  return status_from_cuda();
}

// ---- dense fp32 GEMM on the same kernel (the reference's density >= 1/4 switch,
// diagcore.py:226-228 / layers.py:150-153, for float32 layers):
//   out (M x N, ldo) = A_eff (M x K) . B_eff (N x K)^T (+ bias)
// with A_eff = A (M x K, lda) or, trans_a, A^T for A given as (K x M, lda); B likewise.
// Transposed or 16-byte-misaligned operands are staged into the workspace first.
static bool tma_ok(const float* p, int ld) { return (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

size_t tf32x3_gemm_workspace(int M, int N, int K, int trans_a, int trans_b) {
  const int kp = pad4(K > 0 ? K : 1);
  const size_t a = trans_a ? align16((size_t)M * kp * 4) : align16((size_t)M * kp * 4);
  const size_t b = trans_b ? align16((size_t)N * kp * 4) : align16((size_t)N * kp * 4);
  return a + b + tf_split_bytes(M > 0 ? M : 1, N > 0 ? N : 1, K > 0 ? K : 1);
}

int run_tf32x3_gemm(int M, int N, int K, const float* A, int lda, int trans_a, const float* B, int ldb, int trans_b,
                    const float* bias, float* out, int ldo, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (M < 1 || N < 1 || K < 1 || ldo < N) return DIAGMM_ESHAPE;
  if (lda < (trans_a ? M : K) || ldb < (trans_b ? N : K)) return DIAGMM_ESHAPE;
  if (ws_bytes < tf32x3_gemm_workspace(M, N, K, trans_a, trans_b)) return DIAGMM_EWORKSPACE;
  const int kp = pad4(K);
  char* p = static_cast<char*>(ws);
  float* sa = reinterpret_cast<float*>(p);
  float* sb = reinterpret_cast<float*>(p + align16((size_t)M * kp * 4));
  float* part = reinterpret_cast<float*>(p + align16((size_t)M * kp * 4) + align16((size_t)N * kp * 4));
  const float* a = A;
  int la = lda;
  if (trans_a) {
    k_transpose_pad<<<dim3(ceil_div(M, 32), ceil_div(kp, 32)), 256, 0, st>>>(K, M, A, lda, sa, kp);
    note_launch();
    a = sa, la = kp;
  } else if (!tma_ok(A, lda)) {
    k_pad_rows<<<grid_1d((long long)M * kp), 256, 0, st>>>(M, K, A, lda, sa, kp);
    note_launch();
    a = sa, la = kp;
  }
  const float* b = B;
  int lb = ldb;
  if (trans_b) {
    k_transpose_pad<<<dim3(ceil_div(N, 32), ceil_div(kp, 32)), 256, 0, st>>>(K, N, B, ldb, sb, kp);
    note_launch();
    b = sb, lb = kp;
  } else if (!tma_ok(B, ldb)) {
    k_pad_rows<<<grid_1d((long long)N * kp), 256, 0, st>>>(N, K, B, ldb, sb, kp);
    note_launch();
    b = sb, lb = kp;
  }
  return tf_gemm(M, N, K, a, la, b, lb, bias, out, ldo, part, true, nullptr, st);
}

}  // namespace diagmm

// tc_kernels.cu — tensor-core (tcgen05) GEMM for the dense-equivalent DiagMM
// route: out[m, n] = sum_k A[m, k] * B[n, k] (+ bias[n]), bf16 in, fp32
// accumulate in TMEM, bf16 out.  Forward: A = x (tokens x in), B = W_K
// (out x in); input gradient: A = dy, B = W_K^T.  See tc_gemm.cuh.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "tc_gemm.cuh"

namespace diagmm {
namespace tc {

// GELU (tanh form) in the GEMM epilogues.  tanh comes from the SFU
// (tanh.approx.f32, |rel err| < 2^-10.9): the results are rounded to bf16
// (2^-8) right after, and a full-precision tanhf made the epilogue warps,
// not the tensor cores, the bottleneck of the fused fc1/fc2 tiles.
__device__ __forceinline__ float tanh_sfu(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_sfu(k0 * fmaf(k1 * x, x * x, x)), hx);
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {  // d gelu_tanh / dx (PyTorch's formula)
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float t = tanh_sfu(k0 * fmaf(k1 * x, x2, x));
  const float hx = 0.5f * x;
  return fmaf(hx * (1.f - t * t), k0 * fmaf(3.f * k1, x2, 1.f), 0.5f * (1.f + t));
}

// MN-major operand, 128-byte swizzle: 64-element MN boxes 8 KB apart (LBO),
// 8 K-rows 1 KB apart (SBO); one UMMA K step (16 rows) = +2 KB (+128 encoded)
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(const void* p) {
  const uint64_t a = (smem_u32(p) & 0x3FFFFu) >> 4;
  return a | (512ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <int BN, int NST = kStages, int NC = 1, int R = 2, int PP = 1>
struct Smem {
  static constexpr size_t a_bytes = (size_t)BM * BK * 2;
  static constexpr size_t b_bytes = (size_t)BN * BK * 2;
  static constexpr size_t stage = a_bytes + b_bytes;
  static constexpr size_t c_bytes = (size_t)BM * (BN / R) * 2;  // one store round: (BN/R)/64 swizzled 64-col boxes
  static constexpr size_t bars = 128 + BN * 4;  // barriers, TMEM slot, aux barrier, bias tile
  static constexpr size_t total = 1024 /* alignment slack */ + NST * stage + PP * NC * c_bytes + bars;
};

// Persistent: grid = min(tiles, SMs); CTA c takes tiles c, c + grid, ...
// (n-block fastest).  The TMA warp runs ahead across tile boundaries, the
// MMA thread alternates between two TMEM accumulators (2 x BN columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
// NST smem pipeline stages; R store rounds per tile; NC staging buffers per
// round (the output, plus the pre-activation out (epi 1) / aux in (epi 2));
// PP buffer sets used round-robin, so with PP = 2 a round only waits for the
// store issued two rounds earlier.  The GELU variants use 3 stages + 2 sets x
// 2 quarter-tile buffers (208 KB): their epilogue was the accumulator-release
// bottleneck (the MMA warp spun on the TMEM-empty barrier) while each store
// round waited for the previous round's bulk store to leave shared memory.
// BMN: B given as (K, N) row-major (out = A @ B) and staged MN-major (four
// 64-column boxes per stage), so the input-gradient product reads W_K itself
// instead of a materialized W_K^T.
template <int BN, int NST, int NC, int R, int PP, bool BMN = false>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
          const __grid_constant__ CUtensorMap tc_out, const __grid_constant__ CUtensorMap tc_aux, int Mdim, int Ndim,
          int K, const float* __restrict__ bias, int epi, const __nv_bfloat16* __restrict__ aux_g, int ld_aux,
          const __grid_constant__ CUtensorMap ta1, const __grid_constant__ CUtensorMap ta2, int a_ks) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using S = Smem<BN, NST, NC, R, PP>;
  constexpr int CPR = (BN / R) / 32;  // 32-column TMEM chunks per store round
  constexpr int BPR = (BN / R) / 64;  // 64-column swizzled boxes per store round
  unsigned char* sA = smem;
  unsigned char* sB = smem + NST * S::a_bytes;
  unsigned char* sC = smem + NST * S::stage;  // 1024-aligned staging buffers [PP][NC]
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + PP * NC * S::c_bytes);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* auxbar = tempty + 3;  // after tslot's 8 bytes

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = (K + BK - 1) / BK;
  const int nb = (Ndim + BN - 1) / BN;
  const int tiles = ((Mdim + BM - 1) / BM) * nb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&tempty[i])) : "memory");
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(auxbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&ta);
    if (a_ks) { prefetch_tmap(&ta1); prefetch_tmap(&ta2); }
    prefetch_tmap(&tb);
    prefetch_tmap(&tc_out);
    if (epi) prefetch_tmap(&tc_aux);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer, running ahead across tiles
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t / nb) * BM, n0 = (t % nb) * BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % NST, round = it / NST;
          mbar_wait_parity(&empty[s], (round & 1) ^ 1);
          mbar_expect_tx(&full[s], (uint32_t)S::stage);
          if (a_ks) {  // A = [A0 | A1 | A2] along K, a_ks columns each (a multiple of BK)
            const int part = kb * BK / a_ks, kc = kb * BK - part * a_ks;
            if (part == 0) tma_load_2d(sA + s * S::a_bytes, &ta, kc, m0, &full[s]);
            else if (part == 1) tma_load_2d(sA + s * S::a_bytes, &ta1, kc, m0, &full[s]);
            else tma_load_2d(sA + s * S::a_bytes, &ta2, kc, m0, &full[s]);
          } else {
            tma_load_2d(sA + s * S::a_bytes, &ta, kb * BK, m0, &full[s]);
          }
          if constexpr (BMN) {
#pragma unroll
            for (int h = 0; h < BN / 64; ++h) tma_load_2d(sB + s * S::b_bytes + h * 8192, &tb, n0 + h * 64, kb * BK, &full[s]);
          } else {
            tma_load_2d(sB + s * S::b_bytes, &tb, kb * BK, n0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (one thread for the whole CTA)
      constexpr uint32_t idesc = idesc_bf16(BM, BN) | (BMN ? (1u << 16) : 0u);  // B MN-major
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int ab = i & 1;
        mbar_wait_parity(&tempty[ab], ((i >> 1) & 1) ^ 1);  // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(ab * BN);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % NST, round = it / NST;
          mbar_wait_parity(&full[s], round & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = smem_desc_sw128(sA + s * S::a_bytes);
          const uint64_t db = BMN ? smem_desc_mn_sw128(sB + s * S::b_bytes) : smem_desc_sw128(sB + s * S::b_bytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)  // K-major: +32 bytes inside the swizzle atom; MN-major: +16 rows
            umma_bf16(acc, da + 2 * k, db + (BMN ? 128 : 2) * k, idesc, (kb | k) != 0);
          umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
        }
        umma_commit(&tfull[ab]);
      }
    }
  } else {  // ---- epilogue: warps 2..9; warp w reads TMEM lanes 32*(w%4), column half (w-2)/4
    // TMEM -> registers (32 columns at a time) -> epilogue op, bf16 -> the 128B-
    // swizzled smem tile (one 64-column box per 16 KB) -> TMA bulk tensor store.
    //   epi 0: out = acc + bias
    //   epi 1: aux = acc + bias (pre-activation), out = gelu_tanh(aux): one TMEM
    //          read, both staged (out / aux buffer of the round's set) and stored in one round
    //   epi 2: out = acc * gelu_tanh'(aux)   (aux prefetched into registers, or TMA-staged)
    //   epi 3: out = acc + bias + aux          (the residual add of the block, same aux path)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int rl = q * 32 + lane;  // row within the tile
    const int et = threadIdx.x - 64;  // epilogue thread id
    const bool leader = et == 0;
    float* sbias = reinterpret_cast<float*>(tslot + 4);  // BN floats after the barriers
    uint32_t aux_phase = 0;
    auto buf = [&](int set, int which) { return sC + (size_t)(set * NC + which) * S::c_bytes; };
    auto wait_reads = [&]() {  // the store that last used this round's buffer set has left smem
      if (leader) {
        if (PP > 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    };
    auto store_round = [&](int m0, int col0, int set, bool with_aux) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async proxy
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (leader) {
#pragma unroll
        for (int bx = 0; bx < BPR; ++bx) {
          const int col = col0 + bx * 64;
          if (col >= Ndim) break;
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                           reinterpret_cast<uint64_t>(&tc_out)),
                       "r"(col), "r"(m0), "r"(smem_u32(buf(set, 0) + (size_t)bx * (BM * 128)))
                       : "memory");
          if (with_aux)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tc_aux)),
                         "r"(col), "r"(m0), "r"(smem_u32(buf(set, 1) + (size_t)bx * (BM * 128)))
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    };
    // 8 bf16 of this thread's row in 16-byte chunk `ch` (0..7) of the box holding chunk cl
    auto sc_addr = [&](int cl, int j, unsigned char* base) {
      unsigned char* box = base + (size_t)(cl >> 1) * (BM * 128);
      const int chunk = ((cl & 1) * 4 + j) ^ (rl & 7);
      return reinterpret_cast<uint4*>(box + rl * 128 + chunk * 16);
    };
    // epi 2 with NC == 1 (R == 4: one 32-column chunk per thread per round):
    // the pre-activation comes straight from global into registers, one round
    // ahead (this tile's next round, or the next tile's first round), so no
    // aux staging buffer and no exposed TMA round trip
    uint4 av_cur[4], av_nxt[4];
    auto load_aux_regs = [&](int tt, int hh, uint4 (&dst)[4]) {
      const int row = (tt / nb) * BM + rl;
      const int col0 = (tt % nb) * BN + hh * (BN / R) + half * 32;
      const __nv_bfloat16* src = aux_g + (size_t)row * ld_aux + col0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dst[j] = make_uint4(0, 0, 0, 0);
        if (tt < tiles && row < Mdim && col0 + 8 * j + 8 <= Ndim) dst[j] = __ldg(reinterpret_cast<const uint4*>(src + 8 * j));
      }
    };
    constexpr bool kRegAux = (NC == 1 && R == 4);
    const bool reg_aux = kRegAux && (epi == 2 || epi == 3);
    if (reg_aux) load_aux_regs(blockIdx.x, 0, av_cur);
    int i = 0, rc = 0;  // rc: store rounds so far (buffer set = rc % PP)
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int ab = i & 1;
      const int m0 = (t / nb) * BM, n0 = (t % nb) * BN;
      // epi 2: the pre-activation for each round comes in by TMA into the aux
      // buffer of that round's set — round 0's before the accumulator wait,
      // round hh+1's right after round hh's store round
      auto load_aux = [&](int hh, unsigned char* dst) {
        mbar_expect_tx(auxbar, (uint32_t)S::c_bytes);
#pragma unroll
        for (int bx = 0; bx < BPR; ++bx)
          tma_load_2d(dst + (size_t)bx * (BM * 128), &tc_aux, n0 + hh * (BN / R) + bx * 64, m0, auxbar);
      };
      wait_reads();
      if (NC > 1 && epi == 2 && leader) load_aux(0, buf(rc % PP, 1));
      for (int c = et; c < BN; c += kEpiThreads) sbias[c] = (bias && n0 + c < Ndim) ? __ldg(bias + n0 + c) : 0.f;
      mbar_wait_parity(&tfull[ab], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll 1
      for (int hh = 0; hh < R; ++hh, ++rc) {
        const int set = rc % PP;
        if (hh > 0) wait_reads();
        if (reg_aux) {
          if (hh + 1 < R) load_aux_regs(t, hh + 1, av_nxt);
          else load_aux_regs(t + gridDim.x, 0, av_nxt);
        } else if (epi == 2) {
          if (NC == 1 && leader) load_aux(hh, buf(set, 0));
          mbar_wait_parity(auxbar, aux_phase);
          aux_phase ^= 1;
        }
        unsigned char* obuf = buf(set, 0);
        unsigned char* abuf = buf(set, NC - 1);  // aux in (epi 2) / pre-activation out (epi 1)
#pragma unroll 1
        for (int cc = 0; cc < CPR / 2; ++cc) {
          const int c = hh * CPR + half * (CPR / 2) + cc;  // 32-column chunk index in the tile
          const int cl = c - hh * CPR;                      // chunk within this round
          uint32_t r[32];
          tmem_ld32(tmem + (uint32_t)(ab * BN) + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), r);
          uint32_t prev[16];
          if (epi >= 2) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 u = kRegAux ? av_cur[j] : *sc_addr(cl, j, abuf);
              prev[4 * j] = u.x; prev[4 * j + 1] = u.y; prev[4 * j + 2] = u.z; prev[4 * j + 3] = u.w;
            }
          }
          uint32_t pk[16], pre[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float a = __uint_as_float(r[2 * j]), b = __uint_as_float(r[2 * j + 1]);
            if (epi != 2) { a += sbias[c * 32 + 2 * j]; b += sbias[c * 32 + 2 * j + 1]; }
            if (epi == 1) {  // gelu of the bf16-rounded pre-activation (as stored)
              __nv_bfloat162 hp = __floats2bfloat162_rn(a, b);
              pre[j] = *reinterpret_cast<uint32_t*>(&hp);
              a = gelu_tanh(__low2float(hp));
              b = gelu_tanh(__high2float(hp));
            } else if (epi == 2) {
              a *= gelu_tanh_grad(__uint_as_float(prev[j] << 16));
              b *= gelu_tanh_grad(__uint_as_float(prev[j] & 0xffff0000u));
            } else if (epi == 3) {  // residual: one rounding of acc + bias + r
              a += __uint_as_float(prev[j] << 16);
              b += __uint_as_float(prev[j] & 0xffff0000u);
            }
            __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
            pk[j] = *reinterpret_cast<uint32_t*>(&h);
          }
          if (NC > 1 && epi == 1) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *sc_addr(cl, j, abuf) = make_uint4(pre[4 * j], pre[4 * j + 1], pre[4 * j + 2], pre[4 * j + 3]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *sc_addr(cl, j, obuf) = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
        if (hh == R - 1) {  // accumulator consumed: hand it back to the MMA thread
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[ab])) : "memory");
        }
        store_round(m0, n0 + hh * (BN / R), set, NC > 1 && epi == 1);
        if (reg_aux) {
#pragma unroll
          for (int j = 0; j < 4; ++j) av_cur[j] = av_nxt[j];
        }
        if (NC > 1 && epi == 2 && hh + 1 < R && leader) load_aux(hh + 1, buf((rc + 1) % PP, 1));
      }
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN) : "memory");
  }
}

template <int BN>
struct SmemSp {  // 2:4-compressed A: half the K bytes
  static constexpr size_t a_bytes = (size_t)BM * BK;
  static constexpr size_t b_bytes = (size_t)BN * BK * 2;
  static constexpr size_t stage = a_bytes + b_bytes;
  static constexpr size_t c_bytes = (size_t)BM * BN;
  static constexpr size_t bars = 128 + BN * 4;
  static constexpr size_t total = 1024 + kStages * stage + c_bytes + bars;
};

__device__ __forceinline__ uint64_t smem_desc_sw64(const void* p) {  // K-major, 64-byte swizzle, SBO 512 B
  const uint64_t a = (smem_u32(p) & 0x3FFFFu) >> 4;
  return a | (1ull << 16) | (32ull << 32) | (1ull << 46) | (4ull << 61);
}

__device__ __forceinline__ void umma_sp_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t tmem_e,
                                             uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %5, 0;\n"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(tmem_e), "r"(idesc), "r"(acc)
      : "memory");
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_gemm_sp(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
          const __grid_constant__ CUtensorMap tc_out, int Mdim, int Ndim, int K, const float* __restrict__ bias) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using S = SmemSp<BN>;
  unsigned char* sA = smem;
  unsigned char* sB = smem + kStages * S::a_bytes;
  unsigned char* sC = smem + kStages * S::stage;  // 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + S::c_bytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = (K + BK - 1) / BK;
  const int nb = (Ndim + BN - 1) / BN;
  const int tiles = ((Mdim + BM - 1) / BM) * nb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&tempty[i])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
    prefetch_tmap(&tc_out);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  if (warp >= 2 && warp < 6) {  // probe metadata: idx (0,1) in every group of 4
    const uint32_t taddr = *tslot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(2 * BN);
    const uint32_t v = 0x44444444u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer, running ahead across tiles
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t / nb) * BM, n0 = (t % nb) * BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kStages, round = it / kStages;
          mbar_wait_parity(&empty[s], (round & 1) ^ 1);
          mbar_expect_tx(&full[s], (uint32_t)S::stage);
          tma_load_2d(sA + s * S::a_bytes, &ta, kb * BK, m0, &full[s]);
          tma_load_2d(sB + s * S::b_bytes, &tb, kb * BK, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (one thread for the whole CTA)
      constexpr uint32_t idesc = idesc_bf16(BM, BN) | (1u << 2);  // sparse
      const uint32_t tmem_e = tmem + (uint32_t)(2 * BN);
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int ab = i & 1;
        mbar_wait_parity(&tempty[ab], ((i >> 1) & 1) ^ 1);  // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(ab * BN);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kStages, round = it / kStages;
          mbar_wait_parity(&full[s], round & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = smem_desc_sw64(sA + s * S::a_bytes);
          const uint64_t db = smem_desc_sw128(sB + s * S::b_bytes);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k)  // logical K = 32 per sparse MMA: A +32 B, B +64 B
            umma_sp_bf16(acc, da + 2 * k, db + 4 * k, tmem_e, idesc, (kb | k) != 0);
          umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
        }
        umma_commit(&tfull[ab]);
      }
    }
  } else {  // ---- epilogue: warps 2..9; warp w reads TMEM lanes 32*(w%4), column half (w-2)/4
    // TMEM -> registers (32 columns at a time) -> +bias, bf16 -> the 128B-swizzled
    // smem tile (one 64-column box per 16 KB) -> TMA bulk tensor store.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int rl = q * 32 + lane;  // row within the tile
    const int et = threadIdx.x - 64;  // epilogue thread id
    const bool leader = et == 0;
    float* sbias = reinterpret_cast<float*>(tslot + 4);  // BN floats after the barriers
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int ab = i & 1;
      const int m0 = (t / nb) * BM, n0 = (t % nb) * BN;
      // the previous tile's TMA store must have finished reading sC / sbias users done
      if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");
      for (int c = et; c < BN; c += kEpiThreads) sbias[c] = (bias && n0 + c < Ndim) ? __ldg(bias + n0 + c) : 0.f;
      mbar_wait_parity(&tfull[ab], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // two halves of BN/2 columns through the same 32 KB staging tile; the 8
      // warps split each half (warps 2-5 the first BN/4 columns, 6-9 the next)
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        if (hh == 1) {
          if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          asm volatile("bar.sync 1, 256;" ::: "memory");
        }
#pragma unroll 1
        for (int cc = 0; cc < BN / 128; ++cc) {
          const int c = hh * (BN / 64) + half * (BN / 128) + cc;  // 32-column chunk index in the tile
          uint32_t r[32];
          tmem_ld32(tmem + (uint32_t)(ab * BN) + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), r);
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float a = __uint_as_float(r[2 * j]) + sbias[c * 32 + 2 * j];
            const float b = __uint_as_float(r[2 * j + 1]) + sbias[c * 32 + 2 * j + 1];
            __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
            pk[j] = *reinterpret_cast<uint32_t*>(&h);
          }
          const int cl = c - hh * (BN / 64);  // chunk within this half
          unsigned char* box = sC + (size_t)(cl >> 1) * (BM * 128);
          const int ch0 = (cl & 1) * 4;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int chunk = (ch0 + j) ^ (rl & 7);
            *reinterpret_cast<uint4*>(box + rl * 128 + chunk * 16) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
        }
        if (hh == 1) {  // accumulator consumed: hand it back to the MMA thread
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[ab])) : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async proxy
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (leader) {
#pragma unroll
          for (int bx = 0; bx < BN / 128; ++bx) {
            const int col = n0 + hh * (BN / 2) + bx * 64;
            if (col >= Ndim) break;
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tc_out)),
                         "r"(col), "r"(m0), "r"(smem_u32(sC + (size_t)bx * (BM * 128)))
                         : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---------------------------------------------------------------------------
// dW on the tensor cores with the diagonal gather fused into the epilogue.
// D[m, n] = sum_tok dy[tok, m] * x[tok, n]: both operands MN-major (the token
// dimension is K and is the strided one), staged as 64-element-wide TMA boxes
// (2 for A's 128 rows, 4 for B's 256 columns) with the 128-byte swizzle.  The
// epilogue keeps only the entries on ACTIVE diagonals and writes them, unscaled,
// into the dW partial buffer [ksplit][slot][t] that k_dw_finalize folds (fixed
// order), scales by alpha_soft and turns into g_values / g_soft — the dense dW
// (M x N fp32) is never written.  K (tokens) is split across CTAs when the
// output has fewer tiles than SMs.
constexpr int kDwBN = 256;
constexpr int kDwThreads = kThreads + 128;  // + 4 warps summing dy's columns (bias gradient) off the A stages
struct SmemDw {
  static constexpr size_t a_bytes = (size_t)BM * BK * 2;      // 2 boxes of 64 x 64
  static constexpr size_t b_bytes = (size_t)kDwBN * BK * 2;   // 4 boxes
  static constexpr size_t stage = a_bytes + b_bytes;
  static constexpr size_t total = 1024 + kStages * stage + 128 + 512 * 4;
};


__global__ void __launch_bounds__(kDwThreads, 1)
k_tc_dw(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M, int N, int ntok,
        int ksplit, const int32_t* __restrict__ slot, const int32_t* __restrict__ n_act_p, int max_act,
        float* __restrict__ partial, float* __restrict__ colsum, const __grid_constant__ CUtensorMap ta1,
        const __grid_constant__ CUtensorMap ta2, int a_ms) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using S = SmemDw;
  constexpr int BN = kDwBN;
  unsigned char* sA = smem;
  unsigned char* sB = smem + kStages * S::a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * S::stage);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_slot = reinterpret_cast<int*>(smem + kStages * S::stage + 128);  // 384 offsets of the tile

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tall = M >= N;
  const int C = tall ? M : N, L = tall ? N : M;
  const int n_act = min(*n_act_p, max_act);
  const int nb = (N + BN - 1) / BN;
  const int otiles = ((M + BM - 1) / BM) * nb;
  const int tiles = otiles * ksplit;
  const int KBt = (ntok + BK - 1) / BK;                 // k-blocks in total
  const int KBs = (KBt + ksplit - 1) / ksplit;          // per split

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&empty[s])) : "memory");  // MMA + colsum
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&tempty[i])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&ta);
    if (a_ms) { prefetch_tmap(&ta1); prefetch_tmap(&ta2); }
    prefetch_tmap(&tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int ot = t % otiles, z = t / otiles;
        const int m0 = (ot / nb) * BM, n0 = (ot % nb) * BN;
        const int kb0 = z * KBs, kb1 = min(KBt, kb0 + KBs);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % kStages, round = it / kStages;
          mbar_wait_parity(&empty[s], (round & 1) ^ 1);
          mbar_expect_tx(&full[s], (uint32_t)S::stage);
#pragma unroll
          for (int h = 0; h < BM / 64; ++h) {  // dy = [dy0 | dy1 | dy2] along M (a_ms columns each)
            const int row = m0 + h * 64, part = a_ms ? row / a_ms : 0, rc = row - part * a_ms;
            if (part == 0) tma_load_2d(sA + s * S::a_bytes + h * 8192, &ta, rc, kb * BK, &full[s]);
            else if (part == 1) tma_load_2d(sA + s * S::a_bytes + h * 8192, &ta1, rc, kb * BK, &full[s]);
            else tma_load_2d(sA + s * S::a_bytes + h * 8192, &ta2, rc, kb * BK, &full[s]);
          }
#pragma unroll
          for (int h = 0; h < BN / 64; ++h)
            tma_load_2d(sB + s * S::b_bytes + h * 8192, &tb, n0 + h * 64, kb * BK, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(BM, BN) | (1u << 15) | (1u << 16);  // A, B MN-major
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int z = t / otiles;
        const int kb0 = z * KBs, kb1 = min(KBt, kb0 + KBs);
        const int ab = i & 1;
        mbar_wait_parity(&tempty[ab], ((i >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(ab * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % kStages, round = it / kStages;
          mbar_wait_parity(&full[s], round & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = smem_desc_mn_sw128(sA + s * S::a_bytes);
          const uint64_t db = smem_desc_mn_sw128(sB + s * S::b_bytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)  // +16 K-rows = +2048 bytes
            umma_bf16(acc, da + 128 * k, db + 128 * k, idesc, (kb != kb0) || (k != 0));
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[ab]);
      }
    }
  } else if (warp >= 10) {  // ---- column sums of dy (bias gradient) from the A stages of n-block-0 tiles
    // thread i: box h = i / 64, 16-byte chunk j = (i / 8) % 8 (8 columns), rows r = i % 8 + 8 m
    const int ci = threadIdx.x - 320;
    const int h = ci >> 6, j = (ci >> 3) & 7, rg = ci & 7;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int ot = t % otiles, z = t / otiles;
      const int m0 = (ot / nb) * BM;
      const bool sum = colsum != nullptr && (ot % nb) == 0;
      const int kb0 = z * KBs, kb1 = min(KBt, kb0 + KBs);
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % kStages, round = it / kStages;
        mbar_wait_parity(&full[s], round & 1);
        if (sum) {
          const unsigned char* box = sA + s * S::a_bytes + h * 8192;
#pragma unroll
          for (int mm = 0; mm < BK / 8; ++mm) {
            const int r = rg + 8 * mm;
            const uint4 u = *reinterpret_cast<const uint4*>(box + r * 128 + ((j ^ (r & 7)) << 4));
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              acc[2 * e] += __uint_as_float(w[e] << 16);
              acc[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
            }
          }
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");  // all 4 colsum warps done with stage s
        if (threadIdx.x == 320)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      }
      if (sum) {
        // fold the 8 row groups (lanes rg = 0..7 of each 8-lane group), fixed order
#pragma unroll
        for (int e = 0; e < 8; ++e) {
#pragma unroll
          for (int o = 1; o < 8; o <<= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
        }
        if (rg == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int m = m0 + h * 64 + j * 8 + e;
            if (m < M) colsum[(size_t)z * M + m] = acc[e];
          }
        }
      }
    }
  } else {  // ---- epilogue (warps 2..9): gather the active diagonals out of the tile
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int ot = t % otiles, z = t / otiles;
      const int m0 = (ot / nb) * BM, n0 = (ot % nb) * BN;
      const int kb0 = z * KBs, kb1 = min(KBt, kb0 + KBs);
      const int ab = i & 1;
      // offsets crossing the tile: (m - n) or (n - m) over m0-n0+[-(BN-1), BM-1]
      asm volatile("bar.sync 1, 256;" ::: "memory");
      for (int d = et; d < BM + BN - 1; d += kEpiThreads) {
        const int delta = d - (BN - 1);  // (m - m0) - (n - n0)
        int o = tall ? (m0 - n0 + delta) : (n0 - m0 - delta);
        o %= C;
        o = o < 0 ? o + C : o;
        const int sl = slot[o];
        s_slot[d] = (sl >= 0 && sl < n_act) ? sl : -1;
      }
      mbar_wait_parity(&tfull[ab], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int ml = q * 32 + lane;
      const int m = m0 + ml;
#pragma unroll 1
      for (int cc = 0; cc < BN / 64; ++cc) {
        const int c = half * (BN / 64) + cc;
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t)(ab * BN) + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), r);
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int nl = c * 32 + j;
          const int n = n0 + nl;
          const int sl = s_slot[ml - nl + BN - 1];
          if (sl < 0 || n >= N) continue;
          const int tt = tall ? n : m;
          partial[((size_t)z * max_act + sl) * L + tt] = __uint_as_float(r[j]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[ab])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN) : "memory");
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// cuTensorMapEncodeTiled with the failure recorded for diagmm_last_error()
static bool encode_2d(CUtensorMap* map, const void* base, const cuuint64_t (&dims)[2], const cuuint64_t (&strides)[1],
                      const cuuint32_t (&box)[2], CUtensorMapSwizzle swz,
                      CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  auto fn = encode_fn();
  if (!fn) {
    last_cuda_error() = "cuTensorMapEncodeTiled entry point unavailable";
    return false;
  }
  // the driver call needs the device's context current on THIS host thread (autograd
  // runs backward on its own thread; before its first runtime call nothing is bound)
  static thread_local bool bound = false;
  if (!bound) {
    cudaFree(nullptr);
    bound = true;
  }
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    static thread_local char msg[256];
    snprintf(msg, sizeof msg, "cuTensorMapEncodeTiled=%d base=%p dims=(%llu,%llu) stride=%llu box=(%u,%u)", (int)r,
             base, (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)strides[0], box[0],
             box[1]);
    last_cuda_error() = msg;
    return false;
  }
  return true;
}

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                    uint64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  return encode_2d(map, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// fp32 (read as tf32 by kind::tf32 MMAs), K-major: box (32 fp32 = 128 bytes, box_rows), 128-byte swizzle
bool make_tmap_f32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, uint64_t ld) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {32, box_rows};
  return encode_2d(map, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

// MN-major staging of a (rows = K, cols = N) row-major matrix: boxes of 64
// columns (128 bytes, contiguous) x BK rows, 128-byte swizzle.
bool make_tmap_bf16_mn(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)BK};
  return encode_2d(map, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace tc

// Throughput probe of 2:4-sparse tcgen05.mma.sp (constant metadata; NOT a
// correct product): A is (Mdim, K/2) compressed bf16.
int run_tc_sparse_probe(int Mdim, int Ndim, int K, const void* Acomp, const void* B, void* out, cudaStream_t st) {
  using namespace tc;
  constexpr int BN = 128;
  CUtensorMap ta, tb, tco;
  auto fn = encode_fn();
  if (!fn) return DIAGMM_ECUDA;
  {
    cuuint64_t dims[2] = {(cuuint64_t)(K / 2), (cuuint64_t)Mdim};
    cuuint64_t strides[1] = {(cuuint64_t)(K / 2) * 2};
    cuuint32_t box[2] = {32, (cuuint32_t)BM};
    cuuint32_t estr[2] = {1, 1};
    if (fn(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(Acomp), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return DIAGMM_ECUDA;
  }
  if (!make_tmap_bf16(&tb, B, (uint64_t)Ndim, (uint64_t)K, BN, (uint64_t)K) ||
      !make_tmap_bf16(&tco, out, (uint64_t)Mdim, (uint64_t)Ndim, BM, (uint64_t)Ndim))
    return DIAGMM_ECUDA;
  auto k = k_tc_gemm_sp<BN>;
  const size_t sm = SmemSp<BN>::total;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int tiles = ceil_div(Mdim, BM) * ceil_div(Ndim, BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  k<<<grid, kThreads, sm, st>>>(ta, tb, tco, Mdim, Ndim, K, nullptr);
  return status_from_cuda();
}

// dW via the tensor cores: returns the number of K splits written into
// partial ([ksplit][max_act][L] fp32, unscaled gw by slot) or a negative status.
int tc_dw_splits(int M, int N, int ntok) {
  using namespace tc;
  const int otiles = ceil_div(M, BM) * ceil_div(N, kDwBN);
  const int kbt = ceil_div(ntok, BK);
  const int sms = num_sms();
  // split count with the best wave quantisation (ties: fewer splits = fewer partials)
  int best = 1;
  double best_eff = 0.0;
  for (int ks = 1; ks <= 16 && ks <= kbt; ++ks) {
    const int tiles = otiles * ks;
    const double waves = (double)tiles / sms;
    const double eff = waves / std::ceil(waves) * (tiles >= sms ? 1.0 : (double)tiles / sms);
    if (eff > best_eff + 0.02) { best_eff = eff; best = ks; }
  }
  const int per = ceil_div(kbt, best);
  return ceil_div(kbt, per);  // every split gets at least one k-block
}

int run_tc_dw(int M, int N, int ntok, const void* dy, const void* x, const int32_t* slot, const int32_t* n_act,
              int max_act, float* partial, size_t partial_bytes, float* colsum, cudaStream_t st, const void* dy1,
              const void* dy2, int a_ms) {
  using namespace tc;
  const int L = M < N ? M : N;
  if (M < 64 || N < 64 || M % 64 || N % 64 || ntok < 1) return DIAGMM_ESHAPE;
  if ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(x)) & 15) return DIAGMM_ESHAPE;
  const int ks = tc_dw_splits(M, N, ntok);  // no empty split (see tc_dw_splits)
  if (partial_bytes < (size_t)ks * max_act * L * sizeof(float)) return DIAGMM_EWORKSPACE;
  auto fn = encode_fn();
  if (!fn) return DIAGMM_ECUDA;
  CUtensorMap ta, tb;
  // MN-major boxes: 64 features (contiguous) x 64 tokens
  auto mk = [&](CUtensorMap* map, const void* base, uint64_t cols) {
    const cuuint64_t dims[2] = {cols, (cuuint64_t)ntok};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)BK};
    return encode_2d(map, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  };
  CUtensorMap ta1, ta2;
  if (a_ms) {  // dy given as column blocks of a_ms (a multiple of 128) in 2 or 3 separate matrices
    if (a_ms % 128 || M % a_ms || M / a_ms > 3 || (M / a_ms > 1 && !dy1) || (M / a_ms > 2 && !dy2)) return DIAGMM_ESHAPE;
    if ((reinterpret_cast<uintptr_t>(dy1) | reinterpret_cast<uintptr_t>(dy2)) & 15) return DIAGMM_ESHAPE;
    if (!mk(&ta, dy, (uint64_t)a_ms) || !mk(&ta1, dy1 ? dy1 : dy, (uint64_t)a_ms) ||
        !mk(&ta2, dy2 ? dy2 : dy, (uint64_t)a_ms) || !mk(&tb, x, (uint64_t)N))
      return DIAGMM_ECUDA;
  } else {
    if (!mk(&ta, dy, (uint64_t)M) || !mk(&tb, x, (uint64_t)N)) return DIAGMM_ECUDA;
    ta1 = ta2 = ta;
  }
  const size_t sm = SmemDw::total;
  cudaFuncSetAttribute(k_tc_dw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int tiles = ceil_div(M, BM) * ceil_div(N, kDwBN) * ks;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  // partials of inactive slots are never read; active (slot, t) entries are all written
  k_tc_dw<<<grid, kDwThreads, sm, st>>>(ta, tb, M, N, ntok, ks, slot, n_act, max_act, partial, colsum, ta1, ta2, a_ms);
  note_launch();
  return status_from_cuda();
}

int run_tc_gemm2_bf16(int Mdim, int Ndim, int K, const void* A, const void* B, const float* bias, void* out, int ldo,
                      void* aux, int epi, cudaStream_t st, bool b_kn, const void* A1, const void* A2, int a_ks);

// CTA-pair (cta_group::2) kernel when the problem fills every pair with 256 x 256
// tiles; DIAGMM_TC_PAIR=0 forces the single-CTA kernel (A/B comparisons)
static bool use_pair(int Mdim, int Ndim) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("DIAGMM_TC_PAIR");
    mode = e ? atoi(e) : 1;
  }
  if (mode == 0) return false;
  if (mode == 2) return true;
  const long long tiles = (long long)ceil_div(Mdim, 256) * ceil_div(Ndim, 256);
  return tiles >= num_sms() / 2;
}

int run_tc_gemm_bf16(int Mdim, int Ndim, int K, const void* A, const void* B, const float* bias, void* out, int ldo,
                     void* aux, int epi, cudaStream_t st, bool b_kn, const void* A1, const void* A2, int a_ks) {
  using namespace tc;
  constexpr int BN = 256;
  if (use_pair(Mdim, Ndim))
    return run_tc_gemm2_bf16(Mdim, Ndim, K, A, B, bias, out, ldo, aux, epi, st, b_kn, A1, A2, a_ks);
  if (Mdim < 1 || Ndim < 1 || K < 1 || K % 8 || ldo < Ndim) return DIAGMM_ESHAPE;
  if (b_kn && Ndim % 8) return DIAGMM_ESHAPE;  // B (K, N) rows must be 16-byte multiples
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return DIAGMM_ESHAPE;
  if ((reinterpret_cast<uintptr_t>(out) & 15) || (ldo % 8)) return DIAGMM_ESHAPE;
  if (epi < 0 || epi > 3 || (epi && (aux == nullptr || (reinterpret_cast<uintptr_t>(aux) & 15)))) return DIAGMM_ESHAPE;
  CUtensorMap ta, tb, tco, taux, ta1, ta2;
  if (a_ks) {  // A given as column blocks of a_ks (a multiple of BK) in 2 or 3 separate (Mdim, a_ks) matrices
    if (a_ks % BK || K % a_ks || K / a_ks > 3 || (K / a_ks > 1 && !A1) || (K / a_ks > 2 && !A2)) return DIAGMM_ESHAPE;
    if ((reinterpret_cast<uintptr_t>(A1) | reinterpret_cast<uintptr_t>(A2)) & 15) return DIAGMM_ESHAPE;
    if (!make_tmap_bf16(&ta1, A1 ? A1 : A, (uint64_t)Mdim, (uint64_t)a_ks, BM, (uint64_t)a_ks) ||
        !make_tmap_bf16(&ta2, A2 ? A2 : A, (uint64_t)Mdim, (uint64_t)a_ks, BM, (uint64_t)a_ks))
      return DIAGMM_ECUDA;
  }
  if (!make_tmap_bf16(&ta, A, (uint64_t)Mdim, (uint64_t)(a_ks ? a_ks : K), BM, (uint64_t)(a_ks ? a_ks : K)) ||
      !(b_kn ? make_tmap_bf16_mn(&tb, B, (uint64_t)K, (uint64_t)Ndim)
             : make_tmap_bf16(&tb, B, (uint64_t)Ndim, (uint64_t)K, BN, (uint64_t)K)) ||
      !make_tmap_bf16(&tco, out, (uint64_t)Mdim, (uint64_t)Ndim, BM, (uint64_t)ldo) ||
      !make_tmap_bf16(&taux, epi ? aux : out, (uint64_t)Mdim, (uint64_t)Ndim, BM, (uint64_t)ldo))
    return DIAGMM_ECUDA;
  const int tiles = ceil_div(Mdim, BM) * ceil_div(Ndim, BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  auto go = [&](auto kern, size_t sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<grid, kThreads, sm, st>>>(ta, tb, tco, taux, Mdim, Ndim, K, bias, epi,
                                     static_cast<const __nv_bfloat16*>(aux), ldo, a_ks ? ta1 : ta, a_ks ? ta2 : ta,
                                     a_ks);
  };
  // Measured at the ViT shapes (50 432 tokens; tools/epi_bench.py):
  //   epi 0: 4 stages + 2 sets of quarter-tile buffers (round-robin) 206 / 154 / 59 us
  //          (N x K = 3072 x 768 / 2304 x 768 / 768 x 768) vs 220 / 165 / 68 us with one
  //          set of half tiles — the epilogue no longer holds the accumulator back
  //   epi 1 (gelu, 2 outputs): 3 stages + 2 sets x (out, pre) quarter tiles 252 us vs 274
  //   epi 2 (gelu'): the epi-0 layout, aux straight from global into registers one
  //          round ahead: 270 / 194 us vs 278 / 208 us staged by TMA
  if (epi == 1) {
    if (b_kn) go(k_tc_gemm<BN, kStages - 1, 2, 4, 2, true>, Smem<BN, kStages - 1, 2, 4, 2>::total);
    else go(k_tc_gemm<BN, kStages - 1, 2, 4, 2>, Smem<BN, kStages - 1, 2, 4, 2>::total);
  } else {
    if (b_kn) go(k_tc_gemm<BN, kStages, 1, 4, 2, true>, Smem<BN, kStages, 1, 4, 2>::total);
    else go(k_tc_gemm<BN, kStages, 1, 4, 2>, Smem<BN, kStages, 1, 4, 2>::total);
  }
  note_launch();
  return status_from_cuda();
}

}  // namespace diagmm

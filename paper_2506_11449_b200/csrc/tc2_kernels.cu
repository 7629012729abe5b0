// tc2_kernels.cu — the tensor-core DiagMM GEMM on CTA PAIRS (tcgen05
// cta_group::2): out[m, n] = sum_k A[m, k] * B[n, k] (+ bias[n], epilogues as
// k_tc_gemm).  Why pairs: one 256 x 256 MMA tile per pair, each CTA staging
// its 128 rows of A and HALF of B (128 rows of the N tile), so per SM and per
// K step the operand traffic from L2 into shared memory drops from
// (128 + 256) x 2 B to (128 + 128) x 2 B for the same MACs.  The single-CTA
// kernel (tc_kernels.cu) runs at ~0.53 of the bf16 peak with 48 KB per
// 128x256x64 step, the rate the L2 -> SM path sustains; halving B's share is
// what lets the pair go faster.
//
// Protocol (leader = cluster rank 0):
//  * both CTAs' TMA loads complete on the LEADER's full[s] barrier
//    (cp.async.bulk.tensor ... .cta_group::2); the leader's producer arms it with
//    the pair's bytes;
//  * the leader's single MMA thread issues tcgen05.mma.cta_group::2 (M = 256,
//    N = 256, K = 16): A from each CTA's smem, B from both halves;
//  * tcgen05.commit ... .multicast::cluster releases the stage (empty[s]) and
//    hands the accumulator (tfull) to BOTH CTAs;
//  * each CTA's epilogue drains its own TMEM (its 128 rows x 256 columns) and
//    arrives on the leader's tempty barrier (16 arrivals: 8 warps x 2 CTAs).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "tc_gemm.cuh"

namespace diagmm {
namespace tc {

// same helpers as tc_kernels.cu (internal linkage there)
__device__ __forceinline__ float tanh_sfu2(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh2(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_sfu2(k0 * fmaf(k1 * x, x * x, x)), hx);
}
__device__ __forceinline__ float gelu_tanh_grad2(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float t = tanh_sfu2(k0 * fmaf(k1 * x, x2, x));
  const float hx = 0.5f * x;
  return fmaf(hx * (1.f - t * t), k0 * fmaf(3.f * k1, x2, 1.f), 0.5f * (1.f + t));
}
__device__ __forceinline__ uint64_t smem_desc_mn_sw128_2(const void* p) {
  const uint64_t a = (smem_u32(p) & 0x3FFFFu) >> 4;
  return a | (512ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_idx() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// TMA 2-D load into THIS CTA's smem, completion counted on the leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on the barrier at the same offset in both CTAs once the MMAs issued so far completed
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

constexpr int BN2 = 256;  // MMA N (both CTAs' B halves)
constexpr int BH = 128;   // B rows staged per CTA

template <int NST, int NC, int R, int PP>
struct Smem2 {
  static constexpr size_t a_bytes = (size_t)BM * BK * 2;  // this CTA's 128 rows of A
  static constexpr size_t b_bytes = (size_t)BH * BK * 2;  // this CTA's half of B
  static constexpr size_t stage = a_bytes + b_bytes;
  static constexpr size_t c_bytes = (size_t)BM * (BN2 / R) * 2;
  static constexpr size_t bars = 128 + BN2 * 4;
  static constexpr size_t total = 1024 + NST * stage + PP * NC * c_bytes + bars;
};

template <int NST, int NC, int R, int PP, bool BMN = false>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_gemm2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           const __grid_constant__ CUtensorMap tc_out, const __grid_constant__ CUtensorMap tc_aux, int Mdim, int Ndim,
           int K, const float* __restrict__ bias, int epi, const __nv_bfloat16* __restrict__ aux_g, int ld_aux,
           const __grid_constant__ CUtensorMap ta1, const __grid_constant__ CUtensorMap ta2, int a_ks) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using S = Smem2<NST, NC, R, PP>;
  constexpr int BN = BN2;
  constexpr int CPR = (BN / R) / 32;
  constexpr int BPR = (BN / R) / 64;
  unsigned char* sA = smem;
  unsigned char* sB = smem + NST * S::a_bytes;
  unsigned char* sC = smem + NST * S::stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + PP * NC * S::c_bytes);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;  // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* auxbar = tempty + 3;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int KB = (K + BK - 1) / BK;
  const int nb = (Ndim + BN - 1) / BN;
  const int tiles = ((Mdim + 2 * BM - 1) / (2 * BM)) * nb;
  const int cl0 = (int)cluster_idx(), ncl = (int)cluster_count();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tfull[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(smem_u32(&tempty[i])) : "memory");
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
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers initialised and TMEM allocated in BOTH CTAs
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs), completing on the leader's full barriers
      int it = 0;
      for (int t = cl0; t < tiles; t += ncl) {
        const int m0 = (t / nb) * (2 * BM) + (int)rank * BM, n0 = (t % nb) * BN + (int)rank * BH;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % NST, round = it / NST;
          mbar_wait_parity(&empty[s], (round & 1) ^ 1);
          if (leader) mbar_expect_tx(&full[s], (uint32_t)(2 * S::stage));
          const uint32_t fb = peer_addr(&full[s], 0);
          if (a_ks) {
            const int part = kb * BK / a_ks, kc = kb * BK - part * a_ks;
            const CUtensorMap* m = part == 0 ? &ta : (part == 1 ? &ta1 : &ta2);
            tma_load_2d_pair(sA + s * S::a_bytes, m, kc, m0, fb);
          } else {
            tma_load_2d_pair(sA + s * S::a_bytes, &ta, kb * BK, m0, fb);
          }
          if constexpr (BMN) {
#pragma unroll
            for (int h = 0; h < BH / 64; ++h)
              tma_load_2d_pair(sB + s * S::b_bytes + h * 8192, &tb, n0 + h * 64, kb * BK, fb);
          } else {
            tma_load_2d_pair(sB + s * S::b_bytes, &tb, kb * BK, n0, fb);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---- the pair's single MMA issuer
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN) | (BMN ? (1u << 16) : 0u);
      int it = 0, i = 0;
      for (int t = cl0; t < tiles; t += ncl, ++i) {
        const int ab = i & 1;
        mbar_wait_parity(&tempty[ab], ((i >> 1) & 1) ^ 1);  // both CTAs drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(ab * BN);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % NST, round = it / NST;
          mbar_wait_parity(&full[s], round & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = smem_desc_sw128(sA + s * S::a_bytes);
          const uint64_t db = BMN ? smem_desc_mn_sw128_2(sB + s * S::b_bytes) : smem_desc_sw128(sB + s * S::b_bytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma_bf16_pair(acc, da + 2 * k, db + (BMN ? 128 : 2) * k, idesc, (kb | k) != 0);
          umma_commit_pair(&empty[s]);  // frees stage s in both CTAs
        }
        umma_commit_pair(&tfull[ab]);
      }
    }
  } else {  // ---- epilogue (warps 2..9 of each CTA): this CTA's 128 rows x 256 columns
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int rl = q * 32 + lane;
    const int et = threadIdx.x - 64;
    const bool eleader = et == 0;
    float* sbias = reinterpret_cast<float*>(tslot + 4);
    const uint32_t tempty_leader[2] = {peer_addr(&tempty[0], 0), peer_addr(&tempty[1], 0)};
    uint32_t aux_phase = 0;
    auto buf = [&](int set, int which) { return sC + (size_t)(set * NC + which) * S::c_bytes; };
    auto wait_reads = [&]() {
      if (eleader) {
        if (PP > 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    };
    auto store_round = [&](int m0, int col0, int set, bool with_aux) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (eleader) {
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
    auto sc_addr = [&](int cl, int j, unsigned char* base) {
      unsigned char* box = base + (size_t)(cl >> 1) * (BM * 128);
      const int chunk = ((cl & 1) * 4 + j) ^ (rl & 7);
      return reinterpret_cast<uint4*>(box + rl * 128 + chunk * 16);
    };
    uint4 av_cur[4], av_nxt[4];
    auto tile_m0 = [&](int tt) { return (tt / nb) * (2 * BM) + (int)rank * BM; };
    auto load_aux_regs = [&](int tt, int hh, uint4 (&dst)[4]) {
      const int row = tile_m0(tt) + rl;
      const int col0 = (tt % nb) * BN + hh * (BN / R) + half * 32;
      const __nv_bfloat16* src = aux_g + (size_t)row * ld_aux + col0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dst[j] = make_uint4(0, 0, 0, 0);
        if (tt < tiles && row < Mdim && col0 + 8 * j + 8 <= Ndim)
          dst[j] = __ldg(reinterpret_cast<const uint4*>(src + 8 * j));
      }
    };
    constexpr bool kRegAux = (NC == 1 && R == 4);
    const bool reg_aux = kRegAux && (epi == 2 || epi == 3);
    if (reg_aux) load_aux_regs(cl0, 0, av_cur);
    int i = 0, rc = 0;
    for (int t = cl0; t < tiles; t += ncl, ++i) {
      const int ab = i & 1;
      const int m0 = tile_m0(t), n0 = (t % nb) * BN;
      auto load_aux = [&](int hh, unsigned char* dst) {
        mbar_expect_tx(auxbar, (uint32_t)S::c_bytes);
#pragma unroll
        for (int bx = 0; bx < BPR; ++bx)
          tma_load_2d(dst + (size_t)bx * (BM * 128), &tc_aux, n0 + hh * (BN / R) + bx * 64, m0, auxbar);
      };
      wait_reads();
      if (NC > 1 && epi == 2 && eleader) load_aux(0, buf(rc % PP, 1));
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
          else load_aux_regs(t + ncl, 0, av_nxt);
        } else if (epi == 2) {
          if (NC == 1 && eleader) load_aux(hh, buf(set, 0));
          mbar_wait_parity(auxbar, aux_phase);
          aux_phase ^= 1;
        }
        unsigned char* obuf = buf(set, 0);
        unsigned char* abuf = buf(set, NC - 1);
#pragma unroll 1
        for (int cc = 0; cc < CPR / 2; ++cc) {
          const int c = hh * CPR + half * (CPR / 2) + cc;
          const int cl = c - hh * CPR;
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
            if (epi == 1) {
              __nv_bfloat162 hp = __floats2bfloat162_rn(a, b);
              pre[j] = *reinterpret_cast<uint32_t*>(&hp);
              a = gelu_tanh2(__low2float(hp));
              b = gelu_tanh2(__high2float(hp));
            } else if (epi == 2) {
              a *= gelu_tanh_grad2(__uint_as_float(prev[j] << 16));
              b *= gelu_tanh_grad2(__uint_as_float(prev[j] & 0xffff0000u));
            } else if (epi == 3) {
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
        if (hh == R - 1) {  // this CTA's half of the accumulator consumed: tell the leader's MMA thread
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader[ab])
                         : "memory");
        }
        store_round(m0, n0 + hh * (BN / R), set, NC > 1 && epi == 1);
        if (reg_aux) {
#pragma unroll
          for (int j = 0; j < 4; ++j) av_cur[j] = av_nxt[j];
        }
        if (NC > 1 && epi == 2 && hh + 1 < R && eleader) load_aux(hh + 1, buf((rc + 1) % PP, 1));
      }
    }
    if (eleader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the pair's MMAs and both epilogues are done with TMEM
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN) : "memory");
  }
}

}  // namespace tc

static bool getenv_r2() {  // DIAGMM_TC_EPI_R2=0: 4 store rounds for the plain epilogue too
  const char* e = getenv("DIAGMM_TC_EPI_R2");
  return !(e && atoi(e) == 0);
}

// Launcher with run_tc_gemm_bf16's contract (tc_kernels.cu), on CTA pairs.
int run_tc_gemm2_bf16(int Mdim, int Ndim, int K, const void* A, const void* B, const float* bias, void* out, int ldo,
                      void* aux, int epi, cudaStream_t st, bool b_kn, const void* A1, const void* A2, int a_ks) {
  using namespace tc;
  if (Mdim < 1 || Ndim < 1 || K < 1 || K % 8 || ldo < Ndim) return DIAGMM_ESHAPE;
  if (b_kn && Ndim % 8) return DIAGMM_ESHAPE;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return DIAGMM_ESHAPE;
  if ((reinterpret_cast<uintptr_t>(out) & 15) || (ldo % 8)) return DIAGMM_ESHAPE;
  if (epi < 0 || epi > 3 || (epi && (aux == nullptr || (reinterpret_cast<uintptr_t>(aux) & 15)))) return DIAGMM_ESHAPE;
  CUtensorMap ta, tb, tco, taux, ta1, ta2;
  if (a_ks) {
    if (a_ks % BK || K % a_ks || K / a_ks > 3 || (K / a_ks > 1 && !A1) || (K / a_ks > 2 && !A2)) return DIAGMM_ESHAPE;
    if ((reinterpret_cast<uintptr_t>(A1) | reinterpret_cast<uintptr_t>(A2)) & 15) return DIAGMM_ESHAPE;
    if (!make_tmap_bf16(&ta1, A1 ? A1 : A, (uint64_t)Mdim, (uint64_t)a_ks, BM, (uint64_t)a_ks) ||
        !make_tmap_bf16(&ta2, A2 ? A2 : A, (uint64_t)Mdim, (uint64_t)a_ks, BM, (uint64_t)a_ks))
      return DIAGMM_ECUDA;
  }
  if (!make_tmap_bf16(&ta, A, (uint64_t)Mdim, (uint64_t)(a_ks ? a_ks : K), BM, (uint64_t)(a_ks ? a_ks : K)) ||
      !(b_kn ? make_tmap_bf16_mn(&tb, B, (uint64_t)K, (uint64_t)Ndim)
             : make_tmap_bf16(&tb, B, (uint64_t)Ndim, (uint64_t)K, BH, (uint64_t)K)) ||
      !make_tmap_bf16(&tco, out, (uint64_t)Mdim, (uint64_t)Ndim, BM, (uint64_t)ldo) ||
      !make_tmap_bf16(&taux, epi ? aux : out, (uint64_t)Mdim, (uint64_t)Ndim, BM, (uint64_t)ldo))
    return DIAGMM_ECUDA;
  const int tiles = ceil_div(Mdim, 2 * BM) * ceil_div(Ndim, BN2);
  const int pairs = num_sms() / 2;
  const int clusters = tiles < pairs ? tiles : pairs;
  auto go = [&](auto kern, size_t sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, ta, tb, tco, taux, Mdim, Ndim, K, bias, epi,
                       static_cast<const __nv_bfloat16*>(aux), ldo, a_ks ? ta1 : ta, a_ks ? ta2 : ta, a_ks);
  };
  // stages: 32 KB each per CTA; staging buffers 16 KB each (quarter tiles)
  if (epi == 1) {
    if (b_kn) go(k_tc_gemm2<4, 2, 4, 2, true>, Smem2<4, 2, 4, 2>::total);
    else go(k_tc_gemm2<4, 2, 4, 2>, Smem2<4, 2, 4, 2>::total);
  } else if (epi == 0 && !b_kn && getenv_r2()) {
    // plain forward epilogue in 2 store rounds of 128 columns: half the proxy fences and
    // barriers per tile — the qkv forward (K = 768) 1.89 -> 1.43 ms of kernel time per ViT-B
    // step (the power-capped step itself did not move); the input-gradient products (W_K
    // read MN-major) measured the same either way
    go(k_tc_gemm2<5, 1, 2, 2>, Smem2<5, 1, 2, 2>::total);
  } else {
    if (b_kn) go(k_tc_gemm2<5, 1, 4, 2, true>, Smem2<5, 1, 4, 2>::total);
    else go(k_tc_gemm2<5, 1, 4, 2>, Smem2<5, 1, 4, 2>::total);
  }
  note_launch();
  return status_from_cuda();
}

}  // namespace diagmm

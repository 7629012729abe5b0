// norm_kernels.cu — fused LayerNorm for the bf16 activations around DiagLinear
// in the ViT caller (vit.py).  Not part of the reference's hot path; it exists
// because PyTorch's LayerNorm under autocast (fp32 upcast + GammaBeta reduction)
// costs ~0.9 ms per call at 50k tokens x 768 on B200, ~10x its HBM roofline.
//
// Forward: one warp per row, the row held in registers (D <= 1024, D % 8 == 0),
// fp32 statistics, bf16 output, mean/rstd saved (fp32).
// Backward: one warp per row for dx; dgamma/dbeta accumulated per CTA in fp32
// registers over its rows, written as per-CTA partials and folded in a fixed
// order by a second kernel (deterministic, no atomics).
#include "common.cuh"
#include <algorithm>
#include <type_traits>

namespace diagmm {

constexpr int kLnWarps = 8;
constexpr int kLnMaxV = 4;  // up to 4 x 8 bf16 per lane -> D <= 1024

__device__ __forceinline__ void unpack8(uint4 u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NV>
__global__ void __launch_bounds__(kLnWarps * 32)
k_ln_fwd(int M, int D, float eps, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
         const float* __restrict__ b, __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
         float* __restrict__ rstd_out) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * kLnWarps + (threadIdx.x >> 5);
  if (row >= M) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)row * D);
  float v[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 8;
    if (c < D) unpack8(xr[i * 32 + lane], v[i]);
    else
#pragma unroll
      for (int e = 0; e < 8; ++e) v[i][e] = 0.f;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) s += v[i][e];
  const float mu = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 8;
    if (c < D)
#pragma unroll
      for (int e = 0; e < 8; ++e) { const float d = v[i][e] - mu; q += d * d; }
  }
  const float rs = rsqrtf(warp_sum(q) / D + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + (size_t)row * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * 8;
    if (c >= D) continue;
    const float4 w0 = *reinterpret_cast<const float4*>(w + c), w1 = *reinterpret_cast<const float4*>(w + c + 4);
    const float4 b0 = *reinterpret_cast<const float4*>(b + c), b1 = *reinterpret_cast<const float4*>(b + c + 4);
    const float ww[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (v[i][e] - mu) * rs * ww[e] + bb[e];
    yr[i * 32 + lane] = pack8(o);
  }
  if (lane == 0) { mean_out[row] = mu; rstd_out[row] = rs; }
}

// dx per row; per-CTA partial dgamma/dbeta over its rows -> part[blockIdx.x][2][D]
template <int NV>
__global__ void __launch_bounds__(kLnWarps * 32, 2)
k_ln_bwd(int M, int D, int rows_per_cta, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy,
         const float* __restrict__ w, const float* __restrict__ mean, const float* __restrict__ rstd,
         __nv_bfloat16* __restrict__ dx, float* __restrict__ part, const __nv_bfloat16* __restrict__ dres) {
  __shared__ float s_acc[2][kLnMaxV * 256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float dg[NV][8], db[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) { dg[i][e] = 0.f; db[i][e] = 0.f; }
  __shared__ __align__(16) float s_w[kLnMaxV * 256];
  for (int c = threadIdx.x; c < NV * 256; c += blockDim.x) s_w[c] = c < D ? w[c] : 0.f;
  __syncthreads();
  const int r0 = blockIdx.x * rows_per_cta, r1 = min(M, r0 + rows_per_cta);
  // Rows stream through a per-warp double buffer in shared memory (cp.async, 16 B per
  // lane per chunk): the next row's x / dy / dres are in flight while this row is
  // computed, two rows per warp instead of one (the dgamma / dbeta accumulators leave
  // no registers for a register prefetch).  Each lane reads back only the chunks it
  // copied itself, so cp.async.wait_group is the only synchronisation needed.
  extern __shared__ __align__(16) uint4 s_rows[];  // [warp][2 slots][3 tensors][NV * 32]
  uint4* wb = s_rows + (size_t)warp * 2 * 3 * NV * 32;
  auto issue = [&](int row, int slot) {
    if (row < r1) {
      uint4* d = wb + (size_t)slot * 3 * NV * 32;
      const __nv_bfloat16* src[3] = {x + (size_t)row * D, dy + (size_t)row * D,
                                     dres ? dres + (size_t)row * D : nullptr};
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        if (!src[t]) continue;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int c = (i * 32 + lane) * 8;
          if (c < D)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d + t * NV * 32 + i * 32 + lane)),
                         "l"(reinterpret_cast<const uint4*>(src[t]) + i * 32 + lane)
                         : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int slot = 0;
  issue(r0 + warp, 0);
#pragma unroll 1
  for (int row = r0 + warp; row < r1; row += kLnWarps, slot ^= 1) {
    issue(row + kLnWarps, slot ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    const uint4* bx = wb + (size_t)slot * 3 * NV * 32;
    const uint4* bg = bx + NV * 32;
    const uint4* br = bg + NV * 32;
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c >= D) continue;
      float xh[8], g[8];
      unpack8(bx[i * 32 + lane], xh);
      unpack8(bg[i * 32 + lane], g);
      const float* wr = s_w + c;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xh[e] = (xh[e] - mu) * rs;
        const float gw = g[e] * wr[e];
        s1 += gw;
        s2 += gw * xh[e];
        dg[i][e] += g[e] * xh[e];
        db[i][e] += g[e];
      }
    }
    s1 = warp_sum(s1) / D;
    s2 = warp_sum(s2) / D;
    uint4* dr = reinterpret_cast<uint4*>(dx + (size_t)row * D);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c >= D) continue;
      float xh[8], g[8], o[8];
      unpack8(bx[i * 32 + lane], xh);
      unpack8(bg[i * 32 + lane], g);
      const float* wr = s_w + c;
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = rs * (g[e] * wr[e] - s1 - (xh[e] - mu) * rs * s2);
      if (dres) {  // the skip connection's gradient, summed here instead of by a separate add
        float rr[8];
        unpack8(br[i * 32 + lane], rr);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] += rr[e];
      }
      dr[i * 32 + lane] = pack8(o);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // fold the warps of this CTA in a fixed order (warp 0, 1, ...), then one
  // partial row per CTA
  for (int k = 0; k < kLnWarps; ++k) {
    if (warp == k) {
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = (i * 32 + lane) * 8 + e;
          if (c < D) {
            s_acc[0][c] = k == 0 ? dg[i][e] : s_acc[0][c] + dg[i][e];
            s_acc[1][c] = k == 0 ? db[i][e] : s_acc[1][c] + db[i][e];
          }
        }
    }
    __syncthreads();
  }
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    part[((size_t)blockIdx.x * 2 + 0) * D + c] = s_acc[0][c];
    part[((size_t)blockIdx.x * 2 + 1) * D + c] = s_acc[1][c];
  }
}

// 32 columns per CTA; the 32 warps take parts w, w+32, ... (4 loads in flight each) and
// are folded in warp order (fixed, deterministic): with ~300 partial rows every warp
// walks ~10 of them, so the fold costs ~3 memory latencies instead of ~10.
constexpr int kFoldWarps = 32;
__global__ void __launch_bounds__(kFoldWarps * 32)
k_ln_fold(int D, int nparts, const float* __restrict__ part, float* __restrict__ dw, float* __restrict__ dbias) {
  __shared__ float red[2][kFoldWarps][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float a = 0.f, b = 0.f;
  if (c < D)
    for (int p0 = w; p0 < nparts; p0 += 4 * kFoldWarps) {  // 4 parts' loads in flight, summed in part order
      float va[4], vb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int p = p0 + kFoldWarps * k;
        va[k] = p < nparts ? part[((size_t)p * 2 + 0) * D + c] : 0.f;
        vb[k] = p < nparts ? part[((size_t)p * 2 + 1) * D + c] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) { a += va[k]; b += vb[k]; }
    }
  red[0][w][lane] = a;
  red[1][w][lane] = b;
  __syncthreads();
  if (w == 0 && c < D) {
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int k = 0; k < kFoldWarps; ++k) { sa += red[0][k][lane]; sb += red[1][k][lane]; }
    dw[c] = sa;
    dbias[c] = sb;
  }
}

// ---- packed qkv gradient: dh (B, T, 3, H, hd) <- dq, dk, dv (B, H, T, hd) with
// arbitrary (b, h, t) strides and unit hd stride; one pass, 16-byte accesses.
__global__ void __launch_bounds__(256)
k_pack_qkv(int B, int T, int H, int hd, const __nv_bfloat16* __restrict__ dq, const __nv_bfloat16* __restrict__ dk,
           const __nv_bfloat16* __restrict__ dv, long long sb, long long sh, long long st,
           __nv_bfloat16* __restrict__ dh) {
  const int v8 = hd / 8;
  const long long total = (long long)B * T * 3 * H * v8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    long long r = i;
    const int c = (int)(r % v8); r /= v8;
    const int h = (int)(r % H); r /= H;
    const int w = (int)(r % 3); r /= 3;
    const int t = (int)(r % T);
    const int b = (int)(r / T);
    const __nv_bfloat16* src = w == 0 ? dq : (w == 1 ? dk : dv);
    const uint4 u = *reinterpret_cast<const uint4*>(src + b * sb + h * sh + t * st + c * 8);
    reinterpret_cast<uint4*>(dh)[i] = u;
  }
}

int run_pack_qkv(int B, int T, int H, int hd, const void* dq, const void* dk, const void* dv, long long sb,
                 long long sh, long long st, void* dh, cudaStream_t stream) {
  if (B < 0 || T < 0 || H < 1 || hd < 8 || hd % 8) return DIAGMM_ESHAPE;
  if ((sb | sh | st) % 8) return DIAGMM_ESHAPE;
  const long long total = (long long)B * T * 3 * H * (hd / 8);
  if (total == 0) return DIAGMM_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 16LL * num_sms()) blocks = 16LL * num_sms();
  k_pack_qkv<<<(int)blocks, 256, 0, stream>>>(B, T, H, hd, static_cast<const __nv_bfloat16*>(dq),
                                             static_cast<const __nv_bfloat16*>(dk), static_cast<const __nv_bfloat16*>(dv),
                                             sb, sh, st, static_cast<__nv_bfloat16*>(dh));
  note_launch();
  return status_from_cuda();
}

static int ln_nv(int D) { return (D + 255) / 256; }

int run_ln_fwd(int M, int D, float eps, const void* x, const float* w, const float* b, void* y, float* mean,
               float* rstd, cudaStream_t st) {
  if (M < 0 || D < 8 || D % 8 || D > kLnMaxV * 256) return DIAGMM_ESHAPE;
  if (M == 0) return DIAGMM_OK;
  const int blocks = ceil_div(M, kLnWarps);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto Y = static_cast<__nv_bfloat16*>(y);
  switch (ln_nv(D)) {
    case 1: k_ln_fwd<1><<<blocks, kLnWarps * 32, 0, st>>>(M, D, eps, X, w, b, Y, mean, rstd); break;
    case 2: k_ln_fwd<2><<<blocks, kLnWarps * 32, 0, st>>>(M, D, eps, X, w, b, Y, mean, rstd); break;
    case 3: k_ln_fwd<3><<<blocks, kLnWarps * 32, 0, st>>>(M, D, eps, X, w, b, Y, mean, rstd); break;
    default: k_ln_fwd<4><<<blocks, kLnWarps * 32, 0, st>>>(M, D, eps, X, w, b, Y, mean, rstd); break;
  }
  note_launch();
  return status_from_cuda();
}

// one wave at 2 CTAs/SM: half the dgamma/dbeta partials of 4 per SM, same dx time
static int ln_bwd_ctas() { return 2 * num_sms(); }

size_t ln_bwd_workspace(int M, int D) {
  const int ctas = ln_bwd_ctas();
  return (size_t)ctas * 2 * D * sizeof(float);
}

int run_ln_bwd(int M, int D, const void* x, const void* dy, const float* w, const float* mean, const float* rstd,
               void* dx, float* dw, float* db, void* ws, size_t ws_bytes, cudaStream_t st, const void* dres) {
  if (M < 0 || D < 8 || D % 8 || D > kLnMaxV * 256) return DIAGMM_ESHAPE;
  if (ws_bytes < ln_bwd_workspace(M, D)) return DIAGMM_EWORKSPACE;
  int ctas = ln_bwd_ctas();
  const int rpc = ceil_div(M > 0 ? M : 1, ctas);
  ctas = ceil_div(M > 0 ? M : 1, rpc);
  float* part = static_cast<float*>(ws);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto G = static_cast<const __nv_bfloat16*>(dy);
  auto DX = static_cast<__nv_bfloat16*>(dx);
  auto R = static_cast<const __nv_bfloat16*>(dres);
  auto go = [&](auto NVc) {
    constexpr int NV = decltype(NVc)::value;
    const size_t sm = (size_t)kLnWarps * 2 * 3 * NV * 32 * sizeof(uint4);
    cudaFuncSetAttribute(k_ln_bwd<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_ln_bwd<NV><<<ctas, kLnWarps * 32, sm, st>>>(M, D, rpc, X, G, w, mean, rstd, DX, part, R);
  };
  switch (ln_nv(D)) {
    case 1: go(std::integral_constant<int, 1>{}); break;
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    default: go(std::integral_constant<int, 4>{}); break;
  }
  note_launch();
  k_ln_fold<<<ceil_div(D, 32), kFoldWarps * 32, 0, st>>>(D, ctas, part, dw, db);
  note_launch();
  return status_from_cuda();
}


// ---------------------------------------------------------------- ViT patch embedding
// (caller-side, around the DiagLinear blocks): the patchify copy, the cls / position
// assembly and their backward as three streaming kernels instead of framework
// permute-copy, cat, broadcast-add, slice-copy and two reductions.

// images (B, Cin, H, W) bf16 -> patches (B * (H/p) * (W/p), Cin * p * p) bf16, column
// order (c, i, j) = conv2d's weight layout; one 16-byte chunk (8 pixels of a patch row)
// per thread: 16-byte loads and stores (p % 8 == 0).
__global__ void __launch_bounds__(256)
k_vit_patchify(int B, int Cin, int H, int W, int p, const uint4* __restrict__ img, uint4* __restrict__ out) {
  const int gh = H / p, gw = W / p, cpr = p / 8;  // 16-byte chunks per patch row
  const long long per_patch = (long long)Cin * p * cpr;
  const long long n = (long long)B * gh * gw * per_patch;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < n; e += (long long)gridDim.x * 256) {
    const long long pi = e / per_patch;
    const int r = (int)(e - pi * per_patch);
    const int c = r / (p * cpr), rem = r - c * p * cpr, i = rem / cpr, j8 = rem - i * cpr;
    const int b = (int)(pi / (gh * gw)), pp = (int)(pi - (long long)b * gh * gw), ph = pp / gw, pw = pp - ph * gw;
    const long long src = ((((long long)b * Cin + c) * H + ph * p + i) * W + pw * p) / 8 + j8;
    out[e] = __ldcs(img + src);
  }
}

__device__ __forceinline__ float bf16r(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// x (B, T, D) bf16: x[b, 0] = bf16(cls) + bf16(pos[0]), x[b, t] = y[b, t-1] + bf16(pos[t]) —
// one bf16 rounding of each sum, as the framework's cat + broadcast add of bf16 operands.
__global__ void __launch_bounds__(256)
k_vit_embed_fwd(int B, int T, int D, const __nv_bfloat16* __restrict__ y, const float* __restrict__ cls,
                const float* __restrict__ pos, __nv_bfloat16* __restrict__ x) {
  const int d8 = D / 8;
  const long long n = (long long)B * T * d8;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < n; e += (long long)gridDim.x * 256) {
    const long long row = e / d8;
    const int c = (int)(e - row * d8) * 8;
    const int b = (int)(row / T), t = (int)(row - (long long)b * T);
    float a[8];
    if (t == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = bf16r(__ldg(cls + c + k));
    } else {
      unpack8(__ldg(reinterpret_cast<const uint4*>(y + ((size_t)b * (T - 1) + t - 1) * D + c)), a);
    }
    const float4 p0 = __ldg(reinterpret_cast<const float4*>(pos + (size_t)t * D + c));
    const float4 p1 = __ldg(reinterpret_cast<const float4*>(pos + (size_t)t * D + c + 4));
    const float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] += bf16r(pv[k]);
    reinterpret_cast<uint4*>(x)[e] = pack8(a);
  }
}

// Backward, pass 1: dy[b, t-1] = gx[b, t] (t >= 1, contiguous for the patch GEMM's
// weight gradient) and per-group column sums part[g][t][d] = sum_{b in group g} gx[b, t, d]
// (fp32, batches in index order).  grid (T, groups), D/8 threads.
constexpr int kEmbGroups = 16;
__global__ void __launch_bounds__(128)
k_vit_embed_bwd(int B, int T, int D, const __nv_bfloat16* __restrict__ gx, __nv_bfloat16* __restrict__ dy,
                float* __restrict__ part) {
  const int t = blockIdx.x, g = blockIdx.y, d8 = D / 8;
  const int bpg = (B + gridDim.y - 1) / gridDim.y, b0 = g * bpg, b1 = min(B, b0 + bpg);
  for (int c8 = threadIdx.x; c8 < d8; c8 += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int b = b0; b < b1; ++b) {
      const uint4 u = __ldcs(reinterpret_cast<const uint4*>(gx + ((size_t)b * T + t) * D) + c8);
      if (t > 0) reinterpret_cast<uint4*>(dy + ((size_t)b * (T - 1) + t - 1) * D)[c8] = u;
      float f[8];
      unpack8(u, f);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += f[k];
    }
    float* pr = part + ((size_t)g * T + t) * D + c8 * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) pr[k] = acc[k];
  }
}

// pass 2: fold the groups in order, one thread per (t, d).  dpos[t] = bf16-rounded sum
// (the framework reduces the bf16 broadcast gradient to bf16), dcls = the fp32 sum at
// t = 0; the fp32 per-t sums go to tsum for the bias gradient.
__global__ void __launch_bounds__(256)
k_vit_embed_fold(int T, int D, int groups, const float* __restrict__ part, float* __restrict__ tsum,
                 float* __restrict__ dpos, float* __restrict__ dcls) {
  const int t = blockIdx.y, d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= D) return;
  float s = 0.f;
  for (int g = 0; g < groups; ++g) s += __ldcg(part + ((size_t)g * T + t) * D + d);
  tsum[(size_t)t * D + d] = s;
  if (dpos) dpos[(size_t)t * D + d] = bf16r(s);
  if (t == 0 && dcls) dcls[d] = s;
}

// pass 3: dbias = bf16-rounded sum over t >= 1 (the patch GEMM's bias gradient in bf16):
// 32 columns per CTA, warp w takes t = 1 + w, 1 + w + 8, ..., folded in warp order.
__global__ void __launch_bounds__(256)
k_vit_embed_bias(int T, int D, const float* __restrict__ tsum, float* __restrict__ dbias) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, d = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (d < D)
    for (int t = 1 + w; t < T; t += 8) s += __ldcg(tsum + (size_t)t * D + d);
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && d < D) {
    float r = 0.f;
    for (int k = 0; k < 8; ++k) r += red[k][lane];
    dbias[d] = bf16r(r);
  }
}

int run_vit_patchify(int B, int Cin, int H, int W, int p, const void* img, void* out, cudaStream_t st) {
  if (B < 1 || Cin < 1 || p < 8 || p % 8 || H % p || W % p || (reinterpret_cast<uintptr_t>(img) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return DIAGMM_ESHAPE;
  const long long n = (long long)B * Cin * H * W / 8;
  const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 16);
  k_vit_patchify<<<blocks, 256, 0, st>>>(B, Cin, H, W, p, static_cast<const uint4*>(img), static_cast<uint4*>(out));
  note_launch();
  return status_from_cuda();
}

int run_vit_embed_fwd(int B, int T, int D, const void* y, const float* cls, const float* pos, void* x,
                      cudaStream_t st) {
  if (B < 1 || T < 2 || D % 8 || (reinterpret_cast<uintptr_t>(y) & 15) || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(pos) & 15))
    return DIAGMM_ESHAPE;
  const long long n = (long long)B * T * (D / 8);
  const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 16);
  k_vit_embed_fwd<<<blocks, 256, 0, st>>>(B, T, D, static_cast<const __nv_bfloat16*>(y), cls, pos,
                                          static_cast<__nv_bfloat16*>(x));
  note_launch();
  return status_from_cuda();
}

size_t vit_embed_bwd_workspace(int T, int D) { return (size_t)(kEmbGroups + 1) * T * D * sizeof(float); }

int run_vit_embed_bwd(int B, int T, int D, const void* gx, void* dy, float* dpos, float* dcls, float* dbias,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
  if (B < 1 || T < 2 || D % 8 || (reinterpret_cast<uintptr_t>(gx) & 15) || (reinterpret_cast<uintptr_t>(dy) & 15))
    return DIAGMM_ESHAPE;
  if (ws_bytes < vit_embed_bwd_workspace(T, D)) return DIAGMM_EWORKSPACE;
  float* part = static_cast<float*>(ws);
  k_vit_embed_bwd<<<dim3(T, kEmbGroups), 128, 0, st>>>(B, T, D, static_cast<const __nv_bfloat16*>(gx),
                                                      static_cast<__nv_bfloat16*>(dy), part);
  float* tsum = part + (size_t)kEmbGroups * T * D;
  k_vit_embed_fold<<<dim3(ceil_div(D, 256), T), 256, 0, st>>>(T, D, kEmbGroups, part, tsum, dpos, dcls);
  note_launch(2);
  if (dbias) {
    k_vit_embed_bias<<<ceil_div(D, 32), 256, 0, st>>>(T, D, tsum, dbias);
    note_launch();
  }
  return status_from_cuda();
}

}  // namespace diagmm

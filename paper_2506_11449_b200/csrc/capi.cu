// capi.cu — extern "C" entry points declared in include/diagmm.h.
// Validates arguments (mirroring the reference's exceptions) and dispatches
// on dtype to the templated launchers.
#include "common.cuh"
#include <atomic>

namespace diagmm {
template <typename T>
int run_product(bool, int, int, int, const void*, const void*, const double*, const int32_t*,
                const int32_t*, int, const void*, void*, void*, size_t, cudaStream_t);
template <typename T> size_t product_workspace(bool, int, int, int, int);
template <typename T> size_t dw_workspace(int, int, int, int);
template <typename T>
int run_dw(int, int, int, const void*, const void*, const void*, const double*, const int32_t*,
           const int32_t*, const int32_t*, int, void*, double*, void*, void*, size_t, cudaStream_t, void*, int);
template <typename T> int run_materialize_batched(int, const diagmm_materialize_job*, cudaStream_t);
template <typename T>
int run_materialize(int, int, const void*, const double*, const int32_t*, const int32_t*, int, void*,
                    cudaStream_t, bool);  // (slot, n_act, ..., transposed)
template <typename P>
int run_gather_dense(int, int, const void*, const void*, const double*, const int32_t*, const int32_t*,
                     void*, double*, cudaStream_t);
int run_waterfill(int, int, double, const double*, double*, uint8_t*, int32_t*, int32_t*, int32_t*,
                  cudaStream_t);
int run_waterfill_batched(int, const diagmm_topk_job*, cudaStream_t);
int run_select_hard(int, int, const double*, int32_t*, cudaStream_t);
template <typename P>
int run_diagheur_update(int, int, int, int32_t*, int32_t*, int32_t*, void*, int, const int32_t*, cudaStream_t);
int run_active_from_list(int, int, const int32_t*, int32_t*, int32_t*, cudaStream_t);
int run_topk_grad(int, int, double, const double*, const uint8_t*, const double*, double, double*, int,
                  const double*, cudaStream_t);
int run_topk_grad_batched(int, const diagmm_topk_grad_job*, cudaStream_t);
template <typename P>
int run_adamw(size_t, void*, const void*, void*, void*, int, double, double, double, double, double,
              const double*, cudaStream_t);
template <typename P> int run_sumsq(size_t, const void*, double*, double*, cudaStream_t);
int run_clip_scale(int, const double*, double, double*, double*, cudaStream_t);
int run_adamw_multi(int, const diagmm_tensor*, double, double, double, double, const double*, const double*,
                    cudaStream_t);
int mt_sumsq_parts(int, const diagmm_tensor*);
int run_sumsq_multi(int, const diagmm_tensor*, double*, int, cudaStream_t);
int run_clip_scale_tree(int, const double*, double, double*, double*, cudaStream_t);
int run_tc_gemm_bf16(int, int, int, const void*, const void*, const float*, void*, int, void*, int, cudaStream_t,
                     bool b_kn = false, const void* A1 = nullptr, const void* A2 = nullptr, int a_ks = 0);
int run_tc_sparse_probe(int, int, int, const void*, const void*, void*, cudaStream_t);
size_t tc_dw_workspace(int, int, int, int);
int tc_dw_splits(int M, int N, int ntok);
int run_tc_dw(int M, int N, int ntok, const void* dy, const void* x, const int32_t* slot, const int32_t* n_act,
              int max_act, float* partial, size_t partial_bytes, float* colsum, cudaStream_t st, const void* dy1,
              const void* dy2, int a_ms);
int run_dw_finalize_batched(int n, const diagmm_dw_finalize_job* jobs, cudaStream_t st);
int run_tc_dw_full(int, int, int, const void*, const void*, const void*, const double*, const int32_t*,
                   const int32_t*, int, void*, double*, void*, void*, size_t, cudaStream_t, const void* dy1,
                   const void* dy2, int a_ms, void* bucket, int bucket_rows);
int run_pack_qkv(int, int, int, int, const void*, const void*, const void*, long long, long long, long long, void*,
                 cudaStream_t);
int run_ln_fwd(int, int, float, const void*, const float*, const float*, void*, float*, float*, cudaStream_t);
int run_vit_patchify(int, int, int, int, int, const void*, void*, cudaStream_t);
size_t tf32x3_gemm_workspace(int, int, int, int, int);
int run_tf32x3_gemm(int, int, int, const float*, int, int, const float*, int, int, const float*, float*, int, void*,
                    size_t, cudaStream_t);
int run_vit_embed_fwd(int, int, int, const void*, const float*, const float*, void*, cudaStream_t);
size_t vit_embed_bwd_workspace(int, int);
int run_vit_embed_bwd(int, int, int, const void*, void*, float*, float*, float*, void*, size_t, cudaStream_t);
size_t ln_bwd_workspace(int, int);
int run_ln_bwd(int, int, const void*, const void*, const float*, const float*, const float*, void*, float*, float*,
               void*, size_t, cudaStream_t, const void* dres = nullptr);
constexpr int kSumsqScratch = 296;
static std::atomic<unsigned long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
}  // namespace diagmm

using namespace diagmm;

#define DIAGMM_DISPATCH(dtype, FN, ...)                         \
  switch (dtype) {                                              \
    case DIAGMM_F64: return FN<double>(__VA_ARGS__);            \
    case DIAGMM_F32: return FN<float>(__VA_ARGS__);             \
    case DIAGMM_BF16: return FN<__nv_bfloat16>(__VA_ARGS__);    \
    default: return DIAGMM_EDTYPE;                              \
  }

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

static int check_shape(int M, int N, int B, int max_act) {
  if (M < 1 || N < 1 || B < 0) return DIAGMM_ESHAPE;
  const int C = M > N ? M : N;
  if (max_act < 0 || max_act > C) return DIAGMM_ESHAPE;
  return DIAGMM_OK;
}

extern "C" {

const char* diagmm_version(void) { return "diagmm 0.1.0 sm_100a"; }

const char* diagmm_last_error(void) { return diagmm::last_cuda_error(); }

unsigned long long diagmm_launch_count(void) { return g_launches.load(); }

const char* diagmm_status_string(int status) {
  switch (status) {
    case DIAGMM_OK: return "ok";
    case DIAGMM_ESHAPE: return "shape mismatch";
    case DIAGMM_ETEMPERATURE: return "temperature must be positive";
    case DIAGMM_EK: return "k outside [1, C]";
    case DIAGMM_EDTYPE: return "unsupported dtype";
    case DIAGMM_EWORKSPACE: return "workspace too small";
    case DIAGMM_ECUDA: return "CUDA launch failure";
    case DIAGMM_ETOOLARGE: return "problem exceeds kernel limits";
    default: return "unknown status";
  }
}

static size_t product_ws(int dtype, bool gather, int M, int N, int B, int max_act) {
  if (check_shape(M, N, B, max_act)) return 0;
  const int C = M > N ? M : N, L = M < N ? M : N;
  switch (dtype) {
    case DIAGMM_F64: return product_workspace<double>(gather, B, C, L, max_act);
    case DIAGMM_F32: return product_workspace<float>(gather, B, C, L, max_act);
    case DIAGMM_BF16: return product_workspace<__nv_bfloat16>(gather, B, C, L, max_act);
    default: return 0;
  }
}

size_t diagmm_forward_workspace(int dtype, int M, int N, int B, int max_act) {
  return product_ws(dtype, M < N, M, N, B, max_act);
}

size_t diagmm_backward_input_workspace(int dtype, int M, int N, int B, int max_act) {
  return product_ws(dtype, M >= N, M, N, B, max_act);
}

int diagmm_forward(int dtype, int M, int N, int B, const void* x, const void* values,
                   const double* alpha_soft, const int32_t* active, const int32_t* n_act, int max_act,
                   const void* bias, void* y, void* workspace, size_t ws_bytes, void* stream) {
  if (int e = check_shape(M, N, B, max_act)) return e;
  const int C = M > N ? M : N, L = M < N ? M : N;
  // tall/square: scatter form with in width L=N, out width C=M; wide: gather form.
  const bool gather = M < N;
  DIAGMM_DISPATCH(dtype, run_product, gather, B, C, L, x, values, alpha_soft, active, n_act, max_act,
                  bias, y, workspace, ws_bytes, S(stream))
}

int diagmm_backward_input(int dtype, int M, int N, int B, const void* dy, const void* values,
                          const double* alpha_soft, const int32_t* active, const int32_t* n_act,
                          int max_act, void* dx, void* workspace, size_t ws_bytes, void* stream) {
  if (int e = check_shape(M, N, B, max_act)) return e;
  const int C = M > N ? M : N, L = M < N ? M : N;
  // tall/square dX: gather form (in = dy width C=M, out width L=N); wide: scatter.
  const bool gather = M >= N;
  DIAGMM_DISPATCH(dtype, run_product, gather, B, C, L, dy, values, alpha_soft, active, n_act, max_act,
                  nullptr, dx, workspace, ws_bytes, S(stream))
}

size_t diagmm_backward_weight_workspace(int dtype, int M, int N, int B, int max_act) {
  if (check_shape(M, N, B, max_act)) return 0;
  switch (dtype) {
    case DIAGMM_F64: return dw_workspace<double>(M, N, B, max_act);
    case DIAGMM_F32: return dw_workspace<float>(M, N, B, max_act);
    case DIAGMM_BF16: return dw_workspace<__nv_bfloat16>(M, N, B, max_act);
    default: return 0;
  }
}

int diagmm_backward_weight(int dtype, int M, int N, int B, const void* dy, const void* x,
                           const void* values, const double* alpha_soft, const int32_t* active,
                           const int32_t* slot, const int32_t* n_act, int max_act, void* g_values,
                           double* g_soft, void* g_bias, void* workspace, size_t ws_bytes,
                           void* bucket, int bucket_rows, void* stream) {
  if (int e = check_shape(M, N, B, max_act)) return e;
  if (bucket_rows < 0 || (bucket_rows > 0 && !bucket)) return DIAGMM_ESHAPE;
  DIAGMM_DISPATCH(dtype, run_dw, M, N, B, dy, x, values, alpha_soft, active, slot, n_act, max_act,
                  g_values, g_soft, g_bias, workspace, ws_bytes, S(stream), bucket, bucket_rows)
}

int diagmm_topk_waterfill(int C, int k, double temperature, const double* alpha, double* alpha_soft,
                          uint8_t* clamped, int32_t* active, int32_t* slot, int32_t* n_act,
                          void* stream) {
  return run_waterfill(C, k, temperature, alpha, alpha_soft, clamped, active, slot, n_act, S(stream));
}

int diagmm_topk_waterfill_batched(int n, const diagmm_topk_job* jobs, void* stream) {
  return run_waterfill_batched(n, jobs, S(stream));
}

int diagmm_adamw_multi(int n, const diagmm_tensor* tensors, double lr, double beta1, double beta2,
                       double eps, const double* clip_scale, const double* sched, void* stream) {
  return run_adamw_multi(n, tensors, lr, beta1, beta2, eps, clip_scale, sched, S(stream));
}
int diagmm_sumsq_multi_len(int n, const diagmm_tensor* tensors) {
  return n > 0 && tensors ? mt_sumsq_parts(n, tensors) : 0;
}
int diagmm_sumsq_multi(int n, const diagmm_tensor* tensors, double* partial, int partial_len, void* stream) {
  return run_sumsq_multi(n, tensors, partial, partial_len, S(stream));
}
int diagmm_clip_scale_tree(int n, const double* partial, double max_norm, double* norm, double* scale,
                           void* stream) {
  if (n < 1) return DIAGMM_ESHAPE;
  return run_clip_scale_tree(n, partial, max_norm, norm, scale, S(stream));
}

int diagmm_tc_gemm_bf16(int Mdim, int Ndim, int K, const void* A, const void* B, const float* bias, void* out,
                        int ldo, void* stream) {
  return run_tc_gemm_bf16(Mdim, Ndim, K, A, B, bias, out, ldo, nullptr, 0, S(stream));
}

int diagmm_tc_gemm_bf16_ex(int Mdim, int Ndim, int K, const void* A, const void* B, const float* bias, void* out,
                           int ldo, void* aux, int epilogue, void* stream) {
  return run_tc_gemm_bf16(Mdim, Ndim, K, A, B, bias, out, ldo, aux, epilogue, S(stream));
}

int diagmm_tc_gemm_bf16_nn(int Mdim, int Ndim, int K, const void* A, const void* B, const float* bias, void* out,
                           int ldo, void* aux, int epilogue, void* stream) {
  return run_tc_gemm_bf16(Mdim, Ndim, K, A, B, bias, out, ldo, aux, epilogue, S(stream), true);
}

size_t diagmm_tc_backward_weight_workspace(int M, int N, int B, int max_act) {
  if (check_shape(M, N, B, max_act)) return 0;
  return tc_dw_workspace(M, N, B, max_act);
}

int diagmm_tc_backward_weight(int M, int N, int B, const void* dy, const void* x, const void* values,
                              const double* alpha_soft, const int32_t* slot, const int32_t* n_act, int max_act,
                              void* g_values, double* g_soft, void* g_bias, void* workspace, size_t ws_bytes,
                              void* bucket, int bucket_rows, void* stream) {
  if (int e = check_shape(M, N, B, max_act)) return e;
  if (bucket_rows < 0 || (bucket_rows > 0 && !bucket)) return DIAGMM_ESHAPE;
  return run_tc_dw_full(M, N, B, dy, x, values, alpha_soft, slot, n_act, max_act, g_values, g_soft, g_bias,
                        workspace, ws_bytes, S(stream), nullptr, nullptr, 0, bucket, bucket_rows);
}

int diagmm_tc_dw_splits(int M, int N, int B) { return tc_dw_splits(M, N, B > 0 ? B : 1); }

int diagmm_tc_backward_weight_partials(int M, int N, int B, const void* dy0, const void* dy1, const void* dy2, int ms,
                                       const void* x, const int32_t* slot, const int32_t* n_act, int max_act,
                                       int need_bias, void* workspace, size_t ws_bytes, void* stream) {
  if (int e = check_shape(M, N, B, max_act)) return e;
  if (ms < 0 || B < 1) return DIAGMM_ESHAPE;
  if (ws_bytes < tc_dw_workspace(M, N, B, max_act)) return DIAGMM_EWORKSPACE;
  const int L = M < N ? M : N;
  const int ks = tc_dw_splits(M, N, B);
  const size_t pbytes = ((size_t)ks * (max_act > 0 ? max_act : 1) * L * sizeof(float) + 15) / 16 * 16;
  float* partial = static_cast<float*>(workspace);
  float* colsum = reinterpret_cast<float*>(static_cast<char*>(workspace) + pbytes);
  return run_tc_dw(M, N, B, dy0, x, slot, n_act, max_act > 0 ? max_act : 1, partial, pbytes,
                   need_bias ? colsum : nullptr, S(stream), dy1, dy2, ms);
}

int diagmm_tc_dw_finalize_batched(int n, const diagmm_dw_finalize_job* jobs, void* stream) {
  if (n < 0) return DIAGMM_ESHAPE;
  return run_dw_finalize_batched(n, jobs, S(stream));
}

int diagmm_tc_gemm_bf16_nn_split(int Mdim, int Ndim, int K, const void* A0, const void* A1, const void* A2, int ks,
                                 const void* B, const float* bias, void* out, int ldo, void* stream) {
  if (ks < 1) return DIAGMM_ESHAPE;
  return run_tc_gemm_bf16(Mdim, Ndim, K, A0, B, bias, out, ldo, nullptr, 0, S(stream), true, A1, A2, ks);
}

int diagmm_tc_backward_weight_split(int M, int N, int B, const void* dy0, const void* dy1, const void* dy2, int ms,
                                    const void* x, const void* values, const double* alpha_soft,
                                    const int32_t* slot, const int32_t* n_act, int max_act, void* g_values,
                                    double* g_soft, void* g_bias, void* workspace, size_t ws_bytes, void* bucket,
                                    int bucket_rows, void* stream) {
  if (int e = check_shape(M, N, B, max_act)) return e;
  if (ms < 1 || bucket_rows < 0 || (bucket_rows > 0 && !bucket)) return DIAGMM_ESHAPE;
  return run_tc_dw_full(M, N, B, dy0, x, values, alpha_soft, slot, n_act, max_act, g_values, g_soft, g_bias,
                        workspace, ws_bytes, S(stream), dy1, dy2, ms, bucket, bucket_rows);
}

// internal (not in the header): 2:4 sparse tensor-core throughput probe
DIAGMM_API int diagmm_internal_tc_sparse_probe(int Mdim, int Ndim, int K, const void* Acomp, const void* B, void* out,
                                               void* stream) {
  return run_tc_sparse_probe(Mdim, Ndim, K, Acomp, B, out, S(stream));
}

size_t diagmm_tf32x3_gemm_workspace(int M, int N, int K, int trans_a, int trans_b) {
  return tf32x3_gemm_workspace(M, N, K, trans_a, trans_b);
}
int diagmm_tf32x3_gemm(int M, int N, int K, const float* A, int lda, int trans_a, const float* B, int ldb,
                       int trans_b, const float* bias, float* out, int ldo, void* workspace, size_t ws_bytes,
                       void* stream) {
  return run_tf32x3_gemm(M, N, K, A, lda, trans_a, B, ldb, trans_b, bias, out, ldo, workspace, ws_bytes, S(stream));
}

int diagmm_vit_patchify(int B, int Cin, int H, int W, int p, const void* images, void* patches, void* stream) {
  return run_vit_patchify(B, Cin, H, W, p, images, patches, S(stream));
}
int diagmm_vit_embed_fwd(int B, int T, int D, const void* y, const float* cls, const float* pos, void* x,
                         void* stream) {
  return run_vit_embed_fwd(B, T, D, y, cls, pos, x, S(stream));
}
size_t diagmm_vit_embed_bwd_workspace(int T, int D) { return vit_embed_bwd_workspace(T, D); }
int diagmm_vit_embed_bwd(int B, int T, int D, const void* gx, void* dy, float* dpos, float* dcls, float* dbias,
                         void* workspace, size_t ws_bytes, void* stream) {
  return run_vit_embed_bwd(B, T, D, gx, dy, dpos, dcls, dbias, workspace, ws_bytes, S(stream));
}

int diagmm_pack_qkv_grad(int B, int T, int H, int hd, const void* dq, const void* dk, const void* dv,
                         long long stride_b, long long stride_h, long long stride_t, void* dqkv, void* stream) {
  return run_pack_qkv(B, T, H, hd, dq, dk, dv, stride_b, stride_h, stride_t, dqkv, S(stream));
}

int diagmm_layernorm_fwd(int M, int D, float eps, const void* x, const float* w, const float* b, void* y,
                         float* mean, float* rstd, void* stream) {
  return run_ln_fwd(M, D, eps, x, w, b, y, mean, rstd, S(stream));
}
size_t diagmm_layernorm_bwd_workspace(int M, int D) { return ln_bwd_workspace(M, D); }
int diagmm_layernorm_bwd(int M, int D, const void* x, const void* dy, const float* w, const float* mean,
                         const float* rstd, void* dx, float* dw, float* db, void* workspace, size_t ws_bytes,
                         void* stream) {
  return run_ln_bwd(M, D, x, dy, w, mean, rstd, dx, dw, db, workspace, ws_bytes, S(stream));
}

int diagmm_layernorm_bwd_res(int M, int D, const void* x, const void* dy, const void* dres, const float* w,
                             const float* mean, const float* rstd, void* dx, float* dw, float* db, void* workspace,
                             size_t ws_bytes, void* stream) {
  if (dres && (reinterpret_cast<uintptr_t>(dres) & 15)) return DIAGMM_ESHAPE;
  return run_ln_bwd(M, D, x, dy, w, mean, rstd, dx, dw, db, workspace, ws_bytes, S(stream), dres);
}

int diagmm_topk_grad(int C, int k, double temperature, const double* alpha, const uint8_t* clamped,
                     const double* g_soft, double l1_coeff, double* g_alpha, int accumulate,
                     const double* params, void* stream) {
  return run_topk_grad(C, k, temperature, alpha, clamped, g_soft, l1_coeff, g_alpha, accumulate, params,
                       S(stream));
}

int diagmm_topk_grad_batched(int n, const diagmm_topk_grad_job* jobs, void* stream) {
  return run_topk_grad_batched(n, jobs, S(stream));
}

int diagmm_diagheur_update(int dtype, int C, int L, int k, int32_t* active, int32_t* slot, int32_t* n_act,
                           void* values, int n_prune, const int32_t* grow_idx, void* stream) {
  if (dtype == DIAGMM_F64)
    return run_diagheur_update<double>(C, L, k, active, slot, n_act, values, n_prune, grow_idx, S(stream));
  if (dtype == DIAGMM_F32)
    return run_diagheur_update<float>(C, L, k, active, slot, n_act, values, n_prune, grow_idx, S(stream));
  return DIAGMM_ESHAPE;
}

int diagmm_select_hard(int C, int k, const double* alpha, int32_t* idx, void* stream) {
  return run_select_hard(C, k, alpha, idx, S(stream));
}

int diagmm_active_from_list(int C, int n, const int32_t* offsets, int32_t* slot, int32_t* n_act,
                            void* stream) {
  return run_active_from_list(C, n, offsets, slot, n_act, S(stream));
}

int diagmm_adamw(int dtype, size_t n, void* param, const void* grad, void* m, void* v, int step,
                 double lr, double beta1, double beta2, double eps, double weight_decay,
                 const double* clip_scale, void* stream) {
  switch (dtype) {
    case DIAGMM_F64:
      return run_adamw<double>(n, param, grad, m, v, step, lr, beta1, beta2, eps, weight_decay,
                               clip_scale, S(stream));
    case DIAGMM_F32:
    case DIAGMM_BF16:
      return run_adamw<float>(n, param, grad, m, v, step, lr, beta1, beta2, eps, weight_decay,
                              clip_scale, S(stream));
    default: return DIAGMM_EDTYPE;
  }
}

int diagmm_sumsq_scratch_len(void) { return kSumsqScratch; }

int diagmm_sumsq(int dtype, size_t n, const void* x, double* out, double* scratch, void* stream) {
  switch (dtype) {
    case DIAGMM_F64: return run_sumsq<double>(n, x, out, scratch, S(stream));
    case DIAGMM_F32:
    case DIAGMM_BF16: return run_sumsq<float>(n, x, out, scratch, S(stream));
    default: return DIAGMM_EDTYPE;
  }
}

int diagmm_clip_scale(int n, const double* partial, double max_norm, double* norm, double* scale,
                      void* stream) {
  return run_clip_scale(n, partial, max_norm, norm, scale, S(stream));
}

int diagmm_materialize(int dtype, int M, int N, const void* values, const double* alpha_soft,
                       const int32_t* active, const int32_t* slot, const int32_t* n_act, int max_act,
                       void* w_dense, void* stream) {
  if (int e = check_shape(M, N, 0, max_act)) return e;
  if (slot == nullptr) return DIAGMM_ESHAPE;
  (void)active;
  DIAGMM_DISPATCH(dtype, run_materialize, M, N, values, alpha_soft, slot, n_act, max_act, w_dense,
                  S(stream), false)
}

int diagmm_materialize_batched(int dtype, int n, const diagmm_materialize_job* jobs, void* stream) {
  if (n < 0) return DIAGMM_ESHAPE;
  if (dtype == DIAGMM_BF16) return run_materialize_batched<__nv_bfloat16>(n, jobs, S(stream));
  if (dtype == DIAGMM_F32) return run_materialize_batched<float>(n, jobs, S(stream));
  return DIAGMM_ESHAPE;
}

int diagmm_materialize_transposed(int dtype, int M, int N, const void* values, const double* alpha_soft,
                                  const int32_t* active, const int32_t* slot, const int32_t* n_act, int max_act,
                                  void* w_dense_t, void* stream) {
  if (int e = check_shape(M, N, 0, max_act)) return e;
  if (slot == nullptr) return DIAGMM_ESHAPE;
  (void)active;
  DIAGMM_DISPATCH(dtype, run_materialize, M, N, values, alpha_soft, slot, n_act, max_act, w_dense_t,
                  S(stream), true)
}

int diagmm_gather_dense_grad(int dtype, int M, int N, const void* dW, const void* values,
                             const double* alpha_soft, const int32_t* active, const int32_t* slot,
                             const int32_t* n_act, void* g_values, double* g_soft, void* stream) {
  (void)active;
  if (int e = check_shape(M, N, 0, 0)) return e;
  switch (dtype) {
    case DIAGMM_F64:
      return run_gather_dense<double>(M, N, dW, values, alpha_soft, slot, n_act, g_values, g_soft,
                                      S(stream));
    case DIAGMM_F32:
    case DIAGMM_BF16:
      return run_gather_dense<float>(M, N, dW, values, alpha_soft, slot, n_act, g_values, g_soft,
                                     S(stream));
    default: return DIAGMM_EDTYPE;
  }
}

}  // extern "C"

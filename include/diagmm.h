/*
 * diagmm.h — C ABI of the B200 (sm_100a) DiagLinear hot path.
 *
 * The reference (DynaDiag, /root/reference/pkg/src/diagsparse) is a float64
 * numpy package whose "FFI" for this path is the custom-op boundary
 * `_record_diag_matmul` (layers.py:108-170) recorded through
 * `Tape.record(out, inputs, backward)` (autodiff.py:43-50), plus the selection
 * functions of selection.py.  Each entry point below replaces one piece of that
 * boundary; the comment on each names the reference symbol (file:line).
 *
 * Conventions
 *   - W is M x N (out x in).  C = max(M, N) candidate diagonals, L = min(M, N)
 *     values per diagonal; candidate i IS offset i (layers.py:199-206).
 *   - Geometry (diagcore.py:106-116): M >= N: value t of offset o sits at
 *     ((o + t) mod M, t);  M < N: at (t, (o + t) mod N).
 *   - Activations are row-major (B, features): x is (B, N), y is (B, M).
 *   - values is the candidate store (C, L) row-major; alpha, alpha_soft are
 *     (C,) float64; `active` is the ascending list of active offsets and
 *     `n_act` its length, both in DEVICE memory (no host sync is needed).
 *   - dtype: DIAGMM_F64 -> activations and parameters double;
 *            DIAGMM_F32 -> activations and parameters float;
 *            DIAGMM_BF16 -> activations bf16, parameters/gradients float,
 *                           fp32 accumulation.
 *   - All pointers are caller-owned device pointers; every call is
 *     stream-ordered on `stream` (a cudaStream_t, NULL = legacy default) and
 *     never synchronizes the host.  Inputs are never written.
 *   - Return value: 0 on success, otherwise a DIAGMM_E* code; the Python
 *     wrapper maps the codes onto the reference's exception classes
 *     (errors.py:8-53): SHAPE -> ShapeMismatch, TEMPERATURE ->
 *     NonPositiveTemperature, K -> ValueError.
 */
#ifndef DIAGMM_H
#define DIAGMM_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DIAGMM_API __attribute__((visibility("default")))
#else
#define DIAGMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum diagmm_dtype { DIAGMM_F64 = 0, DIAGMM_F32 = 1, DIAGMM_BF16 = 2 };

enum diagmm_status {
  DIAGMM_OK = 0,
  DIAGMM_ESHAPE = 1,       /* ShapeMismatch (errors.py:20) */
  DIAGMM_ETEMPERATURE = 2, /* NonPositiveTemperature (errors.py:24) */
  DIAGMM_EK = 3,           /* k outside [1, C] (selection.py:95-96) */
  DIAGMM_EDTYPE = 4,
  DIAGMM_EWORKSPACE = 5,
  DIAGMM_ECUDA = 6,
  DIAGMM_ETOOLARGE = 7,    /* C above the single-CTA selection limit */
};

/* Library identity: "diagmm <version> sm_100a". */
DIAGMM_API const char* diagmm_version(void);
DIAGMM_API const char* diagmm_status_string(int status);
/* The CUDA runtime's message for the last DIAGMM_ECUDA returned on this host thread. */
DIAGMM_API const char* diagmm_last_error(void);
/* Kernels launched by this library since load (for launch accounting). */
DIAGMM_API unsigned long long diagmm_launch_count(void);

/* ---- K1: forward DiagMM --------------------------------------------------
 * y = x @ W_K^T (+ bias), W_K = sum_{o in active} alpha_soft[o] P_o diag(values[o]).
 * Replaces: the forward product of _record_diag_matmul (layers.py:130-137:
 * bcsr_spmm / reference_spmm, diagcore.py:200-238, bcsr.py:362-409), the
 * weight scaling of DynaDiagLayer.forward (layers.py:235) and Tape.add_bias
 * (autodiff.py:72-81).  alpha_soft == NULL means unit scale (DiagHeur /
 * frozen layers, layers.py:354-363, 301-310).  max_act is a host upper bound
 * on *n_act used only to size work (pass C when unknown).  workspace
 * (REQUIRED, >= diagmm_forward_workspace bytes, 16-byte aligned) holds the
 * compact pre-scaled weights alpha_soft[o] * values[o] of the active
 * diagonals (the reference's `weights`, layers.py:235) and, for small
 * batches, the partial sums of the split diagonal list. */
DIAGMM_API size_t diagmm_forward_workspace(int dtype, int M, int N, int B,
                                           int max_act);
DIAGMM_API int diagmm_forward(int dtype, int M, int N, int B, const void* x,
                   const void* values, const double* alpha_soft,
                   const int32_t* active, const int32_t* n_act, int max_act,
                   const void* bias, void* y, void* workspace,
                   size_t ws_bytes, void* stream);

/* ---- K2: input gradient through the (never materialized) transpose -------
 * dx = dy @ W_K.  Replaces layers.py:144-148 (transpose, diagcore.py:162-191,
 * followed by the same spmm).  workspace: as diagmm_forward. */
DIAGMM_API size_t diagmm_backward_input_workspace(int dtype, int M, int N,
                                                  int B, int max_act);
DIAGMM_API int diagmm_backward_input(int dtype, int M, int N, int B, const void* dy,
                          const void* values, const double* alpha_soft,
                          const int32_t* active, const int32_t* n_act,
                          int max_act, void* dx, void* workspace,
                          size_t ws_bytes, void* stream);

/* ---- K3: per-diagonal weight gradient ----------------------------------
 * gw[j,t] = sum_b dy[b, r_jt] * x[b, c_jt]   (layers.py:149-158)
 * g_values (C, L): row active[j] = alpha_soft[active[j]] * gw[j] (unit scale
 * if alpha_soft == NULL), every other row exactly 0 (layers.py:159-163).
 * g_soft (C,) float64, may be NULL: g_soft[active[j]] = sum_t gw[j,t] *
 * values[active[j],t], 0 elsewhere (layers.py:164-165).
 * g_bias (M,), may be NULL: column sums of dy (autodiff.py:77-79).
 * slot (C,) int32 from diagmm_topk_waterfill / diagmm_active_from_list.
 * workspace: at least diagmm_backward_weight_workspace(...) bytes.
 * bucket (bucket_rows, L) in the values' type, may be NULL (bucket_rows 0):
 * the data-parallel exchange buffer — active row j (j < bucket_rows) is ALSO
 * written to bucket row j, so the all-reduce sends [g_values[active]] without
 * a pack pass (inactive rows are exactly 0 on every rank). */
DIAGMM_API size_t diagmm_backward_weight_workspace(int dtype, int M, int N, int B,
                                        int max_act);
DIAGMM_API int diagmm_backward_weight(int dtype, int M, int N, int B, const void* dy,
                           const void* x, const void* values,
                           const double* alpha_soft, const int32_t* active,
                           const int32_t* slot, const int32_t* n_act,
                           int max_act, void* g_values, double* g_soft,
                           void* g_bias, void* workspace, size_t ws_bytes,
                           void* bucket, int bucket_rows, void* stream);

/* ---- K4: soft TopK (capped water-filling) + active set -------------------
 * alpha_soft = soft_topk(alpha, k, T) (selection.py:100-142); clamped[i] = 1
 * for the water-filling's clamped set; active = flatnonzero(alpha_soft >=
 * 1e-3) ascending (layers.py:234, EPS_ACTIVE layers.py:41); slot[i] = index of
 * i in active or -1; *n_act = len(active).  float64 throughout.  Any of
 * clamped/active/slot/n_act may be NULL. */
DIAGMM_API int diagmm_topk_waterfill(int C, int k, double temperature, const double* alpha,
                          double* alpha_soft, uint8_t* clamped,
                          int32_t* active, int32_t* slot, int32_t* n_act,
                          void* stream);

/* Batched K4: n independent selections in one launch (one CTA each), e.g.
 * every DiagLinear layer of a model at the start of a step (the reference
 * runs soft_topk once per layer forward, layers.py:233).  `jobs` is a HOST
 * array; its device pointers follow the diagmm_topk_waterfill conventions. */
typedef struct diagmm_topk_job {
  int C, k;
  double temperature;
  const double* alpha;
  double* alpha_soft;
  uint8_t* clamped;
  int32_t* active;
  int32_t* slot;
  int32_t* n_act;
  /* NULL, or a DEVICE pair {T, (double)k} read by the kernel instead of
   * temperature / k: one captured CUDA graph replays an annealing / sparsity
   * schedule whose per-step values the host writes into that buffer
   * (selection.py:189-214, training.py:608-619).  temperature / k still
   * size and validate the launch. */
  const double* params;
} diagmm_topk_job;
DIAGMM_API int diagmm_topk_waterfill_batched(int n, const diagmm_topk_job* jobs,
                                             void* stream);

/* ---- K5: soft TopK gradient (+ fused l1 penalty gradient) ----------------
 * g = soft_topk_grad(alpha, k, T, g_soft) (selection.py:145-173)
 *     + l1_coeff * sign(alpha) (selection.py:217-222, layers.py:253-257).
 * clamped must come from diagmm_topk_waterfill on the same (alpha, k, T).
 * accumulate != 0 adds into g_alpha (Tape.backward accumulation,
 * autodiff.py:149-155).  params: NULL or the device {T, k} of diagmm_topk_job. */
DIAGMM_API int diagmm_topk_grad(int C, int k, double temperature, const double* alpha,
                     const uint8_t* clamped, const double* g_soft,
                     double l1_coeff, double* g_alpha, int accumulate,
                     const double* params, void* stream);

/* ---- K5 batched: every layer's soft TopK gradient in ONE launch (one CTA each)
 * after the backward (replaces one diagmm_topk_grad launch per layer; same math,
 * bit-identical results).  g_soft must be complete when this is enqueued. */
typedef struct diagmm_topk_grad_job {
  int C, k;
  double temperature;
  const double* alpha;
  const uint8_t* clamped;
  const double* g_soft;
  double l1_coeff;
  double* g_alpha;
  int accumulate;
  const double* params; /* NULL or the device {T, k} of diagmm_topk_job */
} diagmm_topk_grad_job;
DIAGMM_API int diagmm_topk_grad_batched(int n, const diagmm_topk_grad_job* jobs, void* stream);

/* ---- DiagHeur prune / regrow (layers.py:381-413) ------------------------
 * In place on the device: prune the n_prune active diagonals of smallest L2
 * value norm (ties -> smaller offset, np.lexsort((active, norms))), regrow the
 * grow_idx[i]-th (0-based) offsets of the ascending list of offsets inactive
 * before the swap with zero values, and rewrite active (first k entries,
 * ascending) / slot / *n_act.  grow_idx (n_prune,) device int32 =
 * rng.choice(C - k, n_prune, replace=False) on the reference's host RNG
 * (numpy's rng.choice(pool, n) is pool[rng.choice(len(pool), n)]).
 * values (C, L) DIAGMM_F64 or DIAGMM_F32. */
DIAGMM_API int diagmm_diagheur_update(int dtype, int C, int L, int k, int32_t* active, int32_t* slot,
                                      int32_t* n_act, void* values, int n_prune, const int32_t* grow_idx,
                                      void* stream);

/* ---- hard TopK: select_hard (selection.py:176-186) -----------------------
 * idx (k,) = indices of the k largest alpha, ties to the smaller index,
 * ascending. */
DIAGMM_API int diagmm_select_hard(int C, int k, const double* alpha, int32_t* idx,
                       void* stream);

/* Build slot/n_act from an explicit ascending offset list of length n (used
 * by DiagHeur and frozen layers whose active set is not soft-selected,
 * layers.py:381-413, 290-310).  slot (C,) int32. */
DIAGMM_API int diagmm_active_from_list(int C, int n, const int32_t* offsets, int32_t* slot,
                            int32_t* n_act, void* stream);

/* ---- K6: AdamW over the full candidate store ----------------------------
 * adamw_step (training.py:346-358) applied elementwise to n elements:
 * grad is scaled by *clip_scale when clip_scale != NULL (clip_global_norm,
 * training.py:406-417).  step is the 1-based update count t.  param/grad/m/v
 * are float64 when dtype == DIAGMM_F64, else float. */
DIAGMM_API int diagmm_adamw(int dtype, size_t n, void* param, const void* grad, void* m,
                 void* v, int step, double lr, double beta1, double beta2,
                 double eps, double weight_decay, const double* clip_scale,
                 void* stream);

/* Global-norm clipping, device side (training.py:406-417):
 * diagmm_sumsq writes sum(x^2) of one tensor into *out (float64, fixed
 * reduction order, so deterministic run to run); scratch holds at least
 * diagmm_sumsq_scratch_len() doubles.  diagmm_clip_scale reads n partial
 * sums, writes norm = sqrt(sum) to *norm and max_norm/norm (if norm >
 * max_norm and norm > 0, else 1) to *scale. */
DIAGMM_API int diagmm_sumsq_scratch_len(void);
DIAGMM_API int diagmm_sumsq(int dtype, size_t n, const void* x, double* out,
                 double* scratch, void* stream);
DIAGMM_API int diagmm_clip_scale(int n, const double* partial, double max_norm,
                      double* norm, double* scale, void* stream);

/* Multi-tensor K6: one launch per <= 40 tensors instead of one per tensor.
 * diagmm_tensor describes one parameter: dtype DIAGMM_F64 or DIAGMM_F32 for
 * param/grad/m/v alike, its element count, its own weight decay (0 for the
 * reference's no-decay ParamSpecs, layers.py:259-266) and its 1-based step.
 * `tensors` is a HOST array of device pointers.
 *   diagmm_adamw_multi: adamw_step (training.py:346-358) on every tensor,
 *     gradients scaled by *clip_scale when non-NULL; sched NULL, or a DEVICE
 *     {lr, 1 - beta1^t, 1 - beta2^t} (host-computed, the reference's floats)
 *     used instead of lr and the per-tensor steps (one CUDA graph per step).
 *   diagmm_sumsq_multi: per-chunk sum(grad^2) (float64, fixed order) into
 *     partial[0 .. diagmm_sumsq_multi_len(n, tensors)); fold them with
 *     diagmm_clip_scale_tree (clip_global_norm, training.py:406-417). */
typedef struct diagmm_tensor {
  int dtype;
  int step;
  size_t n;
  void* param;
  const void* grad;
  void* m;
  void* v;
  double weight_decay;
} diagmm_tensor;
DIAGMM_API int diagmm_adamw_multi(int n, const diagmm_tensor* tensors, double lr,
                                  double beta1, double beta2, double eps,
                                  const double* clip_scale, const double* sched, void* stream);
DIAGMM_API int diagmm_sumsq_multi_len(int n, const diagmm_tensor* tensors);
DIAGMM_API int diagmm_sumsq_multi(int n, const diagmm_tensor* tensors, double* partial,
                                  int partial_len, void* stream);
DIAGMM_API int diagmm_clip_scale_tree(int n, const double* partial, double max_norm,
                                      double* norm, double* scale, void* stream);

/* ---- tensor-core route (tcgen05 + TMEM + TMA) -----------------------------
 * out[m, n] = sum_k A[m, k] * B[n, k] (+ bias[n]); A (Mdim, K), B (Ndim, K)
 * bf16 row-major (k contiguous, 16-byte aligned, K % 8 == 0), fp32
 * accumulation, out bf16 with row stride ldo.  The dense-equivalent DiagMM:
 * forward with A = x, B = W_K (diagmm_materialize), input gradient with
 * A = dy, B = W_K^T (the reference's dense switch, diagcore.py:226-228). */
DIAGMM_API int diagmm_tc_gemm_bf16(int Mdim, int Ndim, int K, const void* A, const void* B,
                                   const float* bias, void* out, int ldo, void* stream);
/* Same GEMM with a fused epilogue (aux: (Mdim, Ndim) bf16, row stride ldo):
 * epilogue 1: aux = A B^T + bias (pre-activation), out = gelu_tanh(aux);
 * epilogue 2: out = (A B^T) * gelu_tanh'(aux) — the MLP's GELU forward fused
 * into fc1 and its backward into fc2's input gradient;  epilogue 3: out =
 * A B^T + bias + aux — the caller's residual add fused into proj / fc2. */
DIAGMM_API int diagmm_tc_gemm_bf16_ex(int Mdim, int Ndim, int K, const void* A, const void* B,
                                      const float* bias, void* out, int ldo, void* aux,
                                      int epilogue, void* stream);
/* out = A B (+ bias) with B given as (K, Ndim) row-major (Ndim % 8 == 0), staged
 * MN-major: the dense-equivalent input gradient dx = dy W_K reads the forward's
 * W_K (diagmm_materialize) directly, no W_K^T (epilogue 0, or 2 as above). */
DIAGMM_API int diagmm_tc_gemm_bf16_nn(int Mdim, int Ndim, int K, const void* A, const void* B,
                                      const float* bias, void* out, int ldo, void* aux,
                                      int epilogue, void* stream);

/* K3 on the tensor cores (bf16 activations): gw = diagonal entries of
 * dy^T x computed by tcgen05 MMAs over token tiles (split-K across CTAs), the
 * gather onto the active diagonals fused into the epilogue (the dense dW is
 * never written), then finalized exactly like diagmm_backward_weight:
 * g_values (C, L) float (active rows = alpha_soft * gw, others 0), g_soft
 * (may be NULL), g_bias (M,) float (may be NULL): the column sums of dy,
 * accumulated by extra warps from the same dy tiles the MMAs consume
 * (autodiff.py:77-79), so dy is read once.  Replaces the dense branch of
 * layers.py:150-153 + 159-165.  M, N multiples of 64; dy (B, M), x (B, N)
 * bf16, 16-byte aligned.  bucket / bucket_rows: as diagmm_backward_weight. */
/* The same two products with the (B, M)/(B, K) left operand given as 2-3
 * separate row-major column blocks A0 | A1 | A2 of `ks` / `ms` columns each
 * (multiple of 64 / 128): the qkv layer's input and weight gradients read the
 * attention's dq, dk, dv directly — no packed (B, 3*d) gradient is built.
 * diagmm_tc_gemm_bf16_nn_split: out = [A0|A1|A2] B, B (K, Ndim) row-major.
 * diagmm_tc_backward_weight_split: as diagmm_tc_backward_weight with
 * dy = [dy0|dy1|dy2]; workspace from diagmm_tc_backward_weight_workspace. */
DIAGMM_API int diagmm_tc_gemm_bf16_nn_split(int Mdim, int Ndim, int K, const void* A0, const void* A1,
                                            const void* A2, int ks, const void* B, const float* bias,
                                            void* out, int ldo, void* stream);
DIAGMM_API int diagmm_tc_backward_weight_split(int M, int N, int B, const void* dy0, const void* dy1,
                                               const void* dy2, int ms, const void* x, const void* values,
                                               const double* alpha_soft, const int32_t* slot,
                                               const int32_t* n_act, int max_act, void* g_values,
                                               double* g_soft, void* g_bias, void* workspace,
                                               size_t ws_bytes, void* bucket, int bucket_rows,
                                               void* stream);

/* Deferred finalize of the tensor-core dW (single process): _partials runs only the
 * dW GEMM with its fused diagonal gather (split-K partials + bias column partials into
 * `workspace`, the layout of diagmm_tc_backward_weight; dy given whole (ms = 0) or as
 * column blocks), and _finalize_batched later folds every layer's partials into
 * g_values / g_soft / g_bias (+ the bucket rows) in ONE launch — the same fixed-order
 * reductions as diagmm_tc_backward_weight, bit-identical results.  `parts` of a job is
 * diagmm_tc_dw_splits(M, N, B). */
DIAGMM_API int diagmm_tc_dw_splits(int M, int N, int B);
DIAGMM_API int diagmm_tc_backward_weight_partials(int M, int N, int B, const void* dy0, const void* dy1,
                                                  const void* dy2, int ms, const void* x, const int32_t* slot,
                                                  const int32_t* n_act, int max_act, int need_bias,
                                                  void* workspace, size_t ws_bytes, void* stream);
typedef struct diagmm_dw_finalize_job {
  int M, N, parts;
  const float* partial;   /* workspace of the _partials call */
  const float* colsum;    /* its bias column partials (NULL: no bias gradient) */
  int max_act;
  const int32_t* slot;
  const int32_t* n_act;
  const double* alpha_soft;
  const float* values;
  float* g_values;        /* (C, L) */
  double* g_soft;         /* (C,) or NULL */
  float* g_bias;          /* (M,) or NULL */
  float* bucket;          /* or NULL */
  int bucket_rows;
} diagmm_dw_finalize_job;
DIAGMM_API int diagmm_tc_dw_finalize_batched(int n, const diagmm_dw_finalize_job* jobs, void* stream);
DIAGMM_API size_t diagmm_tc_backward_weight_workspace(int M, int N, int B, int max_act);
DIAGMM_API int diagmm_tc_backward_weight(int M, int N, int B, const void* dy, const void* x,
                                         const void* values, const double* alpha_soft,
                                         const int32_t* slot, const int32_t* n_act, int max_act,
                                         void* g_values, double* g_soft, void* g_bias,
                                         void* workspace, size_t ws_bytes, void* bucket,
                                         int bucket_rows, void* stream);

/* ---- fused LayerNorm for the bf16 activations of the ViT caller ----------
 * Not a reference symbol: the caller's LayerNorm (vit.py) around DiagLinear.
 * x, y, dy, dx: (M, D) bf16 row-major; w, b, dw, db: (D,) float; mean, rstd:
 * (M,) float saved by the forward.  D % 8 == 0, D <= 1024.  The backward
 * folds dgamma/dbeta in a fixed order (deterministic); workspace >=
 * diagmm_layernorm_bwd_workspace(M, D) bytes. */
DIAGMM_API int diagmm_layernorm_fwd(int M, int D, float eps, const void* x, const float* w,
                                    const float* b, void* y, float* mean, float* rstd,
                                    void* stream);
DIAGMM_API size_t diagmm_layernorm_bwd_workspace(int M, int D);
DIAGMM_API int diagmm_layernorm_bwd(int M, int D, const void* x, const void* dy, const float* w,
                                    const float* mean, const float* rstd, void* dx, float* dw,
                                    float* db, void* workspace, size_t ws_bytes, void* stream);
/* Same backward with the skip connection's gradient dres ((M, D) bf16, may be
 * NULL) added into dx: x feeds both the norm and the block's residual, so its
 * two gradient contributions are summed inside the kernel. */
DIAGMM_API int diagmm_layernorm_bwd_res(int M, int D, const void* x, const void* dy, const void* dres,
                                        const float* w, const float* mean, const float* rstd, void* dx,
                                        float* dw, float* db, void* workspace, size_t ws_bytes,
                                        void* stream);

/* Packed attention-input gradient for the ViT caller: dqkv (B, T, 3, H, hd)
 * bf16 contiguous <- dq, dk, dv (B, H, T, hd) bf16 sharing the element
 * strides (stride_b, stride_h, stride_t; hd contiguous, all multiples of 8). */
DIAGMM_API int diagmm_pack_qkv_grad(int B, int T, int H, int hd, const void* dq, const void* dk,
                                    const void* dv, long long stride_b, long long stride_h,
                                    long long stride_t, void* dqkv, void* stream);

/* Dense float32 GEMM on the 3xTF32 tensor-core kernel (fp32-accurate): the
 * reference's density >= 1/4 BLAS switch (diagcore.py:226-228, layers.py:150-153)
 * for float32 layers.  out (M x N, row stride ldo) = op(A) (M x K) . op(B) (N x K)^T
 * (+ bias (N,)); op(A) = A given as (M x K, lda), or with trans_a the transpose of
 * A given as (K x M, lda); op(B) likewise (trans_b: B given as (K x N, ldb)). */
DIAGMM_API size_t diagmm_tf32x3_gemm_workspace(int M, int N, int K, int trans_a, int trans_b);
DIAGMM_API int diagmm_tf32x3_gemm(int M, int N, int K, const float* A, int lda, int trans_a, const float* B,
                                  int ldb, int trans_b, const float* bias, float* out, int ldo, void* workspace,
                                  size_t ws_bytes, void* stream);

/* ViT patch embedding for the caller (no reference counterpart on the path):
 * patchify: images (B, Cin, H, W) bf16 -> (B * (H/p) * (W/p), Cin*p*p) bf16 in conv2d
 * weight order (p % 8 == 0); embed_fwd: x (B, T, D) bf16 = [bf16(cls); y] + bf16(pos)
 * with y the (B * (T-1), D) patch projections, cls (D,) and pos (T, D) fp32;
 * embed_bwd: from gx (B, T, D) the contiguous patch gradient dy (B * (T-1), D) and the
 * fp32 gradients of pos (T, D), cls (D,) and the patch bias (D,) (any may be NULL). */
DIAGMM_API int diagmm_vit_patchify(int B, int Cin, int H, int W, int p, const void* images, void* patches,
                                   void* stream);
DIAGMM_API int diagmm_vit_embed_fwd(int B, int T, int D, const void* y, const float* cls, const float* pos,
                                    void* x, void* stream);
DIAGMM_API size_t diagmm_vit_embed_bwd_workspace(int T, int D);
DIAGMM_API int diagmm_vit_embed_bwd(int B, int T, int D, const void* gx, void* dy, float* dpos, float* dcls,
                                    float* dbias, void* workspace, size_t ws_bytes, void* stream);

/* ---- dense-equivalent route (reference's own BLAS switch) ---------------
 * The reference multiplies the materialized matrix with BLAS when the
 * structural density reaches 1/4 (diagcore.py:226-228) and computes dW
 * densely then gathers (layers.py:150-153).  diagmm_materialize writes
 * W_K (M, N) row-major in `dtype` (zeros off the active diagonals) in one
 * coalesced pass, looking offsets up in `slot` (C,) from the selection;
 * diagmm_gather_dense_grad turns a dense dW (M, N, float32/float64 = param
 * type) into g_values / g_soft exactly like diagmm_backward_weight. */
DIAGMM_API int diagmm_materialize(int dtype, int M, int N, const void* values,
                       const double* alpha_soft, const int32_t* active,
                       const int32_t* slot, const int32_t* n_act, int max_act,
                       void* w_dense, void* stream);
/* W_K^T (N, M) row-major: the B operand of the tensor-core input gradient. */
DIAGMM_API int diagmm_materialize_transposed(int dtype, int M, int N, const void* values,
                       const double* alpha_soft, const int32_t* active,
                       const int32_t* slot, const int32_t* n_act, int max_act,
                       void* w_dense_t, void* stream);

/* Every layer's W_K in ONE launch (bf16 or fp32 W, one dtype per call): the
 * model-level pre-pass right after the batched soft TopK, so the tensor-core route
 * does not pay one small launch per layer.  Same values as diagmm_materialize. */
typedef struct diagmm_materialize_job {
  int M, N;
  const void* values;       /* (C, L) float32 candidate store */
  const double* alpha_soft; /* NULL: scale 1 */
  const int32_t* slot;
  const int32_t* n_act;
  int max_act;
  void* w;                  /* (M, N) output */
} diagmm_materialize_job;
DIAGMM_API int diagmm_materialize_batched(int dtype, int n, const diagmm_materialize_job* jobs, void* stream);
DIAGMM_API int diagmm_gather_dense_grad(int dtype, int M, int N, const void* dW,
                             const void* values, const double* alpha_soft,
                             const int32_t* active, const int32_t* slot,
                             const int32_t* n_act, void* g_values,
                             double* g_soft, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DIAGMM_H */

// kd.h -- reward-weighted KL distillation (learner.cpp:10-160) on the device.
#pragma once
#include <vector>

#include <cuda_bf16.h>

#include "engine.h"

namespace rs {

// learner.cpp:10-27
double kd_weight(double r, const std::vector<double> &batch_rewards, const rs_kd_policy &p);

// learner.cpp:98-160 for a tabular drafter. Host: ceil(N/I) partial Fisher-Yates selection
// with the caller's mt19937_64 (state advanced in place), weights, row grouping. Device:
// per-position drafter softmax + KL terms (K5), per-row gradient accumulation in the
// reference's summation order and the SGD step into a new table (version + 1).
void kd_update_tabular(rs_ctx *ctx, const TabularModel *drafter, const rs_kd_sample *buf, int n,
                       const rs_kd_policy &policy, uint64_t *sel_state, double cost, rs_model **out_model,
                       rs_kd_result *out);

std::vector<int> kd_select(int n, int interval, uint64_t *sel_state);
double kd_core(rs_ctx *ctx, const TabularModel *drafter, const std::vector<const rs_kd_sample *> &sel,
               const std::vector<double> &w, double *out_dev, bool grad_only, double scale, bool policy = false);

// K5 for large vocabularies: per position, loss_i = w_i * sum_x p(x)(log p(x) - log q(x)) and
// dZ_i(x) = w_i * (q(x) - p(x)) / tau, with p given as target logits rows (softmax at tau_p)
// and q as drafter logits rows (softmax at tau_q), fp32 rows, fp64 accumulation.
void kd_rows_loss_grad(const float *target_rows, const float *drafter_rows, const double *weights,
                       const double *eos_bias, int rows, int V, double tau_p, double tau_q, double *loss_out,
                       float *dz_out, cudaStream_t st);

// Softmax tile partials (row_stats layout) of KD's target and drafter rows, fp32 exponentials.
void kd_tile_stats(const float *P, const float *Q, int R, int V, double tau_p, double tau_q, double *stP, double *stQ,
                   cudaStream_t st);
// K5 at full-chip parallelism (transformer drafters): per-row log-normalisers from the rows'
// 256-column tile partials, then one pass over 64 x 256 tiles producing the weighted KL per row
// (loss[r] = w_r KL_r) and dZ^T = (w (q - p~) / tau_q * zscale)^T as bf16 [V][ldt].
void kd_rows_lse(const float *rows, const double *stats, int nrows, int V, double tau, const double *bias, double *lse,
                 cudaStream_t st);
void kd_rows_elem(const float *P, const float *Q, const double *lseP, const double *lseQ, const double *w,
                  const double *bias, int R, int V, double tau_p, double tau_q, float zscale, __nv_bfloat16 *dzT, int ldt,
                  double *kl_part, double *loss, cudaStream_t st);
void transpose_pad_bf16(const __nv_bfloat16 *in, int ldi, int R, int C, __nv_bfloat16 *out, int ldo, cudaStream_t st);
void sgd_bf16(const __nv_bfloat16 *w, const float *g, float scale, size_t n, __nv_bfloat16 *out, cudaStream_t st);

// Whole-drafter KD backward (kd_train.cu): element-wise / reduction pieces around the GEMMs.
// rms_bwd: dx = base + dRMSNorm/dx . dy (base / dx / gterm optional), gterm = dy * x * r (the
// per-row gain gradient terms); colsum_f32: out[c] (+)= sum over rows in a fixed order
// (partial needs max_chunks * C floats); swiglu_bwd: pairwise-interleaved gate/up gradient;
// rope_bwd: inverse rotation in place; softmax_bwd: causal rows (row i of a head stack sees keys
// 0 .. i % T), P and dS (times scale) in
// bf16; cast_bf16: fp32 -> bf16 sub-matrix; sgd_f32: out = w + scale * g.
void rms_bwd(const float *x, int ldx, const float *g, const float *dy, int lddy, int M, int d, float eps,
             const float *base, int ldb, float *dx, int lddx, float *gterm, int ldg, cudaStream_t st);
void colsum_f32(const float *in, int ld, int M, int C, float *out, bool accumulate, float *partial, int max_chunks,
                cudaStream_t st);
void swiglu_bwd(const __nv_bfloat16 *gu, int ldgu, const float *dh, int lddh, int M, int F, __nv_bfloat16 *dgu,
                int lddgu, cudaStream_t st);
void rope_bwd(float *x, int ldx, int M, int heads, int hd, const int *pos, const float *rope, cudaStream_t st);
void softmax_bwd(const float *S, const float *dP, int lds, int rows, int T, float scale, __nv_bfloat16 *P,
                 __nv_bfloat16 *dS, int ldo, cudaStream_t st);
// stack_heads: the heads of a GQA group as [heads * T][hd] rows (bf16); unstack_heads: the fp32
// inverse into a [T][ldo] row-major block at the group's first head.
void stack_heads(const __nv_bfloat16 *in, int ldi, int T, int heads, int hd, __nv_bfloat16 *out, cudaStream_t st);
void unstack_heads(const float *in, int T, int heads, int hd, float *out, int ldo, cudaStream_t st);
void cast_bf16(const float *in, int ldi, int M, int C, __nv_bfloat16 *out, int ldo, cudaStream_t st);
void sgd_f32(const float *w, const float *g, float scale, size_t n, float *out, cudaStream_t st);

// L2 norm of a bf16 weight tensor (fp64 accumulation, deterministic order) -- the learner's
// LearnerMetrics::weights_l2 for transformer drafters (learner.cpp:268-272).
double weights_l2_bf16(const __nv_bfloat16 *w, size_t n, cudaStream_t st);

}  // namespace rs

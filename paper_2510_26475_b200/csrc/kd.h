// kd.h -- reward-weighted KL distillation (learner.cpp:10-160) on the device.
#pragma once
#include <vector>

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
               const std::vector<double> &w, double *out_dev, bool grad_only, double scale);

// K5 for large vocabularies: per position, loss_i = w_i * sum_x p(x)(log p(x) - log q(x)) and
// dZ_i(x) = w_i * (q(x) - p(x)) / tau, with p given as target logits rows (softmax at tau_p)
// and q as drafter logits rows (softmax at tau_q), fp32 rows, fp64 accumulation.
void kd_rows_loss_grad(const float *target_rows, const float *drafter_rows, const double *weights,
                       const double *eos_bias, int rows, int V, double tau_p, double tau_q, double *loss_out,
                       float *dz_out, cudaStream_t st);

}  // namespace rs

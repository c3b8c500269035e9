// rl.cpp -- the GRPO stage around the rollout (rl.cpp:8-90 of the reference): reward,
// group-relative advantages and the tabular actor's policy-gradient step. reward/advantages are
// host scalars; the policy step runs on the device through the K5 row machinery of kd.cu (one
// CTA per visited table row, contributions accumulated in the reference's sample/position order).
#include <cmath>
#include <stdexcept>
#include <vector>

#include "abi.h"
#include "engine.h"
#include "kd.h"

using rs_abi::guard;
using rs_abi::need;

extern "C" {

// reward (rl.cpp:8-19): fraction of adjacent pairs equal to (golden_a, golden_b).
int rs_reward(const int32_t *y, int32_t n, int32_t golden_a, int32_t golden_b, double *out) {
    return guard([&] {
        need(out, "rs_reward");
        if (n > 0) need(y, "rs_reward: response");
        if (n < 2) {
            *out = 0.0;
            return;
        }
        int matches = 0;
        for (int i = 0; i + 1 < n; ++i)
            if (y[i] == golden_a && y[i + 1] == golden_b) ++matches;
        *out = static_cast<double>(matches) / static_cast<double>(n - 1);
    });
}

// group_advantages (rl.cpp:21-40): (r - mean) / (population std + 1e-6); G >= 2.
int rs_group_advantages(const double *rewards, int32_t g, double *out) {
    return guard([&] {
        if (g < 2) throw std::invalid_argument("group_advantages: group size must be >= 2");
        need(rewards, "rs_group_advantages");
        need(out, "rs_group_advantages: out");
        double mean = 0.0;
        for (int i = 0; i < g; ++i) mean += rewards[i];
        mean /= static_cast<double>(g);
        double var = 0.0;
        for (int i = 0; i < g; ++i) var += (rewards[i] - mean) * (rewards[i] - mean);
        const double sd = std::sqrt(var / static_cast<double>(g));
        for (int i = 0; i < g; ++i) out[i] = (rewards[i] - mean) / (sd + 1e-6);
    });
}

// policy_update (rl.cpp:74-88): reject off-policy samples, then actor + lr * grad of
// sum_i A_i sum_t log pi(y_t | ctx_t) into a new model (version + 1, model.cpp:161-170).
int rs_policy_update_tabular(rs_ctx *ctx, const rs_model *actor, const rs_kd_sample *samples,
                             const double *advantages, const int32_t *actor_versions, int32_t n, double lr,
                             rs_model **out) {
    return guard([&] {
        need(ctx, "rs_policy_update_tabular");
        need(actor, "rs_policy_update_tabular: actor");
        need(out, "rs_policy_update_tabular: out");
        if (actor->kind != rs_model::Tabular) throw std::invalid_argument("policy_update: tabular actor required");
        if (n > 0) {
            need(samples, "rs_policy_update_tabular: samples");
            need(advantages, "rs_policy_update_tabular: advantages");
        }
        for (int i = 0; i < n; ++i)
            if (actor_versions && actor_versions[i] != actor->version)
                throw std::invalid_argument("policy_update: off-policy update");
        const auto *a = static_cast<const rs::TabularModel *>(actor);
        auto m = std::make_unique<rs::TabularModel>();
        m->ctx = ctx;
        m->vocab = a->vocab;
        m->order = a->order;
        m->rows = a->rows;
        m->temperature = a->temperature;
        m->version = a->version + 1;
        m->host = a->host;
        m->table.alloc(m->host.size());
        std::vector<const rs_kd_sample *> sel(std::max(n, 0));
        std::vector<double> w(std::max(n, 0));
        for (int i = 0; i < n; ++i) {
            sel[i] = &samples[i];
            w[i] = advantages[i];
        }
        rs::kd_core(ctx, a, sel, w, m->table.p, false, lr, true);
        RS_CUDA(cudaMemcpy(m->host.data(), m->table.p, m->host.size() * 8, cudaMemcpyDeviceToHost));
        *out = m.release();
    });
}

}  // extern "C"

// api.cpp -- extern "C" entry points (include/respec_b200.h). Every entry point converts the
// internal C++ exception into the status code of the reference's exception class and
// keeps the message in a thread-local buffer for rs_last_error().
#include <algorithm>
#include <memory>
#include <random>
#include <cstring>
#include <stdexcept>
#include <string>

#include "abi.h"
#include "common.cuh"
#include "engine.h"
#include "gemm.h"
#include "kd.h"
#include "model.h"
#include "prof.h"

namespace rs_abi {
std::string &last_error() {
    thread_local std::string e;
    return e;
}
}  // namespace rs_abi

namespace {
thread_local int64_t g_launches = 0;
using rs_abi::guard;
using rs_abi::need;

void check_cfg(const rs_sdconfig &c) {
    if (!c.enabled) return;
    if (c.rounds < 1 || c.branching < 1 || c.draft_len < 1)
        throw std::invalid_argument("SDConfig: rounds, branching and draft_len must be >= 1");
    if (c.rounds > rs::kMaxRounds || c.branching > rs::kMaxBranch || c.draft_len > rs::kMaxDraft)
        throw std::invalid_argument("SDConfig: exceeds engine limits (s<=8, t<=16, n<=32)");
    // per-cycle RNG consumption must fit one mt19937_64 block (SURVEY App. A maxima)
    if (c.rounds * c.branching * c.draft_len > rs::kMtN || c.rounds * (c.branching + c.draft_len - 1) + 1 > rs::kMtN)
        throw std::invalid_argument("SDConfig: per-cycle draws exceed 312");
}
}  // namespace

namespace {
template <class T>
void copy_out(const std::vector<T> &v, T *out, int32_t cap, int32_t *n) {
    if (n) *n = (int32_t)v.size();
    if (out) std::copy(v.begin(), v.begin() + std::min<size_t>(v.size(), (size_t)std::max(cap, 0)), out);
}

}  // namespace

namespace rs {
thread_local int64_t g_h2d = 0, g_d2h = 0;
void note_launch() { ++g_launches; }
void note_copy(bool h2d, size_t bytes) { (h2d ? g_h2d : g_d2h) += (int64_t)bytes; }
int64_t copy_bytes(bool h2d) { return h2d ? g_h2d : g_d2h; }
void reset_copy_bytes() { g_h2d = g_d2h = 0; }
}  // namespace rs

using namespace rs;

extern "C" {

const char *rs_last_error(void) { return rs_abi::last_error().c_str(); }
int rs_version(void) { return 10000; }
int64_t rs_launch_count(void) { return g_launches; }
void rs_launch_count_reset(void) { g_launches = 0; }

int rs_ctx_create(int device, rs_ctx **out) {
    return guard([&] {
        need(out, "rs_ctx_create");
        auto c = std::make_unique<rs_ctx>();
        c->device = device;
        RS_CUDA(cudaSetDevice(device));
        // the rollout path is latency-critical: its stream gets the GREATEST priority (background
        // work -- an asynchronous learner's update -- runs at the least, learner.cpp)
        int least = 0, greatest = 0;
        RS_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        RS_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, greatest));
        c->own_stream = true;
        RS_CUDA(cudaEventCreate(&c->ev0));
        RS_CUDA(cudaEventCreate(&c->ev1));
        *out = c.release();
    });
}

int rs_ctx_destroy(rs_ctx *ctx) {
    return guard([&] {
        if (!ctx) return;
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
        if (ctx->ev0) cudaEventDestroy(ctx->ev0);
        if (ctx->ev1) cudaEventDestroy(ctx->ev1);
        delete ctx;
    });
}

int rs_ctx_sync(rs_ctx *ctx) {
    return guard([&] {
        need(ctx, "rs_ctx_sync");
        RS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int rs_ctx_set_stream(rs_ctx *ctx, void *s) {
    return guard([&] {
        need(ctx, "rs_ctx_set_stream");
        RS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
        ctx->stream = static_cast<cudaStream_t>(s);
        ctx->own_stream = false;
    });
}

// ---- models --------------------------------------------------------------------------------
int rs_tabular_create(rs_ctx *ctx, int32_t vocab, int32_t order, double temperature, const double *logits,
                      int32_t version, rs_model **out) {
    return guard([&] {
        need(ctx, "rs_tabular_create");
        need(out, "rs_tabular_create");
        // TabularARModel constructor checks (model.cpp:80-94)
        if (vocab < 2) throw std::invalid_argument("TabularARModel: vocab size must be >= 2");
        if (order < 0) throw std::invalid_argument("TabularARModel: negative order");
        if (!(temperature > 0.0)) throw std::invalid_argument("TabularARModel: temperature must be positive");
        auto m = std::make_unique<TabularModel>();
        m->ctx = ctx;
        m->vocab = vocab;
        m->order = order;
        m->temperature = temperature;
        m->version = version;
        size_t rows = 1;
        for (int i = 0; i < order; ++i) rows *= static_cast<size_t>(vocab);
        m->rows = rows;
        const size_t cnt = rows * static_cast<size_t>(vocab);
        if (!logits) throw std::invalid_argument("TabularARModel: logits table has wrong shape");
        m->host.assign(logits, logits + cnt);
        m->table.alloc(cnt);
        RS_CUDA(cudaMemcpy(m->table.p, logits, cnt * sizeof(double), cudaMemcpyHostToDevice));
        *out = m.release();
    });
}

int rs_tabular_logits(const rs_model *m, double *out, int64_t n) {
    return guard([&] {
        need(m, "rs_tabular_logits");
        if (m->kind != rs_model::Tabular) throw std::invalid_argument("rs_tabular_logits: not a tabular model");
        auto *t = static_cast<const TabularModel *>(m);
        if (n < (int64_t)t->host.size()) throw std::invalid_argument("rs_tabular_logits: buffer too small");
        std::memcpy(out, t->host.data(), t->host.size() * sizeof(double));
    });
}

int rs_model_version(const rs_model *m, int32_t *out) {
    return guard([&] { need(m, "rs_model_version"); *out = m->version; });
}
int rs_model_vocab(const rs_model *m, int32_t *out) {
    return guard([&] { need(m, "rs_model_vocab"); *out = m->vocab; });
}
int rs_model_destroy(rs_model *m) {
    return guard([&] {
        if (m && m->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) delete m;
    });
}
int rs_model_retain(rs_model *m) {
    return guard([&] {
        need(m, "rs_model_retain");
        m->refs.fetch_add(1, std::memory_order_relaxed);
    });
}

// ---- ProfileTable ----------------------------------------------------------------------------
int rs_table_create(const int32_t *buckets, int32_t n, rs_table **out) {
    return guard([&] {
        need(out, "rs_table_create");
        std::vector<int> b(buckets, buckets + std::max(0, n));
        *out = new rs_table{ProfileTable(std::move(b))};
    });
}
int rs_table_set_entry(rs_table *t, int32_t bucket, rs_sdconfig cfg, double tpt) {
    return guard([&] { need(t, "rs_table_set_entry"); t->t.set_entry(bucket, cfg, tpt); });
}
int rs_table_finalize(rs_table *t) {
    return guard([&] { need(t, "rs_table_finalize"); t->t.finalize(); });
}
int rs_table_bucket_for(const rs_table *t, int32_t b, int32_t *out) {
    return guard([&] { need(t, "rs_table_bucket_for"); *out = t->t.bucket_for(b); });
}
int rs_table_solve(const rs_table *t, int32_t b, rs_sdconfig *out) {
    return guard([&] { need(t, "rs_table_solve"); *out = t->t.solve(b); });
}
int rs_table_best_for_bucket(const rs_table *t, int32_t b, rs_sdconfig *out) {
    return guard([&] { need(t, "rs_table_best_for_bucket"); *out = t->t.best_for_bucket(b); });
}
int rs_table_entry(const rs_table *t, int32_t b, rs_sdconfig cfg, double *out) {
    return guard([&] { need(t, "rs_table_entry"); *out = t->t.entry(b, cfg); });
}
int rs_table_to_csv(const rs_table *t, char *buf, int64_t cap, int64_t *len) {
    return guard([&] {
        need(t, "rs_table_to_csv");
        const std::string s = t->t.to_csv();
        if (len) *len = (int64_t)s.size();
        if (buf && cap > 0) {
            const size_t k = std::min<size_t>(s.size(), (size_t)cap - 1);
            std::memcpy(buf, s.data(), k);
            buf[k] = 0;
        }
    });
}
int rs_table_destroy(rs_table *t) {
    return guard([&] { delete t; });
}

// ---- engine -----------------------------------------------------------------------------------
int rs_engine_create(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_table *table,
                     const rs_timing_model *tm, const rs_request *reqs, int32_t n, rs_sdconfig forced,
                     int32_t verify_mode, int32_t record_full, rs_engine **out) {
    return guard([&] {
        need(ctx, "rs_engine_create");
        need(target, "rs_engine_create: target");
        need(out, "rs_engine_create");
        if (n < 0 || (n > 0 && !reqs)) throw std::invalid_argument("rs_engine_create: bad request array");
        if (verify_mode != RS_VERIFY_SAMPLE && verify_mode != RS_VERIFY_GREEDY)
            throw std::invalid_argument("rs_engine_create: unknown verify mode");
        if (target->kind == rs_model::Drafter) throw std::invalid_argument("rs_engine_create: target must not be a drafter");
        check_cfg(forced);
        auto e = std::make_unique<rs_engine>();
        e->ctx = ctx;
        e->target = target;
        e->pending_drafter = drafter;
        e->table = table ? &table->t : nullptr;
        if (tm) e->tm = *tm;
        else e->tm = rs_timing_model{{1.0, 32, 2.0}, {0.1, 32, 0.4}};
        e->mode = forced;
        e->verify_mode = verify_mode;
        e->record_full = record_full != 0;
        e->n = n;
        e->V = target->vocab;
        // sizes for every config this engine may run
        std::vector<rs_sdconfig> cfgs{forced};
        if (e->table) {
            auto more = e->table->all_configs();
            cfgs.insert(cfgs.end(), more.begin(), more.end());
        }
        for (const auto &c : cfgs) {
            check_cfg(c);
            if (!c.enabled) continue;
            e->t_max = std::max(e->t_max, (int)c.branching);
            e->n_max = std::max(e->n_max, (int)c.draft_len);
            e->s_max = std::max(e->s_max, (int)c.rounds);
            e->slots_max = std::max(e->slots_max, 1 + c.branching * c.draft_len);
        }
        int tok_cap = 1, steps_cap = 1;
        std::vector<int32_t> h_tok;
        std::vector<std::vector<int>> prompts;
        for (int i = 0; i < n; ++i) {
            const rs_request &r = reqs[i];
            if (r.prompt_len < 0 || (r.prompt_len > 0 && !r.prompt)) throw std::invalid_argument("rs_request: bad prompt");
            for (int k = 0; k < r.prompt_len; ++k)
                if (r.prompt[k] < 0 || r.prompt[k] >= e->V) throw std::invalid_argument("row_index: token out of vocabulary");
            tok_cap = std::max(tok_cap, r.prompt_len + std::max(r.max_len, 0) + 1);
            steps_cap = std::max(steps_cap, std::max(r.max_len, 1));
        }
        e->tok_cap = tok_cap;
        e->steps_cap = steps_cap;
        h_tok.assign((size_t)std::max(n, 1) * tok_cap, 0);
        std::vector<uint64_t> seeds(n), sids(n);
        for (int i = 0; i < n; ++i) {
            const rs_request &r = reqs[i];
            e->ids.push_back(r.id);
            e->prompt_len.push_back(r.prompt_len);
            e->max_len.push_back(r.max_len);
            e->len.push_back(r.prompt_len);
            // a request with max_len <= 0 can never step (BatchEngine keeps it active; we
            // mark it done so the engine cannot spin on it)
            e->done.push_back(r.max_len <= 0 ? 1 : 0);
            e->eos_bias.push_back(r.eos_bias);
            std::copy(r.prompt, r.prompt + r.prompt_len, h_tok.begin() + (size_t)i * tok_cap);
            seeds[i] = r.seed;
            sids[i] = r.stream_id;
            prompts.emplace_back(r.prompt, r.prompt + r.prompt_len);
        }
        e->accept_lens.resize(n);
        const int N = std::max(n, 1);
        e->d_tok.alloc((size_t)N * tok_cap);
        RS_CUDA(cudaMemcpy(e->d_tok.p, h_tok.data(), h_tok.size() * 4, cudaMemcpyHostToDevice));
        auto up_i = [&](DBuf<int32_t> &b, const std::vector<int> &v) {
            b.alloc(N);
            if (!v.empty()) RS_CUDA(cudaMemcpy(b.p, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
        };
        up_i(e->d_len, e->len);
        up_i(e->d_plen, e->prompt_len);
        up_i(e->d_maxlen, e->max_len);
        up_i(e->d_done, e->done);
        e->d_active.alloc(N);
        e->d_bias.alloc(N);
        if (n) RS_CUDA(cudaMemcpy(e->d_bias.p, e->eos_bias.data(), n * 8, cudaMemcpyHostToDevice));
        e->d_rng.alloc(2 * (size_t)N);
        DBuf<uint64_t> dseed(N), dsid(N);
        if (n) {
            RS_CUDA(cudaMemcpy(dseed.p, seeds.data(), n * 8, cudaMemcpyHostToDevice));
            RS_CUDA(cudaMemcpy(dsid.p, sids.data(), n * 8, cudaMemcpyHostToDevice));
            rng_init(e->d_rng.p, dseed.p, dsid.p, n, ctx->stream);
        }
        e->d_st_tok.alloc((size_t)N * steps_cap);
        e->d_st_logp.alloc((size_t)N * steps_cap);
        e->d_st_logq.alloc((size_t)N * steps_cap);
        e->d_st_drafted.alloc((size_t)N * steps_cap);
        if (e->record_full) e->d_st_full.alloc((size_t)N * steps_cap * e->V);
        e->d_cyc.alloc((size_t)N * 17);  // + [N][6] two-stage acceptance state
        e->d_round_cost.alloc((size_t)N * kMaxRounds * 3);
        e->d_chain.alloc((size_t)N * e->t_max * (e->n_max + 3));
        RS_CUDA(cudaMemset(e->d_chain.p, 0, e->d_chain.bytes()));
        e->d_err.alloc(1);
        e->d_flag.alloc(1);
        RS_CUDA(cudaMemset(e->d_err.p, 0, 4));
        RS_CUDA(cudaMemset(e->d_flag.p, 0, 4));
        e->d_summary.alloc((size_t)N * (kSummaryFixed + 3 * kMaxRounds));
        RS_CUDA(cudaMallocHost(&e->h_summary, (size_t)N * (kSummaryFixed + 3 * kMaxRounds) * 4));
        e->newtok_cap = kMaxRounds * e->n_max + 1;  // a cycle emits <= s * n + 1 tokens
        e->d_newtok.alloc((size_t)N * e->newtok_cap);
        RS_CUDA(cudaMallocHost(&e->h_newtok, (size_t)N * e->newtok_cap * 4));
        RS_CUDA(cudaMallocHost(&e->h_active, (size_t)N * 4));
        RS_CUDA(cudaMallocHost(&e->h_misc, 16));
        std::memset(e->h_misc, 0, 16);

        if (target->kind == rs_model::Tabular) {
            if (drafter && drafter->kind != rs_model::Tabular) throw std::invalid_argument("tabular target needs a tabular drafter");
            const size_t rows = (size_t)N * e->slots_max * e->V * sizeof(double);
            e->d_P.alloc(rows);
            e->d_Q.alloc(rows);
            e->pair = make_tabular_pair(static_cast<const TabularModel *>(target), static_cast<const TabularModel *>(drafter));
        } else {
            const size_t rows = (size_t)N * e->slots_max * e->V * sizeof(float);
            e->d_P.alloc(rows);
            e->d_Q.alloc(rows);
            const size_t nst = (size_t)N * e->slots_max * ((e->V + 255) / 256) * 2;
            e->d_Pst.alloc(nst);
            e->d_Qst.alloc(nst);
            e->pair = make_transformer_pair(ctx, e.get(), target, drafter, n, e->slots_max, e->prompt_len, prompts, tok_cap);
        }
        e->d_pq.alloc((size_t)N * 2 * e->V);
        if (drafter && drafter->vocab != e->V) throw std::invalid_argument("BatchEngine: drafter vocabulary differs from target");
        RS_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = e.release();
    });
}

int rs_engine_set_drafter(rs_engine *e, const rs_model *drafter) {
    return guard([&] { need(e, "rs_engine_set_drafter"); e->pending_drafter = drafter; });
}
int rs_engine_step(rs_engine *e, rs_step_info *info) {
    return guard([&] {
        need(e, "rs_engine_step");
        e->check_unpinned("BatchEngine::step");
        std::unique_lock<std::mutex> lk(e->use_mu, std::try_to_lock);
        if (!lk) throw std::runtime_error("BatchEngine::step: engine in use by another thread");
        e->step(info);
    });
}
int rs_engine_all_done(const rs_engine *e, int32_t *out) {
    return guard([&] {
        need(e, "rs_engine_all_done");
        *out = std::all_of(e->done.begin(), e->done.end(), [](int d) { return d != 0; });
    });
}
int rs_engine_active_batch(const rs_engine *e, int32_t *out) {
    return guard([&] {
        need(e, "rs_engine_active_batch");
        *out = (int32_t)std::count(e->done.begin(), e->done.end(), 0);
    });
}
int rs_engine_cycles(const rs_engine *e, int32_t *out) {
    return guard([&] { need(e, "rs_engine_cycles"); *out = e->cycle; });
}
int rs_engine_prefill_events(const rs_engine *e, int32_t *out) {
    return guard([&] { need(e, "rs_engine_prefill_events"); *out = e->prefill_events; });
}
int rs_engine_ledger_time(const rs_engine *e, double *out) {
    return guard([&] {
        need(e, "rs_engine_ledger_time");
        // ledger_time / forward_time (costsim.cpp:13-27)
        double total = 0.0;
        for (const auto &ev : e->ledger) {
            const rs_role_timing &t = ev.role ? e->tm.target : e->tm.drafter;
            if (ev.batch_tokens < 1) throw std::invalid_argument("forward_time: total_tokens must be >= 1");
            total += t.latency_floor + t.unit_cost * (double)std::max(ev.batch_tokens, t.saturation_tokens);
        }
        *out = total;
    });
}

int rs_engine_ledger(const rs_engine *e, rs_forward_event *out, int32_t cap, int32_t *n) {
    return guard([&] { need(e, "rs_engine_ledger"); copy_out(e->ledger, out, cap, n); });
}
int rs_engine_switches(const rs_engine *e, rs_switch_event *out, int32_t cap, int32_t *n) {
    return guard([&] { need(e, "rs_engine_switches"); copy_out(e->switches, out, cap, n); });
}
int rs_engine_active_trace(const rs_engine *e, int32_t *out, int32_t cap, int32_t *n) {
    return guard([&] { need(e, "rs_engine_active_trace"); copy_out(e->active_trace, (int *)out, cap, n); });
}
int rs_engine_drafter_versions(const rs_engine *e, int32_t *out, int32_t cap, int32_t *n) {
    return guard([&] { need(e, "rs_engine_drafter_versions"); copy_out(e->drafter_versions, (int *)out, cap, n); });
}

static void check_req(const rs_engine *e, int32_t req) {
    if (req < 0 || req >= e->n) throw std::invalid_argument("request index out of range");
}

int rs_engine_response(rs_engine *e, int32_t req, int32_t *tokens, int32_t cap, int32_t *len) {
    return guard([&] {
        need(e, "rs_engine_response");
        check_req(e, req);
        const int gen = e->len[req] - e->prompt_len[req];
        if (len) *len = gen;
        const int k = std::min(gen, std::max(cap, 0));
        if (tokens && k > 0)
            RS_CUDA(cudaMemcpy(tokens, e->d_tok.p + (size_t)req * e->tok_cap + e->prompt_len[req], k * 4, cudaMemcpyDeviceToHost));
    });
}

int rs_profile_measured(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const int32_t *buckets,
                        int32_t nb, const rs_sdconfig *cfgs, int32_t nc, int32_t prompt_len, int32_t warmup,
                        int32_t cycles, uint64_t seed, double *tpt) {
    return guard([&] {
        need(ctx, "rs_profile_measured");
        need(target, "rs_profile_measured: target");
        need(tpt, "rs_profile_measured: out");
        if (nb <= 0 || nc <= 0 || cycles <= 0 || prompt_len <= 0)
            throw std::invalid_argument("profile: empty grid");
        const int V = target->vocab;
        for (int ib = 0; ib < nb; ++ib) {
            const int b = buckets[ib];
            if (b <= 0) throw std::invalid_argument("profile: bucket sizes must be positive");
            // synthetic prompts (splitmix64 over [0, V-1)), the same for every config of a bucket
            std::vector<std::vector<int32_t>> prompts(b, std::vector<int32_t>(prompt_len));
            uint64_t x = seed * 0x9E3779B97F4A7C15ull + (uint64_t)b;
            for (auto &p : prompts)
                for (auto &t : p) {
                    x += 0x9E3779B97F4A7C15ull;
                    uint64_t z = x;
                    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
                    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
                    t = (int32_t)((z ^ (z >> 31)) % (uint64_t)(V - 1));
                }
            for (int ic = 0; ic < nc; ++ic) {
                const rs_sdconfig c = cfgs[ic];
                if (c.enabled && !drafter) throw std::invalid_argument("profile: spec configs need a drafter");
                const int per = c.enabled ? c.rounds * c.draft_len + 1 : 1;
                const int max_len = (warmup + cycles) * per + 8;
                std::vector<rs_request> reqs(b);
                for (int i = 0; i < b; ++i)
                    reqs[i] = {i, prompts[i].data(), prompt_len, -1e4, max_len, seed, (uint64_t)i};
                rs_timing_model tm{{1.0, 32, 2.0}, {0.1, 32, 0.4}};
                rs_engine *e = nullptr;
                int rc = rs_engine_create(ctx, target, c.enabled ? drafter : nullptr, nullptr, &tm, reqs.data(), b, c,
                                          RS_VERIFY_SAMPLE, 0, &e);
                if (rc != RS_OK) throw std::runtime_error(std::string("profile: ") + rs_last_error());
                double ms = 0.0;
                long long toks = 0;
                for (int k = 0; k < warmup + cycles; ++k) {
                    rs_step_info info{};
                    rc = rs_engine_step(e, &info);
                    if (rc != RS_OK) {
                        const std::string m = rs_last_error();
                        rs_engine_destroy(e);
                        throw std::runtime_error("profile: " + m);
                    }
                    if (k >= warmup) {
                        ms += info.step_ms;
                        toks += info.emitted_tokens;
                    }
                }
                rs_engine_destroy(e);
                tpt[(size_t)ib * nc + ic] = toks > 0 ? ms / (double)toks : 1e30;
            }
        }
    });
}

int rs_engine_step_tokens(rs_engine *e, int32_t *req, int32_t *count, int32_t *tokens, int32_t cap_per_req,
                          int32_t *n) {
    return guard([&] {
        need(e, "rs_engine_step_tokens");
        const int na = (int)e->last_active.size();
        if (n) *n = na;
        for (int a = 0; a < na; ++a) {
            if (req) req[a] = e->last_active[a];
            const int c = std::min(e->last_emitted[a], e->newtok_cap);
            if (count) count[a] = c;
            if (tokens)
                for (int k = 0; k < std::min(c, cap_per_req); ++k)
                    tokens[(size_t)a * cap_per_req + k] = e->h_newtok[(size_t)a * e->newtok_cap + k];
        }
    });
}

int rs_engine_steps(rs_engine *e, int32_t req, double *logp, uint8_t *drafted, double *logq, int32_t cap, int32_t *n) {
    return guard([&] {
        need(e, "rs_engine_steps");
        check_req(e, req);
        const int gen = e->len[req] - e->prompt_len[req];
        if (n) *n = gen;
        const int k = std::min(gen, std::max(cap, 0));
        if (k <= 0) return;
        const size_t off = (size_t)req * e->steps_cap;
        if (logp) RS_CUDA(cudaMemcpy(logp, e->d_st_logp.p + off, k * 8, cudaMemcpyDeviceToHost));
        if (drafted) RS_CUDA(cudaMemcpy(drafted, e->d_st_drafted.p + off, k, cudaMemcpyDeviceToHost));
        if (logq) RS_CUDA(cudaMemcpy(logq, e->d_st_logq.p + off, k * 8, cudaMemcpyDeviceToHost));
    });
}

int rs_engine_step_logprobs(rs_engine *e, int32_t req, double *out, int64_t cap, int32_t *rows) {
    return guard([&] {
        need(e, "rs_engine_step_logprobs");
        check_req(e, req);
        if (!e->record_full) throw std::invalid_argument("engine was created without record_full_logprobs");
        const int gen = e->len[req] - e->prompt_len[req];
        if (rows) *rows = gen;
        const int64_t k = std::min<int64_t>((int64_t)gen * e->V, cap);
        if (out && k > 0)
            RS_CUDA(cudaMemcpy(out, e->d_st_full.p + (size_t)req * e->steps_cap * e->V, k * 8, cudaMemcpyDeviceToHost));
    });
}

int rs_engine_accept_lens(rs_engine *e, int32_t req, int32_t *out, int32_t cap, int32_t *n) {
    return guard([&] {
        need(e, "rs_engine_accept_lens");
        check_req(e, req);
        copy_out(e->accept_lens[req], (int *)out, cap, n);
    });
}

int rs_engine_destroy(rs_engine *e) {
    return guard([&] {
        if (e && e->ctx) cudaStreamSynchronize(e->ctx->stream);
        delete e;
    });
}

int rs_engine_set_stop_at_eos(rs_engine *e, int32_t stop) {
    return guard([&] {
        need(e, "rs_engine_set_stop_at_eos");
        if (e->cycle > 0) throw std::runtime_error("rs_engine_set_stop_at_eos: engine already stepped");
        e->stop_at_eos = stop != 0;
    });
}

// profile() (server.cpp:182-239) on the GPU engine with the SIMULATED cost model: per bucket and
// config (the non-spec entry first), waves of exactly `batch` requests over a pool of
// num_requests (prompt rid % n_prompts, DecodeRng::from_seed(seed, rid), eos_bias 0), each
// running cycles_per_request engine cycles with stop_at_eos = false; every wave's forward
// events are appended to one ledger, and time_per_token = ledger_time / emitted tokens.
int rs_profile_simulated(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_sdconfig *grid,
                         int32_t ng, const int32_t *prompts, const int32_t *prompt_off, int32_t n_prompts,
                         const rs_timing_model *tm, const int32_t *buckets, int32_t nb, int32_t cycles_per_request,
                         int32_t num_requests, uint64_t seed, double *time_per_token) {
    return guard([&] {
        need(ctx, "rs_profile_simulated");
        need(target, "rs_profile_simulated: target");
        need(tm, "rs_profile_simulated: timing");
        need(time_per_token, "rs_profile_simulated: out");
        if (n_prompts <= 0) throw std::invalid_argument("profile: no eval prompts");
        need(prompts, "rs_profile_simulated: prompts");
        need(prompt_off, "rs_profile_simulated: prompt offsets");
        if (nb > 0) need(buckets, "rs_profile_simulated: buckets");
        std::vector<rs_sdconfig> cfgs{rs_sdconfig{1, 1, 1, 0}};
        for (int i = 0; i < ng; ++i) {
            check_cfg(grid[i]);
            cfgs.push_back(grid[i]);
        }
        const int nc = (int)cfgs.size();
        for (int ib = 0; ib < nb; ++ib) {
            const int batch = buckets[ib];
            if (batch < 1) throw std::invalid_argument("profile: batch sizes must be >= 1");
            for (int ic = 0; ic < nc; ++ic) {
                const rs_sdconfig c = cfgs[ic];
                if (c.enabled && !drafter) throw std::invalid_argument("profile: spec configs need a drafter");
                const int per = c.enabled ? c.rounds * c.draft_len + 1 : 1;
                const int max_len = cycles_per_request * per + (c.enabled ? c.draft_len : 0) + 8;
                // Every wave of the pool runs side by side in ONE engine (a request's trajectory
                // depends only on its own RNG streams and context); the engine charges each wave's
                // lockstep cycles into that wave's own ledger, concatenated in wave order below --
                // the reference's single ledger, event for event.
                std::vector<rs_forward_event> ledger;
                long long tokens = 0;
                const int waves = num_requests > 0 ? (num_requests + batch - 1) / batch : 0;
                if (waves > 0) {
                    std::vector<rs_request> reqs((size_t)waves * batch);
                    for (int rid = 0; rid < waves * batch; ++rid) {
                        const int p = rid % n_prompts;
                        reqs[rid] = {rid, prompts + prompt_off[p], prompt_off[p + 1] - prompt_off[p], 0.0, max_len,
                                     seed, (uint64_t)rid};
                    }
                    rs_engine *e = nullptr;
                    rs_abi::rethrow(rs_engine_create(ctx, target, c.enabled ? drafter : nullptr, nullptr, tm,
                                                     reqs.data(), (int32_t)reqs.size(), c, RS_VERIFY_SAMPLE, 0, &e));
                    std::unique_ptr<rs_engine, int (*)(rs_engine *)> hold(e, rs_engine_destroy);
                    e->stop_at_eos = false;
                    e->ledger_group = batch;
                    for (int k = 0; k < cycles_per_request; ++k) {
                        rs_step_info info{};
                        rs_abi::rethrow(rs_engine_step(e, &info));
                        tokens += info.emitted_tokens;
                    }
                    for (const auto &gl : e->group_ledgers) ledger.insert(ledger.end(), gl.begin(), gl.end());
                }
                double total = 0.0;  // ledger_time (costsim.cpp:13-27) over the whole pool, in order
                for (const auto &ev : ledger) {
                    const rs_role_timing &t = ev.role ? tm->target : tm->drafter;
                    total += t.latency_floor + t.unit_cost * (double)std::max(ev.batch_tokens, t.saturation_tokens);
                }
                time_per_token[(size_t)ib * nc + ic] = total / (double)tokens;
            }
        }
    });
}

// TabularARModel::random (model.cpp:102-111): scale * N(0, 1) logits drawn with
// std::normal_distribution from std::mt19937_64(seed) -- the host standard library's own
// algorithms (the same libstdc++ as the reference build), so the table is bit-identical.
int rs_tabular_random(rs_ctx *ctx, int32_t vocab, int32_t order, double temperature, double scale, uint64_t seed,
                      rs_model **out) {
    return guard([&] {
        need(out, "rs_tabular_random");
        if (vocab < 2 || order < 0) throw std::invalid_argument("TabularARModel: bad vocab/order");
        size_t rows = 1;
        for (int i = 0; i < order; ++i) rows *= (size_t)vocab;
        std::vector<double> logits(rows * (size_t)vocab);
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> gauss(0.0, 1.0);
        for (double &z : logits) z = scale * gauss(rng);
        rs_abi::rethrow(rs_tabular_create(ctx, vocab, order, temperature, logits.data(), 0, out));
    });
}

// make_skew_requests' EOS hazards (scenarios.cpp:175-189): 2.5 - 2.2 * Exp(1) draws from
// std::exponential_distribution over std::mt19937_64(seed).
int rs_skew_eos_biases(uint64_t seed, int32_t n, double *out) {
    return guard([&] {
        if (n > 0) need(out, "rs_skew_eos_biases");
        std::mt19937_64 rng(seed);
        std::exponential_distribution<double> tail(1.0);
        for (int i = 0; i < n; ++i) out[i] = 2.5 - 2.2 * tail(rng);
    });
}

// DecodeRng continuation (rng.hpp:33-47): the two mt19937_64 streams of a request as an opaque
// image -- exported after a step, imported into a fresh engine before its first step -- so a
// caller can run spec_step_tree cycle by cycle on one DecodeRng& like the reference.
int rs_engine_rng_export(const rs_engine *e, int32_t req, uint64_t *out, int64_t cap, int64_t *n) {
    return guard([&] {
        need(e, "rs_engine_rng_export");
        check_req(e, req);
        const int64_t words = (int64_t)(2 * sizeof(rs::MtStream) / 8);
        if (n) *n = words;
        if (!out || cap <= 0) return;
        if (cap < words) throw std::invalid_argument("rs_engine_rng_export: buffer too small");
        RS_CUDA(cudaStreamSynchronize(e->ctx->stream));
        RS_CUDA(cudaMemcpy(out, e->d_rng.p + 2 * (size_t)req, 2 * sizeof(rs::MtStream), cudaMemcpyDeviceToHost));
    });
}
int rs_engine_rng_import(rs_engine *e, int32_t req, const uint64_t *in, int64_t n) {
    return guard([&] {
        need(e, "rs_engine_rng_import");
        need(in, "rs_engine_rng_import: state");
        check_req(e, req);
        if (e->cycle > 0) throw std::runtime_error("rs_engine_rng_import: engine already stepped");
        if (n != (int64_t)(2 * sizeof(rs::MtStream) / 8)) throw std::invalid_argument("rs_engine_rng_import: bad state size");
        RS_CUDA(cudaStreamSynchronize(e->ctx->stream));
        RS_CUDA(cudaMemcpy(e->d_rng.p + 2 * (size_t)req, in, 2 * sizeof(rs::MtStream), cudaMemcpyHostToDevice));
    });
}

int rs_engine_set_capture(rs_engine *e, int32_t enable) {
    return guard([&] { need(e, "rs_engine_set_capture"); e->capture = enable != 0; });
}
int rs_engine_capture_count(const rs_engine *e, int64_t *rows, int32_t *vocab, int32_t *ext_width) {
    return guard([&] {
        need(e, "rs_engine_capture_count");
        *rows = (int64_t)e->cap_role.size();
        *vocab = e->V;
        if (ext_width) *ext_width = e->n_max;
    });
}
int rs_engine_capture_read(rs_engine *e, int64_t first, int64_t count, int32_t *role, int32_t *req, int32_t *ctx_len,
                           int32_t *ext, double *logits) {
    return guard([&] {
        need(e, "rs_engine_capture_read");
        const int64_t total = (int64_t)e->cap_role.size();
        if (first < 0 || count < 0 || first + count > total) throw std::invalid_argument("capture range");
        for (int64_t i = 0; i < count; ++i) {
            const int64_t k = first + i;
            if (role) role[i] = e->cap_role[k];
            if (req) req[i] = e->cap_req[k];
            if (ctx_len) ctx_len[i] = e->cap_ctx_len[k];
            if (ext) std::copy_n(&e->cap_ext[k * e->n_max], e->n_max, ext + i * e->n_max);
            if (logits) {
                if (!e->cap_logits.empty()) std::copy_n(&e->cap_logits[k * e->V], e->V, logits + i * e->V);
                else std::copy_n(&e->cap_f32[k * e->V], e->V, logits + i * e->V);
            }
        }
    });
}
int rs_engine_capture_read_f32(rs_engine *e, int64_t first, int64_t count, float *logits) {
    return guard([&] {
        need(e, "rs_engine_capture_read_f32");
        need(logits, "rs_engine_capture_read_f32: logits");
        const int64_t total = (int64_t)e->cap_role.size();
        if (first < 0 || count < 0 || first + count > total) throw std::invalid_argument("capture range");
        if (!e->cap_logits.empty()) throw std::invalid_argument("rs_engine_capture_read_f32: rows are fp64");
        std::copy_n(&e->cap_f32[first * e->V], count * e->V, logits);
    });
}

// ---- KD ---------------------------------------------------------------------------------------
double rs_kd_weight(double r, const double *br, int32_t n, rs_kd_policy p, int *status) {
    double w = 0.0;
    const int s = guard([&] { w = kd_weight(r, std::vector<double>(br, br + std::max(n, 0)), p); });
    if (status) *status = s;
    return w;
}

int rs_kd_update_tabular(rs_ctx *ctx, const rs_model *drafter, const rs_kd_sample *buf, int32_t n, rs_kd_policy policy,
                         uint64_t *sel_state, double cost, rs_model **new_drafter, rs_kd_result *out) {
    return guard([&] {
        need(ctx, "rs_kd_update_tabular");
        need(drafter, "rs_kd_update_tabular: drafter");
        need(sel_state, "rs_kd_update_tabular: selection rng");
        need(new_drafter, "rs_kd_update_tabular: out");
        if (drafter->kind != rs_model::Tabular) throw std::invalid_argument("rs_kd_update_tabular: tabular drafter required");
        kd_update_tabular(ctx, static_cast<const TabularModel *>(drafter), buf, n, policy, sel_state, cost, new_drafter, out);
    });
}

namespace {
std::vector<rs::KdSeq> kd_seqs(const rs_kd_sample *buf, const std::vector<int> &idx, const std::vector<double> &w) {
    std::vector<rs::KdSeq> seqs;
    for (size_t i = 0; i < idx.size(); ++i) {
        const rs_kd_sample &x = buf[idx[i]];
        if (x.response_len <= 0) continue;  // nothing to distil (learner.cpp:40-53 sums over steps)
        rs::KdSeq q;
        q.tokens.assign(x.prompt, x.prompt + x.prompt_len);
        q.tokens.insert(q.tokens.end(), x.response, x.response + x.response_len);
        q.prompt_len = x.prompt_len;
        q.eos_bias = x.eos_bias;
        q.weight = w[i];
        seqs.push_back(std::move(q));
    }
    return seqs;
}
const rs::TransformerModel *as_target(const rs_model *m) {
    if (!m || m->kind != rs_model::Transformer) throw std::invalid_argument("kd: transformer target required");
    return static_cast<const rs::TransformerModel *>(m);
}
const rs::DrafterModel *as_drafter(const rs_model *m) {
    if (!m || m->kind != rs_model::Drafter) throw std::invalid_argument("kd: EAGLE drafter required");
    return static_cast<const rs::DrafterModel *>(m);
}
}  // namespace

int rs_kd_grad_transformer(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_kd_sample *samples,
                           int32_t n, const double *weights, float *grad_dev, int32_t zero_grad, double *loss_out) {
    return guard([&] {
        need(ctx, "rs_kd_grad_transformer");
        need(grad_dev, "rs_kd_grad_transformer: grad");
        if (n > 0) need(samples, "rs_kd_grad_transformer: samples");
        std::vector<int> idx(std::max(n, 0));
        std::vector<double> w(std::max(n, 0), 1.0);
        for (int i = 0; i < n; ++i) {
            idx[i] = i;
            if (weights) w[i] = weights[i];
        }
        const double loss = rs::kd_grad_transformer(ctx, as_target(target), as_drafter(drafter),
                                                    kd_seqs(samples, idx, w), grad_dev, zero_grad != 0);
        if (loss_out) *loss_out = loss;
    });
}

int rs_drafter_grad_layout(const rs_model *drafter, const char *name, int64_t *offset, int64_t *count) {
    return guard([&] {
        need(drafter, "rs_drafter_grad_layout");
        if (drafter->kind != rs_model::Drafter) throw std::invalid_argument("rs_drafter_grad_layout: EAGLE drafter required");
        const auto *d = static_cast<const rs::DrafterModel *>(drafter);
        const rs::TfShape &s = d->s;
        const rs::DrafterGradLayout g = rs::drafter_grad_layout(s);
        const size_t q = s.qkv_dim(), HD = (size_t)s.H * s.hd;
        size_t off = 0, n = g.total;
        if (name) {
            const std::string nm(name);
            if (nm == "lm_w") { off = g.lm; n = (size_t)s.V * s.d; }
            else if (nm == "fc_w") { off = g.fc; n = (size_t)s.d * 3 * s.d; }
            else if (nm == "norm_emb") { off = g.norm_emb; n = s.d; }
            else if (nm == "norm_hid") { off = g.norm_hid; n = s.d; }
            else if (nm == "qkv_w") { off = g.qkv_w; n = q * 2 * s.d; }
            else if (nm == "qkv_b") { off = g.qkv_b; n = q; }
            else if (nm == "o_w") { off = g.o_w; n = (size_t)s.d * HD; }
            else if (nm == "ln2") { off = g.ln2; n = s.d; }
            else if (nm == "gu_w") { off = g.gu_w; n = (size_t)2 * s.dff * s.d; }
            else if (nm == "down_w") { off = g.down_w; n = (size_t)s.d * s.dff; }
            else if (nm == "final_norm") { off = g.final_norm; n = s.d; }
            else throw std::invalid_argument("rs_drafter_grad_layout: unknown tensor " + nm);
        }
        if (offset) *offset = (int64_t)off;
        if (count) *count = (int64_t)n;
    });
}

int rs_drafter_apply_grad(rs_ctx *ctx, const rs_model *drafter, const float *grad_dev, double scale, rs_model **out) {
    return guard([&] {
        need(ctx, "rs_drafter_apply_grad");
        need(out, "rs_drafter_apply_grad: out");
        *out = rs::drafter_apply_lm_grad(ctx, as_drafter(drafter), grad_dev, scale);
    });
}

int rs_engine_kd_grad(rs_engine *e, const rs_model *drafter, const int32_t *req, int32_t n, const double *weights,
                      float *grad_dev, int32_t zero_grad, double *loss_out) {
    return guard([&] {
        need(e, "rs_engine_kd_grad");
        need(grad_dev, "rs_engine_kd_grad: grad");
        std::unique_lock<std::mutex> lk(e->use_mu, std::try_to_lock);
        if (!lk) throw std::runtime_error("rs_engine_kd_grad: engine in use by another thread");
        if (n > 0) need(req, "rs_engine_kd_grad: requests");
        if (!e->pair) throw std::runtime_error("rs_engine_kd_grad: engine has no model pair");
        const auto *t = static_cast<const rs::TransformerModel *>(e->target);
        if (e->target->kind != rs_model::Transformer) throw std::invalid_argument("kd from the engine needs a transformer target");
        if (zero_grad)
            RS_CUDA(cudaMemsetAsync(grad_dev, 0, rs::drafter_grad_layout(t->s).total * sizeof(float), e->ctx->stream));
        std::vector<rs::KdRef> refs;
        for (int i = 0; i < n; ++i) {
            if (req[i] < 0 || req[i] >= e->n) throw std::invalid_argument("kd: request index out of range");
            if (e->len[req[i]] - e->prompt_len[req[i]] <= 0) continue;  // nothing generated: nothing to distil
            refs.push_back(rs::KdRef{req[i], weights ? weights[i] : 1.0, e->eos_bias[req[i]]});
        }
        const double loss = refs.empty() ? 0.0 : e->pair->kd_cached(refs, drafter, grad_dev);
        RS_CUDA(cudaStreamSynchronize(e->ctx->stream));
        rs::prof_collect();
        if (loss_out) *loss_out = loss;
    });
}

int rs_kd_update_transformer(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_kd_sample *buf,
                             int32_t n, rs_kd_policy policy, uint64_t *sel_state, double cost, rs_model **new_drafter,
                             rs_kd_result *out) {
    return guard([&] {
        need(ctx, "rs_kd_update_transformer");
        need(sel_state, "rs_kd_update_transformer: selection rng");
        need(new_drafter, "rs_kd_update_transformer: out");
        const auto *t = as_target(target);
        const auto *d = as_drafter(drafter);
        if (policy.mode == 2) throw std::logic_error("kd_update: frozen drafter takes no updates");
        if (policy.interval < 1) throw std::invalid_argument("kd_update: interval must be >= 1");
        rs_kd_result res{};
        if (n <= 0) {  // empty buffer: no-op (learner.cpp:103-105) -- an unchanged snapshot
            *new_drafter = rs::drafter_apply_lm_grad(ctx, d, nullptr, 0.0);
            static_cast<rs::DrafterModel *>(*new_drafter)->version = d->version;
            if (out) *out = res;
            return;
        }
        const std::vector<int> idx = rs::kd_select(n, policy.interval, sel_state);
        std::vector<double> br(idx.size()), w(idx.size());
        for (size_t i = 0; i < idx.size(); ++i) br[i] = buf[idx[i]].reward;
        double wsum = 0, wmin = 0, wmax = 0;
        size_t distilled = 0;
        for (size_t i = 0; i < idx.size(); ++i) {
            w[i] = rs::kd_weight(buf[idx[i]].reward, br, policy);
            wsum += w[i];
            wmin = i == 0 ? w[i] : std::min(wmin, w[i]);
            wmax = i == 0 ? w[i] : std::max(wmax, w[i]);
            distilled += static_cast<size_t>(std::max(0, buf[idx[i]].response_len));
        }
        rs::DBuf<float> grad(rs::drafter_grad_layout(t->s).total);
        const double loss = rs::kd_grad_transformer(ctx, t, d, kd_seqs(buf, idx, w), grad.p, true);
        *new_drafter = rs::drafter_apply_lm_grad(ctx, d, grad.p, -policy.lr);
        res.updated = 1;
        res.samples_used = static_cast<int>(idx.size());
        res.loss = loss;
        res.weight_mean = wsum / static_cast<double>(idx.size());
        res.weight_min = wmin;
        res.weight_max = wmax;
        res.sim_time = cost * static_cast<double>(distilled);
        if (out) *out = res;
    });
}

int rs_model_tensor(const rs_model *m, const char *name, int32_t layer, void **ptr, int64_t *bytes) {
    return guard([&] {
        need(m, "rs_model_tensor");
        need(name, "rs_model_tensor: name");
        const std::string nm(name);
        void *p = nullptr;
        size_t b = 0;
        auto layer_tensor = [&](const LayerW &w, const TfShape &s, int d_in) {
            const size_t q = s.qkv_dim();
            if (nm == "qkv_w") { p = w.qkv_w; b = q * d_in * 2; }
            else if (nm == "qkv_b") { p = w.qkv_b; b = q * 2; }
            else if (nm == "o_w") { p = w.o_w; b = (size_t)s.d * s.H * s.hd * 2; }
            else if (nm == "gu_w") { p = w.gu_w; b = 2 * (size_t)s.dff * s.d * 2; }
            else if (nm == "down_w") { p = w.down_w; b = (size_t)s.d * s.dff * 2; }
            else if (nm == "ln1") { p = w.ln1; b = (size_t)d_in * 4; }
            else if (nm == "ln2") { p = w.ln2; b = (size_t)s.d * 4; }
        };
        if (m->kind == rs_model::Transformer) {
            const auto *t = static_cast<const TransformerModel *>(m);
            const TfShape &s = t->s;
            if (nm == "emb") { p = t->emb; b = (size_t)s.V * s.d * 2; }
            else if (nm == "final_norm") { p = t->final_norm; b = (size_t)s.d * 4; }
            else if (nm == "rope") { p = t->rope; b = (size_t)s.max_ctx * s.hd * 4; }
            else {
                if (layer < 0 || layer >= s.L) throw std::invalid_argument("rs_model_tensor: layer out of range");
                layer_tensor(t->layers[layer], s, s.d);
            }
        } else if (m->kind == rs_model::Drafter) {
            const auto *dm = static_cast<const DrafterModel *>(m);
            const TfShape &s = dm->s;
            if (nm == "fc_w") { p = dm->fc_w; b = (size_t)s.d * 3 * s.d * 2; }
            else if (nm == "norm_emb") { p = dm->norm_emb; b = (size_t)s.d * 4; }
            else if (nm == "norm_hid") { p = dm->norm_hid; b = (size_t)s.d * 4; }
            else if (nm == "final_norm") { p = dm->final_norm; b = (size_t)s.d * 4; }
            else if (nm == "lm_w") { p = dm->lm_w; b = (size_t)s.V * s.d * 2; }
            else layer_tensor(dm->layer, s, 2 * s.d);
        } else {
            throw std::invalid_argument("rs_model_tensor: tabular models have no named tensors");
        }
        if (!p) throw std::invalid_argument("rs_model_tensor: unknown tensor " + nm);
        *ptr = p;
        *bytes = (int64_t)b;
    });
}

namespace {
// A checkpoint tensor (Hugging Face Qwen2 / EAGLE-3 naming) as a strided view of the arena:
// `rows` rows of `cols` elements, row r at dev + r * row_stride (elements of the device dtype).
// q/k/v_proj are row slices of the fused QKV matrix; gate/up_proj are the even / odd rows of
// the pairwise-interleaved gate/up matrix.
struct CkptView {
    char *dev = nullptr;
    bool f32 = false;  // device dtype: fp32 (norm gains) or bf16
    int64_t rows = 0, cols = 0, row_stride = 0;
};

CkptView ckpt_view(const rs_model *m, const std::string &nm, int layer) {
    CkptView v;
    auto bf = [&](void *p, int64_t rows, int64_t cols, int64_t stride) {
        v.dev = static_cast<char *>(p);
        v.rows = rows;
        v.cols = cols;
        v.row_stride = stride;
    };
    auto gain = [&](float *p, int64_t n) {
        bf(p, 1, n, n);
        v.f32 = true;
    };
    auto layer_view = [&](const LayerW &w, const TfShape &s, int d_in) -> bool {
        const int64_t hq = (int64_t)s.H * s.hd, hk = (int64_t)s.KV * s.hd;
        if (nm == "q_proj.weight") bf(w.qkv_w, hq, d_in, d_in);
        else if (nm == "k_proj.weight") bf(w.qkv_w + hq * d_in, hk, d_in, d_in);
        else if (nm == "v_proj.weight") bf(w.qkv_w + (hq + hk) * d_in, hk, d_in, d_in);
        else if (nm == "q_proj.bias") bf(w.qkv_b, 1, hq, hq);
        else if (nm == "k_proj.bias") bf(w.qkv_b + hq, 1, hk, hk);
        else if (nm == "v_proj.bias") bf(w.qkv_b + hq + hk, 1, hk, hk);
        else if (nm == "o_proj.weight") bf(w.o_w, s.d, hq, hq);
        else if (nm == "gate_proj.weight") bf(w.gu_w, s.dff, s.d, 2 * (int64_t)s.d);
        else if (nm == "up_proj.weight") bf(w.gu_w + s.d, s.dff, s.d, 2 * (int64_t)s.d);
        else if (nm == "down_proj.weight") bf(w.down_w, s.d, s.dff, s.dff);
        else if (nm == "post_attention_layernorm.weight") gain(w.ln2, s.d);
        else return false;
        return true;
    };
    if (m->kind == rs_model::Transformer) {
        const auto *t = static_cast<const TransformerModel *>(m);
        const TfShape &s = t->s;
        if (nm == "embed_tokens.weight") bf(t->emb, s.V, s.d, s.d);
        else if (nm == "norm.weight") gain(t->final_norm, s.d);
        else {
            if (layer < 0 || layer >= s.L) throw std::invalid_argument("rs_model_load_tensor: layer out of range");
            const LayerW &w = t->layers[layer];
            if (nm == "input_layernorm.weight") gain(w.ln1, s.d);
            else if (!layer_view(w, s, s.d)) throw std::invalid_argument("rs_model_load_tensor: unknown tensor " + nm);
        }
    } else if (m->kind == rs_model::Drafter) {
        const auto *dm = static_cast<const DrafterModel *>(m);
        const TfShape &s = dm->s;
        if (nm == "fc.weight") bf(dm->fc_w, s.d, 3 * (int64_t)s.d, 3 * (int64_t)s.d);
        else if (nm == "input_layernorm.weight") gain(dm->norm_emb, s.d);  // EAGLE-3: norm of emb(x)
        else if (nm == "hidden_norm.weight") gain(dm->norm_hid, s.d);      // EAGLE-3: norm of f
        else if (nm == "norm.weight") gain(dm->final_norm, s.d);
        else if (nm == "lm_head.weight") bf(dm->lm_w, s.V, s.d, s.d);
        else if (!layer_view(dm->layer, s, 2 * s.d)) throw std::invalid_argument("rs_model_load_tensor: unknown tensor " + nm);
    } else {
        throw std::invalid_argument("rs_model_load_tensor: tabular models have no named tensors");
    }
    return v;
}

uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // quiet NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
float bf16_to_f32(uint16_t h) {
    const uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// host rows (dtype 0 = bf16 bits, 1 = fp32; row-major, `cols` per row) <-> the strided view
void ckpt_copy(rs_ctx *ctx, const CkptView &v, void *host, int dtype, int64_t n, bool load) {
    if (dtype != RS_DTYPE_BF16 && dtype != RS_DTYPE_F32) throw std::invalid_argument("rs_model_load_tensor: dtype must be bf16 or f32");
    if (n != v.rows * v.cols)
        throw std::invalid_argument("rs_model_load_tensor: element count " + std::to_string(n) + " != " +
                                    std::to_string(v.rows) + " x " + std::to_string(v.cols));
    const size_t des = v.f32 ? 4 : 2;
    const bool same = (dtype == RS_DTYPE_F32) == v.f32;
    std::vector<char> conv;
    char *h = static_cast<char *>(host);
    if (!same) conv.resize((size_t)n * des);
    if (load && !same) {
        for (int64_t i = 0; i < n; ++i) {
            if (v.f32) {
                const float f = bf16_to_f32(static_cast<const uint16_t *>(host)[i]);
                std::memcpy(conv.data() + 4 * i, &f, 4);
            } else {
                const uint16_t b = f32_to_bf16_rne(static_cast<const float *>(host)[i]);
                std::memcpy(conv.data() + 2 * i, &b, 2);
            }
        }
    }
    char *src = same ? h : conv.data();
    const size_t row_bytes = (size_t)v.cols * des, pitch = (size_t)v.row_stride * des;
    if (load)
        RS_CUDA(cudaMemcpy2DAsync(v.dev, pitch, src, row_bytes, row_bytes, (size_t)v.rows, cudaMemcpyHostToDevice, ctx->stream));
    else
        RS_CUDA(cudaMemcpy2DAsync(src, row_bytes, v.dev, pitch, row_bytes, (size_t)v.rows, cudaMemcpyDeviceToHost, ctx->stream));
    RS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!load && !same) {
        for (int64_t i = 0; i < n; ++i) {
            if (v.f32) {
                float f;
                std::memcpy(&f, conv.data() + 4 * i, 4);
                static_cast<uint16_t *>(host)[i] = f32_to_bf16_rne(f);
            } else {
                uint16_t b;
                std::memcpy(&b, conv.data() + 2 * i, 2);
                static_cast<float *>(host)[i] = bf16_to_f32(b);
            }
        }
    }
}
}  // namespace

int rs_model_tensor_shape(const rs_model *m, const char *name, int32_t layer, int64_t *rows, int64_t *cols) {
    return guard([&] {
        need(m, "rs_model_tensor_shape");
        need(name, "rs_model_tensor_shape: name");
        const CkptView v = ckpt_view(m, name, layer);
        if (rows) *rows = v.rows;
        if (cols) *cols = v.cols;
    });
}

int rs_model_load_tensor(rs_ctx *ctx, rs_model *m, const char *name, int32_t layer, const void *host, int32_t dtype,
                         int64_t n) {
    return guard([&] {
        need(ctx, "rs_model_load_tensor");
        need(m, "rs_model_load_tensor");
        need(name, "rs_model_load_tensor: name");
        need(host, "rs_model_load_tensor: host buffer");
        ckpt_copy(ctx, ckpt_view(m, name, layer), const_cast<void *>(host), dtype, n, true);
        // engines key their drafter-cache invalidation on the snapshot id: new weights = new snapshot
        m->uid = rs_model::next_uid();
    });
}

int rs_model_store_tensor(rs_ctx *ctx, const rs_model *m, const char *name, int32_t layer, void *host, int32_t dtype,
                          int64_t n) {
    return guard([&] {
        need(ctx, "rs_model_store_tensor");
        need(m, "rs_model_store_tensor");
        need(name, "rs_model_store_tensor: name");
        need(host, "rs_model_store_tensor: host buffer");
        ckpt_copy(ctx, ckpt_view(m, name, layer), host, dtype, n, false);
    });
}

void rs_prof_enable(int32_t on) { prof_enable(on != 0); }
int rs_set_tuning(const char *key, int64_t value) {
    return guard([&] {
        const std::string k = key ? key : "";
        if (k == "accept_cluster") {
            if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
                throw std::invalid_argument("accept_cluster must be 0, 1, 2, 4 or 8");
            rs::tuning().accept_cluster = static_cast<int>(value);
        } else if (k == "fused_stats") {
            rs::tuning().fused_stats = value != 0 ? 1 : -1;
        } else if (k == "gemm2") {
            rs::tuning().gemm2 = static_cast<int>(value);
        } else if (k == "pdl") {
            rs::tuning().pdl = static_cast<int>(value);
        } else if (k == "lazy_lm") {
            rs::tuning().lazy_lm = static_cast<int>(value);
        } else if (k == "epi3") {
            rs::tuning().epi3 = static_cast<int>(value);
        } else if (k == "kd_rows") {
            if (value < 0) throw std::invalid_argument("kd_rows must be >= 0");
            rs::tuning().kd_rows = static_cast<int>(value);
        } else {
            throw std::invalid_argument("unknown tuning key: " + k);
        }
    });
}
void rs_prof_reset(void) { prof_reset(); }
int rs_prof_json(char *buf, int64_t cap, int64_t *len) {
    return guard([&] {
        const std::string s = prof_json();
        if (len) *len = (int64_t)s.size();
        if (buf && cap > 0) {
            const size_t k = std::min<size_t>(s.size(), (size_t)cap - 1);
            std::memcpy(buf, s.data(), k);
            buf[k] = 0;
        }
    });
}

int rs_memcpy_d2d(rs_ctx *ctx, void *dst, const void *src, int64_t bytes) {
    return guard([&] {
        need(ctx, "rs_memcpy_d2d");
        RS_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, ctx->stream));
        RS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int rs_model_params(const rs_model *m, int64_t *out) {
    return guard([&] {
        need(m, "rs_model_params");
        if (m->kind == rs_model::Transformer) *out = (int64_t) static_cast<const TransformerModel *>(m)->n_params;
        else if (m->kind == rs_model::Drafter) *out = (int64_t) static_cast<const DrafterModel *>(m)->n_params;
        else *out = (int64_t) static_cast<const TabularModel *>(m)->host.size();
    });
}

int rs_gemm_bf16(rs_ctx *ctx, const void *A, const void *B, void *Cp, const void *bias, int32_t M, int32_t N, int32_t K,
                 int32_t epilogue, float scale, int32_t block_n, int32_t splits) {
    return guard([&] {
        need(ctx, "rs_gemm_bf16");
        GemmArgs g;
        g.A = A;
        g.B = B;
        g.M = M;
        g.N = N;
        g.K = K;
        g.lda = K;
        g.ldb = K;
        g.block_n = block_n;
        g.splits = std::max(1, (int)splits);
        g.epi.kind = epilogue;
        g.epi.out = Cp;
        g.epi.ldo = epilogue == kEpiSwiGLU || epilogue == kEpiSwiGLU2 ? N / 2 : N;
        g.epi.bias = bias;
        g.epi.scale = scale;
        gemm_bf16(g, ctx->stream);
    });
}

int rs_lm_head_bf16(rs_ctx *ctx, const void *A, const void *B, float *Cp, double *stats, int32_t M, int32_t N,
                    int32_t K, float scale, double tau) {
    return guard([&] {
        need(ctx, "rs_lm_head_bf16");
        GemmArgs g;
        g.A = A;
        g.B = B;
        g.M = M;
        g.N = N;
        g.K = K;
        g.lda = K;
        g.ldb = K;
        g.epi.kind = kEpiF32;
        g.epi.out = Cp;
        g.epi.ldo = N;
        g.epi.scale = scale;
        g.epi.stats = stats;
        g.epi.tau = tau;
        gemm_bf16(g, ctx->stream);
    });
}

int rs_row_stats(rs_ctx *ctx, const float *rows, int32_t nrows, int32_t V, double tau, double *stats) {
    return guard([&] {
        need(ctx, "rs_row_stats");
        row_stats(rows, nullptr, nrows, V, tau, stats, ctx->stream);
    });
}

int rs_transformer_create(rs_ctx *ctx, const rs_transformer_shape *sh, uint64_t seed, rs_model **out) {
    return guard([&] {
        need(ctx, "rs_transformer_create");
        need(sh, "rs_transformer_create: shape");
        need(out, "rs_transformer_create");
        *out = create_transformer(ctx, *sh, seed);
    });
}

int rs_drafter_create(rs_ctx *ctx, const rs_model *target, uint64_t seed, int32_t version, rs_model **out) {
    return guard([&] {
        need(ctx, "rs_drafter_create");
        need(target, "rs_drafter_create: target");
        need(out, "rs_drafter_create");
        *out = create_drafter(ctx, target, seed, version);
    });
}

int rs_kd_select(int32_t n, int32_t interval, uint64_t *state, int32_t *out_idx, int32_t *take) {
    return guard([&] {
        need(state, "rs_kd_select: selection rng");
        const std::vector<int> idx = kd_select(n, interval, state);
        if (take) *take = (int32_t)idx.size();
        if (out_idx) std::copy(idx.begin(), idx.end(), out_idx);
    });
}

int rs_kd_grad_tabular(rs_ctx *ctx, const rs_model *drafter, const rs_kd_sample *samples, int32_t n,
                       const double *weights, double *grad_out, double *loss_out) {
    return guard([&] {
        need(ctx, "rs_kd_grad_tabular");
        need(drafter, "rs_kd_grad_tabular: drafter");
        if (drafter->kind != rs_model::Tabular) throw std::invalid_argument("rs_kd_grad_tabular: tabular drafter required");
        const auto *t = static_cast<const TabularModel *>(drafter);
        std::vector<const rs_kd_sample *> sel;
        std::vector<double> w;
        for (int i = 0; i < n; ++i) {
            sel.push_back(&samples[i]);
            w.push_back(weights[i]);
        }
        DBuf<double> g(t->host.size());
        const double loss = kd_core(ctx, t, sel, w, g.p, true, 1.0);
        if (grad_out) RS_CUDA(cudaMemcpy(grad_out, g.p, g.bytes(), cudaMemcpyDeviceToHost));
        if (loss_out) *loss_out = loss;
    });
}

int rs_tabular_apply_delta(rs_ctx *ctx, const rs_model *m, const double *grad, double scale, rs_model **out) {
    return guard([&] {
        need(ctx, "rs_tabular_apply_delta");
        need(m, "rs_tabular_apply_delta: model");
        need(out, "rs_tabular_apply_delta: out");
        if (m->kind != rs_model::Tabular) throw std::invalid_argument("rs_tabular_apply_delta: tabular model required");
        const auto *t = static_cast<const TabularModel *>(m);
        // with_logits_delta (model.cpp:161-170): z[i] += delta[i], delta = grad * scale
        std::vector<double> z = t->host;
        for (size_t i = 0; i < z.size(); ++i) z[i] += grad[i] * scale;
        rs_model *nm = nullptr;
        const int rc = rs_tabular_create(ctx, t->vocab, t->order, t->temperature, z.data(), t->version + 1, &nm);
        if (rc != RS_OK) throw std::runtime_error(rs_last_error());
        *out = nm;
    });
}

int rs_mt19937_64_seed(uint64_t seed, uint64_t *state) {
    return guard([&] {
        need(state, "rs_mt19937_64_seed");
        HostMt m;
        m.seed(seed);
        std::copy(m.mt, m.mt + kMtN, state);
        state[kMtN] = (uint64_t)m.idx;
    });
}

}  // extern "C"

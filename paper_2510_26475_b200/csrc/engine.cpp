// engine.cpp -- host orchestration of the B200 rollout engine.
// ProfileTable follows server.cpp:21-145; rs_engine::step follows BatchEngine::step
// (server.cpp:266-349) with the per-request spec_step_tree calls replaced by batched device
// launches (drafting by depth, one verify forward, one fused acceptance per round).
#include <cstdlib>
#include "engine.h"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "common.cuh"
#include "prof.h"

namespace rs {

std::string cfg_key(const rs_sdconfig &c) {
    if (!c.enabled) return "off";
    return "s" + std::to_string(c.rounds) + "_t" + std::to_string(c.branching) + "_n" + std::to_string(c.draft_len);
}

// Defaults can be overridden for A/B measurements with RS_TUNE="key=value,key=value".
Tuning &tuning() {
    static Tuning t = [] {
        Tuning x;
        if (const char *env = std::getenv("RS_TUNE")) {
            std::string s(env);
            size_t p = 0;
            while (p < s.size()) {
                size_t e = s.find(',', p);
                if (e == std::string::npos) e = s.size();
                const std::string kv = s.substr(p, e - p);
                const size_t eq = kv.find('=');
                if (eq != std::string::npos) {
                    const std::string k = kv.substr(0, eq);
                    const int v = std::atoi(kv.c_str() + eq + 1);
                    if (k == "accept_cluster") x.accept_cluster = v;
                    else if (k == "fused_stats") x.fused_stats = v;
                    else if (k == "accept_minb") x.accept_minb = v;
                    else if (k == "lazy_lm") x.lazy_lm = v;
                    else if (k == "epi3") x.epi3 = v;
                    else if (k == "attn_trace") x.attn_trace = v;
                    else if (k == "attn_skip") x.attn_skip = v;
                    else if (k == "pdl") x.pdl = v;
                    else if (k == "gemm2") x.gemm2 = v;
                    else if (k == "gemm_trace") x.gemm_trace = v;
                    else if (k == "kd_rows") x.kd_rows = v;
                }
                p = e + 1;
            }
        }
        return x;
    }();
    return t;
}

const char *dev_err_message(int code) {
    switch (code) {
        case kErrAcceptQ: return "accept_prob: drafted token must have q > 0";
        case kErrAcceptRange: return "accept_prob: probabilities out of range";
        case kErrResidual: return "residual_dist: degenerate residual (p == q)";
        case kErrAllZero: return "sample_from: all-zero distribution";
        case kErrRowIndex: return "row_index: token out of vocabulary";
        case kErrCapacity: return "BatchEngine: context exceeds engine capacity";
        default: return "unknown device error";
    }
}

// ---- ProfileTable ---------------------------------------------------------------------
ProfileTable::ProfileTable(std::vector<int> buckets) : buckets_(std::move(buckets)) {
    if (buckets_.empty()) throw std::invalid_argument("ProfileTable: no buckets");
    std::sort(buckets_.begin(), buckets_.end());
}

void ProfileTable::set_entry(int bucket, const rs_sdconfig &cfg, double tpt) { entries_[bucket].emplace_back(cfg, tpt); }

void ProfileTable::finalize() {
    best_.clear();
    for (int b : buckets_) {
        auto it = entries_.find(b);
        if (it == entries_.end()) throw std::invalid_argument("ProfileTable: bucket has no entries");
        bool has_base = false;
        const rs_sdconfig *best = nullptr;
        double best_t = 0.0;
        for (const auto &[cfg, t] : it->second) {
            if (!cfg.enabled) has_base = true;
            bool better = false;
            if (best == nullptr || t < best_t) {
                better = true;
            } else if (t == best_t) {  // ties: fewer drafted tokens, then non-spec
                const int cur = cfg.enabled ? cfg_drafted(cfg) : 0;
                const int old = best->enabled ? cfg_drafted(*best) : 0;
                better = cur < old || (cur == old && !cfg.enabled && best->enabled);
            }
            if (better) {
                best = &cfg;
                best_t = t;
            }
        }
        if (!has_base) throw std::invalid_argument("ProfileTable: bucket missing non-spec baseline");
        best_[b] = *best;
    }
}

int ProfileTable::bucket_for(int active_batch) const {
    if (active_batch < 1) throw std::invalid_argument("bucket_for: batch must be >= 1");
    for (int b : buckets_)
        if (active_batch <= b) return b;
    return buckets_.back();
}

rs_sdconfig ProfileTable::best_for_bucket(int bucket) const {
    auto it = best_.find(bucket);
    if (it == best_.end()) throw std::invalid_argument("ProfileTable: table not finalized or unknown bucket");
    return it->second;
}

double ProfileTable::entry(int bucket, const rs_sdconfig &cfg) const {
    auto it = entries_.find(bucket);
    if (it == entries_.end()) throw std::invalid_argument("ProfileTable: unknown bucket");
    for (const auto &[c, t] : it->second)
        if (cfg_eq(c, cfg)) return t;
    throw std::invalid_argument("ProfileTable: no entry for config " + cfg_key(cfg));
}

std::string ProfileTable::to_csv() const {
    std::string out = "batch,s,t,n,time_per_token,speedup\n";
    char buf[128];
    for (int b : buckets_) {
        const double base = entry(b, rs_sdconfig{1, 1, 1, 0});
        for (const auto &[cfg, t] : entries_.at(b)) {
            std::snprintf(buf, sizeof(buf), "%d,%d,%d,%d,%.12g,%.12g\n", b, cfg.enabled ? cfg.rounds : 0,
                          cfg.enabled ? cfg.branching : 0, cfg.enabled ? cfg.draft_len : 0, t, base / t);
            out += buf;
        }
    }
    return out;
}

std::vector<rs_sdconfig> ProfileTable::all_configs() const {
    std::vector<rs_sdconfig> v;
    for (const auto &[b, es] : entries_)
        for (const auto &e : es) v.push_back(e.first);
    return v;
}

// ---- tabular model pair -----------------------------------------------------------------
namespace {
struct TabularPair : ModelPair {
    const TabularModel *target;
    const TabularModel *drafter;
    TabularPair(const TabularModel *t, const TabularModel *d) : target(t), drafter(d) {}
    RowType row_type() const override { return RowType::F64; }
    void draft_rows(const SdDev &d, int depth, cudaStream_t st) override { tab_draft_rows(d, drafter->dev(), depth, st); }
    void verify_rows(const SdDev &d, bool naive, cudaStream_t st) override { tab_verify_rows(d, target->dev(), naive, st); }
    void set_drafter(const rs_model *m) override {
        if (m && m->kind != rs_model::Tabular) throw std::invalid_argument("tabular target needs a tabular drafter");
        drafter = static_cast<const TabularModel *>(m);
    }
};
}  // namespace

std::unique_ptr<ModelPair> make_tabular_pair(const TabularModel *target, const TabularModel *drafter) {
    return std::make_unique<TabularPair>(target, drafter);
}

}  // namespace rs

using namespace rs;

rs_engine::~rs_engine() {
    if (h_summary) cudaFreeHost(h_summary);
    if (h_newtok) cudaFreeHost(h_newtok);
    if (h_active) cudaFreeHost(h_active);
    if (h_misc) cudaFreeHost(h_misc);
}

SdDev rs_engine::dev(const rs_sdconfig &cfg, int nact) {
    SdDev d{};
    d.tok = d_tok.p;
    d.tok_cap = tok_cap;
    d.len = d_len.p;
    d.prompt_len = d_plen.p;
    d.max_len = d_maxlen.p;
    d.eos_bias = d_bias.p;
    d.rng = d_rng.p;
    d.done = d_done.p;
    d.st_tok = d_st_tok.p;
    d.st_logp = d_st_logp.p;
    d.st_drafted = d_st_drafted.p;
    d.st_logq = d_st_logq.p;
    d.st_full = record_full ? d_st_full.p : nullptr;
    d.steps_cap = steps_cap;
    d.active = d_active.p;
    d.nact = nact;
    int32_t *c = d_cyc.p;
    d.n_eff = c + 0 * n;
    d.d_used = c + 1 * n;
    d.a_used = c + 2 * n;
    d.cont = c + 3 * n;
    d.ended = c + 4 * n;
    d.accept_len = c + 5 * n;
    d.drafted = c + 6 * n;
    d.emitted = c + 7 * n;
    d.n_rounds = c + 8 * n;
    d.rsel = c + 9 * n;
    d.racc = c + 10 * n;
    d.stg = c + 11 * n;
    d.round_cost = d_round_cost.p;
    const size_t ch = (size_t)n * t_max;
    d.chain_tok = d_chain.p;
    d.chain_len = d_chain.p + ch * n_max;
    d.chain_stop = d.chain_len + ch;
    d.chain_off = d.chain_stop + ch;
    d.t_max = t_max;
    d.n_max = n_max;
    d.s = cfg.enabled ? cfg.rounds : 1;
    d.t = cfg.enabled ? cfg.branching : 1;
    d.n = cfg.enabled ? cfg.draft_len : 1;
    d.V = V;
    d.eos = stop_at_eos ? V - 1 : -1;  // -1 matches no token: spec_step_tree(stop_at_eos = false)
    d.tau_p = target->temperature;
    d.tau_q = pending_drafter ? pending_drafter->temperature : target->temperature;
    d.slots = cfg.enabled ? 1 + d.t * d.n : 1;  // rows per active sequence in P / Q
    d.P = d_P.p;
    d.Q = d_Q.p;
    d.Pst = d_Pst.n ? d_Pst.p : nullptr;
    d.Qst = d_Qst.n ? d_Qst.p : nullptr;
    d.ntiles = (V + 255) / 256;
    d.lazy_pst = d.Pst ? 1 : 0;
    d.pq_cache = d_pq.n ? d_pq.p : nullptr;  // target rows: stats on demand inside the acceptance kernel
    d.verify_mode = verify_mode;
    d.record_full = record_full ? 1 : 0;
    d.err = d_err.p;
    d.flag = d_flag.p;
    d.summary = d_summary.p;
    d.newtok = d_newtok.n ? d_newtok.p : nullptr;
    d.newtok_cap = newtok_cap;
    return d;
}

// which (verify rows): 0 every row, 1 the roots only, 2 the selected chains only (lazy verify LM
// head: the chains' rows exist after the branch point picked them, the others are never computed)
void rs_engine::capture_rows(const SdDev &d, bool verify, int depth, int which) {
    // Debug path: copies the rows this launch produced plus their contexts to the host.
    RS_CUDA(cudaStreamSynchronize(ctx->stream));
    const int nact = d.nact;
    std::vector<int32_t> lens(n), neff(n), clen((size_t)n * t_max), ctok((size_t)n * t_max * n_max);
    RS_CUDA(cudaMemcpy(lens.data(), d.len, n * 4, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(neff.data(), d.n_eff, n * 4, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(clen.data(), d.chain_len, clen.size() * 4, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(ctok.data(), d.chain_tok, ctok.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<int32_t> stg((size_t)n * 6, -1);
    if (which == 2) RS_CUDA(cudaMemcpy(stg.data(), d.stg, stg.size() * 4, cudaMemcpyDeviceToHost));
    const size_t es = pair->row_type() == RowType::F64 ? 8 : 4;
    std::vector<char> row(V * es);
    auto grab = [&](const void *base, int a, int slot, int role, int r, const int *ext, int e) {
        const char *src = static_cast<const char *>(base) + ((size_t)a * d.slots + slot) * V * es;
        RS_CUDA(cudaMemcpy(row.data(), src, V * es, cudaMemcpyDeviceToHost));
        cap_role.push_back(role);
        cap_req.push_back(r);
        cap_ctx_len.push_back(lens[r]);
        for (int k = 0; k < n_max; ++k) cap_ext.push_back(k < e ? ext[k] : -1);
        if (es == 8) {
            const double *x = reinterpret_cast<const double *>(row.data());
            cap_logits.insert(cap_logits.end(), x, x + V);
        } else {
            const float *x = reinterpret_cast<const float *>(row.data());
            cap_f32.insert(cap_f32.end(), x, x + V);
        }
    };
    const bool naive = !mode.enabled;
    for (int a = 0; a < nact; ++a) {
        const int r = active[a];
        const int ne = naive ? 0 : neff[r];
        if (!naive && ne < 0) continue;
        if (verify) {
            if (which != 2) grab(d.P, a, 0, 1, r, nullptr, 0);
            if (naive || which == 1) continue;
            for (int i = 0; i < d.t; ++i) {
                if (which == 2 && stg[(size_t)r * 6] != i) continue;
                const int *ch = &ctok[((size_t)r * t_max + i) * n_max];
                for (int j = 0; j < clen[(size_t)r * t_max + i]; ++j) grab(d.P, a, 1 + i * d.n + j, 1, r, ch, j + 1);
            }
        } else {
            if (depth >= ne) continue;
            if (depth == 0) {
                grab(d.Q, a, 0, 0, r, nullptr, 0);
                continue;
            }
            for (int i = 0; i < d.t; ++i) {
                const int *ch = &ctok[((size_t)r * t_max + i) * n_max];
                if (clen[(size_t)r * t_max + i] == depth + 1) grab(d.Q, a, 1 + i * d.n + depth, 0, r, ch, depth);
            }
        }
    }
}

// One round's target verification + acceptance. Transformer pairs with a lazy verify LM head
// (TransformerPair::lazy_lm_head) compute the root rows' logits, run the branch point (acceptance
// stage 1), then the selected chains' logits and the chain verification (stage 2): the other
// chains' rows -- most of the tree -- never go through the LM head.
void rs_engine::verify_accept(const SdDev &d, int round, RowType rt, cudaStream_t st) {
    prof_set_scope("verify");
    pair->verify_rows(d, false, st);
    if (!pair->lazy_lm_head(d)) {
        if (capture) capture_rows(d, true, 0, 0);
        prof_set_scope("accept");
        sd_accept(d, round, false, rt, st);
        return;
    }
    if (capture) capture_rows(d, true, 0, 1);
    prof_set_scope("accept");
    sd_accept(d, round, false, rt, st, 1);
    prof_set_scope("verify");
    pair->verify_rows_selected(d, st);
    if (capture) capture_rows(d, true, 0, 2);
    prof_set_scope("accept");
    sd_accept(d, round, false, rt, st, 2);
}

// BatchEngine::step (server.cpp:266-349)
void rs_engine::step(rs_step_info *info) {
    active.clear();
    for (int r = 0; r < n; ++r)
        if (!done[r]) active.push_back(r);
    if (active.empty()) throw std::runtime_error("BatchEngine: empty batch");
    const int batch = static_cast<int>(active.size());
    active_trace.push_back(batch);

    const rs_sdconfig desired = table ? table->solve(batch) : mode;
    bool enabling = false;
    if (mode_init && !cfg_eq(desired, mode)) {
        if (!mode.enabled && desired.enabled) {
            // non-spec -> spec: drafter prefill over all active contexts (server.cpp:280-290)
            int ctx_tokens = 0;
            for (int r : active) ctx_tokens += len[r];
            ledger.push_back({0, ctx_tokens, ctx_tokens});
            ++prefill_events;
            enabling = true;
        }
        switches.push_back({cycle, batch, mode, desired});
    }
    mode = desired;
    if (!mode_init && mode.enabled) enabling = true;
    mode_init = true;

    const rs_model *drafter = nullptr;
    if (mode.enabled) {
        drafter = pending_drafter;
        if (!drafter) throw std::runtime_error("BatchEngine: spec mode requires a drafter snapshot");
        if (drafter->vocab != V) throw std::invalid_argument("BatchEngine: drafter vocabulary differs from target");
        pair->set_drafter(drafter);
    }
    drafter_versions.push_back(drafter ? drafter->version : -1);

    cudaStream_t st = ctx->stream;
    pair->begin_step();
    reset_copy_bytes();
    for (int a = 0; a < batch; ++a) h_active[a] = active[a];
    RS_CUDA(cudaMemcpyAsync(d_active.p, h_active, batch * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    note_copy(true, batch * sizeof(int32_t));
    RS_CUDA(cudaEventRecord(ctx->ev0, st));
    SdDev d = dev(mode, batch);
    if (enabling) pair->on_spec_enable(d, st);
    rng_refill(d_rng.p, 2 * n, st);
    sd_cycle_begin(d, st);
    const RowType rt = pair->row_type();
    int redraft_passes = 0;
    // Single-round cycles run OPTIMISTICALLY with no host synchronisation inside the step: the
    // redraft check (EOS-shortened chain -> later chains' draft-stream offsets move) only raises a
    // device flag that turns acceptance and the cycle end into no-ops; the flag is read back
    // with the step summary and, in that rare case, the cycle is redone synchronously below.
    const bool optimistic = mode.enabled && mode.rounds == 1 && verify_mode != RS_VERIFY_GREEDY &&
                            mode.branching > 1 && !capture;
    bool redo = false;
    if (optimistic) {
        sd_round_setup(d, 0, st);
        for (int depth = 0; depth < mode.draft_len; ++depth) {
            prof_set_scope("draft");
            pair->draft_rows(d, depth, st);
            sd_draft_sample(d, depth, rt, st);
        }
        sd_redraft_check(d, st);
        verify_accept(d, 0, rt, st);
        pair->after_accept(d, false, st);
        sd_cycle_end(d, false, st);
        RS_CUDA(cudaEventRecord(ctx->ev1, st));
        RS_CUDA(cudaMemcpyAsync(h_misc + 1, d_flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        note_copy(false, sizeof(int32_t));
        RS_CUDA(cudaStreamSynchronize(st));
        redo = h_misc[1] != 0;
        if (redo) {
            RS_CUDA(cudaMemsetAsync(d_flag.p, 0, sizeof(int32_t), st));
            ++redraft_passes;
        }
    }
    if (optimistic && !redo) {
        // done: summary below
    } else if (mode.enabled) {
        for (int round = 0; round < mode.rounds; ++round) {
            if (!redo) sd_round_setup(d, round, st);  // a redo keeps the corrected offsets
            redo = false;
            for (;;) {
                for (int depth = 0; depth < mode.draft_len; ++depth) {
                    prof_set_scope("draft");
                    pair->draft_rows(d, depth, st);
                    sd_draft_sample(d, depth, rt, st);
                    if (capture) capture_rows(d, false, depth, 0);
                }
                if (verify_mode == RS_VERIFY_GREEDY || mode.branching == 1) break;
                sd_redraft_check(d, st);
                RS_CUDA(cudaMemcpyAsync(h_misc + 1, d_flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                note_copy(false, sizeof(int32_t));
                RS_CUDA(cudaStreamSynchronize(st));
                if (!h_misc[1]) break;
                RS_CUDA(cudaMemsetAsync(d_flag.p, 0, sizeof(int32_t), st));
                ++redraft_passes;
            }
            verify_accept(d, round, rt, st);
            pair->after_accept(d, false, st);
            if (round + 1 < mode.rounds) {
                // any request continuing into the next round? (lockstep, server.cpp:154-178)
                std::vector<int32_t> cont(n), lens(n);
                RS_CUDA(cudaMemcpyAsync(cont.data(), d.cont, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                RS_CUDA(cudaMemcpyAsync(lens.data(), d.len, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                note_copy(false, 2 * n * sizeof(int32_t));
                RS_CUDA(cudaStreamSynchronize(st));
                bool any = false;
                for (int r : active) any |= cont[r] != 0;
                if (!any) break;
                for (int r : active) len[r] = lens[r];  // next round's forwards start from here
            }
        }
    } else {
        prof_set_scope("naive");
        pair->verify_rows(d, true, st);
        if (capture) capture_rows(d, true, 0, 0);
        sd_accept(d, 0, true, rt, st);
        pair->after_accept(d, true, st);
    }
    if (!(optimistic && !redo && redraft_passes == 0)) {
        sd_cycle_end(d, !mode.enabled, st);
        RS_CUDA(cudaEventRecord(ctx->ev1, st));
    }
    const int sw = kSummaryFixed + 3 * kMaxRounds;
    RS_CUDA(cudaMemcpyAsync(h_summary, d_summary.p, (size_t)batch * sw * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (h_newtok) {  // this cycle's tokens ride along with the summary (one synchronisation)
        RS_CUDA(cudaMemcpyAsync(h_newtok, d_newtok.p, (size_t)batch * newtok_cap * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st));
        note_copy(false, (size_t)batch * newtok_cap * sizeof(int32_t));
    }
    RS_CUDA(cudaMemcpyAsync(h_misc, d_err.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    note_copy(false, (size_t)batch * sw * sizeof(int32_t) + sizeof(int32_t));
    RS_CUDA(cudaStreamSynchronize(st));
    prof_collect();
    prof_set_scope("step");
    if (h_misc[0] != 0) {
        const int code = h_misc[0];
        h_misc[0] = 0;
        RS_CUDA(cudaMemset(d_err.p, 0, sizeof(int32_t)));
        throw std::invalid_argument(dev_err_message(code));
    }

    // host bookkeeping: accept lens, done flags, ledger (charge_batched_cycle, server.cpp:154-178)
    int emitted = 0, drafted_cycles = 0, accepted = 0;
    size_t max_rounds = 0;
    for (int a = 0; a < batch; ++a) max_rounds = std::max<size_t>(max_rounds, h_summary[a * sw + 4]);
    last_active.assign(active.begin(), active.begin() + batch);
    last_emitted.assign(batch, 0);
    for (int a = 0; a < batch; ++a) {
        const int32_t *s = h_summary + a * sw;
        const int r = active[a];
        last_emitted[a] = s[1];
        done[r] = s[0];
        len[r] = s[5];
        emitted += s[1];
        if (mode.enabled && s[3]) {
            accept_lens[r].push_back(s[2]);
            ++drafted_cycles;
            accepted += s[2];
        }
    }
    // charge_batched_cycle over the whole active batch, or -- ledger_group > 0 (the profiler's
    // fixed-width waves run side by side) -- separately per group of ledger_group requests into
    // that group's own ledger.
    auto charge = [&](std::vector<rs_forward_event> &out, int a0, int a1) {
        const int width = a1 - a0;
        if (mode.enabled) {
            size_t rounds = 0;
            for (int a = a0; a < a1; ++a) rounds = std::max<size_t>(rounds, h_summary[a * sw + 4]);
            for (size_t rr = 0; rr < rounds; ++rr) {
                int max_fw = 0, each = 0, max_target = 0;
                for (int a = a0; a < a1; ++a) {
                    const int32_t *s = h_summary + a * sw;
                    if ((size_t)s[4] > rr) {
                        const int32_t *rc = s + kSummaryFixed + 3 * rr;
                        max_fw = std::max(max_fw, rc[0]);
                        each = std::max(each, rc[1]);
                        max_target = std::max(max_target, rc[2]);
                    }
                }
                for (int f = 0; f < max_fw; ++f) out.push_back({0, width * each, width * each});
                if (max_target > 0) out.push_back({1, width * max_target, width * max_target});
            }
        } else {
            out.push_back({1, width, width});
        }
    };
    if (ledger_group > 0) {
        group_ledgers.resize((n + ledger_group - 1) / ledger_group);
        for (int a0 = 0; a0 < batch;) {
            const int g = active[a0] / ledger_group;
            int a1 = a0;
            while (a1 < batch && active[a1] / ledger_group == g) ++a1;
            charge(group_ledgers[g], a0, a1);
            a0 = a1;
        }
    } else {
        charge(ledger, 0, batch);
    }
    (void)max_rounds;
    ++cycle;
    if (info) {
        float ms = 0.f;
        RS_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        info->active_batch = batch;
        info->mode = mode;
        info->drafter_version = drafter ? drafter->version : -1;
        info->emitted_tokens = emitted;
        info->drafted_cycles = drafted_cycles;
        info->accepted_drafted = accepted;
        info->redraft_passes = redraft_passes;
        info->step_ms = ms;
        info->h2d_bytes = copy_bytes(true);
        info->d2h_bytes = copy_bytes(false);
    }
}

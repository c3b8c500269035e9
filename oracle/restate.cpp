// oracle/restate.cpp -- TEST INFRASTRUCTURE ONLY (see restate.hpp header).
// Line-by-line restatement of the reference decision logic; every function cites the
// reference file:line it follows (paths relative to /root/reference/proj/core/src).
#include "restate.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <numeric>

namespace orc {

// model.cpp:113-130
size_t TabularModel::row_index(const std::vector<int> & ctx) const {
    size_t idx = 0;
    const size_t len = ctx.size();
    for (int i = 0; i < order; ++i) {
        const size_t back = static_cast<size_t>(order - i);
        int tok = len >= back ? ctx[len - back] : 0;  // left-pad with token 0
        if (tok < 0 || tok >= vocab) throw std::invalid_argument("row_index: token out of vocabulary");
        idx = idx * static_cast<size_t>(vocab) + static_cast<size_t>(tok);
    }
    return idx;
}

std::vector<double> TabularModel::logits(const std::vector<int> & ctx) const {
    const size_t r = row_index(ctx), V = static_cast<size_t>(vocab);
    return std::vector<double>(table.begin() + static_cast<long>(r * V),
                               table.begin() + static_cast<long>((r + 1) * V));
}

std::vector<double> LookupModel::logits_at(const std::vector<int> & ctx, int depth) const {
    const std::pair<std::vector<int>, int> key{ctx, depth_aware ? depth : 0};
    auto it = rows.find(key);
    if (it == rows.end()) {
        auto f = rows32.find(key);
        if (f != rows32.end()) return std::vector<double>(f->second.begin(), f->second.end());
        std::string s = "LookupModel: no row for context of length " + std::to_string(ctx.size()) + " [";
        for (size_t i = ctx.size() > 6 ? ctx.size() - 6 : 0; i < ctx.size(); ++i) s += std::to_string(ctx[i]) + " ";
        throw std::out_of_range(s + "]");
    }
    return it->second;
}

// model.cpp:53-68: max of z/tau, exp(z/tau - max), sequential sum, divide.
std::vector<double> softmax(const std::vector<double> & z, double tau) {
    std::vector<double> out(z.size());
    double m = -std::numeric_limits<double>::infinity();
    for (double v : z) m = std::max(m, v / tau);
    double sum = 0.0;
    for (size_t i = 0; i < z.size(); ++i) {
        out[i] = std::exp(z[i] / tau - m);
        sum += out[i];
    }
    for (double & p : out) p /= sum;
    return out;
}

// model.cpp:132-139: EOS bias added to z[V-1] before the temperature division.
std::vector<double> dist(const Model & m, const std::vector<int> & ctx, double eos_bias, int depth) {
    std::vector<double> z = m.logits_at(ctx, depth);
    if (static_cast<int>(z.size()) != m.vocab) throw std::invalid_argument("dist: row has wrong width");
    z[z.size() - 1] += eos_bias;
    return softmax(z, m.temperature);
}

// model.cpp:23-40
int sample_from(const std::vector<double> & p, double u) {
    double cum = 0.0;
    const int n = static_cast<int>(p.size());
    for (int i = 0; i < n; ++i) {
        cum += p[static_cast<size_t>(i)];
        if (u < cum) return i;
    }
    for (int i = n - 1; i >= 0; --i)
        if (p[static_cast<size_t>(i)] > 0.0) return i;
    throw std::invalid_argument("sample_from: all-zero distribution");
}

int argmax_first(const std::vector<double> & p) {
    int best = 0;
    for (int i = 1; i < static_cast<int>(p.size()); ++i)
        if (p[static_cast<size_t>(i)] > p[static_cast<size_t>(best)]) best = i;
    return best;
}

// specdec.cpp:25-33
double accept_prob(double p, double q) {
    if (!(q > 0.0)) throw std::invalid_argument("accept_prob: drafted token must have q > 0");
    if (p < 0.0 || p > 1.0 || q > 1.0) throw std::invalid_argument("accept_prob: probabilities out of range");
    return std::min(1.0, p / q);
}

// specdec.cpp:35-52
std::vector<double> residual_dist(const std::vector<double> & p, const std::vector<double> & q) {
    if (p.size() != q.size()) throw std::invalid_argument("residual_dist: size mismatch");
    std::vector<double> r(p.size());
    double norm = 0.0;
    for (size_t x = 0; x < p.size(); ++x) {
        r[x] = std::max(0.0, p[x] - q[x]);
        norm += r[x];
    }
    if (norm <= 1e-12) throw std::invalid_argument("residual_dist: degenerate residual (p == q)");
    for (double & v : r) v /= norm;
    return r;
}

std::string SDConfig::key() const {  // specdec.cpp:8-14
    if (!enabled) return "off";
    return "s" + std::to_string(rounds) + "_t" + std::to_string(branching) + "_n" + std::to_string(draft_len);
}

namespace {

StepRecord make_step(int token, const std::vector<double> & pd, bool drafted, double logq, bool full) {
    // specdec.cpp:62-74
    StepRecord s;
    s.token = token;
    s.logp = std::log(pd[static_cast<size_t>(token)]);
    s.drafted = drafted;
    s.logq = logq;
    if (full) {
        s.target_logprobs.resize(pd.size());
        for (size_t i = 0; i < pd.size(); ++i) s.target_logprobs[i] = std::log(pd[i]);
    }
    return s;
}

std::vector<int> extend(const std::vector<int> & base, const std::vector<int> & ext) {
    std::vector<int> c = base;
    c.insert(c.end(), ext.begin(), ext.end());
    return c;
}

// Greedy tree expansion at the root: the t most likely first tokens (ties -> lower id).
std::vector<int> top_k_first(const std::vector<double> & q, int k) {
    std::vector<int> idx(q.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return q[static_cast<size_t>(a)] > q[static_cast<size_t>(b)]; });
    idx.resize(static_cast<size_t>(std::min<int>(k, static_cast<int>(q.size()))));
    return idx;
}

}  // namespace

// specdec.cpp:146-269 (sampling); greedy variant per SURVEY.md §8 A6.
VerifyOutcome spec_step_tree(const Model & target, const Model & drafter, const std::vector<int> & ctx,
                             const SDConfig & cfg, DecodeRng & rng, double eos_bias, bool stop_at_eos,
                             int max_emit, VerifyMode mode, bool full) {
    if (!cfg.enabled) throw std::invalid_argument("spec_step_tree: config is disabled");
    const int eos = target.eos();
    const bool greedy = mode == VerifyMode::Greedy;
    VerifyOutcome out;
    std::vector<int> accepted;

    auto emit = [&](int tok, const std::vector<double> & pd, bool drafted, double logq) {
        out.steps.push_back(make_step(tok, pd, drafted, logq, full));
        out.accepted_tokens.push_back(tok);
        accepted.push_back(tok);
        if (stop_at_eos && tok == eos) out.ended = true;
    };

    for (int round = 0; round < cfg.rounds && !out.ended; ++round) {
        const int remaining = max_emit - static_cast<int>(accepted.size());
        if (remaining < 2) break;  // specdec.cpp:166-169
        const int n_eff = std::min(cfg.draft_len, remaining - 1);
        const std::vector<int> round_ctx = extend(ctx, accepted);

        // drafting (specdec.cpp:173-195)
        std::vector<std::vector<int>> chains(static_cast<size_t>(cfg.branching));
        size_t longest = 0;
        int tree_tokens = 0;
        std::vector<int> roots;
        if (greedy) roots = top_k_first(dist(drafter, round_ctx, eos_bias, 0), cfg.branching);
        for (size_t ci = 0; ci < chains.size(); ++ci) {
            auto & chain = chains[ci];
            for (int pos = 0; pos < n_eff; ++pos) {
                std::vector<double> qd = dist(drafter, extend(round_ctx, chain), eos_bias, static_cast<int>(chain.size()));
                int d;
                if (greedy) d = pos == 0 ? roots[std::min(ci, roots.size() - 1)] : argmax_first(qd);
                else d = sample_from(qd, rng.du());
                ++out.draft_records;
                chain.push_back(d);
                ++tree_tokens;
                if (stop_at_eos && d == eos) break;
            }
            longest = std::max(longest, chain.size());
        }
        out.rounds.push_back({static_cast<int>(longest), cfg.branching, tree_tokens + 1});

        // branch point (specdec.cpp:197-217)
        const std::vector<double> p1 = dist(target, round_ctx, eos_bias);
        const std::vector<double> q1 = dist(drafter, round_ctx, eos_bias, 0);
        int selected = -1;
        if (greedy) {
            const int a1 = argmax_first(p1);
            for (int i = 0; i < cfg.branching; ++i)
                if (chains[static_cast<size_t>(i)][0] == a1) { selected = i; break; }
            if (selected < 0) {
                emit(a1, p1, false, 0.0);
                out.bonus_token = a1;
                return out;
            }
        } else {
            std::vector<double> p_cur = p1;
            for (int i = 0; i < cfg.branching; ++i) {
                const int cand = chains[static_cast<size_t>(i)][0];
                const double a = std::min(1.0, p_cur[static_cast<size_t>(cand)] / q1[static_cast<size_t>(cand)]);
                if (rng.au() < a) { selected = i; break; }
                p_cur = residual_dist(p_cur, q1);
            }
            if (selected < 0) {
                int x = sample_from(p_cur, rng.au());
                emit(x, p1, false, 0.0);  // record keeps the original p1 (specdec.cpp:214)
                out.bonus_token = x;
                return out;
            }
        }
        const std::vector<int> & chain = chains[static_cast<size_t>(selected)];
        emit(chain[0], p1, true, std::log(q1[static_cast<size_t>(chain[0])]));
        out.accept_len += 1;
        if (out.ended) return out;

        // chain-style verification of the rest (specdec.cpp:226-245)
        bool rejected = false;
        for (size_t pos = 1; pos < chain.size() && !out.ended; ++pos) {
            const std::vector<int> c = extend(ctx, accepted);
            const std::vector<double> pd = dist(target, c, eos_bias);
            const std::vector<double> qd = dist(drafter, c, eos_bias, static_cast<int>(pos));
            const int d = chain[pos];
            bool ok;
            int repl = -1;
            if (greedy) {
                repl = argmax_first(pd);
                ok = d == repl;
            } else {
                ok = rng.au() < accept_prob(pd[static_cast<size_t>(d)], qd[static_cast<size_t>(d)]);
            }
            if (ok) {
                emit(d, pd, true, std::log(qd[static_cast<size_t>(d)]));
                out.accept_len += 1;
            } else {
                int x = greedy ? repl : sample_from(residual_dist(pd, qd), rng.au());
                emit(x, pd, false, 0.0);
                out.bonus_token = x;
                rejected = true;
                break;
            }
        }
        if (rejected || out.ended) return out;
    }

    // bonus (specdec.cpp:256-267)
    if (!out.ended && static_cast<int>(accepted.size()) < max_emit) {
        const std::vector<double> pd = dist(target, extend(ctx, accepted), eos_bias);
        int x = greedy ? argmax_first(pd) : sample_from(pd, rng.au());
        emit(x, pd, false, 0.0);
        out.bonus_token = x;
        if (out.rounds.empty()) out.rounds.push_back({0, 0, 1});
    }
    return out;
}

// costsim.cpp:13-27
double forward_time(const TimingModel & tm, bool target, int tokens) {
    if (tokens < 1) throw std::invalid_argument("forward_time: total_tokens must be >= 1");
    const RoleTiming & t = target ? tm.target : tm.drafter;
    return t.latency_floor + t.unit_cost * static_cast<double>(std::max(tokens, t.saturation_tokens));
}

double ledger_time(const TimingModel & tm, const std::vector<ForwardEvent> & ev) {
    double total = 0.0;
    for (const auto & e : ev) total += forward_time(tm, e.target, e.batch_tokens);
    return total;
}

// server.cpp:154-178
void charge_batched_cycle(std::vector<ForwardEvent> & ledger, const std::vector<VerifyOutcome> & outs) {
    const int width = static_cast<int>(outs.size());
    size_t max_rounds = 0;
    for (const auto & o : outs) max_rounds = std::max(max_rounds, o.rounds.size());
    for (size_t r = 0; r < max_rounds; ++r) {
        int max_fw = 0, each = 0, max_target = 0;
        for (const auto & o : outs) {
            if (o.rounds.size() > r) {
                max_fw = std::max(max_fw, o.rounds[r].drafter_forwards);
                each = std::max(each, o.rounds[r].drafter_tokens_each);
                max_target = std::max(max_target, o.rounds[r].target_tokens);
            }
        }
        for (int f = 0; f < max_fw; ++f) ledger.push_back({false, width * each, width * each});
        if (max_target > 0) ledger.push_back({true, width * max_target, width * max_target});
    }
}

// server.cpp:21-78
ProfileTable::ProfileTable(std::vector<int> buckets) : buckets_(std::move(buckets)) {
    if (buckets_.empty()) throw std::invalid_argument("ProfileTable: no buckets");
    std::sort(buckets_.begin(), buckets_.end());
}

void ProfileTable::set_entry(int bucket, const SDConfig & cfg, double tpt) { entries_[bucket].emplace_back(cfg, tpt); }

void ProfileTable::finalize() {
    best_.clear();
    for (int b : buckets_) {
        auto it = entries_.find(b);
        if (it == entries_.end()) throw std::invalid_argument("ProfileTable: bucket has no entries");
        bool has_base = false;
        const SDConfig * best = nullptr;
        double best_t = 0.0;
        for (const auto & [cfg, t] : it->second) {
            if (!cfg.enabled) has_base = true;
            bool better = false;
            if (best == nullptr || t < best_t) better = true;
            else if (t == best_t) {
                const int cur = cfg.enabled ? cfg.drafted_per_cycle() : 0;
                const int old = best->enabled ? best->drafted_per_cycle() : 0;
                better = cur < old || (cur == old && !cfg.enabled && best->enabled);
            }
            if (better) { best = &cfg; best_t = t; }
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

SDConfig ProfileTable::solve(int active_batch) const { return best_for_bucket(bucket_for(active_batch)); }

SDConfig ProfileTable::best_for_bucket(int bucket) const {
    auto it = best_.find(bucket);
    if (it == best_.end()) throw std::invalid_argument("ProfileTable: table not finalized or unknown bucket");
    return it->second;
}

const std::vector<std::pair<SDConfig, double>> & ProfileTable::entries_for(int b) const {
    auto it = entries_.find(b);
    if (it == entries_.end()) throw std::invalid_argument("ProfileTable: unknown bucket");
    return it->second;
}

double ProfileTable::entry(int bucket, const SDConfig & cfg) const {
    for (const auto & [c, t] : entries_for(bucket))
        if (c == cfg) return t;
    throw std::invalid_argument("ProfileTable: no entry for config " + cfg.key());
}

std::string ProfileTable::to_csv() const {  // server.cpp:136-145
    std::string out = "batch,s,t,n,time_per_token,speedup\n";
    char buf[128];
    for (int b : buckets_) {
        const double base = entry(b, SDConfig{});
        for (const auto & [cfg, t] : entries_.at(b)) {
            std::snprintf(buf, sizeof(buf), "%d,%d,%d,%d,%.12g,%.12g\n", b, cfg.enabled ? cfg.rounds : 0,
                          cfg.enabled ? cfg.branching : 0, cfg.enabled ? cfg.draft_len : 0, t, base / t);
            out += buf;
        }
    }
    return out;
}

std::vector<int> RequestState::full_ctx() const { return extend(prompt, generated); }

BatchEngine::BatchEngine(const Model & target, std::function<std::shared_ptr<const Model>()> drafter,
                         const ProfileTable * table, std::vector<RequestState> reqs, SDConfig forced,
                         VerifyMode mode, bool record_full)
    : target_(target), drafter_(std::move(drafter)), table_(table), reqs_(std::move(reqs)), mode_(forced),
      vmode_(mode), record_full_(record_full) {}

bool BatchEngine::all_done() const {
    return std::all_of(reqs_.begin(), reqs_.end(), [](const RequestState & r) { return r.done; });
}

// server.cpp:266-349
void BatchEngine::step() {
    std::vector<RequestState *> active;
    for (auto & r : reqs_)
        if (!r.done) active.push_back(&r);
    if (active.empty()) throw std::runtime_error("BatchEngine: empty batch");
    const int batch = static_cast<int>(active.size());
    active_trace_.push_back(batch);

    const SDConfig desired = table_ ? table_->solve(batch) : mode_;
    if (mode_init_ && !(desired == mode_)) {
        if (!mode_.enabled && desired.enabled) {
            int ctx_tokens = 0;
            for (auto * r : active) ctx_tokens += static_cast<int>(r->prompt.size() + r->generated.size());
            ledger_.push_back({false, ctx_tokens, ctx_tokens});
            ++prefill_events_;
        }
        switches_.push_back({cycle_, batch, mode_, desired});
    }
    mode_ = desired;
    mode_init_ = true;
    for (auto * r : active) r->spec_flag = mode_.enabled;

    std::shared_ptr<const Model> drafter;
    if (mode_.enabled) {
        drafter = drafter_ ? drafter_() : nullptr;
        if (!drafter) throw std::runtime_error("BatchEngine: spec mode requires a drafter snapshot");
    }
    drafter_versions_.push_back(drafter ? drafter->version : -1);

    if (mode_.enabled) {
        std::vector<VerifyOutcome> outs;
        for (auto * r : active) {
            VerifyOutcome o = spec_step_tree(target_, *drafter, r->full_ctx(), mode_, r->rng, r->eos_bias, true,
                                             r->remaining(), vmode_, record_full_);
            for (int t : o.accepted_tokens) r->generated.push_back(t);
            r->steps.insert(r->steps.end(), o.steps.begin(), o.steps.end());
            if (o.draft_records > 0) r->accept_lens.push_back(o.accept_len);
            if (o.ended || r->remaining() == 0) r->done = true;
            outs.push_back(std::move(o));
        }
        charge_batched_cycle(ledger_, outs);
    } else {
        const int eos = target_.eos();
        for (auto * r : active) {
            const std::vector<double> pd = dist(target_, r->full_ctx(), r->eos_bias);
            const int tok = vmode_ == VerifyMode::Greedy ? argmax_first(pd) : sample_from(pd, r->rng.du());
            r->steps.push_back(make_step(tok, pd, false, 0.0, record_full_));
            r->generated.push_back(tok);
            if (tok == eos || r->remaining() == 0) r->done = true;
        }
        ledger_.push_back({true, batch, batch});
    }
    ++cycle_;
}

// learner.cpp:10-27
double kd_weight(double r, const std::vector<double> & br, const KDPolicy & p) {
    switch (p.mode) {
        case WeightMode::Uniform: return 1.0;
        case WeightMode::Frozen: throw std::logic_error("kd_weight: frozen drafter takes no updates");
        case WeightMode::Reward: break;
    }
    if (br.empty()) throw std::invalid_argument("kd_weight: empty batch");
    const double mean = std::accumulate(br.begin(), br.end(), 0.0) / static_cast<double>(br.size());
    return std::clamp(r / std::max(1e-6, mean), p.clip_lo, p.clip_hi);
}

// learner.cpp:33-60
double kd_loss(const TabularModel & drafter, const Rollout & s, double w) {
    if (s.target_logprobs.size() != s.response.size()) throw std::invalid_argument("kd_loss: steps/response length mismatch");
    double total = 0.0;
    std::vector<int> ctx = s.prompt;
    for (size_t t = 0; t < s.response.size(); ++t) {
        const auto & lp = s.target_logprobs[t];
        std::vector<double> q = dist(drafter, ctx, s.eos_bias);
        if (lp.size() != q.size()) throw std::invalid_argument("kd_loss: vocab size mismatch");
        for (size_t x = 0; x < lp.size(); ++x) {
            if (std::isinf(lp[x])) continue;
            total += std::exp(lp[x]) * (lp[x] - std::log(q[x]));
        }
        ctx.push_back(s.response[t]);
    }
    return w * total;
}

// learner.cpp:62-82
std::vector<double> kd_loss_gradient(const TabularModel & drafter,
                                     const std::vector<std::pair<const Rollout *, double>> & ws) {
    const size_t V = static_cast<size_t>(drafter.vocab);
    std::vector<double> grad(drafter.table.size(), 0.0);
    const double inv_tau = 1.0 / drafter.temperature;
    for (const auto & [s, w] : ws) {
        std::vector<int> ctx = s->prompt;
        for (size_t t = 0; t < s->response.size(); ++t) {
            const size_t row = drafter.row_index(ctx);
            const std::vector<double> q = dist(drafter, ctx, s->eos_bias);
            const auto & lp = s->target_logprobs[t];
            for (size_t x = 0; x < V; ++x) {
                const double p = std::isinf(lp[x]) ? 0.0 : std::exp(lp[x]);
                grad[row * V + x] += w * (q[x] - p) * inv_tau;
            }
            ctx.push_back(s->response[t]);
        }
    }
    return grad;
}

// learner.cpp:98-160
KDUpdateResult kd_update(const TabularModel & drafter, const std::vector<Rollout> & buf, const KDPolicy & p,
                         std::mt19937_64 & sel, double cost) {
    if (p.mode == WeightMode::Frozen) throw std::logic_error("kd_update: frozen drafter takes no updates");
    if (p.interval < 1) throw std::invalid_argument("kd_update: interval must be >= 1");
    KDUpdateResult res;
    res.logits = drafter.table;
    if (buf.empty()) return res;
    const size_t n = buf.size();
    const size_t take = (n + static_cast<size_t>(p.interval) - 1) / static_cast<size_t>(p.interval);
    std::vector<size_t> idx(n);
    std::iota(idx.begin(), idx.end(), size_t{0});
    for (size_t i = 0; i < take; ++i) {
        const size_t j = i + static_cast<size_t>(sel() % (n - i));
        std::swap(idx[i], idx[j]);
    }
    std::vector<double> br(take);
    for (size_t i = 0; i < take; ++i) br[i] = buf[idx[i]].reward;
    std::vector<std::pair<const Rollout *, double>> ws;
    double wsum = 0, wmin = 0, wmax = 0;
    size_t tokens = 0;
    for (size_t i = 0; i < take; ++i) {
        const Rollout & s = buf[idx[i]];
        const double w = kd_weight(s.reward, br, p);
        ws.emplace_back(&s, w);
        wsum += w;
        wmin = i == 0 ? w : std::min(wmin, w);
        wmax = i == 0 ? w : std::max(wmax, w);
        tokens += s.response.size();
        res.selected.push_back(idx[i]);
    }
    double loss = 0.0;
    for (const auto & [s, w] : ws) loss += kd_loss(drafter, *s, w);
    std::vector<double> g = kd_loss_gradient(drafter, ws);
    for (size_t i = 0; i < g.size(); ++i) res.logits[i] += g[i] * -p.lr;
    res.updated = true;
    res.loss = loss;
    res.samples_used = static_cast<int>(take);
    res.weight_mean = wsum / static_cast<double>(take);
    res.weight_min = wmin;
    res.weight_max = wmax;
    res.sim_time = cost * static_cast<double>(tokens);
    return res;
}

}  // namespace orc

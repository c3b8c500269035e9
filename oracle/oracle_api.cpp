// oracle/oracle_api.cpp -- TEST INFRASTRUCTURE ONLY.
// JSON-in / JSON-out C entry point over the CPU restatement (restate.cpp), so the Python
// tests can drive it with ctypes. oracle/ref_shim.cpp exposes the SAME schema over the
// compiled reference, which is how the restatement is pinned (tests/test_oracle.py).
#include <cstdlib>
#include <cstring>
#include <json.hpp>
#include <map>
#include <memory>
#include <mutex>

#include "restate.hpp"
#include "tf_cpu.hpp"
#include <chrono>
#include <omp.h>

using nlohmann::json;
using namespace orc;

namespace {

SDConfig cfg_of(const json & j) {
    SDConfig c;
    c.rounds = j.value("s", 1);
    c.branching = j.value("t", 1);
    c.draft_len = j.value("n", 1);
    c.enabled = j.value("enabled", false);
    return c;
}
json cfg_json(const SDConfig & c) { return {{"s", c.rounds}, {"t", c.branching}, {"n", c.draft_len}, {"enabled", c.enabled}}; }

// Lookup models filled through the binary entry points below (oracle_lookup_*), referenced
// from a JSON request as {"kind": "lookup_ref", "id": k}.
std::mutex g_reg_mu;
std::map<int, std::shared_ptr<LookupModel>> g_reg;
int g_reg_next = 1;

// CPU transformer ports (tf_cpu.hpp), created by op "tf_cpu_create" and referenced as
// {"kind": "tf_cpu_target" | "tf_cpu_drafter", "id": k}.
struct TfPair {
    std::shared_ptr<TfWeights> w;
    std::shared_ptr<CpuTransformer> target;
    std::shared_ptr<CpuEagleDrafter> drafter;
};
std::map<int, TfPair> g_tf;
int g_tf_next = 1;

TfPair & tf_of(const json & j) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = g_tf.find(j.at("id").get<int>());
    if (it == g_tf.end()) throw std::invalid_argument("tf_cpu: unknown id");
    return it->second;
}

std::shared_ptr<Model> model_of(const json & j) {
    const std::string kind = j.value("kind", "tabular");
    if (kind == "tf_cpu_target") return tf_of(j).target;
    if (kind == "tf_cpu_drafter") return tf_of(j).drafter;
    if (kind == "lookup_ref") {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        auto it = g_reg.find(j.at("id").get<int>());
        if (it == g_reg.end()) throw std::invalid_argument("lookup_ref: unknown id");
        return it->second;
    }
    if (kind == "tabular") {
        auto m = std::make_shared<TabularModel>();
        m->vocab = j.at("vocab");
        m->order = j.at("order");
        m->temperature = j.value("temperature", 1.0);
        m->version = j.value("version", 0);
        m->table = j.at("logits").get<std::vector<double>>();
        size_t rows = 1;
        for (int i = 0; i < m->order; ++i) rows *= static_cast<size_t>(m->vocab);
        if (m->table.size() != rows * static_cast<size_t>(m->vocab)) throw std::invalid_argument("tabular: wrong table size");
        return m;
    }
    if (kind == "lookup") {
        auto m = std::make_shared<LookupModel>();
        m->vocab = j.at("vocab");
        m->temperature = j.value("temperature", 1.0);
        m->version = j.value("version", 0);
        m->depth_aware = j.value("depth_aware", false);
        for (const auto & r : j.at("rows"))
            m->rows.emplace(std::make_pair(r.at("ctx").get<std::vector<int>>(), m->depth_aware ? r.value("depth", 0) : 0),
                            r.at("logits").get<std::vector<double>>());
        return m;
    }
    throw std::invalid_argument("unknown model kind " + kind);
}

TimingModel timing_of(const json & j) {
    TimingModel tm;
    if (j.is_object()) {
        auto rt = [](const json & a) { return RoleTiming{a.at(0).get<double>(), a.at(1).get<int>(), a.at(2).get<double>()}; };
        if (j.contains("target")) tm.target = rt(j.at("target"));
        if (j.contains("drafter")) tm.drafter = rt(j.at("drafter"));
    }
    return tm;
}

ProfileTable table_of(const json & j) {
    ProfileTable t(j.at("buckets").get<std::vector<int>>());
    for (const auto & e : j.at("entries")) t.set_entry(e.at("bucket"), cfg_of(e), e.at("time_per_token"));
    t.finalize();
    return t;
}

json step_json(const StepRecord & s) {
    json j = {{"token", s.token}, {"logp", s.logp}, {"drafted", s.drafted}, {"logq", s.logq}};
    if (!s.target_logprobs.empty()) j["target_logprobs"] = s.target_logprobs;
    return j;
}

VerifyMode mode_of(const json & req) { return req.value("verify_mode", "sample") == "greedy" ? VerifyMode::Greedy : VerifyMode::Sample; }

json op_run_generation(const json & req) {
    auto target = model_of(req.at("target"));
    std::shared_ptr<const Model> drafter;
    if (req.contains("drafter") && !req.at("drafter").is_null()) drafter = model_of(req.at("drafter"));
    std::unique_ptr<ProfileTable> table;
    if (req.contains("table") && !req.at("table").is_null()) table = std::make_unique<ProfileTable>(table_of(req.at("table")));
    const TimingModel tm = timing_of(req.value("timing", json()));
    const bool full = req.value("record_logprobs", true);
    std::vector<RequestState> reqs;
    for (const auto & r : req.at("requests")) {
        RequestState s;
        s.id = r.value("id", 0);
        s.prompt = r.at("prompt").get<std::vector<int>>();
        s.eos_bias = r.value("eos_bias", 0.0);
        s.max_len = r.at("max_len");
        s.rng = DecodeRng::from_seed(r.at("seed").get<uint64_t>(), r.at("stream").get<uint64_t>());
        reqs.push_back(std::move(s));
    }
    std::function<std::shared_ptr<const Model>()> snap;
    if (drafter) snap = [drafter]() { return drafter; };
    BatchEngine eng(*target, snap, table.get(), std::move(reqs), cfg_of(req.value("forced", json::object())),
                    mode_of(req), full);
    const int max_cycles = req.value("max_cycles", -1);
    while (!eng.all_done() && (max_cycles < 0 || eng.cycles() < max_cycles)) eng.step();
    json out;
    out["cycles"] = eng.cycles();
    out["total_time"] = ledger_time(tm, eng.ledger());
    out["active_trace"] = eng.active_trace();
    out["prefill_events"] = eng.prefill_events();
    out["drafter_versions"] = eng.drafter_versions();
    json sw = json::array();
    for (const auto & s : eng.switches()) sw.push_back({{"cycle", s.cycle}, {"active_batch", s.active_batch}, {"from", cfg_json(s.from)}, {"to", cfg_json(s.to)}});
    out["switches"] = sw;
    json ledger = json::array();
    for (const auto & e : eng.ledger()) ledger.push_back({e.target ? 1 : 0, e.positions, e.batch_tokens});
    out["ledger"] = ledger;
    json samples = json::array();
    std::vector<int> all_al;
    for (const auto & r : eng.requests()) {
        json steps = json::array();
        for (const auto & s : r.steps) steps.push_back(step_json(s));
        samples.push_back({{"prompt", r.prompt}, {"response", r.generated}, {"steps", steps}, {"eos_bias", r.eos_bias},
                           {"accept_lens", r.accept_lens}, {"done", r.done}, {"draws", {r.rng.n_draft, r.rng.n_accept}}});
        all_al.insert(all_al.end(), r.accept_lens.begin(), r.accept_lens.end());
    }
    out["samples"] = samples;
    out["accept_lens"] = all_al;
    return out;
}

json op_spec_step_tree(const json & req) {
    auto target = model_of(req.at("target"));
    auto drafter = model_of(req.at("drafter"));
    std::vector<int> ctx = req.at("ctx").get<std::vector<int>>();
    DecodeRng rng = DecodeRng::from_seed(req.at("seed").get<uint64_t>(), req.value("stream", uint64_t{0}));
    const int cycles = req.value("cycles", 1);
    json outs = json::array();
    for (int c = 0; c < cycles; ++c) {
        VerifyOutcome o = spec_step_tree(*target, *drafter, ctx, cfg_of(req.at("cfg")), rng, req.value("eos_bias", 0.0),
                                         req.value("stop_at_eos", true), req.value("max_emit", 1 << 30), mode_of(req),
                                         req.value("record_logprobs", false));
        json rounds = json::array();
        for (const auto & r : o.rounds) rounds.push_back({r.drafter_forwards, r.drafter_tokens_each, r.target_tokens});
        json steps = json::array();
        for (const auto & s : o.steps) steps.push_back(step_json(s));
        outs.push_back({{"accepted_tokens", o.accepted_tokens}, {"accept_len", o.accept_len}, {"bonus_token", o.bonus_token},
                        {"ended", o.ended}, {"rounds", rounds}, {"steps", steps}, {"draft_records", o.draft_records}});
        if (req.value("advance_ctx", false)) ctx.insert(ctx.end(), o.accepted_tokens.begin(), o.accepted_tokens.end());
    }
    return {{"outcomes", outs}, {"draws", {rng.n_draft, rng.n_accept}}};
}

json op_kd_update(const json & req) {
    auto dm = model_of(req.at("drafter"));
    auto * drafter = dynamic_cast<TabularModel *>(dm.get());
    if (!drafter) throw std::invalid_argument("kd_update: tabular drafter required");
    std::vector<Rollout> buf;
    for (const auto & s : req.at("buffer")) {
        Rollout r;
        r.prompt = s.at("prompt").get<std::vector<int>>();
        r.response = s.at("response").get<std::vector<int>>();
        for (const auto & st : s.at("steps")) r.target_logprobs.push_back(st.at("target_logprobs").get<std::vector<double>>());
        r.eos_bias = s.value("eos_bias", 0.0);
        r.reward = s.value("reward", 0.0);
        buf.push_back(std::move(r));
    }
    const json & pj = req.at("policy");
    KDPolicy p;
    p.interval = pj.value("interval", 1);
    const std::string mode = pj.value("mode", "reward");
    p.mode = mode == "uniform" ? WeightMode::Uniform : mode == "frozen" ? WeightMode::Frozen : WeightMode::Reward;
    p.clip_lo = pj.value("clip_lo", 0.0);
    p.clip_hi = pj.value("clip_hi", 4.0);
    p.lr = pj.value("lr", 0.1);
    std::mt19937_64 sel(req.at("selection_seed").get<uint64_t>());
    KDUpdateResult r = kd_update(*drafter, buf, p, sel, req.value("cost_per_token", 0.0));
    json losses = json::array();
    for (size_t i = 0; i < buf.size(); ++i) losses.push_back(kd_loss(*drafter, buf[i], 1.0));
    return {{"updated", r.updated}, {"loss", r.loss}, {"samples_used", r.samples_used}, {"weight_mean", r.weight_mean},
            {"weight_min", r.weight_min}, {"weight_max", r.weight_max}, {"sim_time", r.sim_time}, {"logits", r.logits},
            {"selected", r.selected}, {"per_sample_loss_w1", losses}};
}

// kd_loss_gradient + weighted kd_loss over an explicit (sample, weight) list (learner.cpp:58-82).
json op_kd_grad(const json & req) {
    auto dm = model_of(req.at("drafter"));
    auto * drafter = dynamic_cast<TabularModel *>(dm.get());
    if (!drafter) throw std::invalid_argument("kd_grad: tabular drafter required");
    std::vector<Rollout> buf;
    for (const auto & s : req.at("samples")) {
        Rollout r;
        r.prompt = s.at("prompt").get<std::vector<int>>();
        r.response = s.at("response").get<std::vector<int>>();
        for (const auto & st : s.at("steps")) r.target_logprobs.push_back(st.at("target_logprobs").get<std::vector<double>>());
        r.eos_bias = s.value("eos_bias", 0.0);
        buf.push_back(std::move(r));
    }
    const std::vector<double> w = req.at("weights").get<std::vector<double>>();
    std::vector<std::pair<const Rollout *, double>> ws;
    double loss = 0.0;
    for (size_t i = 0; i < buf.size(); ++i) {
        ws.emplace_back(&buf[i], w.at(i));
        loss += kd_loss(*drafter, buf[i], w[i]);
    }
    return {{"grad", kd_loss_gradient(*drafter, ws)}, {"loss", loss}};
}

json op_profile_table(const json & req) {
    ProfileTable t(req.at("buckets").get<std::vector<int>>());
    for (const auto & e : req.at("entries")) t.set_entry(e.at("bucket"), cfg_of(e), e.at("time_per_token"));
    t.finalize();
    json best = json::array();
    for (int b : t.buckets()) best.push_back({{"bucket", b}, {"cfg", cfg_json(t.best_for_bucket(b))}});
    json solved = json::array();
    for (int b : req.value("solve", std::vector<int>{})) solved.push_back({{"batch", b}, {"bucket", t.bucket_for(b)}, {"cfg", cfg_json(t.solve(b))}});
    return {{"best", best}, {"solve", solved}, {"csv", t.to_csv()}};
}

// {"shape": {V, d, L, H, KV, dff, [rope_theta, eps, std, logit_scale]}, "seed", "drafter_seed",
// "temperature", "drafter_version"} -> {"id"}: target + drafter weights generated like model.cu
json op_tf_cpu_create(const json & req) {
    const json & sh = req.at("shape");
    TfShape s;
    s.V = sh.at("V");
    s.d = sh.at("d");
    s.L = sh.at("L");
    s.H = sh.at("H");
    s.KV = sh.at("KV");
    s.dff = sh.at("dff");
    s.hd = sh.value("hd", 128);
    s.rope_theta = sh.value("rope_theta", 1e6f);
    s.eps = sh.value("eps", 1e-6f);
    s.std = sh.value("std", 0.02f);
    s.logit_scale = sh.value("logit_scale", 1.0f);
    if (s.hd != 128 || s.H % s.KV) throw std::invalid_argument("tf_cpu: head_dim 128 and H % KV == 0 required");
    TfPair p;
    p.w = std::make_shared<TfWeights>();
    p.w->init_target(s, req.at("seed").get<uint64_t>(), 0);
    if (req.contains("drafter_seed")) p.w->init_drafter(req.at("drafter_seed").get<uint64_t>());
    p.target = std::make_shared<CpuTransformer>(p.w, req.value("temperature", 1.0));
    if (req.contains("drafter_seed")) p.drafter = std::make_shared<CpuEagleDrafter>(p.w, p.target, req.value("drafter_version", 0));
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_tf[g_tf_next] = std::move(p);
    return {{"id", g_tf_next++}};
}

// {"id", "role": "target" | "drafter", "ctx", "depth"} -> {"logits"} (raw row, fp32 values)
json op_tf_cpu_logits(const json & req) {
    TfPair & p = tf_of(req);
    const std::vector<int> ctx = req.at("ctx").get<std::vector<int>>();
    if (req.value("role", "target") == "drafter") {
        if (!p.drafter) throw std::invalid_argument("tf_cpu: no drafter");
        return {{"logits", p.drafter->logits_at(ctx, req.value("depth", 0))}};
    }
    return {{"logits", p.target->logits(ctx)}};
}

// {"id", "name", "layer", "drafter": bool} -> {"bits"} bf16 bit patterns, or {"f32"} for gains
json op_tf_cpu_tensor(const json & req) {
    TfPair & p = tf_of(req);
    const TfWeights & w = *p.w;
    const std::string nm = req.at("name");
    const bool dr = req.value("drafter", false);
    const TfLayer & L = dr ? w.dl : w.layers.at(req.value("layer", 0));
    if (nm == "emb") return {{"bits", w.emb}};
    if (nm == "lm_w") return {{"bits", w.lm_w}};
    if (nm == "fc_w") return {{"bits", w.fc_w}};
    if (nm == "qkv_w") return {{"bits", L.qkv_w}};
    if (nm == "qkv_b") return {{"bits", L.qkv_b}};
    if (nm == "o_w") return {{"bits", L.o_w}};
    if (nm == "gu_w") return {{"bits", L.gu_w}};
    if (nm == "down_w") return {{"bits", L.down_w}};
    throw std::invalid_argument("tf_cpu: unknown tensor " + nm);
}

// Timing sample of the SAME workload as the GPU bench, on the host cores: the target's and the
// drafter's caches hold `ctx` synthetic context positions, then `steps` engine steps (each one SD
// cycle of the restated engine over the CPU transformer port) run for `batch` requests.
json op_tf_cpu_bench(const json & req) {
    TfPair & p = tf_of(req);
    const int ctx = req.at("ctx"), batch = req.value("batch", 1), steps = req.value("steps", 1);
    if (req.contains("threads")) omp_set_num_threads(req.at("threads").get<int>());
    std::vector<RequestState> reqs;
    for (int b = 0; b < batch; ++b) {
        RequestState r;
        r.id = b;
        uint64_t st = 0x5eed + b;
        for (int i = 0; i < ctx; ++i) r.prompt.push_back(static_cast<int>(splitmix64(st) % (p.w->s.V - 1)));
        r.eos_bias = req.value("eos_bias", -20.0);
        r.max_len = req.value("max_len", 256);
        r.rng = DecodeRng::from_seed(req.value("seed", uint64_t{1}), b);
        // every context position but the last is synthetic: the first step computes the last
        // prompt row and then runs real SD cycles over the cache
        p.target->synthetic_prefix(r.prompt, ctx - 1, 1000 + b);
        if (p.drafter) p.drafter->synthetic_prefix(r.prompt, ctx - 1, 2000 + b);
        reqs.push_back(std::move(r));
    }
    std::function<std::shared_ptr<const Model>()> snap;
    if (p.drafter) {
        auto d = p.drafter;
        snap = [d]() { return d; };
    }
    BatchEngine eng(*p.target, snap, nullptr, std::move(reqs), cfg_of(req.at("cfg")), mode_of(req), false);
    eng.step();  // prompt rows (not timed): the engine's prefill of the last context position
    size_t before = 0;
    for (const auto & r : eng.requests()) before += r.generated.size();
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps && !eng.all_done(); ++i) eng.step();
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    size_t after = 0;
    for (const auto & r : eng.requests()) after += r.generated.size();
    return {{"seconds", sec}, {"tokens", after - before}, {"threads", omp_get_max_threads()}, {"steps", steps}};
}

json dispatch(const json & req) {
    const std::string op = req.at("op");
    if (op == "tf_cpu_create") return op_tf_cpu_create(req);
    if (op == "tf_cpu_logits") return op_tf_cpu_logits(req);
    if (op == "tf_cpu_tensor") return op_tf_cpu_tensor(req);
    if (op == "tf_cpu_bench") return op_tf_cpu_bench(req);
    if (op == "tf_cpu_free") {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        g_tf.erase(req.at("id").get<int>());
        return json::object();
    }
    if (op == "run_generation") return op_run_generation(req);
    if (op == "spec_step_tree") return op_spec_step_tree(req);
    if (op == "kd_update") return op_kd_update(req);
    if (op == "profile_table") return op_profile_table(req);
    if (op == "kd_grad") return op_kd_grad(req);
    throw std::invalid_argument("oracle: unknown op " + op);
}

char * dup(const std::string & s) {
    char * p = static_cast<char *>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

}  // namespace

extern "C" {
// Returns a malloc'd JSON string; {"error": {"type": ..., "what": ...}} on exception.
char * oracle_call(const char * req) {
    try {
        return dup(dispatch(json::parse(req)).dump());
    } catch (const std::invalid_argument & e) {
        return dup(json{{"error", {{"type", "invalid_argument"}, {"what", e.what()}}}}.dump());
    } catch (const std::logic_error & e) {
        return dup(json{{"error", {{"type", "logic_error"}, {"what", e.what()}}}}.dump());
    } catch (const std::runtime_error & e) {
        return dup(json{{"error", {{"type", "runtime_error"}, {"what", e.what()}}}}.dump());
    } catch (const std::exception & e) {
        return dup(json{{"error", {{"type", "exception"}, {"what", e.what()}}}}.dump());
    }
}
void oracle_free(char * p) { std::free(p); }

// Binary transport for captured full-vocabulary rows (V ~ 152K fp32 per row).
int oracle_lookup_new(int vocab, double temperature, int depth_aware) {
    auto m = std::make_shared<LookupModel>();
    m->vocab = vocab;
    m->temperature = temperature;
    m->depth_aware = depth_aware != 0;
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_reg[g_reg_next] = m;
    return g_reg_next++;
}
// Adds one row keyed by (ctx, depth). Returns 0 when added, 1 when an identical row was
// already present, -1 when a DIFFERENT row exists for the same key (row invariance broken),
// -2 for an unknown id.
int oracle_lookup_add_f32(int id, const int * ctx, int n, int depth, const float * logits) {
    std::shared_ptr<LookupModel> m;
    {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        auto it = g_reg.find(id);
        if (it == g_reg.end()) return -2;
        m = it->second;
    }
    std::pair<std::vector<int>, int> key{std::vector<int>(ctx, ctx + n), m->depth_aware ? depth : 0};
    auto it = m->rows32.find(key);
    if (it != m->rows32.end())
        return std::memcmp(it->second.data(), logits, sizeof(float) * m->vocab) == 0 ? 1 : -1;
    m->rows32.emplace(std::move(key), std::vector<float>(logits, logits + m->vocab));
    return 0;
}
void oracle_lookup_free(int id) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_reg.erase(id);
}
}

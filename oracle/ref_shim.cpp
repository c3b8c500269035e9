// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
// Compiled together with the UNMODIFIED reference sources (/root/reference/proj/core/src,
// read in place by oracle/Makefile) into oracle/_ref/librespec_ref.so. Exposes the same
// JSON schema as oracle_api.cpp so tests can diff the restatement against the reference,
// and bench.py --impl reference can time the reference's own CPU engine.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <json.hpp>
#include <memory>
#include <thread>

#include "respec/config.hpp"
#include "respec/learner.hpp"
#include "respec/rl.hpp"
#include "respec/scenarios.hpp"
#include "respec/server.hpp"
#include "respec/specdec.hpp"
#include "respec/verify.hpp"

using nlohmann::json;
using namespace respec;

namespace {

SDConfig cfg_of(const json & j) {
    return SDConfig{j.value("s", 1), j.value("t", 1), j.value("n", 1), j.value("enabled", false)};
}
json cfg_json(const SDConfig & c) { return {{"s", c.rounds}, {"t", c.branching}, {"n", c.draft_len}, {"enabled", c.enabled}}; }

TabularARModel model_of(const json & j) {
    if (j.value("kind", "tabular") != "tabular") throw std::invalid_argument("reference supports tabular models only");
    return TabularARModel(Vocabulary{j.at("vocab").get<int>()}, j.at("order").get<int>(), j.at("logits").get<std::vector<double>>(),
                          j.value("temperature", 1.0), j.value("version", 0));
}
json model_json(const TabularARModel & m) {
    return {{"kind", "tabular"}, {"vocab", m.vocab().size}, {"order", m.order()}, {"temperature", m.temperature()},
            {"version", m.version()}, {"logits", m.logits()}};
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

json step_json(const StepRecord & s, bool full) {
    json j = {{"token", s.token}, {"logp", s.logp}, {"drafted", s.drafted}, {"logq", s.logq}};
    if (full) j["target_logprobs"] = s.target_logprobs;
    return j;
}

std::vector<RequestState> requests_of(const json & arr) {
    std::vector<RequestState> reqs;
    for (const auto & r : arr) {
        RequestState s;
        s.id = r.value("id", 0);
        s.prompt = Context{r.at("prompt").get<std::vector<int>>()};
        s.eos_bias = r.value("eos_bias", 0.0);
        s.max_len = r.at("max_len");
        s.rng = DecodeRng::from_seed(r.at("seed").get<uint64_t>(), r.at("stream").get<uint64_t>());
        reqs.push_back(std::move(s));
    }
    return reqs;
}

json run_json(const GenerationRun & run, const std::vector<std::vector<int>> & per_req_al, bool full) {
    json out;
    out["cycles"] = run.cycles;
    out["total_time"] = run.total_time;
    out["active_trace"] = run.active_trace;
    json sw = json::array();
    for (const auto & s : run.switches) sw.push_back({{"cycle", s.cycle}, {"active_batch", s.active_batch}, {"from", cfg_json(s.from)}, {"to", cfg_json(s.to)}});
    out["switches"] = sw;
    json ledger = json::array();
    for (const auto & e : run.ledger.events) ledger.push_back({e.role == ModelRole::Target ? 1 : 0, e.positions_evaluated, e.concurrent_batch_tokens});
    out["ledger"] = ledger;
    json samples = json::array();
    for (size_t i = 0; i < run.samples.size(); ++i) {
        const auto & s = run.samples[i];
        json steps = json::array();
        for (const auto & st : s.steps) steps.push_back(step_json(st, full));
        samples.push_back({{"prompt", s.prompt}, {"response", s.response}, {"steps", steps}, {"eos_bias", s.eos_bias},
                           {"accept_lens", per_req_al[i]}});
    }
    out["samples"] = samples;
    out["accept_lens"] = run.accept_lens;
    return out;
}

json op_run_generation(const json & req) {
    TabularARModel target = model_of(req.at("target"));
    std::shared_ptr<const TabularARModel> drafter;
    if (req.contains("drafter") && !req.at("drafter").is_null()) drafter = std::make_shared<const TabularARModel>(model_of(req.at("drafter")));
    std::unique_ptr<ProfileTable> table;
    if (req.contains("table") && !req.at("table").is_null()) table = std::make_unique<ProfileTable>(ProfileTable::from_json(req.at("table")));
    if (req.value("verify_mode", "sample") != "sample") throw std::invalid_argument("reference has no greedy mode");
    const TimingModel tm = timing_of(req.value("timing", json()));
    DrafterSnapshotFn snap = nullptr;
    if (drafter) snap = [drafter]() { return drafter; };
    // BatchEngine directly (not run_generation) so per-request accept_lens and the
    // prefill counter are visible; run_generation is exactly this loop (server.cpp:351-376).
    BatchEngine eng(target, snap, table.get(), &tm, requests_of(req.at("requests")), cfg_of(req.value("forced", json::object())));
    while (!eng.all_done()) eng.step();
    GenerationRun run;
    run.ledger = eng.ledger();
    run.total_time = ledger_time(tm, run.ledger);
    run.switches = eng.switches();
    run.active_trace = eng.active_trace();
    run.cycles = eng.cycles();
    std::vector<std::vector<int>> per;
    for (RequestState & r : eng.requests()) {
        run.accept_lens.insert(run.accept_lens.end(), r.accept_lens.begin(), r.accept_lens.end());
        per.push_back(r.accept_lens);
        RolloutSample s;
        s.prompt = r.prompt.tokens;
        s.response = r.generated;
        s.steps = r.steps;
        s.eos_bias = r.eos_bias;
        run.samples.push_back(std::move(s));
    }
    json out = run_json(run, per, req.value("record_logprobs", true));
    out["prefill_events"] = eng.prefill_events();
    std::vector<int> dv;
    for (int c = 0; c < eng.cycles(); ++c) dv.push_back(eng.drafter_version_at_cycle(c));
    out["drafter_versions"] = dv;
    return out;
}

json op_spec_step_tree(const json & req) {
    TabularARModel target = model_of(req.at("target"));
    TabularARModel drafter = model_of(req.at("drafter"));
    Context ctx{req.at("ctx").get<std::vector<int>>()};
    DecodeRng rng = DecodeRng::from_seed(req.at("seed").get<uint64_t>(), req.value("stream", uint64_t{0}));
    const int cycles = req.value("cycles", 1);
    const bool full = req.value("record_logprobs", false);
    json outs = json::array();
    for (int c = 0; c < cycles; ++c) {
        VerifyOutcome o = spec_step_tree(target, drafter, ctx, cfg_of(req.at("cfg")), rng, req.value("eos_bias", 0.0),
                                         req.value("stop_at_eos", true), req.value("max_emit", 1 << 30));
        json rounds = json::array();
        for (const auto & r : o.rounds) rounds.push_back({r.drafter_forwards, r.drafter_tokens_each, r.target_tokens});
        json steps = json::array();
        for (const auto & s : o.steps) steps.push_back(step_json(s, full));
        outs.push_back({{"accepted_tokens", o.accepted_tokens}, {"accept_len", o.accept_len}, {"bonus_token", o.bonus_token},
                        {"ended", o.ended}, {"rounds", rounds}, {"steps", steps}, {"draft_records", static_cast<int>(o.draft_records.size())}});
        if (req.value("advance_ctx", false))
            for (int t : o.accepted_tokens) ctx.push(t);
    }
    return {{"outcomes", outs}};
}

json op_kd_update(const json & req) {
    TabularARModel drafter = model_of(req.at("drafter"));
    std::vector<RolloutSample> buf;
    for (const auto & s : req.at("buffer")) {
        RolloutSample r;
        r.prompt = s.at("prompt").get<std::vector<int>>();
        r.response = s.at("response").get<std::vector<int>>();
        for (const auto & st : s.at("steps")) {
            StepRecord rec;
            rec.token = st.value("token", 0);
            rec.target_logprobs = st.at("target_logprobs").get<std::vector<double>>();
            r.steps.push_back(std::move(rec));
        }
        r.eos_bias = s.value("eos_bias", 0.0);
        r.reward = s.value("reward", 0.0);
        buf.push_back(std::move(r));
    }
    const json & pj = req.at("policy");
    const std::string mode = pj.value("mode", "reward");
    KDPolicy p{pj.value("interval", 1), mode == "uniform" ? WeightMode::Uniform : mode == "frozen" ? WeightMode::Frozen : WeightMode::Reward,
               pj.value("clip_lo", 0.0), pj.value("clip_hi", 4.0), pj.value("lr", 0.1)};
    std::mt19937_64 sel(req.at("selection_seed").get<uint64_t>());
    KDUpdateResult r = kd_update(drafter, buf, p, sel, req.value("cost_per_token", 0.0));
    json losses = json::array();
    for (const auto & s : buf) losses.push_back(kd_loss(drafter, s, 1.0));
    return {{"updated", r.updated}, {"loss", r.loss}, {"samples_used", r.samples_used}, {"weight_mean", r.weight_mean},
            {"weight_min", r.weight_min}, {"weight_max", r.weight_max}, {"sim_time", r.sim_time}, {"logits", r.drafter.logits()},
            {"per_sample_loss_w1", losses}};
}

json op_profile_table(const json & req) {
    ProfileTable t(req.at("buckets").get<std::vector<int>>());
    for (const auto & e : req.at("entries")) t.set_entry(e.at("bucket"), cfg_of(e), e.at("time_per_token"));
    t.finalize();
    json best = json::array();
    for (int b : t.buckets()) best.push_back({{"bucket", b}, {"cfg", cfg_json(t.best_for_bucket(b))}});
    json solved = json::array();
    for (int b : req.value("solve", std::vector<int>{})) solved.push_back({{"batch", b}, {"bucket", t.bucket_for(b)}, {"cfg", cfg_json(t.solve(b))}});
    return {{"best", best}, {"solve", solved}, {"csv", t.to_csv()}, {"json", t.to_json()}};
}

// Default ExperimentConfig env (scenarios.cpp:28-51): actor, KD-warmed drafter, task.
json op_make_env(const json & req) {
    ExperimentConfig cfg;
    cfg.seed = req.value("seed", uint64_t{1});
    Env env = make_env(cfg);
    json prompts = json::array();
    for (const auto & p : env.task.prompts) prompts.push_back(p.tokens);
    json out = {{"actor", model_json(env.actor)}, {"drafter", model_json(env.drafter)},
                {"task", {{"prompts", prompts}, {"eos_biases", env.task.eos_biases}, {"group_size", env.task.group_size},
                          {"max_len", env.task.max_len}}}};
    if (req.value("with_profile", false)) out["table"] = build_profile(cfg, env.actor, env.drafter).to_json();
    return out;
}

json op_make_step_requests(const json & req) {
    ExperimentConfig cfg;
    Task task = cfg.make_task();
    auto reqs = make_step_requests(task, req.value("seed", uint64_t{1}), req.value("step", 0));
    json arr = json::array();
    const uint64_t seed = req.value("seed", uint64_t{1});
    const int step = req.value("step", 0);
    for (const auto & r : reqs)
        arr.push_back({{"id", r.id}, {"prompt", r.prompt.tokens}, {"eos_bias", r.eos_bias}, {"max_len", r.max_len}, {"seed", seed},
                       {"stream", (static_cast<uint64_t>(step) << 24) | static_cast<uint64_t>(r.id)}});
    return {{"requests", arr}};
}

json op_reward(const json & req) {
    RewardSpec spec{req.value("golden_a", 1), req.value("golden_b", 2)};
    json out = json::array();
    for (const auto & y : req.at("responses")) out.push_back(reward(y.get<std::vector<int>>(), spec));
    return {{"rewards", out}};
}

// Wall-clock timing of the reference's own run_generation (server.cpp:351-376) on
// `threads` host threads, each running its own engine on a disjoint request shard
// (SPEC.md:388). Used by bench.py as the reference CPU arm.
json op_time_generation(const json & req) {
    TabularARModel target = model_of(req.at("target"));
    auto drafter = std::make_shared<const TabularARModel>(model_of(req.at("drafter")));
    const TimingModel tm = timing_of(req.value("timing", json()));
    const SDConfig forced = cfg_of(req.value("forced", json::object()));
    std::vector<RequestState> all = requests_of(req.at("requests"));
    const int threads = std::max(1, req.value("threads", 1));
    std::vector<std::vector<RequestState>> shards(static_cast<size_t>(threads));
    for (size_t i = 0; i < all.size(); ++i) shards[i % static_cast<size_t>(threads)].push_back(std::move(all[i]));
    std::vector<long> tokens(static_cast<size_t>(threads), 0), al_sum(static_cast<size_t>(threads), 0), al_n(static_cast<size_t>(threads), 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t]() {
            DrafterSnapshotFn snap = [drafter]() { return drafter; };
            GenerationRun run = run_generation(std::move(shards[static_cast<size_t>(t)]), target, snap, nullptr, tm, forced, 0);
            for (const auto & s : run.samples) tokens[static_cast<size_t>(t)] += static_cast<long>(s.response.size());
            for (int a : run.accept_lens) al_sum[static_cast<size_t>(t)] += a;
            al_n[static_cast<size_t>(t)] += static_cast<long>(run.accept_lens.size());
        });
    }
    for (auto & th : pool) th.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    long tok = 0, as = 0, an = 0;
    for (int t = 0; t < threads; ++t) { tok += tokens[static_cast<size_t>(t)]; as += al_sum[static_cast<size_t>(t)]; an += al_n[static_cast<size_t>(t)]; }
    return {{"seconds", secs}, {"tokens", tok}, {"accept_len_sum", as}, {"accept_len_cycles", an}, {"threads", threads}};
}

RolloutSample sample_of(const json & s) {
    RolloutSample r;
    r.prompt = s.at("prompt").get<std::vector<int>>();
    r.response = s.at("response").get<std::vector<int>>();
    if (s.contains("steps"))
        for (const auto & st : s.at("steps")) {
            StepRecord rec;
            rec.token = st.value("token", 0);
            if (st.contains("target_logprobs")) rec.target_logprobs = st.at("target_logprobs").get<std::vector<double>>();
            r.steps.push_back(std::move(rec));
        }
    r.eos_bias = s.value("eos_bias", 0.0);
    r.reward = s.value("reward", 0.0);
    r.actor_version = s.value("actor_version", 0);
    return r;
}

KDPolicy policy_of(const json & pj) {
    const std::string mode = pj.value("mode", "reward");
    return KDPolicy{pj.value("interval", 1), mode == "uniform" ? WeightMode::Uniform : mode == "frozen" ? WeightMode::Frozen : WeightMode::Reward,
                    pj.value("clip_lo", 0.0), pj.value("clip_hi", 4.0), pj.value("lr", 0.1)};
}

json learner_metrics_json(const std::vector<LearnerMetrics> & ms) {
    json out = json::array();
    for (const auto & m : ms)
        out.push_back({{"update", m.update_idx}, {"drafter_version", m.drafter_version}, {"kd_loss", m.kd_loss},
                       {"samples", m.samples_used}, {"weight_mean", m.weight_mean}, {"weight_min", m.weight_min},
                       {"weight_max", m.weight_max}, {"weights_l2", m.weights_l2}});
    return out;
}

// OnlineLearner driven by a script of iterations: {"feed": [samples], "boundary": it, "await": bool}.
// generate (specdec.cpp:271-316) on one sequence, plus mean_accept_len.
// kd_loss_gradient + per-sample kd_loss over an explicit (sample, weight) list (learner.cpp:33-82).
json op_kd_grad(const json & req) {
    TabularARModel drafter = model_of(req.at("drafter"));
    std::vector<RolloutSample> samples;
    for (const auto & s : req.at("samples")) samples.push_back(sample_of(s));
    const auto w = req.at("weights").get<std::vector<double>>();
    std::vector<std::pair<const RolloutSample *, double>> ws;
    json losses = json::array();
    for (size_t i = 0; i < samples.size(); ++i) {
        ws.emplace_back(&samples[i], w.at(i));
        losses.push_back(kd_loss(drafter, samples[i], w.at(i)));
    }
    return {{"grad", kd_loss_gradient(drafter, ws)}, {"losses", losses}};
}

json op_generate(const json & req) {
    TabularARModel target = model_of(req.at("target"));
    TabularARModel drafter = model_of(req.at("drafter"));
    DecodeRng rng = DecodeRng::from_seed(req.at("seed").get<uint64_t>(), req.value("stream", uint64_t{0}));
    GenerateResult g = generate(target, drafter, Context{req.at("prompt").get<std::vector<int>>()}, cfg_of(req.at("cfg")),
                                req.at("max_len").get<int>(), rng, req.value("eos_bias", 0.0), req.value("stop_at_eos", true));
    json steps = json::array();
    for (const auto & st : g.steps) steps.push_back(step_json(st, false));
    json ledger = json::array();
    for (const auto & e : g.ledger.events) ledger.push_back({e.role == ModelRole::Target ? 1 : 0, e.positions_evaluated, e.concurrent_batch_tokens});
    json out = {{"tokens", g.tokens}, {"steps", steps}, {"accept_lens", g.accept_lens}, {"ledger", ledger}, {"ended_eos", g.ended_eos}};
    if (!g.accept_lens.empty()) out["mean_accept_len"] = mean_accept_len(g.accept_lens);
    return out;
}

json op_online_learner(const json & req) {
    OnlineLearner l(model_of(req.at("drafter")), policy_of(req.at("policy")), req.at("selection_seed").get<uint64_t>(),
                    req.value("cost_per_token", 0.0), req.value("capacity", size_t{4096}), req.value("async", false));
    json states = json::array();
    for (const auto & it : req.at("script")) {
        std::vector<RolloutSample> batch;
        for (const auto & s : it.value("feed", json::array())) batch.push_back(sample_of(s));
        l.feed(std::move(batch));
        json st = {{"buffer_after_feed", l.buffer_size()}};
        if (it.contains("boundary")) l.on_iteration_boundary(it.at("boundary").get<int>());
        if (it.value("await", true)) l.await_pending();
        st["version"] = l.drafter_version();
        st["buffer"] = l.buffer_size();
        st["updates"] = l.metrics().size();
        states.push_back(st);
    }
    l.await_pending();
    json out = {{"states", states}, {"metrics", learner_metrics_json(l.metrics())}, {"total_sim_time", l.total_sim_time()},
                {"logits", l.snapshot()->logits()}, {"version", l.drafter_version()}};
    l.shutdown();
    return out;
}

json op_policy_update(const json & req) {
    TabularARModel actor = model_of(req.at("actor"));
    std::vector<RolloutSample> samples;
    for (const auto & s : req.at("samples")) samples.push_back(sample_of(s));
    std::vector<std::pair<const RolloutSample *, double>> w;
    const auto adv = req.at("advantages").get<std::vector<double>>();
    for (size_t i = 0; i < samples.size(); ++i) w.emplace_back(&samples[i], adv.at(i));
    TabularARModel next = policy_update(actor, w, req.value("lr", 0.2));
    return {{"logits", next.logits()}, {"version", next.version()}, {"objective", policy_objective(actor, w)}};
}

json op_group_advantages(const json & req) {
    return {{"advantages", group_advantages(req.at("rewards").get<std::vector<double>>())}};
}

json op_build_profile(const json & req) {
    ExperimentConfig cfg = ExperimentConfig::from_json(req.at("config"));
    Env env = make_env(cfg);
    ProfileTable t = build_profile(cfg, env.actor, env.drafter);
    return {{"json", t.to_json()}, {"csv", t.to_csv()}};
}

json op_make_env_cfg(const json & req) {
    ExperimentConfig cfg = ExperimentConfig::from_json(req.at("config"));
    Env env = make_env(cfg);
    return {{"actor", model_json(env.actor)}, {"drafter", model_json(env.drafter)}};
}

// run_scenario (scenarios.cpp:330-341) on an ExperimentConfig JSON.
json op_run_scenario(const json & req) {
    ExperimentConfig cfg = ExperimentConfig::from_json(req.at("config"));
    ScenarioResult r = run_scenario(cfg);
    json out = {{"scenario", r.scenario}, {"summary", r.summary}, {"step_lines", r.step_lines},
                {"learner_lines", r.learner_lines}, {"switch_lines", r.switch_lines}};
    if (r.table) out["table"] = {{"json", r.table->to_json()}, {"csv", r.table->to_csv()}};
    return out;
}

json op_config_roundtrip(const json & req) {
    return ExperimentConfig::from_json(req.at("config")).to_json();
}

json dispatch(const json & req) {
    const std::string op = req.at("op");
    if (op == "run_generation") return op_run_generation(req);
    if (op == "spec_step_tree") return op_spec_step_tree(req);
    if (op == "kd_update") return op_kd_update(req);
    if (op == "profile_table") return op_profile_table(req);
    if (op == "make_env") return op_make_env(req);
    if (op == "make_step_requests") return op_make_step_requests(req);
    if (op == "reward") return op_reward(req);
    if (op == "time_generation") return op_time_generation(req);
    if (op == "online_learner") return op_online_learner(req);
    if (op == "generate") return op_generate(req);
    if (op == "kd_grad") return op_kd_grad(req);
    if (op == "policy_update") return op_policy_update(req);
    if (op == "group_advantages") return op_group_advantages(req);
    if (op == "build_profile") return op_build_profile(req);
    if (op == "make_env_cfg") return op_make_env_cfg(req);
    if (op == "run_scenario") return op_run_scenario(req);
    if (op == "config_roundtrip") return op_config_roundtrip(req);
    if (op == "run_verify") return {{"ok", run_verify(req.value("seed", uint64_t{1})).all_pass}};
    throw std::invalid_argument("ref: unknown op " + op);
}

char * dup(const std::string & s) {
    char * p = static_cast<char *>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

}  // namespace

extern "C" {
char * ref_call(const char * req) {
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
void ref_free(char * p) { std::free(p); }
}

// oracle/restate.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the ReSpec rollout hot path (reference: /root/reference/proj/core).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
// code, and only as the checker. The product path (paper_2510_26475_b200/) never links it.
//
// Parity status: PINNED. tests/test_oracle.py checks this restatement against the
// compiled reference (oracle/_ref/librespec_ref.so, built from the reference sources by
// oracle/Makefile) on identical seeds/configs, and against the golden fingerprints of
// SURVEY.md Appendix B (tests/golden/).
//
// The restatement is generic over the model (the reference functions take a concrete
// TabularARModel, so they cannot drive a transformer): any object that returns a raw
// logit row for a context plugs in. It also defines the greedy-verification mode that
// the reference lacks; the reference enforces tau > 0 and has no
// greedy path (model.cpp:88-90).
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---- RNG: rng.hpp:11-47 ------------------------------------------------------------
inline double to_unit_double(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

inline uint64_t splitmix64(uint64_t & s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct DecodeRng {
    std::mt19937_64 draft, accept;
    long n_draft = 0, n_accept = 0;  // draws consumed (not in the reference; diagnostic)
    static DecodeRng from_seed(uint64_t seed, uint64_t stream) {
        uint64_t s = seed ^ (0x51ed270b8d2c7f13ULL * (stream + 1));  // rng.hpp:38
        DecodeRng r;
        r.draft.seed(splitmix64(s));   // rng.hpp:40 (sequential use of the same state)
        r.accept.seed(splitmix64(s));  // rng.hpp:41
        return r;
    }
    double du() { ++n_draft; return to_unit_double(draft()); }
    double au() { ++n_accept; return to_unit_double(accept()); }
};

// ---- models --------------------------------------------------------------------------
// A model returns the raw logit row z(ctx) (no EOS bias, no temperature); dist() applies
// both exactly as TabularARModel::next_dist does (model.cpp:132-139).
struct Model {
    int vocab = 2;
    double temperature = 1.0;
    int version = 0;
    virtual ~Model() = default;
    virtual std::vector<double> logits(const std::vector<int> & ctx) const = 0;
    // `depth` = tokens beyond the current round's root (0 at the root). Tabular models ignore
    // it; an EAGLE drafter's row depends on it (target features at the root, its own hidden
    // state deeper in the tree), so captured drafter rows are keyed by (ctx, depth).
    virtual std::vector<double> logits_at(const std::vector<int> & ctx, int /*depth*/) const { return logits(ctx); }
    int eos() const { return vocab - 1; }  // model.hpp:20
};

struct TabularModel : Model {
    int order = 0;
    std::vector<double> table;  // rows x V
    size_t row_index(const std::vector<int> & ctx) const;  // model.cpp:113-130
    std::vector<double> logits(const std::vector<int> & ctx) const override;
};

// Logit rows captured from another implementation (the CUDA engine), keyed by context.
// Used to replay the acceptance logic bit-for-bit on exactly the rows the GPU computed.
struct LookupModel : Model {
    bool depth_aware = false;
    std::map<std::pair<std::vector<int>, int>, std::vector<double>> rows;  // (ctx, depth or 0)
    // fp32 rows handed over through the binary entry (oracle_lookup_add_f32): full-vocabulary
    // rows at V ~ 152K are too large for the JSON transport
    std::map<std::pair<std::vector<int>, int>, std::vector<float>> rows32;
    std::vector<double> logits(const std::vector<int> & ctx) const override { return logits_at(ctx, 0); }
    std::vector<double> logits_at(const std::vector<int> & ctx, int depth) const override;
};

std::vector<double> softmax(const std::vector<double> & z, double tau);             // model.cpp:53-68
std::vector<double> dist(const Model & m, const std::vector<int> & ctx, double eos_bias, int depth = 0);
int sample_from(const std::vector<double> & p, double u);                           // model.cpp:23-40
int argmax_first(const std::vector<double> & p);                                     // greedy: lowest index wins ties
double accept_prob(double p, double q);                                              // specdec.cpp:25-33
std::vector<double> residual_dist(const std::vector<double> & p, const std::vector<double> & q);  // specdec.cpp:35-52

// ---- SD cycle --------------------------------------------------------------------------
struct SDConfig {
    int rounds = 1, branching = 1, draft_len = 1;
    bool enabled = false;
    int drafted_per_cycle() const { return rounds * branching * draft_len; }
    std::string key() const;
    bool operator==(const SDConfig & o) const {  // specdec.hpp:30-36
        if (!enabled && !o.enabled) return true;
        return enabled == o.enabled && rounds == o.rounds && branching == o.branching &&
               draft_len == o.draft_len;
    }
};

enum class VerifyMode { Sample, Greedy };

struct StepRecord {
    int token = 0;
    double logp = 0.0;
    bool drafted = false;
    double logq = 0.0;
    std::vector<double> target_logprobs;  // full row; kept when record_full is set
};

struct RoundCost { int drafter_forwards = 0, drafter_tokens_each = 0, target_tokens = 0; };

struct VerifyOutcome {
    std::vector<int> accepted_tokens;
    int accept_len = 0;
    int bonus_token = -1;
    int draft_records = 0;
    std::vector<StepRecord> steps;
    std::vector<RoundCost> rounds;
    bool ended = false;
};

VerifyOutcome spec_step_tree(const Model & target, const Model & drafter, const std::vector<int> & ctx,
                             const SDConfig & cfg, DecodeRng & rng, double eos_bias, bool stop_at_eos,
                             int max_emit, VerifyMode mode, bool record_full);

// ---- cost ledger / timing model: costsim.hpp:22-56, costsim.cpp:13-27 -------------------
struct RoleTiming { double unit_cost = 1.0; int saturation_tokens = 32; double latency_floor = 0.0; };
struct TimingModel { RoleTiming target{1.0, 32, 2.0}; RoleTiming drafter{0.1, 32, 0.4}; };
struct ForwardEvent { bool target; int positions; int batch_tokens; };
double forward_time(const TimingModel & tm, bool target, int tokens);
double ledger_time(const TimingModel & tm, const std::vector<ForwardEvent> & ev);

// ---- adaptive server: server.cpp:21-78, :154-178, :266-376 ----------------------------
class ProfileTable {
public:
    ProfileTable() = default;
    explicit ProfileTable(std::vector<int> buckets);
    void set_entry(int bucket, const SDConfig & cfg, double tpt);
    void finalize();
    int bucket_for(int active_batch) const;
    SDConfig solve(int active_batch) const;
    SDConfig best_for_bucket(int bucket) const;
    double entry(int bucket, const SDConfig & cfg) const;
    const std::vector<int> & buckets() const { return buckets_; }
    const std::vector<std::pair<SDConfig, double>> & entries_for(int b) const;
    std::string to_csv() const;
private:
    std::vector<int> buckets_;
    std::map<int, std::vector<std::pair<SDConfig, double>>> entries_;
    std::map<int, SDConfig> best_;
};

struct RequestState {
    int id = 0;
    std::vector<int> prompt, generated;
    double eos_bias = 0.0;
    int max_len = 1;
    bool spec_flag = false, done = false;
    DecodeRng rng;
    std::vector<StepRecord> steps;
    std::vector<int> accept_lens;
    std::vector<int> full_ctx() const;
    int remaining() const { return max_len - static_cast<int>(generated.size()); }
};

struct SwitchEvent { int cycle, active_batch; SDConfig from, to; };

class BatchEngine {
public:
    BatchEngine(const Model & target, std::function<std::shared_ptr<const Model>()> drafter,
                const ProfileTable * table, std::vector<RequestState> reqs, SDConfig forced,
                VerifyMode mode, bool record_full);
    void step();
    bool all_done() const;
    int cycles() const { return cycle_; }
    std::vector<RequestState> & requests() { return reqs_; }
    const std::vector<ForwardEvent> & ledger() const { return ledger_; }
    const std::vector<SwitchEvent> & switches() const { return switches_; }
    const std::vector<int> & active_trace() const { return active_trace_; }
    int prefill_events() const { return prefill_events_; }
    const std::vector<int> & drafter_versions() const { return drafter_versions_; }
private:
    const Model & target_;
    std::function<std::shared_ptr<const Model>()> drafter_;
    const ProfileTable * table_;
    std::vector<RequestState> reqs_;
    SDConfig mode_;
    VerifyMode vmode_;
    bool record_full_;
    bool mode_init_ = false;
    int cycle_ = 0, prefill_events_ = 0;
    std::vector<ForwardEvent> ledger_;
    std::vector<SwitchEvent> switches_;
    std::vector<int> active_trace_, drafter_versions_;
};

void charge_batched_cycle(std::vector<ForwardEvent> & ledger, const std::vector<VerifyOutcome> & outs);

// ---- KD: learner.cpp:10-160 --------------------------------------------------------------
enum class WeightMode { Reward, Uniform, Frozen };
struct KDPolicy { int interval = 1; WeightMode mode = WeightMode::Reward; double clip_lo = 0, clip_hi = 4, lr = 0.1; };
struct Rollout {
    std::vector<int> prompt, response;
    std::vector<std::vector<double>> target_logprobs;  // one full row per response token
    double eos_bias = 0.0, reward = 0.0;
};
double kd_weight(double r, const std::vector<double> & batch_rewards, const KDPolicy & p);
double kd_loss(const TabularModel & drafter, const Rollout & s, double w);
std::vector<double> kd_loss_gradient(const TabularModel & drafter,
                                     const std::vector<std::pair<const Rollout *, double>> & ws);
struct KDUpdateResult {
    std::vector<double> logits;
    bool updated = false;
    double loss = 0, weight_mean = 0, weight_min = 0, weight_max = 0, sim_time = 0;
    int samples_used = 0;
    std::vector<size_t> selected;
};
KDUpdateResult kd_update(const TabularModel & drafter, const std::vector<Rollout> & buf, const KDPolicy & p,
                         std::mt19937_64 & sel, double cost_per_token);

}  // namespace orc

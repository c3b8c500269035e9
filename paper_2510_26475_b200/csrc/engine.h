// engine.h -- host C++ side of the B200 rollout engine. Mirrors the reference's
// ProfileTable / BatchEngine / run_generation (server.hpp:21-148) and drives the device
// kernels through the launchers in sd.h (tabular) and model.h (transformer).
#pragma once
#include <atomic>
#include <mutex>
#include <stdexcept>

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/respec_b200.h"
#include "sd.h"

struct rs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace rs {

// Device buffer with RAII.
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) RS_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void ensure(size_t count) {  // grow-only: keeps the allocation when it is large enough
        if (count > n) alloc(count);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// SDConfig semantics (specdec.hpp:17-37)
inline bool cfg_eq(const rs_sdconfig &a, const rs_sdconfig &b) {
    if (!a.enabled && !b.enabled) return true;
    return (a.enabled != 0) == (b.enabled != 0) && a.rounds == b.rounds && a.branching == b.branching &&
           a.draft_len == b.draft_len;
}
inline int cfg_drafted(const rs_sdconfig &c) { return c.rounds * c.branching * c.draft_len; }
std::string cfg_key(const rs_sdconfig &c);

}  // namespace rs

// ---- models --------------------------------------------------------------------------
struct rs_model {
    enum Kind { Tabular, Transformer, Drafter } kind;
    rs_ctx *ctx = nullptr;
    int vocab = 0;
    double temperature = 1.0;
    int version = 0;
    // Handles are reference-counted: rs_model_retain adds one, rs_model_destroy drops one and
    // frees the weights at zero (learner snapshots are shared between the learner and callers).
    std::atomic<int> refs{1};
    // Process-unique id: a snapshot allocated at a freed snapshot's address is still a new
    // snapshot (engines key their drafter-cache invalidation on it, not on the pointer).
    // Loading checkpoint tensors into a model (rs_model_load_tensor) gives it a fresh id.
    uint64_t uid = next_uid();
    explicit rs_model(Kind k) : kind(k) {}
    static uint64_t next_uid() {
        static std::atomic<uint64_t> n{1};
        return n.fetch_add(1);
    }
    virtual ~rs_model() = default;
};

namespace rs {

struct TabularModel : rs_model {
    int order = 0;
    size_t rows = 1;
    DBuf<double> table;
    std::vector<double> host;  // kept for rs_tabular_logits / KD
    TabularModel() : rs_model(Tabular) {}
    TabDev dev() const { return TabDev{table.p, order, vocab}; }
};

// ProfileTable (server.cpp:21-145)
class ProfileTable {
public:
    explicit ProfileTable(std::vector<int> buckets);
    void set_entry(int bucket, const rs_sdconfig &cfg, double tpt);
    void finalize();
    int bucket_for(int active_batch) const;
    rs_sdconfig solve(int active_batch) const { return best_for_bucket(bucket_for(active_batch)); }
    rs_sdconfig best_for_bucket(int bucket) const;
    double entry(int bucket, const rs_sdconfig &cfg) const;
    std::string to_csv() const;
    const std::vector<int> &buckets() const { return buckets_; }
    std::vector<rs_sdconfig> all_configs() const;

private:
    std::vector<int> buckets_;
    std::map<int, std::vector<std::pair<rs_sdconfig, double>>> entries_;
    std::map<int, rs_sdconfig> best_;
};

// Model-side hooks of one engine (the forwards that produce logit rows).
struct KdRef {  // one request of a finished (or running) engine taking part in a KD update
    int req = 0;
    double weight = 1.0, eos_bias = 0.0;
};

struct ModelPair {
    virtual ~ModelPair() = default;
    virtual RowType row_type() const = 0;
    virtual void draft_rows(const SdDev &d, int depth, cudaStream_t st) = 0;
    virtual void verify_rows(const SdDev &d, bool naive, cudaStream_t st) = 0;
    virtual void after_accept(const SdDev &, bool /*naive*/, cudaStream_t) {}
    // Lazy verify LM head (transformer pairs): verify_rows then produced only the root rows'
    // logits; verify_rows_selected computes the chains the acceptance's branch point selected.
    virtual bool lazy_lm_head(const SdDev &) const { return false; }
    virtual void verify_rows_selected(const SdDev &, cudaStream_t) {}
    virtual void on_spec_enable(const SdDev &, cudaStream_t) {}
    virtual void set_drafter(const rs_model *) {}
    virtual void begin_step() {}
    // Online-KD loss + drafter LM-head gradient over requests' generated tokens from the
    // resident caches (transformer pairs only).
    // `stream` (or null: the engine's) carries the pass -- an asynchronous learner runs it on its own.
    virtual double kd_cached(const std::vector<KdRef> &, const rs_model *, float *, cudaStream_t = nullptr) {
        throw std::invalid_argument("kd from the engine needs a transformer target");
    }
};

std::unique_ptr<ModelPair> make_tabular_pair(const TabularModel *target, const TabularModel *drafter);
}  // namespace rs
struct rs_engine;
namespace rs {
std::unique_ptr<ModelPair> make_transformer_pair(rs_ctx *ctx, rs_engine *eng, const rs_model *target,
                                                 const rs_model *drafter, int n_req, int slots_max,
                                                 const std::vector<int> &prompt_lens,
                                                 const std::vector<std::vector<int>> &prompts, int tok_cap);

}  // namespace rs

struct rs_table {
    rs::ProfileTable t;
};

struct rs_engine {
    rs_ctx *ctx = nullptr;
    // Held while the engine's device state is in use: by step() / kd_grad on the caller's
    // thread and by a KD update that reads the engine's resident caches (possibly on an
    // asynchronous learner's worker). Overlap raises instead of corrupting the rollout.
    std::mutex use_mu;
    // Scheduled KD updates that will read this engine's resident caches: step() refuses to run
    // while any is pending (the rollout state they read must stay as it was fed).
    std::atomic<int> kd_pins{0};
    void check_unpinned(const char *what) const {
        if (kd_pins.load() > 0)
            throw std::runtime_error(std::string(what) + ": engine is read by a pending KD update (await_pending first)");
    }
    const rs_model *target = nullptr;
    const rs_model *pending_drafter = nullptr;  // snapshot read at the next step
    const rs::ProfileTable *table = nullptr;
    rs_timing_model tm{};
    rs_sdconfig mode{};
    int verify_mode = RS_VERIFY_SAMPLE;
    bool record_full = false;
    bool stop_at_eos = true;  // false: EOS neither stops a chain nor ends a request (profile waves)
    bool mode_init = false;
    int cycle = 0;
    int prefill_events = 0;
    int n = 0;
    int V = 0;
    int t_max = 1, n_max = 1, s_max = 1, slots_max = 1;
    int tok_cap = 0, steps_cap = 0;
    std::unique_ptr<rs::ModelPair> pair;

    // host mirrors
    std::vector<int> ids, prompt_len, max_len, len, done;
    std::vector<double> eos_bias;
    std::vector<std::vector<int>> accept_lens;
    std::vector<rs_forward_event> ledger;
    int ledger_group = 0;  // > 0: charge cycles per group of this many requests (profile waves)
    std::vector<std::vector<rs_forward_event>> group_ledgers;
    std::vector<rs_switch_event> switches;
    std::vector<int> active_trace, drafter_versions;
    std::vector<int> active;

    // device state
    rs::DBuf<int32_t> d_tok, d_len, d_plen, d_maxlen, d_done, d_active;
    rs::DBuf<double> d_bias;
    rs::DBuf<rs::MtStream> d_rng;
    rs::DBuf<int32_t> d_st_tok;
    rs::DBuf<double> d_st_logp, d_st_logq, d_st_full;
    rs::DBuf<uint8_t> d_st_drafted;
    rs::DBuf<int32_t> d_cyc;  // n_eff, d_used, a_used, cont, ended, accept_len, drafted, emitted, n_rounds
    rs::DBuf<int32_t> d_round_cost, d_chain;  // chain_tok, chain_len, chain_stop, chain_off
    rs::DBuf<int32_t> d_err, d_flag, d_summary, d_newtok;
    int32_t *h_newtok = nullptr;   // pinned [B][newtok_cap]: last step's emitted tokens per active slot
    int newtok_cap = 0;
    std::vector<int32_t> last_active, last_emitted;  // active slots of the last step and their counts
    rs::DBuf<char> d_P, d_Q;
    rs::DBuf<double> d_pq;          // acceptance scratch: fp64 p1 / q1 rows per active sequence
    rs::DBuf<double> d_Pst, d_Qst;  // LM-head tile softmax partials (transformer engines)
    int32_t *h_summary = nullptr;  // pinned
    int32_t *h_active = nullptr;   // pinned
    int32_t *h_misc = nullptr;     // pinned: err, flag

    // capture (debug replay against the CPU oracle)
    bool capture = false;
    std::vector<int32_t> cap_role, cap_req, cap_ctx_len, cap_ext;  // ext: up to n_max tokens
    std::vector<double> cap_logits;  // fp64 rows (tabular parity mode)
    std::vector<float> cap_f32;      // fp32 rows (transformer logits), stored as produced

    ~rs_engine();
    rs::SdDev dev(const rs_sdconfig &cfg, int nact);
    void step(rs_step_info *info);
    void capture_rows(const rs::SdDev &d, bool verify, int depth, int which);
    void verify_accept(const rs::SdDev &d, int round, rs::RowType rt, cudaStream_t st);
};

// learner.cpp -- OnlineLearner + ReplayBuffer (learner.hpp:39-139, learner.cpp:84-289) on the
// device KD update.
//
// The reference trains on a worker thread that overlaps the trainer's non-generation work and
// publishes a new immutable snapshot under a mutex; the engine picks it up at the next
// rendezvous (await_pending), so async and synchronous learners produce identical drafter
// sequences given the same selection seed. Here the update itself is the device kd_update
// (rs_kd_update_tabular / rs_kd_update_transformer). In async mode the worker owns a second
// rs_ctx -- its own CUDA stream -- so the KD kernels run concurrently with the rollout on the
// caller's stream; the worker synchronises its stream before publishing, which makes the
// published snapshot safe to read from any stream. Snapshots are reference-counted rs_model
// handles shared between the learner and its callers.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "abi.h"
#include "engine.h"
#include "kd.h"
#include "model.h"

using rs_abi::guard;
using rs_abi::need;

namespace {

struct Sample {  // RolloutSample fields the learner reads (rollout.hpp:12-20)
    std::vector<int32_t> prompt, response;
    std::vector<double> lp;  // response_len x V target log-probabilities, or empty
    double eos_bias = 0.0, reward = 0.0;
    rs_engine *eng = nullptr;  // or: request `req` of a live transformer engine (resident caches)
    int req = -1, response_len = 0;
};

struct ModelRef {  // one counted reference to an rs_model
    rs_model *m = nullptr;
    ModelRef() = default;
    explicit ModelRef(rs_model *p) : m(p) {}
    ModelRef(const ModelRef &o) : m(o.m) {
        if (m) m->refs.fetch_add(1, std::memory_order_relaxed);
    }
    ModelRef &operator=(ModelRef o) {
        std::swap(m, o.m);
        return *this;
    }
    ~ModelRef() {
        if (m && m->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) delete m;
    }
};

}  // namespace

// Engines whose resident caches a scheduled update reads are pinned (one count per sample)
// from on_iteration_boundary until that update ends; rs_engine_step refuses to run meanwhile.
void pin_engines(const std::vector<Sample> &batch, int delta) {
    for (const Sample &x : batch)
        if (x.eng) x.eng->kd_pins.fetch_add(delta);
}

struct rs_learner {
    rs_ctx *ctx = nullptr;      // caller's context (synchronous updates run on its stream)
    rs_ctx *own = nullptr;      // async worker's context (its own stream)
    rs_kd_policy policy{};
    uint64_t sel[313] = {};     // std::mt19937_64 selection_rng_ (learner.hpp:124)
    double cost = 0.0;
    size_t capacity = 0;
    std::deque<Sample> buffer;  // ReplayBuffer (learner.hpp:39-51)
    int update_idx = 0;

    mutable std::mutex mu;
    std::condition_variable cv;
    ModelRef snapshot;
    int vocab = 0;                      // of every snapshot version (fixed at creation; read
    rs_model::Kind kind = rs_model::Tabular;  // without `mu` by feed / feed_engine)
    std::vector<rs_learner_metric> metrics;
    double sim_time = 0.0;
    std::deque<std::vector<Sample>> jobs;
    bool busy = false, stopping = false, async = false;
    std::string worker_error;   // an update that failed on the worker, raised at the rendezvous
    rs::DBuf<float> grad_buf;   // drafter gradient of engine-backed updates (grow-only, one updater at a time)
    int worker_status = RS_OK;
    std::thread worker;

    // ReplayBuffer::push (learner.cpp:84-89): drop the oldest entry when full.
    void push(Sample s) {
        if (capacity == 0) return;
        if (buffer.size() == capacity) buffer.pop_front();
        buffer.push_back(std::move(s));
    }

    // kd_update (learner.cpp:98-160) for an EAGLE drafter when samples come from live engines:
    // the same selection and reward weights, the gradient of each engine's selected requests from
    // its resident KV cache / features (rs_engine_kd_grad), detached samples by the teacher-forced
    // recompute; contributions in selection order, grouped by source.
    rs_model *update_from_engines(const std::vector<Sample> &batch, const rs::DrafterModel *d, rs_ctx *c,
                                  rs_kd_result &res) {
        if (policy.mode == 2) throw std::logic_error("kd_update: frozen drafter takes no updates");
        if (policy.interval < 1) throw std::invalid_argument("kd_update: interval must be >= 1");
        const std::vector<int> idx = rs::kd_select((int)batch.size(), policy.interval, sel);
        std::vector<double> br(idx.size()), w(idx.size());
        for (size_t i = 0; i < idx.size(); ++i) br[i] = batch[idx[i]].reward;
        double wsum = 0, wmin = 0, wmax = 0;
        size_t distilled = 0;
        for (size_t i = 0; i < idx.size(); ++i) {
            w[i] = rs::kd_weight(batch[idx[i]].reward, br, policy);
            wsum += w[i];
            wmin = i == 0 ? w[i] : std::min(wmin, w[i]);
            wmax = i == 0 ? w[i] : std::max(wmax, w[i]);
            distilled += (size_t)std::max(0, batch[idx[i]].response_len);
        }
        const auto *t = d->target;
        rs::DBuf<float> &grad = grad_buf;  // kept across updates (1.6 GB at 3B: no per-update cudaMalloc)
        grad.ensure(rs::drafter_grad_layout(t->s).total);
        RS_CUDA(cudaMemsetAsync(grad.p, 0, grad.bytes(), c->stream));
        double loss = 0.0;
        size_t i = 0;
        while (i < idx.size()) {
            const Sample &s0 = batch[idx[i]];
            size_t j = i;
            if (s0.eng) {
                std::vector<rs::KdRef> refs;
                for (; j < idx.size() && batch[idx[j]].eng == s0.eng; ++j)
                    if (batch[idx[j]].response_len > 0)
                        refs.push_back(rs::KdRef{batch[idx[j]].req, w[j], batch[idx[j]].eos_bias});
                if (!refs.empty()) {
                    if (!s0.eng->pair) throw std::runtime_error("OnlineLearner: engine has no model pair");
                    std::lock_guard<std::mutex> lk(s0.eng->use_mu);  // kd_cached uses the engine's scratch
                    loss += s0.eng->pair->kd_cached(refs, d, grad.p, c->stream);
                    RS_CUDA(cudaStreamSynchronize(c->stream));  // its caches are read before the engine moves on
                }
            } else {
                std::vector<rs::KdSeq> seqs;
                for (; j < idx.size() && !batch[idx[j]].eng; ++j) {
                    const Sample &x = batch[idx[j]];
                    if (x.response.empty()) continue;
                    rs::KdSeq q;
                    q.tokens = x.prompt;
                    q.tokens.insert(q.tokens.end(), x.response.begin(), x.response.end());
                    q.prompt_len = (int)x.prompt.size();
                    q.eos_bias = x.eos_bias;
                    q.weight = w[j];
                    seqs.push_back(std::move(q));
                }
                if (!seqs.empty()) loss += rs::kd_grad_transformer(c, t, d, seqs, grad.p, false);
            }
            i = j;
        }
        rs_model *out = rs::drafter_apply_lm_grad(c, d, grad.p, -policy.lr);
        res.updated = 1;
        res.samples_used = (int)idx.size();
        res.loss = loss;
        res.weight_mean = idx.empty() ? 0.0 : wsum / (double)idx.size();
        res.weight_min = wmin;
        res.weight_max = wmax;
        res.sim_time = cost * (double)distilled;
        return out;
    }

    // OnlineLearner::do_update (learner.cpp:256-289).
    void do_update(const std::vector<Sample> &batch, rs_ctx *c) {
        ModelRef base;
        {
            std::lock_guard<std::mutex> lock(mu);
            base = snapshot;
        }
        const bool from_engines =
            base.m->kind == rs_model::Drafter &&
            std::any_of(batch.begin(), batch.end(), [](const Sample &x) { return x.eng != nullptr; });
        std::vector<rs_kd_sample> arr(batch.size());
        for (size_t i = 0; i < batch.size(); ++i) {
            const Sample &s = batch[i];
            arr[i] = rs_kd_sample{s.prompt.data(), (int32_t)s.prompt.size(), s.response.data(),
                                  (int32_t)s.response.size(), s.lp.empty() ? nullptr : s.lp.data(), s.eos_bias,
                                  s.reward};
        }
        rs_model *out = nullptr;
        rs_kd_result res{};
        int st = RS_OK;
        if (from_engines) {
            out = update_from_engines(batch, static_cast<const rs::DrafterModel *>(base.m), c, res);
        } else if (base.m->kind == rs_model::Tabular) {
            st = rs_kd_update_tabular(c, base.m, arr.data(), (int32_t)arr.size(), policy, sel, cost, &out, &res);
        } else {
            const auto *d = static_cast<const rs::DrafterModel *>(base.m);
            st = rs_kd_update_transformer(c, d->target, base.m, arr.data(), (int32_t)arr.size(), policy, sel, cost,
                                          &out, &res);
        }
        rs_abi::rethrow(st);
        ModelRef next(out);
        if (!res.updated) return;
        RS_CUDA(cudaStreamSynchronize(c->stream));  // the snapshot is complete before it is published
        double l2 = 0.0;
        if (next.m->kind == rs_model::Tabular) {
            for (double w : static_cast<const rs::TabularModel *>(next.m)->host) l2 += w * w;
            l2 = std::sqrt(l2);
        } else {
            const auto *d = static_cast<const rs::DrafterModel *>(next.m);
            l2 = rs::weights_l2_bf16(d->lm_w, (size_t)d->s.V * d->s.d, c->stream);
        }
        next.m->ctx = ctx;
        std::lock_guard<std::mutex> lock(mu);
        snapshot = next;
        sim_time += res.sim_time;
        metrics.push_back(rs_learner_metric{update_idx++, snapshot.m->version, res.loss, res.samples_used,
                                             res.weight_mean, res.weight_min, res.weight_max, l2});
    }

    // OnlineLearner::worker_loop (learner.cpp:233-254).
    void worker_loop() {
        cudaSetDevice(own->device);
        for (;;) {
            std::vector<Sample> batch;
            {
                std::unique_lock<std::mutex> lock(mu);
                cv.wait(lock, [this] { return stopping || !jobs.empty(); });
                if (jobs.empty()) return;  // stopping with the queue drained
                batch = std::move(jobs.front());
                jobs.pop_front();
                busy = true;
            }
            int st = guard([&] { do_update(batch, own); });
            pin_engines(batch, -1);
            {
                std::lock_guard<std::mutex> lock(mu);
                busy = false;
                if (st != RS_OK && worker_status == RS_OK) {
                    worker_status = st;
                    worker_error = rs_abi::last_error();
                }
            }
            cv.notify_all();
        }
    }

    void raise_worker_error() {
        std::lock_guard<std::mutex> lock(mu);
        if (worker_status == RS_OK) return;
        rs_abi::last_error() = worker_error;
        const int st = worker_status;
        worker_status = RS_OK;
        rs_abi::rethrow(st);
    }

    void shutdown() {
        if (async && worker.joinable()) {
            {
                std::lock_guard<std::mutex> lock(mu);
                stopping = true;
            }
            cv.notify_all();
            worker.join();
        }
    }

    ~rs_learner() {
        shutdown();
        if (own) rs_ctx_destroy(own);
    }
};

extern "C" {

int rs_learner_create(rs_ctx *ctx, const rs_model *drafter, rs_kd_policy policy, uint64_t selection_seed,
                      double sim_cost_per_token, int64_t buffer_capacity, int32_t async, rs_learner **out) {
    return guard([&] {
        need(ctx, "rs_learner_create");
        need(drafter, "rs_learner_create: drafter");
        need(out, "rs_learner_create: out");
        if (drafter->kind == rs_model::Transformer)
            throw std::invalid_argument("OnlineLearner: drafter must be a tabular or EAGLE drafter model");
        if (buffer_capacity < 0) throw std::invalid_argument("OnlineLearner: buffer capacity must be >= 0");
        auto l = std::make_unique<rs_learner>();
        l->ctx = ctx;
        l->policy = policy;
        rs_abi::rethrow(rs_mt19937_64_seed(selection_seed, l->sel));
        l->cost = sim_cost_per_token;
        l->capacity = (size_t)buffer_capacity;
        auto *m = const_cast<rs_model *>(drafter);
        m->refs.fetch_add(1, std::memory_order_relaxed);
        l->snapshot = ModelRef(m);
        l->vocab = m->vocab;
        l->kind = m->kind;
        l->async = async != 0;
        if (l->async) {
            rs_abi::rethrow(rs_ctx_create(ctx->device, &l->own));
            // the update is background work: its stream gets the LEAST priority, so the block
            // scheduler hands freed SMs to the rollout's kernels first and the KD kernels fill the
            // gaps (with equal priorities the two streams' kernels interleave and every rollout
            // step waits behind KD CTAs)
            int least = 0, greatest = 0;
            RS_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            RS_CUDA(cudaStreamDestroy(l->own->stream));
            RS_CUDA(cudaStreamCreateWithPriority(&l->own->stream, cudaStreamNonBlocking, least));
            rs_learner *raw = l.get();
            l->worker = std::thread([raw] { raw->worker_loop(); });
        }
        *out = l.release();
    });
}

int rs_learner_destroy(rs_learner *l) {
    return guard([&] { delete l; });
}

// OnlineLearner::feed (learner.cpp:178-182): every sample is copied into the replay buffer.
int rs_learner_feed(rs_learner *l, const rs_kd_sample *samples, int32_t n) {
    return guard([&] {
        need(l, "rs_learner_feed");
        if (n > 0) need(samples, "rs_learner_feed: samples");
        const int V = l->vocab;
        for (int i = 0; i < n; ++i) {
            const rs_kd_sample &x = samples[i];
            if (x.prompt_len < 0 || x.response_len < 0) throw std::invalid_argument("feed: negative length");
            Sample s;
            s.prompt.assign(x.prompt, x.prompt + x.prompt_len);
            s.response.assign(x.response, x.response + x.response_len);
            if (x.target_logprobs) s.lp.assign(x.target_logprobs, x.target_logprobs + (size_t)x.response_len * V);
            s.eos_bias = x.eos_bias;
            s.reward = x.reward;
            s.response_len = x.response_len;
            l->push(std::move(s));
        }
    });
}

// Samples backed by a live transformer engine: request req[i] (prompt = its prompt, response =
// its generated tokens, its EOS bias) with reward[i]. Updates then read the engine's resident
// caches instead of recomputing the prompts; the engine must outlive them and must not be
// stepped while one is pending.
int rs_learner_feed_engine(rs_learner *l, rs_engine *e, const int32_t *req, const double *reward, int32_t n) {
    return guard([&] {
        need(l, "rs_learner_feed_engine");
        need(e, "rs_learner_feed_engine: engine");
        if (n > 0) {
            need(req, "rs_learner_feed_engine: requests");
            need(reward, "rs_learner_feed_engine: rewards");
        }
        if (l->kind != rs_model::Drafter || e->target->kind != rs_model::Transformer)
            throw std::invalid_argument("OnlineLearner: engine samples need an EAGLE drafter and a transformer engine");
        for (int i = 0; i < n; ++i) {
            if (req[i] < 0 || req[i] >= e->n) throw std::invalid_argument("feed: request index out of range");
            Sample s;
            s.eng = e;
            s.req = req[i];
            s.response_len = e->len[req[i]] - e->prompt_len[req[i]];
            s.eos_bias = e->eos_bias[req[i]];
            s.reward = reward[i];
            l->push(std::move(s));
        }
    });
}

// OnlineLearner::on_iteration_boundary (learner.cpp:184-203).
int rs_learner_on_iteration_boundary(rs_learner *l, int32_t iteration) {
    return guard([&] {
        need(l, "rs_learner_on_iteration_boundary");
        l->raise_worker_error();
        if (l->policy.mode == 2) return;  // Frozen
        if (l->policy.interval < 1) throw std::invalid_argument("kd_update: interval must be >= 1");
        if ((iteration + 1) % l->policy.interval != 0) return;
        std::vector<Sample> batch(std::make_move_iterator(l->buffer.begin()), std::make_move_iterator(l->buffer.end()));
        l->buffer.clear();
        if (batch.empty()) return;
        pin_engines(batch, +1);
        if (!l->async) {
            struct Unpin {
                std::vector<Sample> &b;
                ~Unpin() { pin_engines(b, -1); }
            } unpin{batch};
            l->do_update(batch, l->ctx);
            return;
        }
        {
            std::lock_guard<std::mutex> lock(l->mu);
            l->jobs.push_back(std::move(batch));
        }
        l->cv.notify_all();
    });
}

// OnlineLearner::await_pending (learner.cpp:205-211).
int rs_learner_await_pending(rs_learner *l) {
    return guard([&] {
        need(l, "rs_learner_await_pending");
        if (l->async) {
            std::unique_lock<std::mutex> lock(l->mu);
            l->cv.wait(lock, [l] { return l->jobs.empty() && !l->busy; });
        }
        l->raise_worker_error();
    });
}

// OnlineLearner::shutdown (learner.cpp:213-222): drains pending updates, no final partial update.
int rs_learner_shutdown(rs_learner *l) {
    return guard([&] {
        need(l, "rs_learner_shutdown");
        l->shutdown();
        l->raise_worker_error();
    });
}

int rs_learner_snapshot(const rs_learner *l, rs_model **out) {
    return guard([&] {
        need(l, "rs_learner_snapshot");
        need(out, "rs_learner_snapshot: out");
        std::lock_guard<std::mutex> lock(l->mu);
        l->snapshot.m->refs.fetch_add(1, std::memory_order_relaxed);
        *out = l->snapshot.m;
    });
}

int rs_learner_drafter_version(const rs_learner *l, int32_t *out) {
    return guard([&] {
        need(l, "rs_learner_drafter_version");
        std::lock_guard<std::mutex> lock(l->mu);
        *out = l->snapshot.m->version;
    });
}

int rs_learner_total_sim_time(const rs_learner *l, double *out) {
    return guard([&] {
        need(l, "rs_learner_total_sim_time");
        std::lock_guard<std::mutex> lock(l->mu);
        *out = l->sim_time;
    });
}

int rs_learner_buffer_size(const rs_learner *l, int64_t *out) {
    return guard([&] {
        need(l, "rs_learner_buffer_size");
        *out = (int64_t)l->buffer.size();
    });
}

int rs_learner_metrics(const rs_learner *l, rs_learner_metric *out, int32_t cap, int32_t *n) {
    return guard([&] {
        need(l, "rs_learner_metrics");
        need(n, "rs_learner_metrics: n");
        std::lock_guard<std::mutex> lock(l->mu);
        *n = (int32_t)l->metrics.size();
        for (int32_t i = 0; i < std::min<int32_t>(cap, *n); ++i) out[i] = l->metrics[i];
    });
}

}  // extern "C"

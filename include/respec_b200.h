/*
 * respec_b200.h -- C-ABI of the B200-native ReSpec rollout hot path.
 *
 * The reference (/root/reference/proj/core) exposes this path as C++ value-type functions
 * in the static library respec_core; it has no FFI. These entry points
 * are what a reference-side binding would call instead; each one names the reference
 * interface it replaces. Conventions:
 *   - every function returns RS_OK (0) or an error code; rs_last_error() returns the
 *     thread-local message, verbatim from the reference where the reference throws
 *     (e.g. "BatchEngine: empty batch", server.cpp:274).
 *   - plain pointers + sizes only; all buffers passed in are HOST memory unless the
 *     parameter name ends in _dev.
 *   - handles are not thread-safe; use one rs_ctx per host thread / GPU.
 */
#ifndef RESPEC_B200_H
#define RESPEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_OK 0
#define RS_EINVAL 1 /* std::invalid_argument in the reference */
#define RS_ESTATE 2 /* std::runtime_error */
#define RS_ELOGIC 3 /* std::logic_error */
#define RS_ECUDA 4  /* CUDA launch / runtime failure */
#define RS_ENOMEM 5

#define RS_VERIFY_SAMPLE 0 /* lossless rejection sampling, specdec.cpp:197-267 */
#define RS_VERIFY_GREEDY 1 /* greedy verification (not in the reference) */

#define RS_DTYPE_BF16 0 /* host tensor elements: bf16 bit patterns (uint16) */
#define RS_DTYPE_F32 1  /* host tensor elements: fp32 */

typedef struct rs_ctx rs_ctx;       /* one GPU + stream + scratch */
typedef struct rs_model rs_model;   /* immutable device-resident model (tabular or transformer) */
typedef struct rs_table rs_table;   /* ProfileTable, server.hpp:21-49 */
typedef struct rs_engine rs_engine; /* BatchEngine, server.hpp:98-132 */
typedef struct rs_learner rs_learner; /* OnlineLearner, learner.hpp:87-139 */
typedef struct rs_comm rs_comm;     /* one rank of an NCCL communicator (drafter-gradient all-reduce) */

/* SDConfig (specdec.hpp:17-37). enabled=0 is the non-spec configuration. */
typedef struct {
    int32_t rounds;    /* s */
    int32_t branching; /* t */
    int32_t draft_len; /* n */
    int32_t enabled;
} rs_sdconfig;

/* RoleTiming / TimingModel (costsim.hpp:34-53): the simulated ledger is kept for parity. */
typedef struct {
    double unit_cost;
    int32_t saturation_tokens;
    double latency_floor;
} rs_role_timing;
typedef struct {
    rs_role_timing target;
    rs_role_timing drafter;
} rs_timing_model;

/* RequestState (server.hpp:69-83); rng = DecodeRng::from_seed(seed, stream_id) (rng.hpp:37-43). */
typedef struct {
    int32_t id;
    const int32_t *prompt;
    int32_t prompt_len;
    double eos_bias;
    int32_t max_len;
    uint64_t seed;
    uint64_t stream_id;
} rs_request;

/* SwitchEvent (server.hpp:85-90). */
typedef struct {
    int32_t cycle;
    int32_t active_batch;
    rs_sdconfig from;
    rs_sdconfig to;
} rs_switch_event;

/* ForwardEvent (costsim.hpp:14-20); role 1 = target, 0 = drafter. */
typedef struct {
    int32_t role;
    int32_t positions;
    int32_t batch_tokens;
} rs_forward_event;

/* Per-step summary returned by rs_engine_step (not in the reference: measured, not simulated). */
typedef struct {
    int32_t active_batch;
    rs_sdconfig mode;
    int32_t drafter_version;
    int32_t emitted_tokens;   /* tokens appended across the batch this step */
    int32_t drafted_cycles;   /* sequences whose cycle drafted (accept_len recorded) */
    int32_t accepted_drafted; /* sum of accept_len over those sequences */
    int32_t redraft_passes;   /* extra drafting passes for EOS-truncated chains (sampling) */
    float step_ms;            /* device time of the step, CUDA events on the engine stream */
    int64_t h2d_bytes;        /* host->device bytes copied during the step (descriptors, active set) */
    int64_t d2h_bytes;        /* device->host bytes copied during the step (summary, flags) */
} rs_step_info;

/* Transformer shape (Qwen2-style target; EAGLE-3-style drafter uses the same d/heads). */
typedef struct {
    int32_t vocab;
    int32_t d_model;
    int32_t n_layers;
    int32_t n_heads;
    int32_t n_kv_heads;
    int32_t head_dim;
    int32_t d_ff;
    int32_t max_ctx;   /* KV capacity per sequence (prompt + max_len + tree slots) */
    float rope_theta;
    float rms_eps;
    float init_std;    /* synthetic weights ~ N(0, init_std) */
    float logit_scale; /* LM-head output scale (synthetic weights) */
    double temperature;
} rs_transformer_shape;

/* KDPolicy (learner.hpp:17-23); mode 0 = Reward, 1 = Uniform, 2 = Frozen. */
typedef struct {
    int32_t interval;
    int32_t mode;
    double clip_lo;
    double clip_hi;
    double lr;
} rs_kd_policy;

/* One RolloutSample (rollout.hpp:12-20) for the KD learner; target_logprobs is
   response_len x vocab (the StepRecord::target_logprobs rows, specdec.hpp:42). */
typedef struct {
    const int32_t *prompt;
    int32_t prompt_len;
    const int32_t *response;
    int32_t response_len;
    const double *target_logprobs;
    double eos_bias;
    double reward;
} rs_kd_sample;

/* KDUpdateResult (learner.hpp:53-62). */
typedef struct {
    int32_t updated;
    int32_t samples_used;
    double loss;
    double weight_mean;
    double weight_min;
    double weight_max;
    double sim_time;
} rs_kd_result;

/* ---- errors / version ---------------------------------------------------------------- */
const char *rs_last_error(void);
int rs_version(void);
/* Number of CUDA kernel launches issued by this thread since the last reset. */
int64_t rs_launch_count(void);
void rs_launch_count_reset(void);

/* ---- context ------------------------------------------------------------------------- */
/* A context owns a non-blocking stream at the device's GREATEST priority (the rollout path is
   latency-critical); an asynchronous learner's worker context runs at the LEAST priority, so its
   update fills gaps instead of delaying rollout kernels. rs_ctx_set_stream replaces the stream. */
int rs_ctx_create(int device, rs_ctx **out);
int rs_ctx_destroy(rs_ctx *ctx);
int rs_ctx_sync(rs_ctx *ctx);
/* Run subsequent work on an externally owned cudaStream_t (e.g. torch's current stream). */
int rs_ctx_set_stream(rs_ctx *ctx, void *cuda_stream);

/* ---- models -------------------------------------------------------------------------- */
/* TabularARModel(vocab, order, logits, temperature, version) -- model.hpp:105-108. The
   rows x vocab table is copied to HBM in fp64 ("parity mode"). */
int rs_tabular_create(rs_ctx *ctx, int32_t vocab, int32_t order, double temperature, const double *logits,
                      int32_t version, rs_model **out);
/* TabularARModel::logits() -- model.hpp:118 */
int rs_tabular_logits(const rs_model *m, double *out, int64_t n);
/* Qwen2-shaped target with synthetic N(0, init_std) weights generated on device from seed. */
int rs_transformer_create(rs_ctx *ctx, const rs_transformer_shape *shape, uint64_t seed, rs_model **out);
/* EAGLE-3-style drafter bound to a target (consumes the target's low/mid/high hidden states). */
int rs_drafter_create(rs_ctx *ctx, const rs_model *target, uint64_t seed, int32_t version, rs_model **out);
int rs_model_version(const rs_model *m, int32_t *out);
int rs_model_vocab(const rs_model *m, int32_t *out);
/* Model handles are reference-counted: destroy drops one reference (the weights are freed at
   zero), retain adds one (learner snapshots are shared between the learner and its callers). */
int rs_model_destroy(rs_model *m);
/* TabularARModel::random (model.cpp:102-111): scale * N(0,1) logits from std::mt19937_64(seed)
   through std::normal_distribution (host standard library; bit-identical to the reference build). */
int rs_tabular_random(rs_ctx *ctx, int32_t vocab, int32_t order, double temperature, double scale, uint64_t seed,
                      rs_model **out);
/* make_skew_requests' per-request EOS biases (scenarios.cpp:175-189): 2.5 - 2.2 * Exp(1) draws
   from std::exponential_distribution over std::mt19937_64(seed). */
int rs_skew_eos_biases(uint64_t seed, int32_t n, double *out);
int rs_model_retain(rs_model *m);

/* ---- ProfileTable (server.hpp:21-49, server.cpp:21-145) -------------------------------- */
/* profile() (server.cpp:182-239) with MEASURED latency instead of ledger_time: for every bucket
   b and config c, a wave of exactly b synthetic requests (prompt_len tokens, EOS suppressed so no
   request finishes, as stop_at_eos = false does in the reference) runs `warmup` + `cycles` engine
   steps with c forced; time_per_token[ib * nc + ic] = measured device ms of the `cycles` steps /
   tokens they emitted. The caller builds the ProfileTable from it (rs_table_set_entry). */
int rs_profile_measured(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const int32_t *buckets,
                        int32_t nb, const rs_sdconfig *cfgs, int32_t nc, int32_t prompt_len, int32_t warmup,
                        int32_t cycles, uint64_t seed, double *time_per_token);
/* profile() (server.cpp:182-239) with the reference's SIMULATED cost model on the GPU engine:
   configs = {off} + grid; per bucket b and config, waves of exactly b requests over a pool of
   num_requests (prompt rid % n_prompts from the flattened `prompts` with n_prompts + 1
   `prompt_off` offsets, DecodeRng::from_seed(seed, rid), eos_bias 0) run cycles_per_request
   cycles with stop_at_eos = false; time_per_token[ib * (ng + 1) + ic] = ledger_time of all
   waves' forward events / emitted tokens. */
int rs_profile_simulated(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_sdconfig *grid,
                         int32_t ng, const int32_t *prompts, const int32_t *prompt_off, int32_t n_prompts,
                         const rs_timing_model *tm, const int32_t *buckets, int32_t nb, int32_t cycles_per_request,
                         int32_t num_requests, uint64_t seed, double *time_per_token);
int rs_table_create(const int32_t *buckets, int32_t n, rs_table **out);
int rs_table_set_entry(rs_table *t, int32_t bucket, rs_sdconfig cfg, double time_per_token);
int rs_table_finalize(rs_table *t);
int rs_table_bucket_for(const rs_table *t, int32_t active_batch, int32_t *out);
int rs_table_solve(const rs_table *t, int32_t active_batch, rs_sdconfig *out);
int rs_table_best_for_bucket(const rs_table *t, int32_t bucket, rs_sdconfig *out);
int rs_table_entry(const rs_table *t, int32_t bucket, rs_sdconfig cfg, double *out);
/* ProfileTable::to_csv (server.cpp:136-145); writes at most cap bytes incl. NUL, *len = full length. */
int rs_table_to_csv(const rs_table *t, char *buf, int64_t cap, int64_t *len);
int rs_table_destroy(rs_table *t);

/* ---- BatchEngine / run_generation (server.hpp:98-148, server.cpp:266-376) ------------- */
/* table == NULL selects fixed mode with `forced`; drafter may be NULL when forced is off.
   The target is borrowed and must outlive the engine (server.hpp:119). */
int rs_engine_create(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_table *table,
                     const rs_timing_model *tm, const rs_request *reqs, int32_t n, rs_sdconfig forced,
                     int32_t verify_mode, int32_t record_full_logprobs, rs_engine **out);
/* DrafterSnapshotFn (server.hpp:92): the snapshot is read once, at the next step boundary. */
int rs_engine_set_drafter(rs_engine *e, const rs_model *drafter);
/* stop_at_eos = 0 (before the first step): EOS neither stops a drafted chain nor ends a request
   (spec_step_tree(..., stop_at_eos = false), as profile() runs it, server.cpp:215). */
int rs_engine_set_stop_at_eos(rs_engine *e, int32_t stop);
/* A request's DecodeRng (draft + accept mt19937_64 streams) as an opaque image of `n` words
   (query n with out = NULL): export after a step, import into a new engine before its first
   step -- spec_step_tree's DecodeRng& continuation across calls (rng.hpp:33-47). */
int rs_engine_rng_export(const rs_engine *e, int32_t req, uint64_t *out, int64_t cap, int64_t *n);
int rs_engine_rng_import(rs_engine *e, int32_t req, const uint64_t *in, int64_t n);
/* BatchEngine::step (server.cpp:266-349); throws "BatchEngine: empty batch" when done. */
int rs_engine_step(rs_engine *e, rs_step_info *info);
int rs_engine_all_done(const rs_engine *e, int32_t *out);
int rs_engine_active_batch(const rs_engine *e, int32_t *out);
int rs_engine_cycles(const rs_engine *e, int32_t *out);
int rs_engine_prefill_events(const rs_engine *e, int32_t *out);
int rs_engine_ledger_time(const rs_engine *e, double *out);
int rs_engine_ledger(const rs_engine *e, rs_forward_event *out, int32_t cap, int32_t *n);
int rs_engine_switches(const rs_engine *e, rs_switch_event *out, int32_t cap, int32_t *n);
int rs_engine_active_trace(const rs_engine *e, int32_t *out, int32_t cap, int32_t *n);
int rs_engine_drafter_versions(const rs_engine *e, int32_t *out, int32_t cap, int32_t *n);
/* RolloutSample fields of request `req` (request order, server.cpp:365-374). */
int rs_engine_response(rs_engine *e, int32_t req, int32_t *tokens, int32_t cap, int32_t *len);
/* The tokens emitted by the LAST rs_engine_step, per active request of that step (host copy that
   arrived with the step summary -- no device access): req[a], count[a] and
   tokens[a * cap_per_req + 0 .. count[a]); n = active requests of that step. */
int rs_engine_step_tokens(rs_engine *e, int32_t *req, int32_t *count, int32_t *tokens, int32_t cap_per_req,
                          int32_t *n);
int rs_engine_steps(rs_engine *e, int32_t req, double *logp, uint8_t *drafted, double *logq, int32_t cap, int32_t *n);
int rs_engine_step_logprobs(rs_engine *e, int32_t req, double *out, int64_t cap, int32_t *rows);
int rs_engine_accept_lens(rs_engine *e, int32_t req, int32_t *out, int32_t cap, int32_t *n);
int rs_engine_destroy(rs_engine *e);
/* Debug: capture the logit rows of the next steps (for replay against the CPU oracle). */
int rs_engine_set_capture(rs_engine *e, int32_t enable);
int rs_engine_capture_count(const rs_engine *e, int64_t *rows, int32_t *vocab, int32_t *ext_width);
int rs_engine_capture_read(rs_engine *e, int64_t first, int64_t count, int32_t *role, int32_t *req,
                           int32_t *ctx_len, int32_t *ext, double *logits);
/* Same rows, fp32 as the transformer LM heads produced them (count * vocab floats); fails
   with RS_EINVAL for fp64 (tabular) rows. Metadata via rs_engine_capture_read(..., NULL). */
int rs_engine_capture_read_f32(rs_engine *e, int64_t first, int64_t count, float *logits);

/* ---- KD learner (learner.hpp:27-69, learner.cpp:10-160) -------------------------------- */
double rs_kd_weight(double r, const double *batch_rewards, int32_t n, rs_kd_policy policy, int *status);
/* kd_update on a tabular drafter: host selects ceil(N/I) samples with `selection_rng`
   (an mt19937_64 seeded state advanced in place, 312 words + index), device computes
   loss + analytic gradient and applies one SGD step into a NEW model (version + 1). */
int rs_kd_update_tabular(rs_ctx *ctx, const rs_model *drafter, const rs_kd_sample *buf, int32_t n,
                         rs_kd_policy policy, uint64_t *selection_rng_state, double sim_cost_per_token,
                         rs_model **new_drafter, rs_kd_result *out);
/* ---- kernels exposed for tests / microbenchmarks (device pointers) ------------------------ */
/* C = A . B^T on tcgen05 tensor cores; A [M,K] bf16, B [N,K] bf16 (K-major), epilogue:
   0 = bf16 out (+ bias[N] bf16), 1 = fp32 out * scale, 2 = fp32 out += acc, 3 = SwiGLU bf16 out [M, N/2].
   block_n: 0 (auto) | 128 | 256; splits: deterministic split-K (epilogue 2 only).
   Runs on the context stream. */
int rs_gemm_bf16(rs_ctx *ctx, const void *A_dev, const void *B_dev, void *C_dev, const void *bias_dev, int32_t M,
                 int32_t N, int32_t K, int32_t epilogue, float scale, int32_t block_n, int32_t splits);
/* LM-head GEMM: C_f32[M, N] = scale * A[M, K] . B[N, K]^T with, when stats_dev is non-null,
   the fused fp64 softmax tile partials of C / tau (per 256-column tile, EOS column N-1
   excluded): stats[(m * ceil(N/256) + t) * 2] = max, [.. + 1] = sum exp(. - max). */
int rs_lm_head_bf16(rs_ctx *ctx, const void *A_dev, const void *B_dev, float *C_dev, double *stats_dev, int32_t M,
                    int32_t N, int32_t K, float scale, double tau);
/* The same tile partials from fp32 rows already in HBM (stand-alone full-chip kernel). */
int rs_row_stats(rs_ctx *ctx, const float *rows_dev, int32_t nrows, int32_t V, double tau, double *stats_dev);
/* Device pointer + byte size of a named weight tensor of a transformer target / drafter
   ("emb", "final_norm", "rope", per layer "qkv_w", "qkv_b", "o_w", "gu_w", "down_w", "ln1",
   "ln2"; drafter "fc_w", "norm_emb", "norm_hid", "lm_w"), for export / test references. */
int rs_model_tensor(const rs_model *m, const char *name, int32_t layer, void **dev_ptr, int64_t *bytes);
/* Checkpoint load / store -- the transformer counterpart of TabularARModel::to_json /
   from_json (model.cpp:176-191), so real Qwen2.5 / EAGLE-3 weights can be served. Tensors use
   the Hugging Face names and layouts, row-major [rows][cols] on the host:
     target:  "embed_tokens.weight" [V][d] (tied LM head), "norm.weight" [d], per layer
              "input_layernorm.weight", "post_attention_layernorm.weight" [d],
              "q_proj.weight" [H*hd][d], "k_proj.weight" / "v_proj.weight" [KV*hd][d],
              "q_proj.bias" / "k_proj.bias" / "v_proj.bias", "o_proj.weight" [d][H*hd],
              "gate_proj.weight" / "up_proj.weight" [d_ff][d], "down_proj.weight" [d][d_ff];
     drafter: "fc.weight" [d][3d], "input_layernorm.weight" (norm of the token embedding),
              "hidden_norm.weight" (norm of the fused feature), "norm.weight",
              "lm_head.weight" [V][d], and the decoder-layer names above with QKV input 2d
              (layer argument ignored).
   The library scatters them into its arena (fused QKV rows, pairwise-interleaved gate/up rows).
   dtype RS_DTYPE_BF16 / RS_DTYPE_F32 is the HOST element type; it is converted (fp32 -> bf16
   round-to-nearest-even for bf16 weights, exact otherwise). n must equal rows * cols. Loading
   gives the model a new snapshot identity (engines re-prefill a drafter's cache); do not load
   into a model while an engine is stepping on it. */
int rs_model_tensor_shape(const rs_model *m, const char *name, int32_t layer, int64_t *rows, int64_t *cols);
int rs_model_load_tensor(rs_ctx *ctx, rs_model *m, const char *name, int32_t layer, const void *host, int32_t dtype,
                         int64_t n);
int rs_model_store_tensor(rs_ctx *ctx, const rs_model *m, const char *name, int32_t layer, void *host, int32_t dtype,
                          int64_t n);
/* Device-to-device copy on the context stream (synchronous). */
int rs_memcpy_d2d(rs_ctx *ctx, void *dst_dev, const void *src_dev, int64_t bytes);
/* Parameter count of a model (tabular: table size). */
int rs_model_params(const rs_model *m, int64_t *out);
/* Per-kernel-class device timing (CUDA events around each launch, this thread only):
   JSON {"<scope>.<kernel>": {"launches", "ms", "flops", "bytes"}} with algorithmic work. */
void rs_prof_enable(int32_t on);
/* Process-wide kernel tuning knobs (0 = automatic). Keys: "accept_cluster" -- CTAs per
   sequence in the fused acceptance kernel (1, 2, 4, 8); "fused_stats" -- drafter LM-head softmax
   partials in the GEMM epilogue (1) or a separate row-stats kernel (0); results are bitwise
   independent of both; "gemm2" -- weight GEMMs on SM pairs (0 auto/on, -1 single-SM kernel);
   "pdl" -- programmatic dependent launch on the forward path (0 on, -1 off); "kd_rows" -- cap on
   the KD rows per group of rs_engine_kd_grad (tests of the grouping; 0 = workspace size);
   "lazy_lm" -- verify LM head on the root rows, then only the selected chains (0 on, -1 one pass);
   "epi3" -- single-wave SM-pair GEMMs give a third of the epilogue to the control warps (0 on,
   -1 off). Results are bitwise independent of every key. */
int rs_set_tuning(const char *key, int64_t value);
void rs_prof_reset(void);
int rs_prof_json(char *buf, int64_t cap, int64_t *len);

/* mt19937_64 state helper for rs_kd_update_tabular: 313 uint64 (312 words + index). */
int rs_mt19937_64_seed(uint64_t seed, uint64_t *state313);
/* The pieces of kd_update for a prompt-sharded learner:
   rs_kd_select   -- host: ceil(n / interval) partial Fisher-Yates indices (learner.cpp:107-121),
                     replicated on every rank from the same selection state;
   rs_kd_grad_tabular -- device: sum_i w_i * (q - p~)/tau per visited row (learner.cpp:62-82) and
                     sum_i w_i * KL_i (learner.cpp:33-60) over this rank's selected samples;
   rs_tabular_apply_delta -- logits + grad * scale into a new model, version + 1 (model.cpp:161-170). */
int rs_kd_select(int32_t n, int32_t interval, uint64_t *selection_rng_state, int32_t *out_idx, int32_t *take);
int rs_kd_grad_tabular(rs_ctx *ctx, const rs_model *drafter, const rs_kd_sample *samples, int32_t n,
                       const double *weights, double *grad_out, double *loss_out);
int rs_tabular_apply_delta(rs_ctx *ctx, const rs_model *m, const double *grad, double scale, rs_model **out);

/* Transformer drafters (EAGLE-3-style) -- the same kd_update (learner.cpp:98-160) with the
   drafter's distribution q recomputed by its forward and the target rows p~ recomputed by a
   teacher-forced target forward over prompt + response (StepRecord::target_logprobs are not
   materialised at V = 152K; rs_kd_sample.target_logprobs is ignored and may be NULL). As in the
   reference, where the gradient covers the whole model (learner.cpp:62-82) and the update moves
   every parameter (with_logits_delta, :146-151), EVERY drafter tensor is trained: dZ_t =
   w (q_t - p~_t) / tau at the response positions, backpropagated through the LM head, final
   norm, SwiGLU MLP, post-attention norm, O projection, causal attention (into every position's
   keys / values), RoPE, QKV (+ bias), the two input norms and fc. The target (and the shared
   embedding) is frozen.
   rs_drafter_grad_layout   -- the fp32 gradient buffer: total floats (name NULL) or the
                               (offset, count) of one tensor ("lm_w", "fc_w", "norm_emb",
                               "norm_hid", "qkv_w", "qkv_b", "o_w", "ln2", "gu_w", "down_w",
                               "final_norm"); the LM head comes first ([V][d] at offset 0);
   rs_kd_grad_transformer   -- the per-rank piece: sum_i w_i KL_i and the gradient of the given
                               samples (accumulated into grad_dev unless zero_grad);
   rs_drafter_apply_grad    -- new snapshot (version + 1): every tensor w + scale * grad;
   rs_kd_update_transformer -- single-process kd_update: select, weight, gradient, SGD (-lr). */
int rs_drafter_grad_layout(const rs_model *drafter, const char *name, int64_t *offset, int64_t *count);
int rs_kd_grad_transformer(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_kd_sample *samples,
                           int32_t n, const double *weights, float *grad_dev, int32_t zero_grad, double *loss_out);
int rs_drafter_apply_grad(rs_ctx *ctx, const rs_model *drafter, const float *grad_dev, double scale, rs_model **out);
/* The same per-rank K5 + LM-head gradient as rs_kd_grad_transformer over requests of a live
   transformer engine (prompt = the request's prompt, response = its generated tokens, eos_bias
   its own), computed from the engine's RESIDENT target KV cache and features: only the response
   positions go through the target (no teacher-forced recompute of the prompt); the given drafter
   runs teacher-forced into a private cache (the engine's drafter state is untouched).
   Per-row losses and dZ are bit-identical to rs_kd_grad_transformer on the same sequences; the
   gradient is too whenever both accumulate the KD rows in the same groups (one group when they
   fit the workspace), else it differs only by fp32 summation grouping. */
int rs_engine_kd_grad(rs_engine *e, const rs_model *drafter, const int32_t *req, int32_t n, const double *weights,
                      float *grad_dev, int32_t zero_grad, double *loss_out);
int rs_kd_update_transformer(rs_ctx *ctx, const rs_model *target, const rs_model *drafter, const rs_kd_sample *buf,
                             int32_t n, rs_kd_policy policy, uint64_t *selection_rng_state, double cost,
                             rs_model **new_drafter, rs_kd_result *out);

/* ---- online learner (learner.hpp:39-139, learner.cpp:84-289) ------------------------------
   OnlineLearner over the device kd_update: feed() copies samples into a ReplayBuffer of
   `buffer_capacity` entries (oldest dropped when full, learner.cpp:84-89); an update fires on
   on_iteration_boundary(it) when (it + 1) % interval == 0 and the buffer is non-empty
   (learner.cpp:184-203), consuming the whole buffer through rs_kd_update_tabular or
   rs_kd_update_transformer (chosen by the drafter's kind). async != 0 runs updates on a worker
   thread with its own CUDA stream, overlapping the caller's rollouts; await_pending is the
   rendezvous (learner.cpp:205-211), and async and synchronous learners publish identical
   snapshot sequences. A failed asynchronous update is reported by the next await_pending /
   on_iteration_boundary / shutdown. rs_learner_snapshot returns a NEW reference (release it
   with rs_model_destroy). */
typedef struct {
    int32_t update_idx;
    int32_t drafter_version;
    double kd_loss;
    int32_t samples_used;
    double weight_mean;
    double weight_min;
    double weight_max;
    double weights_l2; /* L2 of the published snapshot's trained weights (tabular logits / drafter LM head) */
} rs_learner_metric;   /* LearnerMetrics, learner.hpp:75-84 */
int rs_learner_create(rs_ctx *ctx, const rs_model *drafter, rs_kd_policy policy, uint64_t selection_seed,
                      double sim_cost_per_token, int64_t buffer_capacity, int32_t async, rs_learner **out);
int rs_learner_destroy(rs_learner *l); /* shutdown (drains queued updates) + free */
int rs_learner_feed(rs_learner *l, const rs_kd_sample *samples, int32_t n);
/* Samples backed by a live transformer engine (EAGLE drafter learners): request req[i] of `e`
   with reward[i]; updates read the engine's resident KV cache and features (as
   rs_engine_kd_grad) instead of recomputing the prompts. The engine must outlive the update and
   must not be stepped while it is pending. */
int rs_learner_feed_engine(rs_learner *l, rs_engine *e, const int32_t *req, const double *reward, int32_t n);
int rs_learner_on_iteration_boundary(rs_learner *l, int32_t iteration);
int rs_learner_await_pending(rs_learner *l);
int rs_learner_shutdown(rs_learner *l);
int rs_learner_snapshot(const rs_learner *l, rs_model **out);
int rs_learner_drafter_version(const rs_learner *l, int32_t *out);
int rs_learner_total_sim_time(const rs_learner *l, double *out);
int rs_learner_buffer_size(const rs_learner *l, int64_t *out);
int rs_learner_metrics(const rs_learner *l, rs_learner_metric *out, int32_t cap, int32_t *n);

/* ---- GRPO stage (rl.hpp:12-50, rl.cpp:8-90) ---------------------------------------------
   rs_reward          -- fraction of adjacent (golden_a, golden_b) pairs in a response (rl.cpp:8-19);
   rs_group_advantages -- (r - mean) / (population std + 1e-6), G >= 2 (rl.cpp:21-40);
   rs_policy_update_tabular -- new actor (version + 1) = actor + lr * sum_i A_i grad log pi(y_i)
                       on the device; samples' target_logprobs are ignored. actor_versions (or
                       NULL) must all equal the actor's version, else "policy_update: off-policy
                       update" (rl.cpp:76-80). */
int rs_reward(const int32_t *y, int32_t n, int32_t golden_a, int32_t golden_b, double *out);
int rs_group_advantages(const double *rewards, int32_t g, double *out);
int rs_policy_update_tabular(rs_ctx *ctx, const rs_model *actor, const rs_kd_sample *samples,
                             const double *advantages, const int32_t *actor_versions, int32_t n, double lr,
                             rs_model **out);

/* ---- multi-GPU: the KD gradient all-reduce ---------------------------
   Replaces the cross-sample sum of kd_loss_gradient (learner.cpp:68-80) when the rollouts are
   sharded by prompt over the GPUs of a box (one process or thread per GPU); the
   generation path itself has no collective. NCCL is loaded at run time (libnccl.so.2).
   rs_comm_unique_id -- rank 0 creates the 128-byte id, the caller ships it to the other ranks;
   rs_comm_create    -- ncclCommInitRank on the context's device (collective over all ranks);
   rs_comm_allreduce -- in-place all-reduce of a device buffer on the context's stream;
   rs_comm_allreduce_host -- synchronous all-reduce of <= 64 host doubles (losses, token
                       counts, max-over-ranks device times). */
#define RS_COMM_ID_BYTES 128
#define RS_DT_F32 0
#define RS_DT_F64 1
#define RS_DT_I64 2
#define RS_OP_SUM 0
#define RS_OP_MAX 1
int rs_nccl_version(int32_t *out);
int rs_comm_unique_id(uint8_t *id);
int rs_comm_create(rs_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t *id, rs_comm **out);
int rs_comm_destroy(rs_comm *c);
int rs_comm_size(const rs_comm *c, int32_t *nranks, int32_t *rank);
int rs_comm_allreduce(rs_comm *c, rs_ctx *ctx, void *buf_dev, int64_t count, int32_t dtype, int32_t op);
int rs_comm_allreduce_host(rs_comm *c, rs_ctx *ctx, double *vals, int32_t n, int32_t op);
/* Library-owned device memory (gradient buffers) and copies on the context's stream; the
   h2d / d2h copies are synchronous. */
int rs_device_alloc(rs_ctx *ctx, int64_t bytes, void **out);
int rs_device_free(rs_ctx *ctx, void *p);
int rs_memset_async(rs_ctx *ctx, void *p, int32_t value, int64_t bytes);
int rs_memcpy_h2d(rs_ctx *ctx, void *dst_dev, const void *src, int64_t bytes);
int rs_memcpy_d2h(rs_ctx *ctx, void *dst, const void *src_dev, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* RESPEC_B200_H */

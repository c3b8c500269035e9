// sd.h -- device state of one BatchEngine and the launchers of the model-agnostic SD
// kernels (drafting sampler, fused softmax + acceptance, cycle bookkeeping).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "rng.cuh"

namespace rs {

constexpr int kMaxBranch = 16;  // t
constexpr int kMaxDraft = 32;   // n
constexpr int kMaxRounds = 8;   // s
constexpr int kSummaryFixed = 6;

// Everything the SD kernels touch. Request-indexed arrays are [B]; row buffers are indexed
// by ACTIVE slot a in [0, nact) (rows are packed the way the model forwards produce them).
struct SdDev {
    // requests
    int32_t *tok;            // [B][tok_cap] prompt + generated
    int32_t tok_cap;
    int32_t *len;            // [B]
    const int32_t *prompt_len;
    const int32_t *max_len;
    const double *eos_bias;
    MtStream *rng;           // [2B]: draft, accept
    int32_t *done;           // [B]
    // step records (StepRecord, specdec.hpp:40-46)
    int32_t *st_tok;         // [B][steps_cap]
    double *st_logp;
    uint8_t *st_drafted;
    double *st_logq;
    double *st_full;         // [B][steps_cap][V] or nullptr
    int32_t steps_cap;
    // active set
    const int32_t *active;   // [nact] request ids
    int32_t nact;
    // cycle state [B]
    int32_t *n_eff, *d_used, *a_used, *cont, *ended, *accept_len, *drafted, *emitted, *n_rounds;
    int32_t *round_cost;     // [B][kMaxRounds][3]
    int32_t *rsel, *racc;    // this round's selected chain (-1 none) and accepted drafted count (K4)
    int32_t *stg;            // [B][6] two-stage acceptance: sel (-1: cycle done), acur, alen, alen0, emitted, len
    // draft tree [B][t_max][n_max]
    int32_t *chain_tok, *chain_len, *chain_stop, *chain_off;
    int32_t t_max, n_max;
    // current SD config
    int32_t s, t, n;
    // model / rows
    int32_t V, eos;
    double tau_p, tau_q;
    int32_t slots;           // 1 + t*n rows per active sequence
    const void *P;           // target logits rows  [nact][slots][V]
    const void *Q;           // drafter logits rows [nact][slots][V]
    const double *Pst;       // LM-head epilogue tile partials for P rows [nact][slots][ntiles][2], or null
    const double *Qst;       // same for Q rows
    int32_t ntiles;          // ceil(V / 256)
    int32_t lazy_pst;
    double *pq_cache;        // [nact][2][V] fp64 p1 / q1 of the branch point (sibling residual passes)        // Pst is scratch: the acceptance kernel fills the rows it touches
    int32_t verify_mode;     // RS_VERIFY_SAMPLE / RS_VERIFY_GREEDY
    int32_t record_full;
    int32_t *err;            // device error word (first error wins)
    int32_t *flag;           // redraft flag
    int32_t *summary;        // [nact][kSummaryFixed + 3*kMaxRounds]
    int32_t *newtok;         // [nact][newtok_cap] tokens emitted by this cycle (returned with the summary)
    int32_t newtok_cap;
};

enum class RowType { F64, F32 };

// Launchers (sd_kernels.cu)
void sd_cycle_begin(const SdDev &d, cudaStream_t st);
void sd_round_setup(const SdDev &d, int round, cudaStream_t st);
void sd_draft_sample(const SdDev &d, int depth, RowType rt, cudaStream_t st);
void sd_redraft_check(const SdDev &d, cudaStream_t st);
// stage 0: whole acceptance; 1 / 2: before / after the LM head of the selected chains (lazy verify LM head)
void sd_accept(const SdDev &d, int round, bool naive, RowType rt, cudaStream_t st, int stage = 0);
void sd_cycle_end(const SdDev &d, bool naive, cudaStream_t st);

// Exact fp64 softmax tile partials of fp32 logit rows (rowstats.cu); row_ids null = rows 0..n-1.
void row_stats(const float *rows, const int32_t *row_ids, int nrows, int V, double tau, double *stats,
               cudaStream_t st);

// Tabular model "forwards": gather logit rows by row_index (model.cpp:113-139).
struct TabDev {
    const double *table;
    int32_t order;
    int32_t V;
};
void tab_draft_rows(const SdDev &d, const TabDev &m, int depth, cudaStream_t st);
void tab_verify_rows(const SdDev &d, const TabDev &m, bool naive, cudaStream_t st);

}  // namespace rs

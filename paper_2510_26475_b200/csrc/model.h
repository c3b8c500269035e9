// model.h -- Qwen2-shaped target and EAGLE-3-style drafter held in HBM (bf16 weights), and
// the device kernels of their forwards (model.cu, attention_tc.cu).
#pragma once
#include <cuda_bf16.h>

#include <vector>

#include "engine.h"

namespace rs {

using bf16 = __nv_bfloat16;

struct TfShape {
    int V = 0, d = 0, L = 0, H = 0, KV = 0, hd = 0, dff = 0, max_ctx = 0;
    float rope_theta = 1e6f, eps = 1e-6f, std = 0.02f, logit_scale = 1.0f;
    int qkv_dim() const { return (H + 2 * KV) * hd; }
};

struct LayerW {
    bf16 *qkv_w = nullptr;   // [(H+2KV)*hd, d_in]
    bf16 *qkv_b = nullptr;   // [(H+2KV)*hd]
    bf16 *o_w = nullptr;     // [d, H*hd]
    bf16 *gu_w = nullptr;    // [2*dff, d], rows interleaved pairwise: 2i gate_i, 2i+1 up_i
    bf16 *down_w = nullptr;  // [d, dff]
    float *ln1 = nullptr;    // [d_in]
    float *ln2 = nullptr;    // [d]
};

// Qwen2 decoder stack: embed -> L x (RMSNorm, QKV+bias, RoPE, GQA attention, O, RMSNorm,
// SwiGLU MLP) -> RMSNorm -> tied LM head. Hidden states after three layers (low/mid/high)
// are the EAGLE-3 features the drafter consumes.
struct TransformerModel : rs_model {
    TfShape s;
    DBuf<char> arena;          // all weights
    bf16 *emb = nullptr;       // [V, d] (tied LM head)
    std::vector<LayerW> layers;
    float *final_norm = nullptr;
    float *rope = nullptr;     // [max_ctx][hd/2][2] cos, sin
    int feat_layers[3] = {0, 0, 0};
    size_t n_params = 0;
    TransformerModel() : rs_model(Transformer) {}
};

// EAGLE-3-style drafter: f = fc([g_low, g_mid, g_high]) (or its own previous hidden state
// when drafting deeper), one decoder layer over [RMSNorm(emb(tok)), RMSNorm(f)], own LM head.
struct DrafterModel : rs_model {
    TfShape s;                 // same d / heads as the target, L = 1
    const TransformerModel *target = nullptr;
    DBuf<char> arena;
    bf16 *fc_w = nullptr;      // [d, 3d]
    float *norm_emb = nullptr, *norm_hid = nullptr;  // [d]
    LayerW layer;              // qkv_w: [(H+2KV)*hd, 2d]
    float *final_norm = nullptr;
    bf16 *lm_w = nullptr;      // [V, d]
    size_t n_params = 0;
    DrafterModel() : rs_model(Drafter) {}
    ~DrafterModel() override;  // the arena goes back to the snapshot pool (model.cu)
};

void init_transformer(TransformerModel &m, uint64_t seed, cudaStream_t st);
TransformerModel *create_transformer(rs_ctx *ctx, const rs_transformer_shape &sh, uint64_t seed);
DrafterModel *create_drafter(rs_ctx *ctx, const rs_model *target, uint64_t seed, int version);
void init_drafter(DrafterModel &m, uint64_t seed, cudaStream_t st);
void carve_drafter(DrafterModel &m);

// Transformer KD (K5 + the drafter LM-head gradient), tf_pair.cpp. One training sequence =
// prompt + response of a RolloutSample; every response position t contributes
// w * KL(p~_t || q_t) with p~ the target and q the drafter at context prompt + response[:t].
struct KdSeq {
    std::vector<int> tokens;
    int prompt_len = 0;
    double eos_bias = 0.0, weight = 1.0;
};
// Accumulates dL/dW_lm (fp32 [V][d]) into grad (zeroed first if zero_grad); returns the loss.
double kd_grad_transformer(rs_ctx *ctx, const TransformerModel *tgt, const DrafterModel *drf,
                           const std::vector<KdSeq> &seqs, float *grad, bool zero_grad);
// New drafter snapshot (version + 1): every tensor w + scale * grad (grad in the layout below).
DrafterModel *drafter_apply_lm_grad(rs_ctx *ctx, const DrafterModel *drf, const float *grad, double scale);

// The drafter gradient (fp32, one buffer): every trainable tensor of the EAGLE drafter, LM head
// first (so a [V][d] prefix is the LM-head gradient), then fc, the two input-norm gains, the
// decoder layer (QKV weight + bias, O, post-attention norm gain, gate/up, down) and the final
// norm gain. The target's embedding (shared by the drafter's input) is frozen.
struct DrafterGradLayout {
    size_t lm = 0, fc = 0, norm_emb = 0, norm_hid = 0, qkv_w = 0, qkv_b = 0, o_w = 0, ln2 = 0, gu_w = 0, down_w = 0,
           final_norm = 0, total = 0;
};
DrafterGradLayout drafter_grad_layout(const TfShape &s);

// One query/update row of a forward pass.
struct RowDesc {
    int seq;     // request id
    int pos;     // logical position (RoPE, causal mask)
    int phys;    // physical KV slot written by this row
    int kind;    // 0: token = tok[seq][pos]; 1: token = chain_tok[seq][chain][cj]
    int chain;   // chain for kind 1 / key mapping (-1: plain causal over the cache)
    int cj;      // chain index of the token for kind 1
    int fsrc;    // drafter feature source: 0 target features at pos-1, 1 drafter hidden (seq, chain) slot
    int fidx;    // hidden-slot index for fsrc == 1
};

// One attention work item: up to 64/G consecutive rows sharing a key mapping.
struct AttnItem {
    int seq, row0, nrows, maxpos;
    int chain, ltree, tbase, nstride;  // keys at logical p >= ltree map to tbase + chain*nstride + (p-ltree)
    int pass0 = 0, npass = 0, grp0 = 0, ngrp = 0;  // tensor-core attention plan (AttnPlan slices)
};

// Host-built pass plan of the tensor-core attention (attention_tc.cu): per item, the key
// chunks it visits in logical order and, for chunks reaching into a draft tree, one replay per
// group of tokens sharing a key mapping (one draft chain; the root rides with chain 0).
struct AttnPass {
    int16_t chunk, grp;  // grp -1: shared by every row of the item
    uint8_t tiles;       // bit i: 128-row M-tile i takes part
    uint8_t manual;      // 1: keys remapped to a chain's slots (cp.async), 0: contiguous (TMA)
    int16_t pad;
};
struct AttnGroup {
    int chain, maxpos;
};
struct AttnPlan {
    const AttnPass *passes = nullptr;
    const AttnGroup *groups = nullptr;
    const int16_t *tok_grp = nullptr;  // per forward row: group index within its item
};
// Tokens of an attention item's first M-tile (tmax = 128 / G): items that need two tiles split
// their tokens evenly (tree items of 1 + t * n tokens would otherwise leave the second tile mostly
// empty while the first carries 128 rows). Host plan and kernel use this one definition.
__host__ __device__ inline int attn_tile_tokens(int ntok, int tmax) { return ntok > tmax ? (ntok + 1) / 2 : tmax; }
constexpr int kAttnChunk = 32;      // keys per pass of the tensor-core attention
constexpr int kAttnMaxPasses = 400;
constexpr int kAttnMaxGroups = 64;

struct KvCache {
    bf16 *k = nullptr, *v = nullptr;  // [layer][B][KV][max_ctx][hd]
    int layers = 0, B = 0, KV = 0, max_ctx = 0, hd = 0;
    __host__ __device__ size_t off(int layer, int seq, int kvh, int phys) const {
        return ((((size_t)layer * B + seq) * KV + kvh) * max_ctx + phys) * hd;
    }
};

// kernels (model.cu)
void k_embed(const RowDesc *rows, int M, const int32_t *tok, int tok_cap, const int32_t *chain_tok, int t_max,
             int n_max, const bf16 *emb, int V, int d, float *x, cudaStream_t st);
void k_rmsnorm(const float *x, int ldx, const float *w, int M, int d, float eps, bf16 *out, int ldo, cudaStream_t st);
void k_rmsnorm_bf16(const bf16 *x, int ldx, const float *w, int M, int d, float eps, bf16 *out, int ldo,
                    cudaStream_t st);
void k_rope_store(const bf16 *qkv, const RowDesc *rows, int M, const TfShape &s, const float *rope, const KvCache &kv,
                  int layer, bf16 *q, cudaStream_t st);
// Target attention on tcgen05/TMEM (attention_tc.cu): items of rows (chain -1 plain causal over the cache, -2 tree),
// at most attn_tc_max_tokens(G) tokens per item.
int attn_tc_max_tokens(int G);
void k_attention_tc(const bf16 *q, const RowDesc *rows, const AttnItem *items, const AttnPlan &plan, int n_items,
                    const KvCache &kv, int layer, const TfShape &s, bf16 *out, cudaStream_t st, double flops = 0,
                    double bytes = 0);
void k_store_features(const float *x, const RowDesc *rows, int M, int d, bf16 *feat, int max_ctx, int slot,
                      cudaStream_t st);
void k_gather_features(const RowDesc *rows, int M, int d, const bf16 *feat, int max_ctx, const float *hid, bf16 *fin,
                       int *use_hidden, cudaStream_t st);
void k_rows_copy_f32(const float *src, int ld_src, const int *src_rows, float *dst, int ld_dst, const int *dst_rows,
                     int n, int d, cudaStream_t st);
// Lazy verify LM head: rows of the selected chains (stg[r * 6]) -> out [nact * n][d], P-row map (-1 none)
void k_gather_selected(const bf16 *xn, const int32_t *active, const int32_t *stg, const int32_t *chain_len, int t_max,
                       int nact, int n, int slots, int d, bf16 *out, int32_t *map, cudaStream_t st);
void k_init_normal(bf16 *p, size_t n, uint64_t seed, uint64_t tensor_id, float std, cudaStream_t st);
void k_fill_f32(float *p, size_t n, float v, cudaStream_t st);
void k_rope_table(float *rope, int max_ctx, int hd, float theta, cudaStream_t st);
void k_compact(const SdDev &d, const int32_t *rsel, const int32_t *racc, const int32_t *rbase, const KvCache &kv,
               bf16 *feat, int feat_w, int max_ctx, cudaStream_t st);

}  // namespace rs

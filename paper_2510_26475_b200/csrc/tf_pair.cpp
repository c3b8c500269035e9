// tf_pair.cpp -- the transformer ModelPair: drafter tree expansion (K1), tree-verify forward
// (K2) and KV compaction (K4) for one BatchEngine, plus the constructors of the transformer
// target and the EAGLE-3-style drafter.
//
// KV invariant per request: after every engine step the target cache holds positions
// 0..len-2 and the newest token (the root of the next round) is not yet processed. A round's
// verify forward writes the root at len-1 and chain i's depth-j token at the tree slot
// len + i*n + j (logical position len + j); K4 then moves the accepted chain's slots to
// len..len+a-1. The drafter cache is caught up lazily: its depth-0 forward processes every
// position it has not seen (all of them at the first spec cycle -- the reference's "drafter
// prefill on off->on", server.cpp:280-290) with the target's low/mid/high features at p-1.
//
// Row / attention-item descriptors are built on the host (the host knows every request's
// length from the previous step's summary) and staged through a pinned arena that is only
// recycled after the engine's end-of-step synchronisation, so no async copy ever reads a
// host buffer that has been overwritten.
#include <algorithm>
#include <cstring>
#include <stdexcept>

#include "common.cuh"
#include "gemm.h"
#include "kd.h"
#include "model.h"
#include "prof.h"

namespace rs {

namespace {

struct Staging {
    char *base = nullptr;
    size_t cap = 0, off = 0;
    void alloc(size_t bytes) {
        cap = bytes;
        RS_CUDA(cudaMallocHost(&base, bytes));
    }
    ~Staging() {
        if (base) cudaFreeHost(base);
    }
    template <class T>
    void upload(T *dst_dev, const std::vector<T> &v, cudaStream_t st) {
        if (v.empty()) return;
        const size_t bytes = v.size() * sizeof(T);
        off = (off + 15) & ~size_t(15);
        if (off + bytes > cap) {  // arena full: drain the stream, then recycle
            RS_CUDA(cudaStreamSynchronize(st));
            off = 0;
            if (bytes > cap) throw std::runtime_error("staging arena too small");
        }
        std::memcpy(base + off, v.data(), bytes);
        RS_CUDA(cudaMemcpyAsync(dst_dev, base + off, bytes, cudaMemcpyHostToDevice, st));
        note_copy(true, bytes);
        off += bytes;
    }
};

struct Workspace {
    int Mcap = 0;
    DBuf<float> x, e32;
    DBuf<bf16> xn, qkv, q, ao, h, fin;
    DBuf<RowDesc> rows;
    DBuf<AttnItem> items;
    DBuf<int32_t> map_a, map_b, idx;
    DBuf<AttnGroup> groups;
    DBuf<int16_t> tok_grp;
    DBuf<AttnPass> passes;
    void ensure_passes(size_t n, cudaStream_t st) {
        if (n <= passes.n) return;
        RS_CUDA(cudaStreamSynchronize(st));
        passes.alloc(std::max(n, 2 * passes.n));
    }
    void alloc(int M, const TfShape &s) {
        Mcap = M;
        x.alloc((size_t)M * s.d);
        e32.alloc((size_t)M * s.d);
        xn.alloc((size_t)M * 2 * s.d);
        qkv.alloc((size_t)M * s.qkv_dim());
        q.alloc((size_t)M * s.H * s.hd);
        ao.alloc((size_t)M * s.H * s.hd);
        h.alloc((size_t)M * s.dff);
        fin.alloc((size_t)M * 3 * s.d);
        rows.alloc(M);
        items.alloc(M);
        map_a.alloc(M);
        map_b.alloc(M);
        idx.alloc((size_t)2 * M);
        groups.alloc(M);
        tok_grp.alloc(M);
        passes.alloc((size_t)M * 8);
    }
};

void gemm(const void *A, int lda, const void *B, int M, int N, int K, GemmEpi epi, cudaStream_t st, int splits = 0) {
    GemmArgs g;
    g.A = A;
    g.B = B;
    g.M = M;
    g.N = N;
    g.K = K;
    g.lda = lda;
    g.ldb = K;
    g.epi = epi;
    g.splits = splits;  // residual epilogue: 0 = split-K by (N, K) only (gemm_2sm.cu), else fixed per weight
    // block_n auto: the tile width that best fills one wave of 148 SMs (gemm_sm100.cu)
    gemm_bf16(g, st);
}

// C[M, N] (+)= A[M, K] . B[N, K]^T with explicit leading dimensions (backward-pass GEMMs:
// transposed activations as operands, K = rows of the training batch).
void gemm_ld(const void *A, int lda, const void *B, int ldb, int M, int N, int K, GemmEpi epi, cudaStream_t st) {
    GemmArgs g;
    g.A = A;
    g.B = B;
    g.M = M;
    g.N = N;
    g.K = K;
    g.lda = lda;
    g.ldb = ldb;
    g.epi = epi;
    g.splits = 1;
    gemm_bf16(g, st);
}

int round64(int x) { return (x + 63) / 64 * 64; }

GemmEpi epi_bf16(void *out, int ldo, const void *bias = nullptr) {
    GemmEpi e;
    e.kind = kEpiBF16;
    e.out = out;
    e.ldo = ldo;
    e.bias = bias;
    return e;
}
GemmEpi epi_resid(float *out, int ldo) {
    GemmEpi e;
    e.kind = kEpiResidual;
    e.out = out;
    e.ldo = ldo;
    return e;
}

// Split-K of the DRAFTER's residual GEMMs (fc, O, down). The drafter runs at 256-ish rows, where
// a 2048-feature output is only 8 SM-pair tiles: without splitting, 8 of 74 pairs walk the whole
// K (down: 172 k-blocks). The count is fixed per weight matrix (a function of K only), never of
// the row count, so a row's partial-sum order -- and its bits -- does not depend on its batch.
// Measured at 256 rows (tools/gemm_split_sweep.py): down 49.8 -> 33.6 us and fc 30.4 -> 24.0 us
// at 2 splits; more splits lose to the last-arriving CTA's reduction of the partials.
int drafter_splits(int K) { return K >= 4096 ? 2 : 1; }
GemmEpi epi_swiglu(void *out, int ldo) {
    GemmEpi e;
    e.kind = kEpiSwiGLU2;  // gate/up rows interleaved pairwise (model layout)
    e.out = out;
    e.ldo = ldo;
    return e;
}
// QKV projection + bias + RoPE + K/V cache store in one SM-pair GEMM epilogue.
GemmEpi epi_qkv_rope(bf16 *q, const bf16 *bias, const RowDesc *rows, const float *rope, const KvCache &kv, int layer,
                     int H) {
    GemmEpi e;
    e.kind = kEpiQKVRope;
    e.bias = bias;
    e.qkv.rows = rows;
    e.qkv.rope = rope;
    e.qkv.q = q;
    e.qkv.k = kv.k;
    e.qkv.v = kv.v;
    e.qkv.H = H;
    e.qkv.KV = kv.KV;
    e.qkv.layer = layer;
    e.qkv.B = kv.B;
    e.qkv.max_ctx = kv.max_ctx;
    return e;
}
bool fused_qkv_rope(const TfShape &s) { return tuning().gemm2 >= 0 && s.hd == 128; }

GemmEpi epi_f32(float *out, int ldo, float scale, const int *row_map, double *stats = nullptr, double tau = 1.0) {
    GemmEpi e;
    e.kind = kEpiF32;
    e.out = out;
    e.ldo = ldo;
    e.scale = scale;
    e.row_map = row_map;
    e.stats = stats;
    e.tau = tau;
    return e;
}

// Host-side description of one forward launch.
struct Batch {
    std::vector<RowDesc> rows;
    std::vector<AttnItem> items;
    std::vector<int32_t> map_a, map_b;
    std::vector<AttnPass> passes;
    std::vector<AttnGroup> groups;
    std::vector<int16_t> tok_grp;
    void clear() {
        rows.clear();
        items.clear();
        map_a.clear();
        map_b.clear();
        passes.clear();
        groups.clear();
        tok_grp.clear();
    }
    // Pass plan of every item for the tensor-core attention (G query heads per kv head).
    void plan_tc(int G) {
        passes.clear();
        groups.clear();
        tok_grp.assign(rows.size(), 0);
        const int Tmax = 128 / G;
        for (auto &it : items) {
            it.pass0 = (int)passes.size();
            it.grp0 = (int)groups.size();
            const int ntok = it.nrows;
            int ng = 0;
            for (int k = 0; k < ntok;) {
                int ch = rows[it.row0 + k].chain, k1 = k + 1;
                if (it.chain == -2) {  // consecutive tokens of one chain; the root joins chain 0
                    if (ch < 0 && k1 < ntok && rows[it.row0 + k1].chain == 0) ch = 0;
                    while (k1 < ntok && rows[it.row0 + k1].chain == ch) ++k1;
                } else {
                    ch = -1;
                    k1 = ntok;
                }
                int gmax = 0;
                for (int j = k; j < k1; ++j) {
                    tok_grp[it.row0 + j] = (int16_t)ng;
                    gmax = std::max(gmax, rows[it.row0 + j].pos);
                }
                groups.push_back(AttnGroup{ch, gmax});
                ++ng;
                k = k1;
            }
            for (int c = 0; c <= it.maxpos / kAttnChunk; ++c) {
                const int c0 = c * kAttnChunk;
                const bool tail = it.chain == -2 && c0 + kAttnChunk - 1 >= it.ltree;
                for (int g = tail ? 0 : -1; g < (tail ? ng : 0); ++g) {
                    uint8_t tiles = 0;
                    for (int k = 0; k < ntok; ++k)
                        if ((g < 0 || tok_grp[it.row0 + k] == g) && rows[it.row0 + k].pos >= c0)
                            tiles |= (uint8_t)(1u << (k / attn_tile_tokens(ntok, Tmax)));
                    if (!tiles) continue;
                    const int ch = g < 0 ? -1 : groups[it.grp0 + g].chain;
                    const bool contiguous = ch < 0 || (ch == 0 && it.tbase == it.ltree);
                    passes.push_back(AttnPass{(int16_t)c, (int16_t)g, tiles, (uint8_t)(contiguous ? 0 : 1), 0});
                }
            }
            it.npass = (int)passes.size() - it.pass0;
            it.ngrp = ng;
            if (it.npass > kAttnMaxPasses || ng > kAttnMaxGroups || ntok > 2 * Tmax)
                throw std::runtime_error("attention plan exceeds the kernel's limits");
        }
    }
    // plain causal attention items over rows [r0, r1) of one sequence (keys = its cache)
    void add_items(int r0, int r1, int per, int chain, int ltree, int tbase, int nstride) {
        for (int a = r0; a < r1; a += per) {
            const int b = std::min(r1, a + per);
            int maxpos = 0;
            for (int k = a; k < b; ++k) maxpos = std::max(maxpos, rows[k].pos);
            items.push_back(AttnItem{rows[a].seq, a, b - a, maxpos, chain, ltree, tbase, nstride});
        }
    }
    // tree items for the tensor-core attention: consecutive runs of at most max_tok tokens (two
    // 128-row M-tiles); the kernel regroups tokens by chain inside an item.
    void add_tree_items_tc(int r0, int r1, int max_tok, int ltree, int tbase, int nstride) {
        for (int a = r0; a < r1; a += max_tok) {
            const int b = std::min(r1, a + max_tok);
            int maxpos = 0;
            for (int k = a; k < b; ++k) maxpos = std::max(maxpos, rows[k].pos);
            items.push_back(AttnItem{rows[a].seq, a, b - a, maxpos, -2, ltree, tbase, nstride});
        }
    }
    int M() const { return static_cast<int>(rows.size()); }
    // algorithmic attention work: every query head attends to pos+1 keys (QK^T and PV);
    // K/V bytes read once per item and kv head
    double attn_flops(const TfShape &s) const {
        double f = 0;
        for (const auto &r : rows) f += 4.0 * s.H * s.hd * (r.pos + 1);
        return f;
    }
    double attn_bytes(const TfShape &s) const {
        double b = 0;
        for (const auto &it : items) b += 4.0 * s.KV * s.hd * (it.maxpos + 1);
        return b;
    }
};

struct TransformerPair : ModelPair {
    rs_ctx *ctx;
    rs_engine *eng;
    const TransformerModel *tgt;
    const DrafterModel *drf = nullptr;
    uint64_t drf_uid = 0;
    TfShape s;
    int B = 0, slots_max = 1, max_ctx = 0, per_item_t = 8;  // per_item_t: tokens per attention item
    KvCache kv_t, kv_d;
    DBuf<bf16> kt, vt, kd, vd, feat;
    DBuf<float> dh;  // drafter hidden per (request, chain) [B][t_max][d]
    DBuf<int32_t> rbase;
    Workspace w;
    Staging stage;
    Batch bt;
    std::vector<int> dkv_len;  // drafter cache valid for positions < dkv_len
    struct KdScratch {         // kd_cached buffers (rows x V logits, stats, dZ^T, h, private drafter KV)
        DBuf<float> Pb, Qb;
        DBuf<double> stP, stQ, lseP, lseQ, kl, lossr, wr, br;
        DBuf<bf16> dzT, hT, hG, tk, tv;
    } kd_scr;

    TransformerPair(rs_ctx *c, rs_engine *e, const TransformerModel *t, const DrafterModel *d)
        : ctx(c), eng(e), tgt(t), drf(d), drf_uid(d ? d->uid : 0), s(t->s) {}

    RowType row_type() const override { return RowType::F32; }
    void begin_step() override { stage.off = 0; }

    void set_drafter(const rs_model *m) override {
        if (m && m->kind != rs_model::Drafter) throw std::invalid_argument("transformer target needs an EAGLE drafter");
        const auto *dm = static_cast<const DrafterModel *>(m);
        if (dm && dm->target != tgt) throw std::invalid_argument("drafter is bound to a different target");
        // new snapshot (by id: a fresh one can reuse a freed one's address): rebuild its cache
        const uint64_t uid = dm ? dm->uid : 0;
        if (uid != drf_uid) std::fill(dkv_len.begin(), dkv_len.end(), 0);
        drf = dm;
        drf_uid = uid;
    }

    void setup(int n_req, int slots, const std::vector<int> &plen, int tok_cap, int t_max) {
        B = std::max(n_req, 1);
        slots_max = slots;
        max_ctx = s.max_ctx;
        per_item_t = attn_tc_max_tokens(s.H / s.KV);
        for (int i = 0; i < n_req; ++i)
            if (plen[i] < 1) throw std::invalid_argument("transformer engine: prompts must be non-empty");
        if (tok_cap + slots > max_ctx)
            throw std::invalid_argument("transformer engine: prompt + max_len + draft tree exceeds max_ctx");
        const size_t kv_elems = (size_t)s.L * B * s.KV * max_ctx * s.hd;
        kt.alloc(kv_elems);
        vt.alloc(kv_elems);
        kv_t = KvCache{kt.p, vt.p, s.L, B, s.KV, max_ctx, s.hd};
        // never-written slots must hold finite values: whole 128-key chunks are multiplied by
        // probabilities that are exactly 0 past a row's position (0 * NaN would poison O)
        RS_CUDA(cudaMemsetAsync(kt.p, 0, kv_elems * sizeof(bf16), ctx->stream));
        RS_CUDA(cudaMemsetAsync(vt.p, 0, kv_elems * sizeof(bf16), ctx->stream));
        const size_t kvd = (size_t)B * s.KV * max_ctx * s.hd;
        kd.alloc(kvd);
        vd.alloc(kvd);
        kv_d = KvCache{kd.p, vd.p, 1, B, s.KV, max_ctx, s.hd};
        RS_CUDA(cudaMemsetAsync(kd.p, 0, kvd * sizeof(bf16), ctx->stream));
        RS_CUDA(cudaMemsetAsync(vd.p, 0, kvd * sizeof(bf16), ctx->stream));
        feat.alloc((size_t)B * max_ctx * 3 * s.d);
        dh.alloc((size_t)B * t_max * s.d);
        rbase.alloc(B);
        w.alloc(std::max(B * slots_max, 2048), s);
        stage.alloc(std::max<size_t>(16u << 20, (size_t)w.Mcap * 64 * 8));
        dkv_len.assign(n_req, 0);
    }

    void upload(Batch &b, cudaStream_t st) {
        if (b.M() > w.Mcap) throw std::runtime_error("forward batch exceeds workspace");
        {  // tensor-core attention plan
            b.plan_tc(s.H / s.KV);
            w.ensure_passes(b.passes.size(), st);
            stage.upload(w.passes.p, b.passes, st);
            stage.upload(w.groups.p, b.groups, st);
            stage.upload(w.tok_grp.p, b.tok_grp, st);
        }
        stage.upload(w.rows.p, b.rows, st);
        stage.upload(w.items.p, b.items, st);
        stage.upload(w.map_a.p, b.map_a, st);
        stage.upload(w.map_b.p, b.map_b, st);
    }

    // Target decoder stack over rows embedded in w.x; optional LM head (row m -> map_a[m]).
    void target_forward(const SdDev &d, int M, int ni, float *logits, bool use_map, cudaStream_t st,
                        double *stats = nullptr) {
        const int qd = s.qkv_dim(), HD = s.H * s.hd;
        const double attn_f = prof_enabled() ? bt.attn_flops(s) : 0, attn_b = prof_enabled() ? bt.attn_bytes(s) : 0;
        k_embed(w.rows.p, M, d.tok, d.tok_cap, d.chain_tok, d.t_max, d.n_max, tgt->emb, s.V, s.d, w.x.p, st);
        int fslot = 0;
        for (int l = 0; l < s.L; ++l) {
            const LayerW &lw = tgt->layers[l];
            k_rmsnorm(w.x.p, s.d, lw.ln1, M, s.d, s.eps, w.xn.p, s.d, st);
            if (fused_qkv_rope(s)) {
                gemm(w.xn.p, s.d, lw.qkv_w, M, qd, s.d, epi_qkv_rope(w.q.p, lw.qkv_b, w.rows.p, tgt->rope, kv_t, l, s.H),
                     st);
            } else {
                gemm(w.xn.p, s.d, lw.qkv_w, M, qd, s.d, epi_bf16(w.qkv.p, qd, lw.qkv_b), st);
                k_rope_store(w.qkv.p, w.rows.p, M, s, tgt->rope, kv_t, l, w.q.p, st);
            }
            k_attention_tc(w.q.p, w.rows.p, w.items.p, AttnPlan{w.passes.p, w.groups.p, w.tok_grp.p}, ni, kv_t, l, s,
                           w.ao.p, st, attn_f, attn_b);
            gemm(w.ao.p, HD, lw.o_w, M, s.d, HD, epi_resid(w.x.p, s.d), st);
            k_rmsnorm(w.x.p, s.d, lw.ln2, M, s.d, s.eps, w.xn.p, s.d, st);
            gemm(w.xn.p, s.d, lw.gu_w, M, 2 * s.dff, s.d, epi_swiglu(w.h.p, s.dff), st);
            gemm(w.h.p, s.dff, lw.down_w, M, s.d, s.dff, epi_resid(w.x.p, s.d), st);
            while (fslot < 3 && tgt->feat_layers[fslot] == l)
                k_store_features(w.x.p, w.rows.p, M, s.d, feat.p, max_ctx, fslot++, st);
        }
        if (logits) {
            k_rmsnorm(w.x.p, s.d, tgt->final_norm, M, s.d, s.eps, w.xn.p, s.d, st);
            gemm(w.xn.p, s.d, tgt->emb, M, s.V, s.d, epi_f32(logits, s.V, s.logit_scale, use_map ? w.map_a.p : nullptr),
                 st);
            if (stats) row_stats(logits, use_map ? w.map_a.p : nullptr, M, s.V, tgt->temperature, stats, st);
        }
    }

    // EAGLE fc: w.x = fin . fc_w^T over the gathered low/mid/high features (split-K into zeroed rows).
    void drafter_fc(int M, cudaStream_t st) {
        RS_CUDA(cudaMemsetAsync(w.x.p, 0, (size_t)M * s.d * sizeof(float), st));
        gemm(w.fin.p, 3 * s.d, drf->fc_w, M, s.d, 3 * s.d, epi_resid(w.x.p, s.d), st, drafter_splits(3 * s.d));
    }

    // EAGLE drafter layer over rows whose residual input f is in w.x.
    void drafter_layer(const SdDev &d, int M, int ni, cudaStream_t st) {
        const int qd = s.qkv_dim(), HD = s.H * s.hd, d2 = 2 * s.d;
        k_embed(w.rows.p, M, d.tok, d.tok_cap, d.chain_tok, d.t_max, d.n_max, tgt->emb, s.V, s.d, w.e32.p, st);
        k_rmsnorm(w.e32.p, s.d, drf->norm_emb, M, s.d, s.eps, w.xn.p, d2, st);
        k_rmsnorm(w.x.p, s.d, drf->norm_hid, M, s.d, s.eps, w.xn.p + s.d, d2, st);
        if (fused_qkv_rope(s)) {
            gemm(w.xn.p, d2, drf->layer.qkv_w, M, qd, d2,
                 epi_qkv_rope(w.q.p, drf->layer.qkv_b, w.rows.p, tgt->rope, kv_d, 0, s.H), st);
        } else {
            gemm(w.xn.p, d2, drf->layer.qkv_w, M, qd, d2, epi_bf16(w.qkv.p, qd, drf->layer.qkv_b), st);
            k_rope_store(w.qkv.p, w.rows.p, M, drf->s, tgt->rope, kv_d, 0, w.q.p, st);
        }
        k_attention_tc(w.q.p, w.rows.p, w.items.p, AttnPlan{w.passes.p, w.groups.p, w.tok_grp.p}, ni, kv_d, 0, drf->s,
                       w.ao.p, st, prof_enabled() ? bt.attn_flops(s) : 0, prof_enabled() ? bt.attn_bytes(s) : 0);
        gemm(w.ao.p, HD, drf->layer.o_w, M, s.d, HD, epi_resid(w.x.p, s.d), st, drafter_splits(HD));
        k_rmsnorm(w.x.p, s.d, drf->layer.ln2, M, s.d, s.eps, w.xn.p, s.d, st);
        gemm(w.xn.p, s.d, drf->layer.gu_w, M, 2 * s.dff, s.d, epi_swiglu(w.h.p, s.dff), st);
        gemm(w.h.p, s.dff, drf->layer.down_w, M, s.d, s.dff, epi_resid(w.x.p, s.d), st, drafter_splits(s.dff));
    }

    // Drafter LM head over n normalised rows in w.xn -> Q rows dst[m]; every drafted row is
    // sampled, so its softmax tile partials come out of the GEMM epilogue (the fp64 exps run
    // on the epilogue warps while the next tile accumulates) unless tuned off.
    void lm_head_q(float *Q, double *qst, const int32_t *dst, int n, cudaStream_t st) {
        // Measured on B200 (cfg2): the fp64 exps do NOT hide under the next tile's MMAs with
        // four epilogue warps (drafter GEMMs 1.76 -> 2.78 ms/step vs 0.41 ms for the separate
        // full-chip kernel), so the separate kernel is the default.
        const bool fused = qst && tuning().fused_stats > 0;
        gemm(w.xn.p, s.d, drf->lm_w, n, s.V, s.d,
             epi_f32(Q, s.V, s.logit_scale, dst, fused ? qst : nullptr, drf->temperature), st);
        if (qst && !fused) row_stats(Q, dst, n, s.V, drf->temperature, qst, st);
    }

    // LM head of the drafter on n selected rows of w.x (src rows, Q destination rows).
    void drafter_head(const int32_t *src_dev, const int32_t *dst_dev, int n, float *Q, double *qst, cudaStream_t st) {
        float *g = w.e32.p;  // gathered rows
        k_rows_copy_f32(w.x.p, s.d, src_dev, g, s.d, nullptr, n, s.d, st);
        k_rmsnorm(g, s.d, drf->final_norm, n, s.d, s.eps, w.xn.p, s.d, st);
        lm_head_q(Q, qst, dst_dev, n, st);
    }

    // ---- ModelPair hooks ---------------------------------------------------------------------
    void draft_rows(const SdDev &d, int depth, cudaStream_t st) override {
        if (!drf) throw std::runtime_error("BatchEngine: spec mode requires a drafter snapshot");
        const int nact = d.nact;
        float *Q = static_cast<float *>(const_cast<void *>(d.Q));
        if (depth == 0) {
            // catch-up rows [dkv_len, len-1] per request; the last one is the round root.
            int a0 = 0;
            while (a0 < nact) {
                bt.clear();
                std::vector<int32_t> head_src, head_dst, hid_src, hid_dst;
                int a = a0;
                for (; a < nact; ++a) {
                    const int r = eng->active[a];
                    const int L = eng->len[r];
                    const int from = std::min(dkv_len[r], L - 1);
                    const int room = w.Mcap - bt.M();
                    if (room <= 0) break;
                    // a catch-up longer than the workspace (the first spec cycle at an 8K context)
                    // runs in consecutive chunks: each chunk's rows attend to the drafter keys the
                    // previous chunks stored, so the result is the same as one pass
                    const int to = std::min(L, from + room);
                    const int r0 = bt.M();
                    for (int p = from; p < to; ++p) bt.rows.push_back(RowDesc{r, p, p, 0, -1, 0, 0, 0});
                    bt.add_items(r0, bt.M(), per_item_t, -1, 0, 0, 0);
                    dkv_len[r] = to;
                    if (to < L) break;  // batch full mid-request: continue it in the next batch
                    head_src.push_back(bt.M() - 1);
                    head_dst.push_back(a * d.slots);
                    for (int i = 0; i < d.t; ++i) {
                        hid_src.push_back(bt.M() - 1);
                        hid_dst.push_back(r * d.t_max + i);
                    }
                }
                bt.map_a = head_src;
                bt.map_b = head_dst;
                upload(bt, st);
                std::vector<int32_t> hid(hid_src);
                hid.insert(hid.end(), hid_dst.begin(), hid_dst.end());
                stage.upload(w.idx.p, hid, st);
                const int M = bt.M();
                k_gather_features(w.rows.p, M, s.d, feat.p, max_ctx, nullptr, w.fin.p, nullptr, st);
                drafter_fc(M, st);
                drafter_layer(d, M, (int)bt.items.size(), st);
                drafter_head(w.map_a.p, w.map_b.p, (int)head_src.size(), Q, const_cast<double *>(d.Qst), st);
                const int nh = (int)hid_src.size();
                k_rows_copy_f32(w.x.p, s.d, w.idx.p, dh.p, s.d, w.idx.p + nh, nh, s.d, st);
                a0 = a;
            }
            return;
        }
        // depth j: one row per (request, chain); token chain_i[j-1] at logical len-1+j
        bt.clear();
        for (int a = 0; a < nact; ++a) {
            const int r = eng->active[a];
            const int L = eng->len[r];
            const int r0 = bt.M();
            for (int i = 0; i < d.t; ++i) {
                bt.rows.push_back(RowDesc{r, L - 1 + depth, L + i * d.n + depth - 1, 1, i, depth - 1, 1, r * d.t_max + i});
                bt.map_a.push_back(r * d.t_max + i);                 // hidden slot in / out
                bt.map_b.push_back(a * d.slots + 1 + i * d.n + depth);  // Q row
            }
            bt.add_tree_items_tc(r0, bt.M(), per_item_t, L, L, d.n);
        }
        upload(bt, st);
        const int M = bt.M();
        k_rows_copy_f32(dh.p, s.d, w.map_a.p, w.x.p, s.d, nullptr, M, s.d, st);
        drafter_layer(d, M, (int)bt.items.size(), st);
        k_rmsnorm(w.x.p, s.d, drf->final_norm, M, s.d, s.eps, w.xn.p, s.d, st);
        lm_head_q(Q, const_cast<double *>(d.Qst), w.map_b.p, M, st);
        k_rows_copy_f32(w.x.p, s.d, nullptr, dh.p, s.d, w.map_a.p, M, s.d, st);
    }

    void verify_rows(const SdDev &d, bool naive, cudaStream_t st) override {
        const int nact = d.nact;
        float *P = static_cast<float *>(const_cast<void *>(d.P));
        bt.clear();
        std::vector<int32_t> base(B, 0);
        for (int a = 0; a < nact; ++a) {
            const int r = eng->active[a];
            const int L = eng->len[r];
            base[r] = L;
            const int r0 = bt.M();
            bt.rows.push_back(RowDesc{r, L - 1, L - 1, 0, -1, 0, 0, 0});
            bt.map_a.push_back(a * d.slots);
            if (naive) {
                bt.add_items(r0, bt.M(), per_item_t, -1, 0, 0, 0);
                continue;
            }
            for (int i = 0; i < d.t; ++i)
                for (int j = 0; j < d.n; ++j) {
                    bt.rows.push_back(RowDesc{r, L + j, L + i * d.n + j, 1, i, j, 0, 0});
                    bt.map_a.push_back(a * d.slots + 1 + i * d.n + j);
                }
            // one CTA per (sequence, kv head) for the whole tree; the root rides with chain 0
            bt.add_tree_items_tc(r0, bt.M(), per_item_t, L, L, d.n);
        }
        upload(bt, st);
        if (!naive) stage.upload(rbase.p, base, st);
        if (!naive && lazy_lm_head(d)) {
            // lazy verify LM head: the final norm of every row, the logits of the ROOT rows only
            // (row a * slots of the batch; P slot 0 of sequence a); the selected chains' rows follow
            // in verify_rows_selected once the acceptance's branch point picked them
            target_forward(d, bt.M(), (int)bt.items.size(), nullptr, false, st);
            k_rmsnorm(w.x.p, s.d, tgt->final_norm, bt.M(), s.d, s.eps, w.xn.p, s.d, st);
            gemm(w.xn.p, d.slots * s.d, tgt->emb, nact, s.V, s.d, epi_f32(P, d.slots * s.V, s.logit_scale, nullptr), st);
            return;
        }
        // no stats pass over the verified rows: acceptance computes the 2-3 rows it touches
        target_forward(d, bt.M(), (int)bt.items.size(), P, true, st, d.lazy_pst ? nullptr : const_cast<double *>(d.Pst));
    }

    bool lazy_lm_head(const SdDev &d) const override { return tuning().lazy_lm >= 0 && d.lazy_pst && d.n > 0; }

    void verify_rows_selected(const SdDev &d, cudaStream_t st) override {
        float *P = static_cast<float *>(const_cast<void *>(d.P));
        const int m = d.nact * d.n;
        k_gather_selected(w.xn.p, d.active, d.stg, d.chain_len, d.t_max, d.nact, d.n, d.slots, s.d, w.h.p, w.idx.p, st);
        gemm(w.h.p, s.d, tgt->emb, m, s.V, s.d, epi_f32(P, s.V, s.logit_scale, w.idx.p), st);
    }

    void after_accept(const SdDev &d, bool naive, cudaStream_t st) override {
        if (naive) return;
        ProfScope prof("compact", 0, 0, st);
        k_compact(d, d.rsel, d.racc, rbase.p, kv_t, feat.p, 3 * s.d, max_ctx, st);
    }

    // ---- whole-drafter KD (kd_update, learner.cpp:62-82 / :146-151) ---------------------------
    // One training sequence = a request slot r of this pair's batch (tokens in d.tok row r) with
    // prompt length plen and length len; its rows are positions 0..len-2, the KD rows (one per
    // response token) positions plen-1..len-2: w * KL(p~ || q) of the next token's distribution.
    struct KdTrainSeq {
        int r, plen, len;
        double w, bias;
    };
    // Activations of the teacher-forced drafter forward, one row per (sequence, position), kept
    // for the backward pass; plus the backward's scratch. Grow-only (repeated updates allocate
    // nothing).
    struct TrainStore {
        DBuf<bf16> fin, hc, q, ao, h2, hs, hf;  // [P][3d] [P][2d] [P][HD] [P][HD] [P][d] [P][dff] [P][d]
        DBuf<float> f, x1, x2;                   // [P][d] fp32 residual stream
        DBuf<float> dhf, dx2, dx1, gterm, wide;  // [P][d] x3, [P][2d], [P][max(dff, 2d, qd)]
        DBuf<bf16> gu, dgu, nb, tA, tB;          // [P][2dff] x2, [P][max(d, HD, qd)], transposes
        DBuf<float> partial;                     // column-sum partials
        DBuf<bf16> WdT, WguT, WoT, WqkvT, lmT;   // transposed drafter weights
        DBuf<float> S, dP;                       // attention backward, per (sequence, GQA group)
        DBuf<bf16> P, dS, PT, dST, KT, QT, dOT, Qs, dOs;  // Qs / dOs: a GQA group's heads stacked
        DBuf<float> dQs;
        DBuf<int32_t> pos, rowmap;
        DBuf<bf16> dz;                           // [Rp][V] dZ row-major
    } trs;

    // Teacher-forced drafter forward over M rows (in w.rows / w.items) whose first global row is
    // o: the drafter_fc + drafter_layer + final-norm ops with every activation the backward pass
    // needs written to the store (same kernels, same arithmetic as the drafting path).
    void drafter_forward_train(const SdDev &d, int M, int ni, size_t o, cudaStream_t st) {
        TrainStore &T = trs;
        const int qd = s.qkv_dim(), HD = s.H * s.hd, d2 = 2 * s.d;
        bf16 *fin = T.fin.p + o * 3 * s.d, *hc = T.hc.p + o * d2, *q = T.q.p + o * HD, *ao = T.ao.p + o * HD;
        bf16 *h2 = T.h2.p + o * s.d, *hs = T.hs.p + o * s.dff, *hf = T.hf.p + o * s.d;
        float *f = T.f.p + o * s.d, *x1 = T.x1.p + o * s.d, *x2 = T.x2.p + o * s.d;
        k_gather_features(w.rows.p, M, s.d, feat.p, max_ctx, nullptr, fin, nullptr, st);
        RS_CUDA(cudaMemsetAsync(f, 0, (size_t)M * s.d * sizeof(float), st));
        gemm(fin, 3 * s.d, drf->fc_w, M, s.d, 3 * s.d, epi_resid(f, s.d), st, drafter_splits(3 * s.d));
        k_embed(w.rows.p, M, d.tok, d.tok_cap, d.chain_tok, d.t_max, d.n_max, tgt->emb, s.V, s.d, w.e32.p, st);
        k_rmsnorm(w.e32.p, s.d, drf->norm_emb, M, s.d, s.eps, hc, d2, st);
        k_rmsnorm(f, s.d, drf->norm_hid, M, s.d, s.eps, hc + s.d, d2, st);
        if (fused_qkv_rope(s)) {
            gemm(hc, d2, drf->layer.qkv_w, M, qd, d2, epi_qkv_rope(q, drf->layer.qkv_b, w.rows.p, tgt->rope, kv_d, 0, s.H),
                 st);
        } else {
            gemm(hc, d2, drf->layer.qkv_w, M, qd, d2, epi_bf16(w.qkv.p, qd, drf->layer.qkv_b), st);
            k_rope_store(w.qkv.p, w.rows.p, M, drf->s, tgt->rope, kv_d, 0, q, st);
        }
        k_attention_tc(q, w.rows.p, w.items.p, AttnPlan{w.passes.p, w.groups.p, w.tok_grp.p}, ni, kv_d, 0, drf->s, ao, st);
        RS_CUDA(cudaMemcpyAsync(x1, f, (size_t)M * s.d * sizeof(float), cudaMemcpyDeviceToDevice, st));
        gemm(ao, HD, drf->layer.o_w, M, s.d, HD, epi_resid(x1, s.d), st, drafter_splits(HD));
        k_rmsnorm(x1, s.d, drf->layer.ln2, M, s.d, s.eps, h2, s.d, st);
        gemm(h2, s.d, drf->layer.gu_w, M, 2 * s.dff, s.d, epi_swiglu(hs, s.dff), st);
        RS_CUDA(cudaMemcpyAsync(x2, x1, (size_t)M * s.d * sizeof(float), cudaMemcpyDeviceToDevice, st));
        gemm(hs, s.dff, drf->layer.down_w, M, s.d, s.dff, epi_resid(x2, s.d), st, drafter_splits(s.dff));
        k_rmsnorm(x2, s.d, drf->final_norm, M, s.d, s.eps, hf, s.d, st);
    }

    // Whole-drafter KD over `seqs`: (1) the drafter forward over every row, teacher-forced from
    // the target's EAGLE features (which must already be in `feat`, with the target KV cache
    // holding every row's keys); (2) per group of <= Mcap KD rows: target logits (P), drafter
    // logits from the stored final-norm rows (Q), K5 (loss, dZ), dW_lm += dZ^T h and dh_final =
    // dZ W_lm; (3) the backward pass of the drafter layer, fc and norms over every row, the
    // causal attention backward per (sequence, head) on the tensor cores. Accumulates into
    // `grad` (drafter_grad_layout); returns sum_rows w KL.
    double kd_train(const SdDev &d, const std::vector<KdTrainSeq> &seqs, float *grad, int Mcap, cudaStream_t st) {
        TrainStore &T = trs;
        const int V = s.V, qd = s.qkv_dim(), HD = s.H * s.hd, d2 = 2 * s.d, G = s.H / s.KV, hd = s.hd;
        const DrafterGradLayout gl = drafter_grad_layout(s);
        std::vector<size_t> row0(seqs.size());
        size_t P = 0;
        long long nkd = 0;
        int Tmax = 1;
        for (size_t j = 0; j < seqs.size(); ++j) {
            row0[j] = P;
            P += (size_t)std::max(0, seqs[j].len - 1);
            nkd += std::max(0, seqs[j].len - seqs[j].plen);
            Tmax = std::max(Tmax, seqs[j].len - 1);
        }
        if (P == 0 || nkd == 0) return 0.0;
        const int Pp = round64((int)P), Tp = round64(Tmax);
        const int Rcap = (int)std::max<long long>(1, std::min<long long>(Mcap, nkd)), Rp = round64(Rcap);
        const int nt = (V + 255) / 256;
        const int wide = std::max({s.dff, d2, qd});
        const int nbw = std::max({s.d, HD, qd});
        const size_t tcols = (size_t)std::max({2 * s.dff, 3 * s.d, qd, HD}) * Pp;
        T.fin.ensure(P * 3 * s.d);
        T.hc.ensure(P * d2);
        T.q.ensure(P * HD);
        T.ao.ensure(P * HD);
        T.h2.ensure(P * s.d);
        T.hs.ensure(P * s.dff);
        T.hf.ensure(P * s.d);
        for (DBuf<float> *b : {&T.f, &T.x1, &T.x2, &T.dhf, &T.dx2, &T.dx1}) b->ensure(P * s.d);
        T.gterm.ensure(P * d2);
        T.wide.ensure(P * wide);
        T.gu.ensure(P * 2 * s.dff);
        T.dgu.ensure(P * 2 * s.dff);
        T.nb.ensure(P * nbw);
        T.tA.ensure(tcols);
        T.tB.ensure(tcols);
        T.partial.ensure((size_t)64 * std::max(qd, d2));
        T.WdT.ensure((size_t)s.dff * s.d);
        T.WguT.ensure((size_t)s.d * 2 * s.dff);
        T.WoT.ensure((size_t)HD * s.d);
        T.WqkvT.ensure((size_t)d2 * qd);
        T.lmT.ensure((size_t)s.d * V);
        const size_t GTp = (size_t)round64(G * Tmax);  // stacked rows of one GQA group
        T.S.ensure(GTp * Tp);
        T.dP.ensure(GTp * Tp);
        for (DBuf<bf16> *b : {&T.P, &T.dS, &T.PT, &T.dST}) b->ensure(GTp * Tp);
        T.KT.ensure((size_t)hd * Tp);
        for (DBuf<bf16> *b : {&T.QT, &T.dOT, &T.Qs, &T.dOs}) b->ensure((size_t)hd * GTp);
        T.dQs.ensure((size_t)hd * GTp);
        T.pos.ensure(P);
        T.rowmap.ensure(Rcap);
        T.dz.ensure((size_t)Rp * V);
        KdScratch &k = kd_scr;
        k.Pb.ensure((size_t)Rcap * V);
        k.Qb.ensure((size_t)Rcap * V);
        k.stP.ensure((size_t)Rcap * nt * 2);
        k.stQ.ensure((size_t)Rcap * nt * 2);
        k.kl.ensure((size_t)Rcap * nt);
        for (DBuf<double> *b : {&k.lseP, &k.lseQ, &k.lossr, &k.wr, &k.br}) b->ensure(Rcap);
        k.dzT.ensure((size_t)V * Rp);
        k.hT.ensure((size_t)s.d * Rp);
        k.hG.ensure((size_t)Rcap * s.d);

        // ---- (1) drafter forward over every row, chunks of <= Mcap rows ----
        prof_set_scope("kd_drafter");
        {
            size_t j = 0;
            int p = 0;
            size_t o = 0;
            while (j < seqs.size()) {
                bt.clear();
                while (j < seqs.size() && bt.M() < Mcap) {
                    const int last = seqs[j].len - 2;
                    if (p > last) {
                        ++j;
                        p = 0;
                        continue;
                    }
                    const int take = std::min(last - p + 1, Mcap - bt.M());
                    const int r0 = bt.M();
                    for (int q = 0; q < take; ++q, ++p) bt.rows.push_back(RowDesc{seqs[j].r, p, p, 0, -1, 0, 0, 0});
                    bt.add_items(r0, bt.M(), per_item_t, -1, 0, 0, 0);
                }
                const int M = bt.M();
                if (M == 0) break;
                upload(bt, st);
                drafter_forward_train(d, M, (int)bt.items.size(), o, st);
                o += (size_t)M;
                RS_CUDA(cudaStreamSynchronize(st));
                stage.off = 0;
            }
        }
        std::vector<int32_t> hpos(P);
        for (size_t j = 0; j < seqs.size(); ++j)
            for (int p = 0; p < seqs[j].len - 1; ++p) hpos[row0[j] + p] = p;
        stage.upload(T.pos.p, hpos, st);

        // weights transposed once per update (the input-gradient GEMMs take W^T as operand)
        transpose_pad_bf16(drf->lm_w, s.d, V, s.d, T.lmT.p, V, st);
        transpose_pad_bf16(drf->layer.down_w, s.dff, s.d, s.dff, T.WdT.p, s.d, st);
        transpose_pad_bf16(drf->layer.gu_w, s.d, 2 * s.dff, s.d, T.WguT.p, 2 * s.dff, st);
        transpose_pad_bf16(drf->layer.o_w, HD, s.d, HD, T.WoT.p, s.d, st);
        transpose_pad_bf16(drf->layer.qkv_w, d2, qd, d2, T.WqkvT.p, qd, st);
        RS_CUDA(cudaMemsetAsync(T.dhf.p, 0, P * s.d * sizeof(float), st));

        // ---- (2) K5 per group of KD rows ----
        double loss = 0.0;
        std::vector<double> lh(Rcap);
        size_t j = 0;
        int p = seqs.empty() ? 0 : seqs[0].plen - 1;
        while (j < seqs.size()) {
            struct Run {
                size_t grow;  // first global row
                int n, k0;    // rows, first group row
            };
            std::vector<Run> runs;
            std::vector<double> kd_w, kd_b;
            std::vector<int32_t> gmap;
            bt.clear();
            while (j < seqs.size() && bt.M() < Mcap) {
                const int last = seqs[j].len - 2;
                if (p > last) {
                    if (++j < seqs.size()) p = seqs[j].plen - 1;
                    continue;
                }
                const int take = std::min(last - p + 1, Mcap - bt.M());
                const int r0 = bt.M();
                runs.push_back(Run{row0[j] + (size_t)p, take, r0});
                for (int q = 0; q < take; ++q, ++p) {
                    bt.rows.push_back(RowDesc{seqs[j].r, p, p, 0, -1, 0, 0, 0});
                    kd_w.push_back(seqs[j].w);
                    kd_b.push_back(seqs[j].bias);
                    gmap.push_back((int32_t)(row0[j] + (size_t)p));
                }
                bt.add_items(r0, bt.M(), per_item_t, -1, 0, 0, 0);
            }
            const int R = bt.M();
            if (R == 0) break;
            prof_set_scope("kd_target");
            upload(bt, st);
            target_forward(d, R, (int)bt.items.size(), k.Pb.p, false, st);
            prof_set_scope("kd_k5");
            for (const Run &u : runs)  // the group's final-norm rows, contiguous
                RS_CUDA(cudaMemcpyAsync(k.hG.p + (size_t)u.k0 * s.d, T.hf.p + u.grow * s.d, (size_t)u.n * s.d * sizeof(bf16),
                                        cudaMemcpyDeviceToDevice, st));
            // drafter logits of the whole group in one LM-head pass (the 622 MB weight streams once
            // per group, not once per rollout; rows are bitwise the per-run GEMM's: token-tile invariance)
            gemm(k.hG.p, s.d, drf->lm_w, R, V, s.d, epi_f32(k.Qb.p, V, s.logit_scale, nullptr), st);
            stage.upload(k.wr.p, kd_w, st);
            stage.upload(k.br.p, kd_b, st);
            stage.upload(T.rowmap.p, gmap, st);
            kd_tile_stats(k.Pb.p, k.Qb.p, R, V, tgt->temperature, drf->temperature, k.stP.p, k.stQ.p, st);
            kd_rows_lse(k.Pb.p, k.stP.p, R, V, tgt->temperature, k.br.p, k.lseP.p, st);
            kd_rows_lse(k.Qb.p, k.stQ.p, R, V, drf->temperature, k.br.p, k.lseQ.p, st);
            const int Rq = round64(R);
            kd_rows_elem(k.Pb.p, k.Qb.p, k.lseP.p, k.lseQ.p, k.wr.p, k.br.p, R, V, tgt->temperature, drf->temperature,
                         s.logit_scale, k.dzT.p, Rq, k.kl.p, k.lossr.p, st);
            prof_set_scope("kd_grad");
            transpose_pad_bf16(k.hG.p, s.d, R, s.d, k.hT.p, Rq, st);
            // dW_lm[V][d] += dZ^T[V][Rq] . (h^T[d][Rq])^T
            gemm_ld(k.dzT.p, Rq, k.hT.p, Rq, V, s.d, Rq, epi_resid(grad + gl.lm, s.d), st);
            // dh_final[row] = dZ[row] . W_lm  (dZ row-major from dZ^T; W_lm^T as the operand)
            transpose_pad_bf16(k.dzT.p, Rq, V, R, T.dz.p, V, st);
            gemm_ld(T.dz.p, V, T.lmT.p, V, R, s.d, V, epi_f32(T.dhf.p, s.d, 1.0f, T.rowmap.p), st);
            RS_CUDA(cudaMemcpyAsync(lh.data(), k.lossr.p, (size_t)R * 8, cudaMemcpyDeviceToHost, st));
            RS_CUDA(cudaStreamSynchronize(st));
            for (int q = 0; q < R; ++q) loss += lh[q];
            stage.off = 0;
        }

        // ---- (3) backward over every row ----
        prof_set_scope("kd_backward");
        const int Pi = (int)P;
        float *dqkv = T.wide.p;  // [P][qd] fp32 (reused below: dhs [P][dff], dh [P][2d])
        // final norm: dx2 = dRMS(x2) . dh_final; d final_norm
        rms_bwd(T.x2.p, s.d, drf->final_norm, T.dhf.p, s.d, Pi, s.d, s.eps, nullptr, 0, T.dx2.p, s.d, T.gterm.p, s.d,
                st);
        colsum_f32(T.gterm.p, s.d, Pi, s.d, grad + gl.final_norm, true, T.partial.p, 64, st);
        // down projection: dhs = dx2 . W_d, dW_d += dx2^T hs
        cast_bf16(T.dx2.p, s.d, Pi, s.d, T.nb.p, s.d, st);
        gemm_ld(T.nb.p, s.d, T.WdT.p, s.d, Pi, s.dff, s.d, epi_f32(T.wide.p, s.dff, 1.0f, nullptr), st);
        transpose_pad_bf16(T.nb.p, s.d, Pi, s.d, T.tA.p, Pp, st);
        transpose_pad_bf16(T.hs.p, s.dff, Pi, s.dff, T.tB.p, Pp, st);
        gemm_ld(T.tA.p, Pp, T.tB.p, Pp, s.d, s.dff, Pp, epi_resid(grad + gl.down_w, s.dff), st);
        // SwiGLU: recompute gate/up, dgu
        gemm(T.h2.p, s.d, drf->layer.gu_w, Pi, 2 * s.dff, s.d, epi_bf16(T.gu.p, 2 * s.dff), st);
        swiglu_bwd(T.gu.p, 2 * s.dff, T.wide.p, s.dff, Pi, s.dff, T.dgu.p, 2 * s.dff, st);
        // gate/up projection: dh2 = dgu . W_gu, dW_gu += dgu^T h2
        gemm_ld(T.dgu.p, 2 * s.dff, T.WguT.p, 2 * s.dff, Pi, s.d, 2 * s.dff, epi_f32(T.wide.p, s.d, 1.0f, nullptr), st);
        transpose_pad_bf16(T.dgu.p, 2 * s.dff, Pi, 2 * s.dff, T.tA.p, Pp, st);
        transpose_pad_bf16(T.h2.p, s.d, Pi, s.d, T.tB.p, Pp, st);
        gemm_ld(T.tA.p, Pp, T.tB.p, Pp, 2 * s.dff, s.d, Pp, epi_resid(grad + gl.gu_w, s.d), st);
        // post-attention norm: dx1 = dx2 + dRMS(x1) . dh2; d ln2
        rms_bwd(T.x1.p, s.d, drf->layer.ln2, T.wide.p, s.d, Pi, s.d, s.eps, T.dx2.p, s.d, T.dx1.p, s.d, T.gterm.p, s.d,
                st);
        colsum_f32(T.gterm.p, s.d, Pi, s.d, grad + gl.ln2, true, T.partial.p, 64, st);
        // O projection: da = dx1 . W_o (bf16, the attention backward's dO), dW_o += dx1^T ao
        cast_bf16(T.dx1.p, s.d, Pi, s.d, T.nb.p, s.d, st);
        transpose_pad_bf16(T.nb.p, s.d, Pi, s.d, T.tA.p, Pp, st);
        transpose_pad_bf16(T.ao.p, HD, Pi, HD, T.tB.p, Pp, st);
        gemm_ld(T.tA.p, Pp, T.tB.p, Pp, s.d, HD, Pp, epi_resid(grad + gl.o_w, HD), st);
        bf16 *da = T.gu.p;  // gate/up no longer needed: [P][HD] bf16
        gemm_ld(T.nb.p, s.d, T.WoT.p, s.d, Pi, HD, s.d, epi_bf16(da, HD), st);
        // attention backward per (sequence, GQA group): the group's G query heads stacked as
        // G*Tn rows, so each step is one GEMM per group instead of one per head: S = Q K^T,
        // dP = dO V^T, softmax backward, dV += P^T dO and dK += dS^T Q (the head sum inside the
        // GEMM's K loop), dQ = dS K (K / V post-RoPE from the private drafter cache)
        RS_CUDA(cudaMemsetAsync(dqkv, 0, P * qd * sizeof(float), st));
        const float scale = 1.0f / sqrtf((float)hd);
        for (size_t jj = 0; jj < seqs.size(); ++jj) {
            const int Tn = seqs[jj].len - 1;
            if (Tn <= 0) continue;
            const int Tq = round64(Tn), GT = G * Tn, GTq = round64(GT);
            const size_t g0 = row0[jj];
            float *rowq = dqkv + g0 * qd;
            for (int g = 0; g < s.KV; ++g) {
                const bf16 *Kg = kv_d.k + kv_d.off(0, seqs[jj].r, g, 0), *Vg = kv_d.v + kv_d.off(0, seqs[jj].r, g, 0);
                stack_heads(T.q.p + g0 * HD + (size_t)g * G * hd, HD, Tn, G, hd, T.Qs.p, st);
                stack_heads(da + g0 * HD + (size_t)g * G * hd, HD, Tn, G, hd, T.dOs.p, st);
                transpose_pad_bf16(Kg, hd, Tn, hd, T.KT.p, Tq, st);
                gemm_ld(T.Qs.p, hd, Kg, hd, GT, Tn, hd, epi_f32(T.S.p, Tq, 1.0f, nullptr), st);
                gemm_ld(T.dOs.p, hd, Vg, hd, GT, Tn, hd, epi_f32(T.dP.p, Tq, 1.0f, nullptr), st);
                softmax_bwd(T.S.p, T.dP.p, Tq, GT, Tn, scale, T.P.p, T.dS.p, Tq, st);
                transpose_pad_bf16(T.P.p, Tq, GT, Tn, T.PT.p, GTq, st);
                transpose_pad_bf16(T.dS.p, Tq, GT, Tn, T.dST.p, GTq, st);
                transpose_pad_bf16(T.dOs.p, hd, GT, hd, T.dOT.p, GTq, st);
                transpose_pad_bf16(T.Qs.p, hd, GT, hd, T.QT.p, GTq, st);
                gemm_ld(T.PT.p, GTq, T.dOT.p, GTq, Tn, hd, GTq, epi_resid(rowq + HD + s.KV * hd + g * hd, qd), st);
                gemm_ld(T.dST.p, GTq, T.QT.p, GTq, Tn, hd, GTq, epi_resid(rowq + HD + g * hd, qd), st);
                gemm_ld(T.dS.p, Tq, T.KT.p, Tq, GT, hd, Tq, epi_f32(T.dQs.p, hd, 1.0f, nullptr), st);
                unstack_heads(T.dQs.p, Tn, G, hd, rowq + (size_t)g * G * hd, qd, st);
            }
        }
        // RoPE backward on dq, dk; QKV bias; dh = dqkv . W_qkv; dW_qkv += dqkv^T h
        rope_bwd(dqkv, qd, Pi, s.H, hd, T.pos.p, tgt->rope, st);
        rope_bwd(dqkv + HD, qd, Pi, s.KV, hd, T.pos.p, tgt->rope, st);
        colsum_f32(dqkv, qd, Pi, qd, grad + gl.qkv_b, true, T.partial.p, 64, st);
        cast_bf16(dqkv, qd, Pi, qd, T.nb.p, qd, st);
        transpose_pad_bf16(T.nb.p, qd, Pi, qd, T.tA.p, Pp, st);
        transpose_pad_bf16(T.hc.p, d2, Pi, d2, T.tB.p, Pp, st);
        gemm_ld(T.tA.p, Pp, T.tB.p, Pp, qd, d2, Pp, epi_resid(grad + gl.qkv_w, d2), st);
        float *dh = T.wide.p;  // [P][2d] (dqkv consumed)
        gemm_ld(T.nb.p, qd, T.WqkvT.p, qd, Pi, d2, qd, epi_f32(dh, d2, 1.0f, nullptr), st);
        // input norms: d norm_emb (the embedding itself is the target's, frozen); df = dx1 +
        // dRMS(f) . dh[:, d:], d norm_hid
        {
            // embedding rows again (fp32), per chunk of <= Mcap rows into the workspace
            for (size_t jj = 0, o = 0; jj < seqs.size(); ++jj) {
                for (int p0 = 0; p0 < seqs[jj].len - 1;) {
                    const int n = std::min(seqs[jj].len - 1 - p0, w.Mcap);
                    bt.clear();
                    for (int q = 0; q < n; ++q) bt.rows.push_back(RowDesc{seqs[jj].r, p0 + q, p0 + q, 0, -1, 0, 0, 0});
                    stage.upload(w.rows.p, bt.rows, st);
                    k_embed(w.rows.p, n, d.tok, d.tok_cap, d.chain_tok, d.t_max, d.n_max, tgt->emb, s.V, s.d, w.e32.p, st);
                    rms_bwd(w.e32.p, s.d, drf->norm_emb, dh + o * d2, d2, n, s.d, s.eps, nullptr, 0, nullptr, 0,
                            T.gterm.p + o * s.d, s.d, st);
                    RS_CUDA(cudaStreamSynchronize(st));
                    stage.off = 0;
                    o += (size_t)n;
                    p0 += n;
                }
            }
            colsum_f32(T.gterm.p, s.d, Pi, s.d, grad + gl.norm_emb, true, T.partial.p, 64, st);
        }
        rms_bwd(T.f.p, s.d, drf->norm_hid, dh + s.d, d2, Pi, s.d, s.eps, T.dx1.p, s.d, T.dx2.p, s.d, T.gterm.p, s.d, st);
        colsum_f32(T.gterm.p, s.d, Pi, s.d, grad + gl.norm_hid, true, T.partial.p, 64, st);
        // fc: dW_fc += df^T fin (df in dx2)
        cast_bf16(T.dx2.p, s.d, Pi, s.d, T.nb.p, s.d, st);
        transpose_pad_bf16(T.nb.p, s.d, Pi, s.d, T.tA.p, Pp, st);
        transpose_pad_bf16(T.fin.p, 3 * s.d, Pi, 3 * s.d, T.tB.p, Pp, st);
        gemm_ld(T.tA.p, Pp, T.tB.p, Pp, s.d, 3 * s.d, Pp, epi_resid(grad + gl.fc, 3 * s.d), st);
        RS_CUDA(cudaStreamSynchronize(st));
        stage.off = 0;
        return loss;
    }

    // kd_pass: detached training sequences (tokens uploaded into d.tok, one batch slot each);
    // the target runs teacher-forced over every row first (its KV cache and EAGLE features),
    // then kd_train.
    double kd_pass(const SdDev &d, const std::vector<KdSeq> &seqs, float *grad) {
        cudaStream_t st = ctx->stream;
        prof_set_scope("kd_target");
        size_t r = 0;
        int p = 0;
        while (r < seqs.size()) {
            bt.clear();
            while (r < seqs.size() && bt.M() < w.Mcap) {
                const int len = (int)seqs[r].tokens.size();
                if (p >= len - 1) {
                    ++r;
                    p = 0;
                    continue;
                }
                const int take = std::min(len - 1 - p, w.Mcap - bt.M());
                const int r0 = bt.M();
                for (int k = 0; k < take; ++k, ++p) bt.rows.push_back(RowDesc{(int)r, p, p, 0, -1, 0, 0, 0});
                bt.add_items(r0, bt.M(), per_item_t, -1, 0, 0, 0);
            }
            if (bt.M() == 0) break;
            upload(bt, st);
            target_forward(d, bt.M(), (int)bt.items.size(), nullptr, false, st);
            RS_CUDA(cudaStreamSynchronize(st));
            stage.off = 0;
        }
        std::vector<KdTrainSeq> ts;
        for (size_t i = 0; i < seqs.size(); ++i)
            ts.push_back(KdTrainSeq{(int)i, seqs[i].prompt_len, (int)seqs[i].tokens.size(), seqs[i].weight,
                                    seqs[i].eos_bias});
        return kd_train(d, ts, grad, w.Mcap, st);
    }

    // KD from the engine's RESIDENT state instead of a teacher-forced recompute of prompt +
    // response: the target KV cache already holds every position 0..len-2 of each request and
    // `feat` its EAGLE features (prefill, verify forwards, K4 compaction); the target re-runs
    // only over the KD rows for their logits (rewriting their keys bit-identically -- every
    // kernel on the path is row-invariant). The drafter (the given snapshot, not the engine's)
    // runs teacher-forced into a private drafter KV cache, so the engine's own drafter state is
    // untouched. Same loss / gradient as kd_pass on the same sequences.
    double kd_cached(const std::vector<KdRef> &refs, const rs_model *m, float *grad,
                     cudaStream_t on = nullptr) override {
        if (!m || m->kind != rs_model::Drafter) throw std::invalid_argument("kd: EAGLE drafter required");
        const auto *kd_drf = static_cast<const DrafterModel *>(m);
        if (kd_drf->target != tgt) throw std::invalid_argument("kd: drafter is bound to a different target");
        for (const auto &x : refs)
            if (x.req < 0 || x.req >= eng->n) throw std::invalid_argument("kd: request index out of range");
        SdDev d{};
        d.tok = eng->d_tok.p;
        d.tok_cap = eng->tok_cap;
        d.t_max = 1;
        d.n_max = 1;
        cudaStream_t st = on ? on : ctx->stream;
        const int Mcap = tuning().kd_rows > 0 ? std::min(w.Mcap, tuning().kd_rows) : w.Mcap;
        KdScratch &k = kd_scr;
        const size_t kvd = (size_t)B * s.KV * max_ctx * s.hd;
        k.tk.ensure(kvd);
        k.tv.ensure(kvd);
        RS_CUDA(cudaMemsetAsync(k.tk.p, 0, kvd * sizeof(bf16), st));
        RS_CUDA(cudaMemsetAsync(k.tv.p, 0, kvd * sizeof(bf16), st));
        struct Swap {  // private drafter cache + the KD snapshot for the duration of the pass
            TransformerPair &t;
            KvCache kv;
            const DrafterModel *m;
            ~Swap() {
                t.kv_d = kv;
                t.drf = m;
            }
        } swap{*this, kv_d, drf};
        kv_d = KvCache{k.tk.p, k.tv.p, 1, B, s.KV, max_ctx, s.hd};
        drf = kd_drf;
        std::vector<KdTrainSeq> ts;
        for (const auto &x : refs)
            ts.push_back(KdTrainSeq{x.req, eng->prompt_len[x.req], eng->len[x.req], x.weight, x.eos_bias});
        return kd_train(d, ts, grad, Mcap, st);
    }

    // Target prefill of prompt positions 0..P-2 (the last prompt token is the first root).
    void prefill(const std::vector<std::vector<int>> &prompts, const SdDev &d) {
        cudaStream_t st = ctx->stream;
        size_t r = 0;
        int p = 0;
        while (r < prompts.size()) {
            bt.clear();
            while (r < prompts.size() && bt.M() < w.Mcap) {
                const int P = (int)prompts[r].size();
                if (p >= P - 1) {
                    ++r;
                    p = 0;
                    continue;
                }
                const int take = std::min(P - 1 - p, w.Mcap - bt.M());
                const int r0 = bt.M();
                for (int k = 0; k < take; ++k, ++p) bt.rows.push_back(RowDesc{(int)r, p, p, 0, -1, 0, 0, 0});
                bt.add_items(r0, bt.M(), per_item_t, -1, 0, 0, 0);
            }
            if (bt.M() == 0) break;
            upload(bt, st);
            target_forward(d, bt.M(), (int)bt.items.size(), nullptr, false, st);
            RS_CUDA(cudaStreamSynchronize(st));
            stage.off = 0;
        }
    }
};

}  // namespace

std::unique_ptr<ModelPair> make_transformer_pair(rs_ctx *ctx, rs_engine *eng, const rs_model *target,
                                                 const rs_model *drafter, int n_req, int slots_max,
                                                 const std::vector<int> &prompt_lens,
                                                 const std::vector<std::vector<int>> &prompts, int tok_cap) {
    if (target->kind != rs_model::Transformer) throw std::invalid_argument("transformer pair: bad target");
    if (drafter && drafter->kind != rs_model::Drafter)
        throw std::invalid_argument("transformer target needs an EAGLE drafter");
    auto p = std::make_unique<TransformerPair>(ctx, eng, static_cast<const TransformerModel *>(target),
                                               static_cast<const DrafterModel *>(drafter));
    if (drafter && static_cast<const DrafterModel *>(drafter)->target != p->tgt)
        throw std::invalid_argument("drafter is bound to a different target");
    p->setup(n_req, slots_max, prompt_lens, tok_cap, eng->t_max);
    p->prefill(prompts, eng->dev(rs_sdconfig{1, 1, 1, 0}, 0));
    return p;
}

DrafterGradLayout drafter_grad_layout(const TfShape &s) {
    DrafterGradLayout g;
    size_t o = 0;
    auto take = [&](size_t n) {
        const size_t at = o;
        o += (n + 63) / 64 * 64;  // 256-byte aligned tensors
        return at;
    };
    const size_t q = s.qkv_dim(), HD = (size_t)s.H * s.hd;
    g.lm = take((size_t)s.V * s.d);
    g.fc = take((size_t)s.d * 3 * s.d);
    g.norm_emb = take(s.d);
    g.norm_hid = take(s.d);
    g.qkv_w = take(q * 2 * s.d);
    g.qkv_b = take(q);
    g.o_w = take((size_t)s.d * HD);
    g.ln2 = take(s.d);
    g.gu_w = take((size_t)2 * s.dff * s.d);
    g.down_w = take((size_t)s.d * s.dff);
    g.final_norm = take(s.d);
    g.total = o;
    return g;
}

double kd_grad_transformer(rs_ctx *ctx, const TransformerModel *tgt, const DrafterModel *drf,
                           const std::vector<KdSeq> &seqs, float *grad, bool zero_grad) {
    if (!tgt || !drf || drf->target != tgt) throw std::invalid_argument("kd: drafter is bound to a different target");
    cudaStream_t st = ctx->stream;
    if (zero_grad) RS_CUDA(cudaMemsetAsync(grad, 0, drafter_grad_layout(drf->s).total * sizeof(float), st));
    if (seqs.empty()) return 0.0;
    int tok_cap = 1;
    std::vector<int> plen;
    for (const auto &q : seqs) {
        if (q.prompt_len < 1 || (int)q.tokens.size() < q.prompt_len)
            throw std::invalid_argument("kd: prompts must be non-empty");
        tok_cap = std::max(tok_cap, (int)q.tokens.size());
        plen.push_back(q.prompt_len);
    }
    if (tok_cap + 1 > tgt->s.max_ctx) throw std::invalid_argument("kd: sequence exceeds the model's max_ctx");
    const int n = (int)seqs.size();
    std::vector<int32_t> htok((size_t)n * tok_cap, 0);
    for (int i = 0; i < n; ++i) std::copy(seqs[i].tokens.begin(), seqs[i].tokens.end(), htok.begin() + (size_t)i * tok_cap);
    DBuf<int32_t> tok(htok.size());
    RS_CUDA(cudaMemcpyAsync(tok.p, htok.data(), htok.size() * 4, cudaMemcpyHostToDevice, st));
    note_copy(true, htok.size() * 4);
    TransformerPair p(ctx, nullptr, tgt, drf);
    p.setup(n, 1, plen, tok_cap, 1);
    SdDev d{};
    d.tok = tok.p;
    d.tok_cap = tok_cap;
    d.t_max = 1;
    d.n_max = 1;
    const double loss = p.kd_pass(d, seqs, grad);
    RS_CUDA(cudaStreamSynchronize(st));
    prof_collect();
    prof_set_scope("step");
    return loss;
}

DrafterModel *drafter_apply_lm_grad(rs_ctx *ctx, const DrafterModel *drf, const float *grad, double scale) {
    auto m = std::make_unique<DrafterModel>();
    m->ctx = ctx;
    m->vocab = drf->vocab;
    m->temperature = drf->temperature;
    m->version = drf->version + 1;
    m->target = drf->target;
    m->s = drf->s;
    carve_drafter(*m);
    if (m->arena.n != drf->arena.n) throw std::logic_error("drafter arena layout mismatch");
    cudaStream_t st = ctx->stream;
    RS_CUDA(cudaMemcpyAsync(m->arena.p, drf->arena.p, m->arena.n, cudaMemcpyDeviceToDevice, st));
    if (grad && scale != 0.0) {  // every drafter tensor: w + scale * grad (drafter_grad_layout)
        const TfShape &s = m->s;
        const DrafterGradLayout gl = drafter_grad_layout(s);
        const float sc = (float)scale;
        const size_t q = s.qkv_dim(), HD = (size_t)s.H * s.hd;
        sgd_bf16(drf->lm_w, grad + gl.lm, sc, (size_t)s.V * s.d, m->lm_w, st);
        sgd_bf16(drf->fc_w, grad + gl.fc, sc, (size_t)s.d * 3 * s.d, m->fc_w, st);
        sgd_f32(drf->norm_emb, grad + gl.norm_emb, sc, s.d, m->norm_emb, st);
        sgd_f32(drf->norm_hid, grad + gl.norm_hid, sc, s.d, m->norm_hid, st);
        sgd_bf16(drf->layer.qkv_w, grad + gl.qkv_w, sc, q * 2 * s.d, m->layer.qkv_w, st);
        sgd_bf16(drf->layer.qkv_b, grad + gl.qkv_b, sc, q, m->layer.qkv_b, st);
        sgd_bf16(drf->layer.o_w, grad + gl.o_w, sc, (size_t)s.d * HD, m->layer.o_w, st);
        sgd_f32(drf->layer.ln2, grad + gl.ln2, sc, s.d, m->layer.ln2, st);
        sgd_bf16(drf->layer.gu_w, grad + gl.gu_w, sc, (size_t)2 * s.dff * s.d, m->layer.gu_w, st);
        sgd_bf16(drf->layer.down_w, grad + gl.down_w, sc, (size_t)s.d * s.dff, m->layer.down_w, st);
        sgd_f32(drf->final_norm, grad + gl.final_norm, sc, s.d, m->final_norm, st);
    }
    RS_CUDA(cudaStreamSynchronize(st));
    return m.release();
}

TransformerModel *create_transformer(rs_ctx *ctx, const rs_transformer_shape &sh, uint64_t seed) {
    TfShape s;
    s.V = sh.vocab;
    s.d = sh.d_model;
    s.L = sh.n_layers;
    s.H = sh.n_heads;
    s.KV = sh.n_kv_heads;
    s.hd = sh.head_dim;
    s.dff = sh.d_ff;
    s.max_ctx = sh.max_ctx;
    s.rope_theta = sh.rope_theta > 0 ? sh.rope_theta : 1e6f;
    s.eps = sh.rms_eps > 0 ? sh.rms_eps : 1e-6f;
    s.std = sh.init_std > 0 ? sh.init_std : 0.02f;
    s.logit_scale = sh.logit_scale > 0 ? sh.logit_scale : 1.0f;
    if (s.V < 2 || s.d <= 0 || s.L <= 0 || s.H <= 0 || s.KV <= 0 || s.max_ctx <= 0)
        throw std::invalid_argument("transformer shape: non-positive dimension");
    if (s.hd != 128) throw std::invalid_argument("transformer shape: head_dim must be 128");
    if (s.H % s.KV || s.H / s.KV > 64)
        throw std::invalid_argument("transformer shape: n_heads must be a multiple of n_kv_heads (group <= 64)");
    if (s.d % 64 || s.dff % 128) throw std::invalid_argument("transformer shape: d_model % 64 and d_ff % 128 required");
    if (s.max_ctx > 14000) throw std::invalid_argument("transformer shape: max_ctx must be <= 14000");
    if (!(sh.temperature > 0.0)) throw std::invalid_argument("TabularARModel: temperature must be positive");
    auto m = std::make_unique<TransformerModel>();
    m->ctx = ctx;
    m->vocab = s.V;
    m->temperature = sh.temperature;
    m->version = 0;
    m->s = s;
    init_transformer(*m, seed, ctx->stream);
    RS_CUDA(cudaStreamSynchronize(ctx->stream));
    return m.release();
}

DrafterModel *create_drafter(rs_ctx *ctx, const rs_model *target, uint64_t seed, int version) {
    if (target->kind != rs_model::Transformer) throw std::invalid_argument("rs_drafter_create: target must be a transformer");
    const auto *t = static_cast<const TransformerModel *>(target);
    auto m = std::make_unique<DrafterModel>();
    m->ctx = ctx;
    m->vocab = t->vocab;
    m->temperature = t->temperature;
    m->version = version;
    m->target = t;
    m->s = t->s;
    m->s.L = 1;
    init_drafter(*m, seed, ctx->stream);
    RS_CUDA(cudaStreamSynchronize(ctx->stream));
    return m.release();
}

}  // namespace rs

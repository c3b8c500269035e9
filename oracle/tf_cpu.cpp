// oracle/tf_cpu.cpp -- TEST INFRASTRUCTURE ONLY. CPU port of the CUDA path's transformer models
// (see tf_cpu.hpp). Compiled with OpenMP; the restated acceptance logic (restate.cpp) is a
// separate translation unit with strict IEEE flags.
#include "tf_cpu.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>

namespace orc {

namespace {

uint16_t f2bf(float f) {  // round to nearest even (__float2bfloat16)
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
inline float bf2f(uint16_t h) {
    const uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
inline float rbf(float x) { return bf2f(f2bf(x)); }

// model.cu init_normal_kernel: splitmix64(seed, tensor id, index) -> two uniforms -> Box-Muller
void init_normal(std::vector<uint16_t> & p, size_t n, uint64_t seed, uint64_t tid, float stdv) {
    p.assign(n, 0);
    const long long pairs = static_cast<long long>((n + 1) / 2);
#pragma omp parallel for schedule(static)
    for (long long pr = 0; pr < pairs; ++pr) {
        const size_t i = static_cast<size_t>(pr) * 2;
        uint64_t s = seed ^ (tid * 0x9E3779B97F4A7C15ULL) ^ (i * 0xD1B54A32D192ED03ULL);
        const uint64_t a = splitmix64(s), b = splitmix64(s);
        const double u1 = (static_cast<double>(a >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        p[i] = f2bf(static_cast<float>(r * std::cos(2.0 * M_PI * u2)) * stdv);
        if (i + 1 < n) p[i + 1] = f2bf(static_cast<float>(r * std::sin(2.0 * M_PI * u2)) * stdv);
    }
}

void init_layer(TfLayer & w, const TfShape & s, int d_in, uint64_t seed, uint64_t tid) {
    const size_t q = static_cast<size_t>(s.qkv());
    init_normal(w.qkv_w, q * d_in, seed, tid + 0, s.std);
    init_normal(w.qkv_b, q, seed, tid + 1, s.std);
    init_normal(w.o_w, static_cast<size_t>(s.d) * s.H * s.hd, seed, tid + 2, s.std);
    init_normal(w.gu_w, 2 * static_cast<size_t>(s.dff) * s.d, seed, tid + 3, s.std);
    init_normal(w.down_w, static_cast<size_t>(s.d) * s.dff, seed, tid + 4, s.std);
    w.ln1.assign(d_in, 1.0f);
    w.ln2.assign(s.d, 1.0f);
}

// y[m][n] (+)= sum_k x[m][k] * W[n][k]   (x fp32 [M][ldx], W bf16 [N][ldw]); 8 partial sums per
// dot in a fixed order (vectorised without reassociation flags)
void matmul(const float * x, int ldx, int M, int K, const uint16_t * W, int ldw, int N, float * y, int ldy, bool acc,
            float scale = 1.0f) {
#pragma omp parallel
    {
        std::vector<float> wf(static_cast<size_t>(K) + 8);
#pragma omp for schedule(static)
        for (int n = 0; n < N; ++n) {
            const uint16_t * w = W + static_cast<size_t>(n) * ldw;
            for (int k = 0; k < K; ++k) wf[k] = bf2f(w[k]);
            for (int m = 0; m < M; ++m) {
                const float * xm = x + static_cast<size_t>(m) * ldx;
                float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                int k = 0;
                for (; k + 8 <= K; k += 8)
                    for (int j = 0; j < 8; ++j) a[j] += xm[k + j] * wf[k + j];
                for (; k < K; ++k) a[k & 7] += xm[k] * wf[k];
                const float dot = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
                float * o = y + static_cast<size_t>(m) * ldy + n;
                *o = acc ? *o + dot * scale : dot * scale;
            }
        }
    }
}

// bf16(x * rsqrt(mean(x^2) + eps) * w) per row
void rmsnorm(const float * x, int ldx, int M, int d, const float * w, float eps, float * out, int ldo) {
    for (int m = 0; m < M; ++m) {
        const float * r = x + static_cast<size_t>(m) * ldx;
        double ss = 0;
        for (int i = 0; i < d; ++i) ss += static_cast<double>(r[i]) * r[i];
        const float inv = 1.0f / std::sqrt(static_cast<float>(ss / d) + eps);
        for (int i = 0; i < d; ++i) out[static_cast<size_t>(m) * ldo + i] = rbf(r[i] * inv * w[i]);
    }
}

// Qwen2 rotate-half RoPE in place on bf16-rounded values (cos / sin from the double table of model.cu)
void rope_row(float * x, int heads, int hd, int pos, float theta) {
    const int half = hd / 2;
    for (int i = 0; i < half; ++i) {
        const double inv = std::pow(static_cast<double>(theta), -2.0 * i / hd);
        const float c = static_cast<float>(std::cos(pos * inv)), sn = static_cast<float>(std::sin(pos * inv));
        for (int h = 0; h < heads; ++h) {
            float * v = x + static_cast<size_t>(h) * hd;
            const float x1 = v[i], x2 = v[i + half];
            v[i] = rbf(x1 * c - x2 * sn);
            v[i + half] = rbf(x2 * c + x1 * sn);
        }
    }
}

// One decoder layer over M new rows (positions pos0 .. pos0 + M - 1) of a sequence whose layer
// cache (k, v: [pos][KV*hd]) holds every earlier position; x is the fp32 residual stream [M][d],
// h the bf16-rounded layer input [M][d_in] (normed by the caller for the drafter).
void layer_forward(const TfShape & s, const TfLayer & w, int d_in, const float * h, float * x, int M, int pos0,
                   std::vector<float> & kc, std::vector<float> & vc, bool norm_input) {
    const int H = s.H, KV = s.KV, hd = s.hd, G = H / KV, q = s.qkv();
    std::vector<float> hn(static_cast<size_t>(M) * d_in), qkv(static_cast<size_t>(M) * q);
    if (norm_input) rmsnorm(x, s.d, M, s.d, w.ln1.data(), s.eps, hn.data(), d_in);
    else std::memcpy(hn.data(), h, sizeof(float) * hn.size());
    matmul(hn.data(), d_in, M, d_in, w.qkv_w.data(), d_in, q, qkv.data(), q, false);
    for (int m = 0; m < M; ++m) {
        float * r = qkv.data() + static_cast<size_t>(m) * q;
        for (int i = 0; i < q; ++i) r[i] = rbf(r[i] + bf2f(w.qkv_b[i]));
        rope_row(r, H + KV, hd, pos0 + m, s.rope_theta);  // q and k heads rotate, v heads do not
        kc.insert(kc.end(), r + H * hd, r + (H + KV) * hd);
        vc.insert(vc.end(), r + (H + KV) * hd, r + q);
    }
    // causal GQA attention over the cache, fp32 softmax, bf16 output
    std::vector<float> ao(static_cast<size_t>(M) * H * hd);
    const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
#pragma omp parallel for schedule(dynamic) collapse(2)
    for (int m = 0; m < M; ++m)
        for (int hh = 0; hh < H; ++hh) {
            const int np = pos0 + m + 1, kvh = hh / G;
            const float * qv = qkv.data() + static_cast<size_t>(m) * q + static_cast<size_t>(hh) * hd;
            std::vector<float> sc(np);
            float mx = -INFINITY;
            for (int p = 0; p < np; ++p) {
                const float * kr = kc.data() + (static_cast<size_t>(p) * KV + kvh) * hd;
                float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int i = 0; i < hd; i += 8)
                    for (int j = 0; j < 8; ++j) a[j] += qv[i + j] * kr[i + j];
                sc[p] = (((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]))) * scale;
                mx = std::max(mx, sc[p]);
            }
            float l = 0;
            for (int p = 0; p < np; ++p) {
                sc[p] = std::exp(sc[p] - mx);
                l += sc[p];
            }
            float o[256] = {0};
            for (int p = 0; p < np; ++p) {
                const float * vr = vc.data() + (static_cast<size_t>(p) * KV + kvh) * hd;
                const float pp = sc[p] / l;
                for (int i = 0; i < hd; ++i) o[i] += pp * vr[i];
            }
            float * dst = ao.data() + (static_cast<size_t>(m) * H + hh) * hd;
            for (int i = 0; i < hd; ++i) dst[i] = rbf(o[i]);
        }
    matmul(ao.data(), H * hd, M, H * hd, w.o_w.data(), H * hd, s.d, x, s.d, true);
    // SwiGLU MLP (gate / up rows interleaved pairwise: 2i gate_i, 2i + 1 up_i)
    std::vector<float> h2(static_cast<size_t>(M) * s.d), gu(static_cast<size_t>(M) * 2 * s.dff),
        mlp(static_cast<size_t>(M) * s.dff);
    rmsnorm(x, s.d, M, s.d, w.ln2.data(), s.eps, h2.data(), s.d);
    matmul(h2.data(), s.d, M, s.d, w.gu_w.data(), s.d, 2 * s.dff, gu.data(), 2 * s.dff, false);
    for (int m = 0; m < M; ++m)
        for (int i = 0; i < s.dff; ++i) {
            const float g = gu[static_cast<size_t>(m) * 2 * s.dff + 2 * i], u = gu[static_cast<size_t>(m) * 2 * s.dff + 2 * i + 1];
            mlp[static_cast<size_t>(m) * s.dff + i] = rbf(g / (1.0f + std::exp(-g)) * u);
        }
    matmul(mlp.data(), s.dff, M, s.dff, w.down_w.data(), s.dff, s.d, x, s.d, true);
}

size_t lcp(const std::vector<int> & a, const std::vector<int> & b) {
    size_t n = 0;
    while (n < a.size() && n < b.size() && a[n] == b[n]) ++n;
    return n;
}

void truncate(TfSeqState & st, size_t n, const TfShape & s, size_t feat_w) {
    const size_t kvw = static_cast<size_t>(s.KV) * s.hd;
    st.tokens.resize(n);
    for (auto & k : st.k) k.resize(n * kvw);
    for (auto & v : st.v) v.resize(n * kvw);
    if (!st.feats.empty() || feat_w == 3) st.feats.resize(n * 3 * s.d);
    if (!st.hidden.empty() || feat_w == 1) st.hidden.resize(n * s.d);
}

// the cached sequence sharing the longest prefix with ctx (a new one when none shares any)
TfSeqState & pick(std::vector<TfSeqState> & cache, const std::vector<int> & ctx, int layers) {
    size_t best = 0, bi = cache.size();
    for (size_t i = 0; i < cache.size(); ++i) {
        const size_t c = lcp(cache[i].tokens, ctx);
        if (c > best) best = c, bi = i;
    }
    if (bi < cache.size()) {
        std::rotate(cache.begin(), cache.begin() + bi, cache.begin() + bi + 1);  // most recent first
        return cache.front();
    }
    if (cache.size() >= 64) cache.pop_back();
    cache.insert(cache.begin(), TfSeqState{});
    cache.front().k.resize(layers);
    cache.front().v.resize(layers);
    return cache.front();
}

void synth(std::vector<float> & v, size_t n, uint64_t seed, float scale) {
    std::vector<uint16_t> b;
    init_normal(b, n, seed, 7, scale);
    v.resize(n);
    for (size_t i = 0; i < n; ++i) v[i] = bf2f(b[i]);
}

}  // namespace

void TfWeights::init_target(const TfShape & sh, uint64_t seed, int) {
    s = sh;
    init_normal(emb, static_cast<size_t>(s.V) * s.d, seed, 1, s.std);
    layers.resize(s.L);
    for (int l = 0; l < s.L; ++l) init_layer(layers[l], s, s.d, seed, 16 + 8 * static_cast<uint64_t>(l));
    final_norm.assign(s.d, 1.0f);
    feat_layers[0] = std::min(1, s.L - 1);
    feat_layers[1] = s.L / 2;
    feat_layers[2] = s.L - 1;
}

void TfWeights::init_drafter(uint64_t seed) {
    init_normal(fc_w, static_cast<size_t>(s.d) * 3 * s.d, seed, 1001, s.std);
    norm_emb.assign(s.d, 1.0f);
    norm_hid.assign(s.d, 1.0f);
    init_layer(dl, s, 2 * s.d, seed, 1010);
    d_final.assign(s.d, 1.0f);
    init_normal(lm_w, static_cast<size_t>(s.V) * s.d, seed, 1020, s.std);
}

// ---- target ------------------------------------------------------------------------------------
CpuTransformer::CpuTransformer(std::shared_ptr<const TfWeights> w, double temperature) : w_(std::move(w)) {
    vocab = w_->s.V;
    this->temperature = temperature;
}

TfSeqState & CpuTransformer::state_for(const std::vector<int> & ctx) const {
    TfSeqState & st = pick(cache_, ctx, w_->s.L);
    truncate(st, lcp(st.tokens, ctx), w_->s, 3);
    return st;
}

void CpuTransformer::extend(TfSeqState & st, const std::vector<int> & ctx, bool want_logits, std::vector<float> * last) const {
    const TfShape & s = w_->s;
    const int pos0 = static_cast<int>(st.tokens.size()), M = static_cast<int>(ctx.size()) - pos0;
    std::vector<float> x(static_cast<size_t>(std::max(M, 0)) * s.d);
    if (M > 0) {
        for (int m = 0; m < M; ++m)
            for (int i = 0; i < s.d; ++i)
                x[static_cast<size_t>(m) * s.d + i] = bf2f(w_->emb[static_cast<size_t>(ctx[pos0 + m]) * s.d + i]);
        st.feats.resize(ctx.size() * 3 * s.d);
        for (int l = 0; l < s.L; ++l) {
            layer_forward(s, w_->layers[l], s.d, nullptr, x.data(), M, pos0, st.k[l], st.v[l], true);
            for (int f = 0; f < 3; ++f)
                if (w_->feat_layers[f] == l)
                    for (int m = 0; m < M; ++m)
                        for (int i = 0; i < s.d; ++i)
                            st.feats[(static_cast<size_t>(pos0 + m) * 3 + f) * s.d + i] = rbf(x[static_cast<size_t>(m) * s.d + i]);
        }
        st.tokens.insert(st.tokens.end(), ctx.begin() + pos0, ctx.end());
    }
    if (want_logits) {
        if (M <= 0) throw std::logic_error("CpuTransformer: the last position is already cached");
        std::vector<float> hn(s.d);
        rmsnorm(x.data() + static_cast<size_t>(M - 1) * s.d, s.d, 1, s.d, w_->final_norm.data(), s.eps, hn.data(), s.d);
        last->resize(s.V);
        matmul(hn.data(), s.d, 1, s.d, w_->emb.data(), s.d, s.V, last->data(), s.V, false, s.logit_scale);
    }
}

std::vector<double> CpuTransformer::logits(const std::vector<int> & ctx) const {
    std::lock_guard<std::mutex> lk(mu_);
    if (ctx.empty()) throw std::invalid_argument("CpuTransformer: empty context");
    TfSeqState & st = pick(cache_, ctx, w_->s.L);
    // the last position is recomputed (its row is what is asked); everything before it is reused
    truncate(st, std::min(lcp(st.tokens, ctx), ctx.size() - 1), w_->s, 3);
    std::vector<float> z;
    extend(st, ctx, true, &z);
    return std::vector<double>(z.begin(), z.end());
}

std::vector<float> CpuTransformer::features(const std::vector<int> & ctx, int p) const {
    std::lock_guard<std::mutex> lk(mu_);
    const std::vector<int> pre(ctx.begin(), ctx.begin() + p + 1);
    TfSeqState & st = state_for(pre);
    extend(st, pre, false, nullptr);
    const size_t o = static_cast<size_t>(p) * 3 * w_->s.d;
    return std::vector<float>(st.feats.begin() + o, st.feats.begin() + o + 3 * w_->s.d);
}

void CpuTransformer::synthetic_prefix(const std::vector<int> & ctx, int n, uint64_t seed) const {
    std::lock_guard<std::mutex> lk(mu_);
    const TfShape & s = w_->s;
    TfSeqState & st = pick(cache_, std::vector<int>(ctx.begin(), ctx.begin() + n), s.L);
    st.tokens.assign(ctx.begin(), ctx.begin() + n);
    const size_t kvw = static_cast<size_t>(s.KV) * s.hd;
    for (int l = 0; l < s.L; ++l) {
        synth(st.k[l], n * kvw, seed + 2 * l, 1.0f);
        synth(st.v[l], n * kvw, seed + 2 * l + 1, 1.0f);
    }
    synth(st.feats, static_cast<size_t>(n) * 3 * s.d, seed + 99991, 1.0f);
}

// ---- drafter -----------------------------------------------------------------------------------
CpuEagleDrafter::CpuEagleDrafter(std::shared_ptr<const TfWeights> w, std::shared_ptr<const CpuTransformer> target,
                                 int version)
    : w_(std::move(w)), tgt_(std::move(target)) {
    vocab = w_->s.V;
    temperature = tgt_->temperature;
    this->version = version;
}

// q(. | ctx) at `depth` tokens beyond the round's root: positions below the root take f =
// fc(target features at p - 1) (zero at p = 0), positions at or beyond it the drafter's own
// hidden state at p - 1; one layer over [norm(emb(x_p)), norm(f_p)] with residual f, own LM head.
std::vector<double> CpuEagleDrafter::logits_at(const std::vector<int> & ctx, int depth) const {
    std::lock_guard<std::mutex> lk(mu_);
    const TfShape & s = w_->s;
    const int T = static_cast<int>(ctx.size()), root = T - depth;
    if (T <= 0 || depth < 0 || root <= 0) throw std::invalid_argument("CpuEagleDrafter: bad context / depth");
    TfSeqState & st = pick(cache_, ctx, 1);
    size_t keep = std::min(lcp(st.tokens, ctx), static_cast<size_t>(T - 1));
    keep = std::min(keep, static_cast<size_t>(std::min(st.root > 0 ? st.root : root, root)));
    truncate(st, keep, s, 1);
    st.root = root;
    const int pos0 = static_cast<int>(keep), M = T - pos0;
    std::vector<float> f(static_cast<size_t>(M) * s.d, 0.0f), x, h(static_cast<size_t>(M) * 2 * s.d), e(s.d);
    for (int m = 0; m < M; ++m) {
        const int p = pos0 + m;
        float * fm = f.data() + static_cast<size_t>(m) * s.d;
        if (p >= root) {
            // own hidden state at p - 1 (computed above in this call or cached)
            const float * hp = p - 1 >= pos0 ? nullptr : st.hidden.data() + static_cast<size_t>(p - 1) * s.d;
            if (hp) std::memcpy(fm, hp, sizeof(float) * s.d);
        } else if (p > 0) {
            const std::vector<float> ft = tgt_->features(ctx, p - 1);
            matmul(ft.data(), 3 * s.d, 1, 3 * s.d, w_->fc_w.data(), 3 * s.d, s.d, fm, s.d, false);
        }
    }
    // rows at or beyond the root chain their own hidden states: run them one at a time
    x.resize(static_cast<size_t>(M) * s.d);
    st.hidden.resize(static_cast<size_t>(T) * s.d);
    auto run_rows = [&](int m0, int m1) {
        const int n = m1 - m0;
        for (int m = m0; m < m1; ++m) {
            const int p = pos0 + m;
            float * fm = f.data() + static_cast<size_t>(m) * s.d;
            if (p >= root && p - 1 >= pos0) std::memcpy(fm, st.hidden.data() + static_cast<size_t>(p - 1) * s.d, sizeof(float) * s.d);
            for (int i = 0; i < s.d; ++i) e[i] = bf2f(w_->emb[static_cast<size_t>(ctx[p]) * s.d + i]);
            rmsnorm(e.data(), s.d, 1, s.d, w_->norm_emb.data(), s.eps, h.data() + static_cast<size_t>(m) * 2 * s.d, 2 * s.d);
            rmsnorm(fm, s.d, 1, s.d, w_->norm_hid.data(), s.eps, h.data() + static_cast<size_t>(m) * 2 * s.d + s.d, 2 * s.d);
            std::memcpy(x.data() + static_cast<size_t>(m) * s.d, fm, sizeof(float) * s.d);
        }
        layer_forward(s, w_->dl, 2 * s.d, h.data() + static_cast<size_t>(m0) * 2 * s.d, x.data() + static_cast<size_t>(m0) * s.d, n,
                      pos0 + m0, st.k[0], st.v[0], false);
        for (int m = m0; m < m1; ++m)
            std::memcpy(st.hidden.data() + static_cast<size_t>(pos0 + m) * s.d, x.data() + static_cast<size_t>(m) * s.d,
                        sizeof(float) * s.d);
    };
    const int mroot = std::max(0, std::min(M, root - pos0));
    if (mroot > 0) run_rows(0, mroot);
    for (int m = mroot; m < M; ++m) run_rows(m, m + 1);
    st.tokens.assign(ctx.begin(), ctx.end());
    std::vector<float> hn(s.d), z(s.V);
    rmsnorm(x.data() + static_cast<size_t>(M - 1) * s.d, s.d, 1, s.d, w_->d_final.data(), s.eps, hn.data(), s.d);
    matmul(hn.data(), s.d, 1, s.d, w_->lm_w.data(), s.d, s.V, z.data(), s.V, false, s.logit_scale);
    return std::vector<double>(z.begin(), z.end());
}

void CpuEagleDrafter::synthetic_prefix(const std::vector<int> & ctx, int n, uint64_t seed) const {
    std::lock_guard<std::mutex> lk(mu_);
    const TfShape & s = w_->s;
    TfSeqState & st = pick(cache_, std::vector<int>(ctx.begin(), ctx.begin() + n), 1);
    st.tokens.assign(ctx.begin(), ctx.begin() + n);
    st.root = n;
    const size_t kvw = static_cast<size_t>(s.KV) * s.hd;
    synth(st.k[0], n * kvw, seed + 5, 1.0f);
    synth(st.v[0], n * kvw, seed + 6, 1.0f);
    synth(st.hidden, static_cast<size_t>(n) * s.d, seed + 7, 1.0f);
}

}  // namespace orc

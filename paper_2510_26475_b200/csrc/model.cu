// model.cu -- weights, synthetic init and the elementwise kernels of the transformer forwards
// (embedding gather, RMSNorm, RoPE + KV-cache store, EAGLE feature capture/gather) and K4, the
// in-place KV-cache compaction of accepted tree paths.
#include <cmath>

#include "common.cuh"
#include "model.h"

#include <mutex>
#include <vector>
#include "launch.cuh"
#include "prof.h"
#include "rng.cuh"

namespace rs {

namespace {

__global__ void init_normal_kernel(bf16 *p, size_t n, uint64_t seed, uint64_t tid, float std) {
    // Portable generator: splitmix64(seed, tensor, index) -> two uniforms -> Box-Muller.
    const size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 2;
    if (i >= n) return;
    uint64_t s = seed ^ (tid * 0x9E3779B97F4A7C15ULL) ^ (i * 0xD1B54A32D192ED03ULL);
    const uint64_t a = splitmix64(s), b = splitmix64(s);
    const double u1 = (static_cast<double>(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    p[i] = __float2bfloat16(static_cast<float>(r * cos(2.0 * M_PI * u2)) * std);
    if (i + 1 < n) p[i + 1] = __float2bfloat16(static_cast<float>(r * sin(2.0 * M_PI * u2)) * std);
}

__global__ void fill_f32_kernel(float *p, size_t n, float v) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void rope_table_kernel(float *rope, int max_ctx, int hd, float theta) {
    const int pos = blockIdx.x, i = threadIdx.x;
    if (i >= hd / 2) return;
    const double inv = pow(static_cast<double>(theta), -2.0 * i / hd);
    const double ang = pos * inv;
    rope[((size_t)pos * (hd / 2) + i) * 2 + 0] = static_cast<float>(cos(ang));
    rope[((size_t)pos * (hd / 2) + i) * 2 + 1] = static_cast<float>(sin(ang));
}

__global__ void embed_kernel(const RowDesc *rows, int M, const int32_t *tok, int tok_cap, const int32_t *chain_tok,
                             int t_max, int n_max, const bf16 *emb, int V, int d, float *x) {
    pdl_trigger();
    pdl_wait();
    const int m = blockIdx.x;
    if (m >= M) return;
    const RowDesc r = rows[m];
    int t = r.kind == 0 ? tok[(size_t)r.seq * tok_cap + r.pos]
                        : chain_tok[((size_t)r.seq * t_max + r.chain) * n_max + r.cj];
    t = min(max(t, 0), V - 1);
    const bf16 *e = emb + (size_t)t * d;
    float *o = x + (size_t)m * d;
    for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
        const int4 raw = *reinterpret_cast<const int4 *>(e + i);
        const bf16 *h = reinterpret_cast<const bf16 *>(&raw);
        float4 a = make_float4(__bfloat162float(h[0]), __bfloat162float(h[1]), __bfloat162float(h[2]),
                               __bfloat162float(h[3]));
        float4 b = make_float4(__bfloat162float(h[4]), __bfloat162float(h[5]), __bfloat162float(h[6]),
                               __bfloat162float(h[7]));
        *reinterpret_cast<float4 *>(o + i) = a;
        *reinterpret_cast<float4 *>(o + i + 4) = b;
    }
}

__device__ __forceinline__ void load8(const float *p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4 *>(p), b = *reinterpret_cast<const float4 *>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const bf16 *p, float (&v)[8]) {
    const int4 raw = *reinterpret_cast<const int4 *>(p);
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&raw);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        v[2 * k] = f.x;
        v[2 * k + 1] = f.y;
    }
}
__device__ __forceinline__ void store8(bf16 *p, const float (&v)[8]) {
    __align__(16) __nv_bfloat162 h[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
    *reinterpret_cast<int4 *>(p) = *reinterpret_cast<const int4 *>(h);
}

// Two rows per 256-thread CTA (128 threads per row, NG groups of 8 elements per thread), so a
// verify batch of ~1.3K rows is a single wave of resident CTAs; the gain vector is read before
// the programmatic-dependency wait (weights never depend on the previous kernel).
// y = x * rsqrt(mean(x^2) + eps) * w (Qwen2RMSNorm, fp32 math); d % 8 == 0, d <= 8192.
template <class T, int NG>
__global__ void __launch_bounds__(256) rmsnorm2_kernel(const T *x, int ldx, const float *w, int M, int d, float eps,
                                                       bf16 *out, int ldo) {
    pdl_trigger();
    const int half = threadIdx.x >> 7, t = threadIdx.x & 127;
    float wv[NG][8];
#pragma unroll
    for (int k = 0; k < NG; ++k) {
        const int i = (t + k * 128) * 8;
        if (i < d) load8(w + i, wv[k]);
    }
    pdl_wait();
    __shared__ float red[8];
    const int row = blockIdx.x * 2 + half;
    const bool live = row < M;
    const T *xr = x + (size_t)(live ? row : 0) * ldx;
    float v[NG][8];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < NG; ++k) {
        const int i = (t + k * 128) * 8;
        if (live && i < d) {
            load8(xr + i, v[k]);
#pragma unroll
            for (int j = 0; j < 8; ++j) ss += v[k][j] * v[k][j];
        }
    }
    ss = warp_sumf(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    const float tot = (red[half * 4] + red[half * 4 + 1]) + (red[half * 4 + 2] + red[half * 4 + 3]);
    if (!live) return;
    const float inv = rsqrtf(tot / d + eps);
    bf16 *o = out + (size_t)row * ldo;
#pragma unroll
    for (int k = 0; k < NG; ++k) {
        const int i = (t + k * 128) * 8;
        if (i < d) {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[k][j] = v[k][j] * inv * wv[k][j];
            store8(o + i, v[k]);
        }
    }
}

template <class T>
void launch_rmsnorm2(const T *x, int ldx, const float *w, int M, int d, float eps, bf16 *out, int ldo, cudaStream_t st) {
    const int ng = (d / 8 + 127) / 128;
    const int grid = (M + 1) / 2;
    switch (ng) {
#define RS_NG(n) \
    case n: launch_pdl(rmsnorm2_kernel<T, n>, grid, 256, 0, st, x, ldx, w, M, d, eps, out, ldo); break;
        RS_NG(1) RS_NG(2) RS_NG(3) RS_NG(4) RS_NG(5) RS_NG(6) RS_NG(7) RS_NG(8)
#undef RS_NG
        default: throw std::invalid_argument("rmsnorm: d must be <= 8192");
    }
}

// RoPE (rotate-half, Qwen2) on q and k; q -> qbuf [M][H][hd]; k, v -> cache at the row's slot.
// One CTA per row; a thread rotates 8 dimension pairs (i, i + hd/2) with 16-byte accesses.
__global__ void __launch_bounds__(256) rope_store_kernel(const bf16 *qkv, const RowDesc *rows, int M, int H, int KV,
                                                         int hd, const float *rope, KvCache kv, int layer, bf16 *q) {
    pdl_trigger();
    pdl_wait();
    const int m = blockIdx.x;
    const RowDesc r = rows[m];
    const int qd = (H + 2 * KV) * hd;
    const bf16 *src = qkv + (size_t)m * qd;
    const int half = hd / 2, groups = half / 8;
    const float *cs = rope + (size_t)r.pos * half * 2;
    for (int idx = threadIdx.x; idx < (H + KV) * groups; idx += blockDim.x) {
        const int head = idx / groups, i = (idx % groups) * 8;
        const bf16 *h = src + head * hd;
        float x1[8], x2[8], c[8], s[8], o1[8], o2[8];
        load8(h + i, x1);
        load8(h + i + half, x2);
        float t[16];
        load8(cs + 2 * i, *reinterpret_cast<float(*)[8]>(t));
        load8(cs + 2 * i + 8, *reinterpret_cast<float(*)[8]>(t + 8));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c[j] = t[2 * j];
            s[j] = t[2 * j + 1];
            o1[j] = x1[j] * c[j] - x2[j] * s[j];
            o2[j] = x2[j] * c[j] + x1[j] * s[j];
        }
        bf16 *dst = head < H ? q + ((size_t)m * H + head) * hd : kv.k + kv.off(layer, r.seq, head - H, r.phys);
        store8(dst + i, o1);
        store8(dst + i + half, o2);
    }
    const int vec = hd / 8;
    for (int idx = threadIdx.x; idx < KV * vec; idx += blockDim.x) {
        const int head = idx / vec, c8 = idx % vec;
        *reinterpret_cast<int4 *>(kv.v + kv.off(layer, r.seq, head, r.phys) + c8 * 8) =
            *reinterpret_cast<const int4 *>(src + (H + KV) * hd + head * hd + c8 * 8);
    }
}

__global__ void store_features_kernel(const float *x, const RowDesc *rows, int M, int d, bf16 *feat, int max_ctx,
                                      int slot) {
    pdl_trigger();
    pdl_wait();
    const int m = blockIdx.x;
    const RowDesc r = rows[m];
    bf16 *dst = feat + (((size_t)r.seq * max_ctx + r.phys) * 3 + slot) * d;
    const float *src = x + (size_t)m * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = __float2bfloat16(src[i]);
}

// fin[m] = [g_low, g_mid, g_high] of the target at logical position pos-1 (zeros at pos 0).
__global__ void gather_features_kernel(const RowDesc *rows, int M, int d, const bf16 *feat, int max_ctx, bf16 *fin) {
    pdl_trigger();
    pdl_wait();
    const int m = blockIdx.x;
    const RowDesc r = rows[m];
    bf16 *dst = fin + (size_t)m * 3 * d;
    if (r.pos == 0) {
        for (int i = threadIdx.x; i < 3 * d; i += blockDim.x) dst[i] = __float2bfloat16(0.f);
        return;
    }
    const bf16 *src = feat + ((size_t)r.seq * max_ctx + (r.pos - 1)) * 3 * d;
    for (int i = threadIdx.x * 8; i < 3 * d; i += blockDim.x * 8)
        *reinterpret_cast<int4 *>(dst + i) = *reinterpret_cast<const int4 *>(src + i);
}

__global__ void rows_copy_kernel(const float *src, int lds, const int *srows, float *dst, int ldd, const int *drows,
                                 int d) {
    pdl_trigger();
    pdl_wait();
    const int k = blockIdx.x;
    const int sr = srows ? srows[k] : k, dr = drows ? drows[k] : k;
    if (sr < 0 || dr < 0) return;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[(size_t)dr * ldd + i] = src[(size_t)sr * lds + i];
}

// K4: move the accepted path of the selected chain from its tree slots to contiguous
// positions, for every layer's K and V and the EAGLE features. One CTA per (sequence, token);
// 16-byte vector moves, each warp streams whole 256-byte head rows.
__global__ void compact_kernel(SdDev d, const int32_t *rsel, const int32_t *racc, const int32_t *rbase, KvCache kv,
                               bf16 *feat, int feat_w, int max_ctx) {
    pdl_trigger();
    pdl_wait();
    const int a = blockIdx.x, j = blockIdx.y;
    const int r = d.active[a];
    const int sel = rsel[r], acc = racc[r];
    if (sel <= 0 || j >= acc) return;  // chain 0 already sits at the contiguous positions
    const int L0 = rbase[r];
    const int src = L0 + sel * d.n + j, dst = L0 + j;
    const int vec = kv.hd / 8;  // int4 per head row
    const int per_layer = kv.KV * vec;
    for (int idx = threadIdx.x; idx < kv.layers * per_layer; idx += blockDim.x) {
        const int layer = idx / per_layer, rem = idx % per_layer, h = rem / vec, c = rem % vec;
        const int4 *ks = reinterpret_cast<const int4 *>(kv.k + kv.off(layer, r, h, src)) + c;
        const int4 *vs = reinterpret_cast<const int4 *>(kv.v + kv.off(layer, r, h, src)) + c;
        reinterpret_cast<int4 *>(kv.k + kv.off(layer, r, h, dst))[c] = *ks;
        reinterpret_cast<int4 *>(kv.v + kv.off(layer, r, h, dst))[c] = *vs;
    }
    if (feat) {
        const int4 *fs = reinterpret_cast<const int4 *>(feat + ((size_t)r * max_ctx + src) * feat_w);
        int4 *fd = reinterpret_cast<int4 *>(feat + ((size_t)r * max_ctx + dst) * feat_w);
        for (int i = threadIdx.x; i < feat_w / 8; i += blockDim.x) fd[i] = fs[i];
    }
}

}  // namespace

void k_init_normal(bf16 *p, size_t n, uint64_t seed, uint64_t tid, float std, cudaStream_t st) {
    if (!n) return;
    const size_t pairs = (n + 1) / 2;
    init_normal_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(p, n, seed, tid, std);
    RS_LAUNCHED();
}

void k_fill_f32(float *p, size_t n, float v, cudaStream_t st) {
    if (!n) return;
    fill_f32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, n, v);
    RS_LAUNCHED();
}

void k_rope_table(float *rope, int max_ctx, int hd, float theta, cudaStream_t st) {
    rope_table_kernel<<<max_ctx, std::max(32, hd / 2), 0, st>>>(rope, max_ctx, hd, theta);
    RS_LAUNCHED();
}

void k_embed(const RowDesc *rows, int M, const int32_t *tok, int tok_cap, const int32_t *chain_tok, int t_max,
             int n_max, const bf16 *emb, int V, int d, float *x, cudaStream_t st) {
    if (M <= 0) return;
    ProfScope prof("embed", 0, (double)M * d * 6.0, st);
    launch_pdl(embed_kernel, M, 128, 0, st, rows, M, tok, tok_cap, chain_tok, t_max, n_max, emb, V, d, x);
    RS_LAUNCHED();
}

void k_rmsnorm(const float *x, int ldx, const float *w, int M, int d, float eps, bf16 *out, int ldo, cudaStream_t st) {
    if (M <= 0) return;
    ProfScope prof("norm", 0, (double)M * d * 6.0, st);
    if (d % 8 || d > 8192) throw std::invalid_argument("rmsnorm: d must be a multiple of 8 and <= 8192");
    launch_rmsnorm2(x, ldx, w, M, d, eps, out, ldo, st);
    RS_LAUNCHED();
}

void k_rmsnorm_bf16(const bf16 *x, int ldx, const float *w, int M, int d, float eps, bf16 *out, int ldo,
                    cudaStream_t st) {
    if (M <= 0) return;
    ProfScope prof("norm", 0, (double)M * d * 4.0, st);
    if (d % 8 || d > 8192) throw std::invalid_argument("rmsnorm: d must be a multiple of 8 and <= 8192");
    launch_rmsnorm2(x, ldx, w, M, d, eps, out, ldo, st);
    RS_LAUNCHED();
}

void k_rope_store(const bf16 *qkv, const RowDesc *rows, int M, const TfShape &s, const float *rope, const KvCache &kv,
                  int layer, bf16 *q, cudaStream_t st) {
    if (M <= 0) return;
    ProfScope prof("rope", 0, (double)M * s.qkv_dim() * 4.0, st);
    launch_pdl(rope_store_kernel, M, 256, 0, st, qkv, rows, M, s.H, s.KV, s.hd, rope, kv, layer, q);
    RS_LAUNCHED();
}

void k_store_features(const float *x, const RowDesc *rows, int M, int d, bf16 *feat, int max_ctx, int slot,
                      cudaStream_t st) {
    if (M <= 0) return;
    ProfScope prof("feat", 0, (double)M * d * 6.0, st);
    launch_pdl(store_features_kernel, M, 256, 0, st, x, rows, M, d, feat, max_ctx, slot);
    RS_LAUNCHED();
}

void k_gather_features(const RowDesc *rows, int M, int d, const bf16 *feat, int max_ctx, const float *, bf16 *fin,
                       int *, cudaStream_t st) {
    if (M <= 0) return;
    ProfScope prof("feat", 0, (double)M * d * 12.0, st);
    launch_pdl(gather_features_kernel, M, 256, 0, st, rows, M, d, feat, max_ctx, fin);
    RS_LAUNCHED();
}

void k_rows_copy_f32(const float *src, int ld_src, const int *src_rows, float *dst, int ld_dst, const int *dst_rows,
                     int n, int d, cudaStream_t st) {
    if (n <= 0) return;
    ProfScope prof("copy", 0, (double)n * d * 8.0, st);
    launch_pdl(rows_copy_kernel, n, 256, 0, st, src, ld_src, src_rows, dst, ld_dst, dst_rows, d);
    RS_LAUNCHED();
}

void k_compact(const SdDev &d, const int32_t *rsel, const int32_t *racc, const int32_t *rbase, const KvCache &kv,
               bf16 *feat, int feat_w, int max_ctx, cudaStream_t st) {
    if (d.nact <= 0) return;
    launch_pdl(compact_kernel, dim3(d.nact, d.n), 256, 0, st, d, rsel, racc, rbase, kv, feat, feat_w, max_ctx);
    RS_LAUNCHED();
}

// ---- weights ------------------------------------------------------------------------------------
namespace {
struct Carver {
    char *base;
    size_t off = 0;
    template <class T>
    T *take(size_t n) {
        off = (off + 255) & ~size_t(255);
        T *p = reinterpret_cast<T *>(base + off);
        off += n * sizeof(T);
        return p;
    }
};

size_t layer_bytes(const TfShape &s, int d_in) {
    const size_t q = s.qkv_dim();
    return (q * d_in + q + (size_t)s.d * s.H * s.hd + 2 * (size_t)s.dff * s.d + (size_t)s.d * s.dff) * 2 +
           (size_t)(d_in + s.d) * 4 + 8 * 256;
}

void carve_layer(Carver &c, LayerW &w, const TfShape &s, int d_in) {
    const size_t q = s.qkv_dim();
    w.qkv_w = c.take<bf16>(q * d_in);
    w.qkv_b = c.take<bf16>(q);
    w.o_w = c.take<bf16>((size_t)s.d * s.H * s.hd);
    w.gu_w = c.take<bf16>(2 * (size_t)s.dff * s.d);
    w.down_w = c.take<bf16>((size_t)s.d * s.dff);
    w.ln1 = c.take<float>(d_in);
    w.ln2 = c.take<float>(s.d);
}

void init_layer(LayerW &w, const TfShape &s, int d_in, uint64_t seed, uint64_t tid, cudaStream_t st) {
    const size_t q = s.qkv_dim();
    k_init_normal(w.qkv_w, q * d_in, seed, tid + 0, s.std, st);
    k_init_normal(w.qkv_b, q, seed, tid + 1, s.std, st);
    k_init_normal(w.o_w, (size_t)s.d * s.H * s.hd, seed, tid + 2, s.std, st);
    k_init_normal(w.gu_w, 2 * (size_t)s.dff * s.d, seed, tid + 3, s.std, st);
    k_init_normal(w.down_w, (size_t)s.d * s.dff, seed, tid + 4, s.std, st);
    k_fill_f32(w.ln1, d_in, 1.0f, st);
    k_fill_f32(w.ln2, s.d, 1.0f, st);
}
}  // namespace

void init_transformer(TransformerModel &m, uint64_t seed, cudaStream_t st) {
    const TfShape &s = m.s;
    size_t bytes = (size_t)s.V * s.d * 2 + (size_t)s.L * layer_bytes(s, s.d) + (size_t)s.d * 4 +
                   (size_t)s.max_ctx * s.hd * 4 + 4096;
    m.arena.alloc(bytes);
    Carver c{m.arena.p};
    m.emb = c.take<bf16>((size_t)s.V * s.d);
    m.layers.resize(s.L);
    for (auto &l : m.layers) carve_layer(c, l, s, s.d);
    m.final_norm = c.take<float>(s.d);
    m.rope = c.take<float>((size_t)s.max_ctx * s.hd);
    k_init_normal(m.emb, (size_t)s.V * s.d, seed, 1, s.std, st);
    for (int l = 0; l < s.L; ++l) init_layer(m.layers[l], s, s.d, seed, 16 + 8 * l, st);
    k_fill_f32(m.final_norm, s.d, 1.0f, st);
    k_rope_table(m.rope, s.max_ctx, s.hd, s.rope_theta, st);
    // EAGLE-3 feature layers: low / mid / high hidden states
    m.feat_layers[0] = std::min(1, s.L - 1);
    m.feat_layers[1] = s.L / 2;
    m.feat_layers[2] = s.L - 1;
    const size_t q = s.qkv_dim();
    m.n_params = (size_t)s.V * s.d + (size_t)s.L * (q * s.d + q + (size_t)s.d * s.H * s.hd + 3 * (size_t)s.dff * s.d);
}

// Drafter snapshot arenas are recycled: an online learner publishes a new snapshot per update and
// drops the previous one; at the 3B drafter (~0.8 GB) cudaMalloc + cudaFree cost ~1.3 ms of host
// time per update (publish 1.84 -> 1.15 ms, release 0.59 -> 0.01 ms; tools/snapshot_cost.py), and
// the bench's KD update went from 21-25 ms to a steady 19.9 ms. A released arena is parked (after a
// device synchronisation, the same ordering guarantee cudaFree gave: no kernel still reads it)
// and handed to the next snapshot of the same size on the same device; at most kArenaPool parked.
namespace {
struct ParkedArena {
    int dev;
    size_t bytes;
    char *p;
};
std::mutex arena_mu;
std::vector<ParkedArena> arena_pool;
constexpr size_t kArenaPool = 2;
}  // namespace

DrafterModel::~DrafterModel() {
    if (!arena.p) return;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, arena.p) != cudaSuccess) return;  // DBuf frees it
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != a.device) cudaSetDevice(a.device);
    const bool idle = cudaDeviceSynchronize() == cudaSuccess;
    if (cur != a.device && cur >= 0) cudaSetDevice(cur);
    if (!idle) return;
    std::lock_guard<std::mutex> lk(arena_mu);
    if (arena_pool.size() >= kArenaPool) return;
    arena_pool.push_back(ParkedArena{a.device, arena.n, arena.p});
    arena.p = nullptr;
    arena.n = 0;
}

// Allocate a drafter's weight arena (a parked one when its size matches) and carve its tensors
// (no initialisation).
void carve_drafter(DrafterModel &m) {
    const TfShape &s = m.s;
    size_t bytes = (size_t)s.d * 3 * s.d * 2 + 2 * (size_t)s.d * 4 + layer_bytes(s, 2 * s.d) + (size_t)s.d * 4 +
                   (size_t)s.V * s.d * 2 + 4096;
    int dev = -1;
    RS_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(arena_mu);
        for (size_t i = 0; i < arena_pool.size(); ++i)
            if (arena_pool[i].dev == dev && arena_pool[i].bytes == bytes) {
                m.arena.release();
                m.arena.p = arena_pool[i].p;
                m.arena.n = bytes;
                arena_pool.erase(arena_pool.begin() + (long)i);
                break;
            }
    }
    if (!m.arena.p) m.arena.alloc(bytes);
    Carver c{m.arena.p};
    m.fc_w = c.take<bf16>((size_t)s.d * 3 * s.d);
    m.norm_emb = c.take<float>(s.d);
    m.norm_hid = c.take<float>(s.d);
    carve_layer(c, m.layer, s, 2 * s.d);
    m.final_norm = c.take<float>(s.d);
    m.lm_w = c.take<bf16>((size_t)s.V * s.d);
    const size_t q = s.qkv_dim();
    m.n_params = (size_t)s.d * 3 * s.d + q * 2 * s.d + q + (size_t)s.d * s.H * s.hd + 3 * (size_t)s.dff * s.d +
                 (size_t)s.V * s.d;
}

void init_drafter(DrafterModel &m, uint64_t seed, cudaStream_t st) {
    const TfShape &s = m.s;
    carve_drafter(m);
    k_init_normal(m.fc_w, (size_t)s.d * 3 * s.d, seed, 1001, s.std, st);
    k_fill_f32(m.norm_emb, s.d, 1.0f, st);
    k_fill_f32(m.norm_hid, s.d, 1.0f, st);
    init_layer(m.layer, s, 2 * s.d, seed, 1010, st);
    k_fill_f32(m.final_norm, s.d, 1.0f, st);
    k_init_normal(m.lm_w, (size_t)s.V * s.d, seed, 1020, s.std, st);
}

namespace {
// Lazy verify LM head: the final-normed rows of each active sequence's SELECTED chain (acceptance
// stage 1 parked its index in stg[r * 6], -1 when the cycle already ended) gathered into n rows per
// sequence, and the P row each maps to (-1: no row; the LM head epilogue drops it).
__global__ void gather_selected_kernel(const bf16 *xn, const int32_t *active, const int32_t *stg,
                                       const int32_t *chain_len, int t_max, int n, int slots, int d, bf16 *out,
                                       int32_t *map) {
    pdl_trigger();
    pdl_wait();
    const int m = blockIdx.x, a = m / n, j = m % n;
    const int r = active[a];
    const int sel = stg[(size_t)r * 6];
    const int L = sel >= 0 ? chain_len[(size_t)r * t_max + sel] : 0;
    const bool live = j < L;
    const int src = a * slots + 1 + sel * n + j;
    if (threadIdx.x == 0) map[m] = live ? src : -1;
    if (!live) return;
    const int4 *s4 = reinterpret_cast<const int4 *>(xn + (size_t)src * d);
    int4 *o4 = reinterpret_cast<int4 *>(out + (size_t)m * d);
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x) o4[i] = s4[i];
}
}  // namespace

void k_gather_selected(const bf16 *xn, const int32_t *active, const int32_t *stg, const int32_t *chain_len, int t_max,
                       int nact, int n, int slots, int d, bf16 *out, int32_t *map, cudaStream_t st) {
    if (nact <= 0) return;
    launch_pdl(gather_selected_kernel, nact * n, 128, 0, st, xn, active, stg, chain_len, t_max, n, slots, d, out, map);
    RS_LAUNCHED();
}

}  // namespace rs

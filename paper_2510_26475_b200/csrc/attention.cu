// attention.cu -- tree-causal GQA attention over the per-sequence KV cache.
//
// A work item is a run of query tokens of one sequence; the CTA for (item, kv head) owns those
// tokens x G query heads as rows (row = token * G + head). Tokens are grouped by key mapping:
// a drafted token of chain i sees the context, the root and exactly its own chain prefix --
// the tree-causal mask of SURVEY.md §8 A3 -- i.e. logical positions 0..pos where positions
// >= ltree live in the chain's own slots (tbase + chain * nstride + p - ltree). Each warp owns
// 16 rows of one group. Keys are visited in LOGICAL order in 64-key chunks: chunks wholly
// below ltree are shared by every group (one K/V tile for all 8 x 21 rows of a tree), the
// 1-2 chunks that reach into the tree are replayed once per group with that group's tile.
// Because every row walks the same chunk sequence with the same key values whatever CTA it
// sits in, a token's output is bit-identical whether it is verified inside a tree, decoded
// alone or prefilled (checked by tests/test_transformer_gpu.py).
// Q.K^T and P.V run on the tensor cores with mma.sync m16n8k16 (bf16 in, fp32 accumulate);
// K/V tiles are double-buffered with cp.async into XOR-swizzled shared memory.
#include <cuda_bf16.h>

#include "common.cuh"
#include "model.h"
#include "launch.cuh"
#include "prof.h"

namespace rs {

namespace {

constexpr int kHD = 128;
constexpr int kChunk = 64;
constexpr int kMaxWarps = 12;  // one 21-token tree at GQA 8; 384 threads -> 170 registers/thread
constexpr int kRowBytes = kHD * 2;                       // 256
constexpr int kTileBytes = kChunk * kRowBytes;           // 16 KB
constexpr int kQBytes = kMaxWarps * 16 * kRowBytes;      // 64 KB
constexpr int kMaxPasses = 256;
constexpr int kSmem = kQBytes + 4 * kTileBytes + 4096;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ int swz(int row, int chunk) { return row * kRowBytes + ((chunk ^ (row & 7)) << 4); }

__device__ __forceinline__ void cp16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

struct Plan {
    int ngroups, nwarps, npasses;
    int g_chain[kMaxWarps], g_maxpos[kMaxWarps];
    int w_group[kMaxWarps], w_r0[kMaxWarps], w_nr[kMaxWarps], w_maxpos[kMaxWarps];
    short p_chunk[kMaxPasses], p_group[kMaxPasses];  // group -1: shared pass (all warps)
};

__global__ void __launch_bounds__(kMaxWarps * 32, 1) attn_kernel(const bf16 *q, const RowDesc *rows,
                                                                 const AttnItem *items, KvCache kv, int layer, int H,
                                                                 int KV, float scale_log2, bf16 *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t *sQ = sm;
    uint8_t *sKV = sm + kQBytes;  // 2 buffers x (K, V)
    Plan &pl = *reinterpret_cast<Plan *>(sm + kQBytes + 4 * kTileBytes);
    __shared__ int rowpos[kMaxWarps * 16];

    pdl_trigger();
    pdl_wait();
    const AttnItem it = items[blockIdx.x];
    const int kvh = blockIdx.y;
    const int G = H / KV;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- plan: groups of tokens sharing a key mapping, warps, pass list --------------------
    if (tid == 0) {
        int ng = 0, nw = 0;
        int k = 0;
        while (k < it.nrows) {
            int ch = rows[it.row0 + k].chain;
            int k1 = k + 1;
            if (it.chain == -2) {  // tree item: consecutive tokens of one chain (root joins chain 0)
                if (ch < 0 && k1 < it.nrows && rows[it.row0 + k1].chain == 0) ch = 0;
                while (k1 < it.nrows && rows[it.row0 + k1].chain == ch) ++k1;
            } else {
                ch = it.chain;
                k1 = it.nrows;
            }
            int gmax = 0;
            for (int j = k; j < k1; ++j) gmax = max(gmax, rows[it.row0 + j].pos);
            pl.g_chain[ng] = ch;
            pl.g_maxpos[ng] = gmax;
            for (int r = k * G; r < k1 * G; r += 16) {
                pl.w_group[nw] = ng;
                pl.w_r0[nw] = r;
                pl.w_nr[nw] = min(16, k1 * G - r);
                int wm = 0;
                for (int rr = r; rr < r + pl.w_nr[nw]; ++rr) wm = max(wm, rows[it.row0 + rr / G].pos);
                pl.w_maxpos[nw] = wm;
                ++nw;
            }
            ++ng;
            k = k1;
        }
        pl.ngroups = ng;
        pl.nwarps = nw;
        int np = 0;
        const int cmax = it.maxpos / kChunk;
        for (int c = 0; c <= cmax; ++c) {
            const bool tail = it.chain != -1 && c * kChunk + kChunk - 1 >= it.ltree;
            if (!tail) {
                pl.p_chunk[np] = c;
                pl.p_group[np++] = -1;
            } else {
                for (int g = 0; g < ng; ++g)
                    if (pl.g_maxpos[g] >= c * kChunk) {
                        pl.p_chunk[np] = c;
                        pl.p_group[np++] = g;
                    }
            }
        }
        pl.npasses = np;
    }
    __syncthreads();

    // ---- Q rows of this warp -> smem (warp-private 16 x 128) --------------------------------
    const bool has_rows = warp < pl.nwarps;
    const int my_group = has_rows ? pl.w_group[warp] : -1;
    const int my_r0 = has_rows ? pl.w_r0[warp] : 0, my_nr = has_rows ? pl.w_nr[warp] : 0;
    uint8_t *qw = sQ + warp * 16 * kRowBytes;
    if (has_rows) {
        for (int idx = lane; idx < 16 * 16; idx += 32) {
            const int r = idx >> 4, c = idx & 15;
            uint8_t *dst = qw + swz(r, c);
            if (r < my_nr) {
                const int rr = my_r0 + r;
                const int tok = it.row0 + rr / G, head = kvh * G + rr % G;
                cp16(dst, q + ((size_t)tok * H + head) * kHD + c * 8);
            } else {
                *reinterpret_cast<int4 *>(dst) = make_int4(0, 0, 0, 0);
            }
        }
        if (lane < 16) rowpos[warp * 16 + lane] = lane < my_nr ? rows[it.row0 + (my_r0 + lane) / G].pos : -1;
    }

    auto load_pass = [&](int pi, int buf) {
        const int c = pl.p_chunk[pi], g = pl.p_group[pi];
        const int ch = g < 0 ? -1 : pl.g_chain[g];
        const int lim = g < 0 ? it.maxpos : pl.g_maxpos[g];
        uint8_t *k = sKV + buf * 2 * kTileBytes, *v = k + kTileBytes;
        for (int idx = tid; idx < kChunk * 16; idx += blockDim.x) {
            const int kk = idx >> 4, cc = idx & 15;
            const int p = c * kChunk + kk;
            if (p <= lim) {
                const int phys = (ch < 0 || p < it.ltree) ? p : it.tbase + ch * it.nstride + (p - it.ltree);
                const size_t o = kv.off(layer, it.seq, kvh, phys) + cc * 8;
                cp16(k + swz(kk, cc), kv.k + o);
                cp16(v + swz(kk, cc), kv.v + o);
            } else {
                *reinterpret_cast<int4 *>(k + swz(kk, cc)) = make_int4(0, 0, 0, 0);
                *reinterpret_cast<int4 *>(v + swz(kk, cc)) = make_int4(0, 0, 0, 0);
            }
        }
    };

    load_pass(0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");

    uint32_t qa[8][4];
    float o[16][4];
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    int pos0 = -1, pos1 = -1;
    const int wmax = has_rows ? pl.w_maxpos[warp] : -1;

    for (int pi = 0; pi < pl.npasses; ++pi) {
        if (pi + 1 < pl.npasses) {
            load_pass(pi + 1, (pi + 1) & 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        if (pi == 0 && has_rows) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int r = lane & 15, ch = 2 * kk + (lane >> 4);
                ldsm_x4(smem_u32(qw + swz(r, ch)), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
            }
            pos0 = rowpos[warp * 16 + (lane >> 2)];
            pos1 = rowpos[warp * 16 + (lane >> 2) + 8];
        }
        const int c = pl.p_chunk[pi], g = pl.p_group[pi];
        if (has_rows && (g < 0 || g == my_group) && wmax >= c * kChunk) {
            const uint8_t *k = sKV + (pi & 1) * 2 * kTileBytes, *v = k + kTileBytes;
            float s[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int key = 16 * jp + (lane & 7) + ((lane >> 4) << 3), ch = 2 * kk + ((lane >> 3) & 1);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(smem_u32(k + swz(key, ch)), b0, b1, b2, b3);
                    mma16816(s[2 * jp], qa[kk], b0, b1);
                    mma16816(s[2 * jp + 1], qa[kk], b2, b3);
                }
            }
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const int p = c * kChunk + nt * 8 + 2 * (lane & 3);
                s[nt][0] = p <= pos0 ? s[nt][0] * scale_log2 : -INFINITY;
                s[nt][1] = p + 1 <= pos0 ? s[nt][1] * scale_log2 : -INFINITY;
                s[nt][2] = p <= pos1 ? s[nt][2] * scale_log2 : -INFINITY;
                s[nt][3] = p + 1 <= pos1 ? s[nt][3] * scale_log2 : -INFINITY;
                mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
                mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
            }
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
            const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
            const float base0 = n0 == -INFINITY ? 0.f : n0, base1 = n1 == -INFINITY ? 0.f : n1;
            const float a0 = exp2f(m0 - base0), a1 = exp2f(m1 - base1);
            m0 = n0;
            m1 = n1;
            l0 *= a0;
            l1 *= a1;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                o[i][0] *= a0;
                o[i][1] *= a0;
                o[i][2] *= a1;
                o[i][3] *= a1;
            }
            uint32_t pa[4][4];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const float p0 = exp2f(s[nt][0] - base0), p1 = exp2f(s[nt][1] - base0);
                const float p2 = exp2f(s[nt][2] - base1), p3 = exp2f(s[nt][3] - base1);
                l0 += p0 + p1;
                l1 += p2 + p3;
                pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
                pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
                for (int dp = 0; dp < 8; ++dp) {
                    const int key = 16 * kk + (lane & 7) + (((lane >> 3) & 1) << 3), ch = 2 * dp + (lane >> 4);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(smem_u32(v + swz(key, ch)), b0, b1, b2, b3);
                    mma16816(o[2 * dp], pa[kk], b0, b1);
                    mma16816(o[2 * dp + 1], pa[kk], b2, b3);
                }
            }
        }
        __syncthreads();
    }
    if (!has_rows) return;
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int r = (lane >> 2) + half * 8;
        if (r >= my_nr) continue;
        const int rr = my_r0 + r;
        const int tok = it.row0 + rr / G, head = kvh * G + rr % G;
        bf16 *dst = out + ((size_t)tok * H + head) * kHD + 2 * (lane & 3);
        const float inv = half ? inv1 : inv0;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            const float x = o[nt][half * 2 + 0] * inv, y = o[nt][half * 2 + 1] * inv;
            *reinterpret_cast<__nv_bfloat162 *>(dst + nt * 8) = __floats2bfloat162_rn(x, y);
        }
    }
}

}  // namespace

int attn_max_tokens(int G) { return kMaxWarps * 16 / G; }
int attn_max_warps() { return kMaxWarps; }

void k_attention(const bf16 *q, const RowDesc *rows, const AttnItem *items, int n_items, const KvCache &kv, int layer,
                 const TfShape &s, bf16 *out, cudaStream_t st, double flops, double bytes) {
    if (n_items <= 0) return;
    ProfScope prof("attn", flops, bytes, st);
    if (s.hd != kHD) throw std::invalid_argument("attention: head_dim must be 128");
    static const bool attr = [] {  // thread-safe one-time init (engine + learner threads)
        static_assert(sizeof(Plan) <= 4096, "plan");
        RS_CUDA(cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        return true;
    }();
    (void)attr;
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(s.hd));
    launch_pdl(attn_kernel, dim3(n_items, s.KV), kMaxWarps * 32, kSmem, st, q, rows, items, kv, layer, s.H, s.KV,
               scale_log2, out);
    RS_LAUNCHED();
}

}  // namespace rs

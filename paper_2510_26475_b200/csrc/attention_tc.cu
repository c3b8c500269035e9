// attention_tc.cu -- tree-causal GQA attention of the TARGET (and the drafter) on 5th-gen tensor
// cores (sm_100a).
//
// A work item = up to two 128-row M-tiles of one (sequence, kv head): row = token * G + head
// (at most 128 / G tokens per tile; an item of more splits its tokens evenly between the two
// tiles, so the two CTAs carry the same softmax load -- attn_tile_tokens). One CTA per (item, M-tile, kv head). Keys are visited in
// LOGICAL order in passes of kAttnChunk = 32 positions; a pass = (key block, key group). Blocks
// wholly below the tree start are shared by every token of the item; the blocks that reach into
// the tree are replayed once per group of tokens sharing a key mapping (the tokens of one draft
// chain, the root riding with chain 0), rows of other groups masked -- the tree-causal mask of
// SURVEY.md §8 A3. Every row therefore sees exactly the key sequence (block boundaries, column
// order, accumulation order) it would see decoded alone or prefilled, so its output is bitwise
// independent of the tree it sits in (tests/test_transformer_gpu.py).
//
// Why this shape (measured on B200, DESIGN.md §4 "target attention"):
//   * Q lives in TENSOR MEMORY and S = Q K^T is a TS-form MMA: the tensor core reads only the
//     K block from shared memory. With Q in shared memory (SS form) every score MMA re-read the
//     128 x 128 Q tile; the MMAs ran at the ~68 B/clk operand rate, ~90 cycles per 128x64x16
//     MMA instead of 32, and the issuing thread -- not HBM -- set the pass rate.
//   * TMEM per CTA = O (128 columns) + Q (64) + two S buffers of 32 keys (2 x 32) = 256, so two
//     CTAs share an SM (shared memory ~100 KB each): one CTA's softmax overlaps the other's MMAs
//     and K/V stream, every SM holds work at the benchmarked grids, and each SM keeps up to
//     2 x 96 KB of K/V in flight.
//   * S is double-buffered: the score MMAs of pass j + 1 run while the softmax of pass j does.
//
// Warp roles (256 threads):
//   warp 0      plan -> shared memory; then one lane issues O += P(j) V(j) (TS: P read from TMEM
//               where it overwrote S(j), V an MN-major smem operand, 2 x 128x128x16)
//   warp 1      one lane issues S(j) = Q K(j)^T (TS, 8 x 128x32x16) into S buffer j & 1
//   warp 2 / 3  K / V producers: one lane issues the two TMA boxes (32 rows x 64 dims, 128B
//               swizzle) of a block whose keys are physically contiguous; for tree blocks whose
//               keys are remapped to a chain's slots the warp copies rows with cp.async in the
//               same swizzled layout. Warp 2 also owns the TMEM allocation.
//   warps 4-7   one thread per row (its TMEM lane): Q row -> TMEM; per pass the row's 32 scores
//               (tcgen05.ld), online softmax in the exp2 domain, P as bf16 over the consumed S
//               columns (tcgen05.st), O rescale in TMEM when the running max moves (after the
//               previous P.V completed); finally O / l as bf16.
// TMEM (256 columns): O [0, 128), Q [128, 192), S(b) at 192 + 32 b.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "gemm.h"
#include "model.h"
#include "prof.h"
#include "launch.cuh"
#include "tc.cuh"

namespace rs {

namespace {

constexpr int kHD = 128;
constexpr int kCk = kAttnChunk;              // keys per pass (32)
constexpr int kNK = 6, kNV = 6;              // K / V ring depths
constexpr int kBox = kCk * 128;              // kCk rows x 64 bf16 dims: one 128B-swizzled TMA box
constexpr int kKVBytes = 2 * kBox;           // kCk keys x 128 dims (K or V of one pass)
constexpr int kMaxPasses = kAttnMaxPasses;
constexpr int kMaxGroups = kAttnMaxGroups;
constexpr int kMaxTok = 128;                 // tokens of one M-tile (G >= 1)
constexpr int kThreads = 256;
constexpr uint32_t kColO = 0, kColQ = 128, kColS = 192, kTmemCols = 256;
static_assert(kCk == 32, "TMEM columns and the P packing assume 32-key passes");
// kind::f16, fp32 accumulate, bf16 A/B, K-major A and B; N at bit 17 (>> 3), M at bit 24 (>> 4)
constexpr uint32_t kIdescBase = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 4) << 24);
constexpr uint32_t kIdescS = kIdescBase | ((uint32_t)(kCk >> 3) << 17);            // 128 x 32 x 16
constexpr uint32_t kIdescPV = kIdescBase | ((128u >> 3) << 17) | (1u << 16);       // 128 x 128 x 16, V MN-major

using Pass = AttnPass;

struct Plan {
    int npasses, ngroups, ntok;
    int g_chain[kMaxGroups], g_maxpos[kMaxGroups];
    short tok_grp[kMaxTok];
    int tok_pos[kMaxTok];
    Pass pass[kMaxPasses];
};

constexpr int kBarBytes = 256;
constexpr int kSmem = 1024 + (kNK + kNV) * kKVBytes + kBarBytes + (int)sizeof(Plan);
// two CTAs per SM: 228 KB per SM, 1 KB of it reserved per CTA
static_assert(2 * (kSmem + 1024) <= 233472, "attention: two CTAs per SM must fit in shared memory");
static_assert((2 * (kNK + kNV) + 2 + 2 + 2 + 1) * 8 + 4 <= kBarBytes, "barrier area");

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
// Packed fp32 pairs (FFMA2 / FADD2 on sm_100): half the issue slots of scalar FFMA / FADD.
__device__ __forceinline__ void fma2(float &d0, float &d1, float a0, float a1, float b0, float b1, float c0, float c1) {
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void add2(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// byte offset of (row r, 16-byte chunk c of 16) in a tile of two 128B-swizzled 64-dim halves
__device__ __forceinline__ uint32_t swz_off(int r, int c) {
    return (uint32_t)((c >> 3) * kBox + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

__global__ void __launch_bounds__(kThreads, 2)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, const bf16 *q,
                   const RowDesc *rows, const AttnItem *items, AttnPlan plan, KvCache kv, int layer, int H, int KV,
                   float scale_log2, bf16 *out, long long *trace, int skip) {
    const int tile = blockIdx.x & 1;
    const AttnItem it = items[blockIdx.x >> 1];  // host-uploaded plan: independent of the previous kernel
    const int G = H / KV;
    const int T = attn_tile_tokens(it.nrows, 128 / G);  // tokens of the first M-tile (tf_pair.cpp plan_tc)
    pdl_trigger();
    if (tile * T >= it.nrows) return;  // the item has no second M-tile (uniform per CTA)
    // trace (diagnostics, CTA (0, 0) only): [0] start; per pass j at 1 + 12 j: K issue, V issue,
    // K landed, V landed, P ready (MMA), -, softmax start / end, -, -, S issue start / end
    const bool tr = trace && blockIdx.x == 0 && blockIdx.y == 0;
    if (tr && threadIdx.x == 0) trace[0] = clock64();
    // per-CTA timeline (diagnostics): [start ns, prologue done ns, end ns, smid] after the pass trace
    long long *ctat = trace ? trace + 1 + 12 * kMaxPasses + 4 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
    if (ctat && threadIdx.x == 0) {
        ctat[0] = (long long)globaltimer_ns();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        ctat[3] = smid;
    }
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // aligned by pointer arithmetic on the shared array (not through an integer), so the compiler
    // keeps the shared address space and emits STS / LDS instead of generic ST / LD
    uint8_t *smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint8_t *sK = smem;
    uint8_t *sV = sK + kNK * kKVBytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sV + kNV * kKVBytes);
    uint64_t *fullK = bars, *emptyK = bars + kNK, *fullV = bars + 2 * kNK, *emptyV = fullV + kNV;
    uint64_t *s_full = emptyV + kNV;  // [buffer]
    uint64_t *p_full = s_full + 2;    // [buffer]
    uint64_t *pv_done = p_full + 2;   // [buffer] P.V(j) completed
    uint64_t *o_done = pv_done + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_done + 1);
    Plan &pl = *reinterpret_cast<Plan *>(reinterpret_cast<uint8_t *>(bars) + kBarBytes);

    const int kvh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tok0 = tile * T, ntok = min(T, it.nrows - tok0);  // this CTA's tokens

    // ---- plan (host-built, tf_pair.cpp Batch::plan_tc) -> smem, by warp 0: this tile's passes
    if (warp == 0) {
        int n = 0;
        for (int j0 = 0; j0 < it.npass; j0 += 32) {
            const int j = j0 + lane;
            const Pass ps = j < it.npass ? plan.passes[it.pass0 + j] : Pass{};
            const bool mine = j < it.npass && ((ps.tiles >> tile) & 1);
            const unsigned m = __ballot_sync(0xffffffffu, mine);
            if (mine) pl.pass[n + __popc(m & ((1u << lane) - 1))] = ps;
            n += __popc(m);
        }
        for (int g = lane; g < it.ngrp; g += 32) {
            const AttnGroup gr = plan.groups[it.grp0 + g];
            pl.g_chain[g] = gr.chain;
            pl.g_maxpos[g] = gr.maxpos;
        }
        for (int k = lane; k < ntok; k += 32) {
            pl.tok_pos[k] = rows[it.row0 + tok0 + k].pos;
            pl.tok_grp[k] = plan.tok_grp[it.row0 + tok0 + k];
        }
        if (lane == 0) {
            pl.npasses = n;
            pl.ngroups = it.ngrp;
            pl.ntok = ntok;
        }
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < kNK; ++s) {
            mbar_init(&fullK[s], 1);
            mbar_init(&emptyK[s], 1);
        }
        for (int s = 0; s < kNV; ++s) {
            mbar_init(&fullV[s], 1);
            mbar_init(&emptyV[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&p_full[b], 4);  // the four softmax warps
        }
        for (int b = 0; b < 2; ++b) mbar_init(&pv_done[b], 1);
        mbar_init(o_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int np = pl.npasses;
    if (ctat && threadIdx.x == 0) ctat[1] = (long long)globaltimer_ns();
    const size_t kvrow0 = (((size_t)layer * kv.B + it.seq) * kv.KV + kvh) * kv.max_ctx;

    if (warp == 0) {
        if (lane == 0) {
            // ---- P.V issuer: O += P(j) V(j) once the softmax wrote P(j); commits free the S
            // buffer for S(j + 2) (pv_done[j & 1]) and the V stage
            for (int j = 0; j < np; ++j) {
                const int s = j % kNV;
                mbar_wait(&fullV[s], (j / kNV) & 1);
                const int b = j & 1;
                mbar_wait(&p_full[b], ((j >> 1) + b) & 1);
                if (tr) trace[5 + 12 * j] = clock64();
                tc_fence_after();
                const uint8_t *vt = sV + s * kKVBytes;
                if (!(skip & 4)) {
#pragma unroll
                    for (int kk = 0; kk < kCk / 16; ++kk)
                        tc_mma_ts(tmem + kColO, tmem + kColS + b * kCk + kk * 8, sw128_desc_mn(vt + kk * 2048, kBox),
                                  kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
                }
                tc_commit(&pv_done[b]);
                tc_commit(&emptyV[s]);
            }
            tc_commit(o_done);
        } else if (tr && lane < 3) {
            // diagnostics: lane 1 / 2 record when each K / V block lands
            const int depth = lane == 1 ? kNK : kNV;
            uint64_t *full = lane == 1 ? fullK : fullV;
            for (int j = 0; j < np; ++j) {
                mbar_wait(&full[j % depth], (j / depth) & 1);
                trace[2 + lane + 12 * j] = clock64();
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ---- producers: warp 2 streams K, warp 3 streams V, each through its own ring in pass
        // order; contiguous blocks by TMA from one lane, tree blocks whose keys are remapped to a
        // chain's slots by cp.async from the warp's 32 lanes in the swizzled layout.
        pdl_wait();  // the K/V cache rows come from the previous kernel (RoPE / KV store)
        const bool isK = warp == 2;
        const int depth = isK ? kNK : kNV;
        uint8_t *ring = isK ? sK : sV;
        uint64_t *full = isK ? fullK : fullV, *empty = isK ? emptyK : emptyV;
        const CUtensorMap *tm = isK ? &tmK : &tmV;
        const bf16 *src = isK ? kv.k : kv.v;
        const uint64_t pol = l2_evict_first_policy();  // the K/V stream is read once
        for (int j = 0, s = 0, ph = 1; j < np; ++j) {
            const Pass ps = pl.pass[j];
            uint8_t *dst = ring + s * kKVBytes;
            mbar_wait(&empty[s], ph);
            if (!ps.manual) {
                if (lane == 0) {
                    if (tr) trace[1 + 12 * j + (isK ? 0 : 1)] = clock64();
                    const int y = (int)(kvrow0 + ps.chunk * kCk);
                    mbar_arrive_expect_tx(&full[s], kKVBytes);
                    tma_load_2d_hint(dst, tm, &full[s], 0, y, pol);
                    tma_load_2d_hint(dst + kBox, tm, &full[s], 64, y, pol);
                }
            } else {
                // keys beyond the group's last position are masked to p = 0 by the softmax; their
                // rows only need finite values, so they are copied from the contiguous position
                const int ch = pl.g_chain[ps.grp], lim = pl.g_maxpos[ps.grp];
                for (int idx = lane; idx < kCk * 16; idx += 32) {
                    const int rr = idx >> 4, c = idx & 15;
                    const int p = ps.chunk * kCk + rr;
                    const int phys = p > lim ? min(p, kv.max_ctx - 1)
                                             : p < it.ltree ? p : it.tbase + ch * it.nstride + (p - it.ltree);
                    cp16(smem_u32(dst + swz_off(rr, c)), src + (kvrow0 + phys) * kHD + c * 8);
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
            if (++s == depth) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 1) {
        // ---- score issuer: S(j) = Q K(j)^T into S buffer j & 1 once P.V(j - 2) has read it ---------
        // (two issuing threads: one thread retires a tcgen05.mma only every ~55 cycles whatever N
        // is -- tools/mma_issue_bench.cu -- so the 8 score MMAs and the 2 P.V MMAs of a pass would
        // serialise on one thread; a third issuer for the odd passes measured no further gain)
        if (lane == 0) {
            // Q is written to TMEM by the softmax warps after their dependency wait; their first
            // arrival on p_full[1] (its phase 0) says "Q ready", so pass j's P completes phase
            // (j >> 1) of p_full[0] or phase (j >> 1) + 1 of p_full[1]
            mbar_wait(&p_full[1], 0);
            tc_fence_after();
            for (int j = 0; j < np; ++j) {
                const int s = j % kNK;
                if (j >= 2) mbar_wait(&pv_done[j & 1], ((j >> 1) - 1) & 1);  // P.V(j - 2) read the buffer
                mbar_wait(&fullK[s], (j / kNK) & 1);
                if (tr) trace[11 + 12 * j] = clock64();
                tc_fence_after();
                const uint8_t *kt = sK + s * kKVBytes;
                const uint32_t d_s = tmem + kColS + (j & 1) * kCk;
                if (!(skip & 2)) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        tc_mma_ts(d_s, tmem + kColQ + kk * 8, sw128_desc(kt + (kk >> 2) * kBox) + 2 * (kk & 3), kIdescS,
                                  kk > 0 ? 1u : 0u);
                }
                tc_commit(&s_full[j & 1]);
                tc_commit(&emptyK[s]);
                if (tr) trace[12 + 12 * j] = clock64();
            }
        }
    } else {
        // ---- softmax warps: one thread per row (row r = token k, head kvh * G + r % G) -------------
        const int r = (warp & 3) * 32 + lane;
        const int k = r / G;
        const bool valid = r < T * G && k < ntok;
        const bool warp_valid = __any_sync(0xffffffffu, valid);
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        pdl_wait();  // Q comes from the previous kernel (QKV + RoPE)
        {
            // Q row -> TMEM columns [128, 192) as bf16 pairs (zero rows beyond the tile's tokens)
            const bf16 *src = q + ((size_t)(it.row0 + tok0 + (valid ? k : 0)) * H + kvh * G + r % G) * kHD;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t w[32];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int4 v = valid ? *reinterpret_cast<const int4 *>(src + h * 64 + c * 8) : make_int4(0, 0, 0, 0);
                    w[4 * c] = (uint32_t)v.x;
                    w[4 * c + 1] = (uint32_t)v.y;
                    w[4 * c + 2] = (uint32_t)v.z;
                    w[4 * c + 3] = (uint32_t)v.w;
                }
                tmem_st32(tmem + lane_off + kColQ + h * 32, w);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[1]);  // "Q ready"
        }
        // Per pass: one TMEM read of the row's 32 scores, the row max, p = 2^(s*scale - m) written
        // as bf16 over the consumed S columns [0, 16) of the buffer. The running max m only moves
        // when the block max exceeds it by more than 2^8 (so p <= 256): O in TMEM is then rescaled
        // once the previous P.V has completed. Row sums are kept as 8 interleaved partials. Every
        // choice depends only on the row's own scores, so the arithmetic is identical whatever
        // item the row sits in.
        const int pos = valid ? pl.tok_pos[k] : -1;
        const int grp = valid ? pl.tok_grp[k] : -2;
        const uint32_t tO = tmem + lane_off + kColO;
        const bool trs = tr && warp == 4 && lane == 0;
        float m = -INFINITY;
        float lp[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) lp[i] = 0.f;
        for (int j = 0; j < np; ++j) {
            const Pass ps = pl.pass[j];
            const int b = j & 1;
            const uint32_t tS = tmem + lane_off + kColS + b * kCk;
            mbar_wait(&s_full[b], (j >> 1) & 1);
            if (trs) trace[7 + 12 * j] = clock64();
            tc_fence_after();
            const int c0 = ps.chunk * kCk;
            const bool mine = valid && (ps.grp < 0 || ps.grp == grp);
            const int lim = mine ? pos - c0 : -1;  // own columns x <= lim are visible
            if (warp_valid && !(skip & 1)) {
                uint32_t v[32];
                tmem_ld32(tS, v);
                float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
                if (lim >= kCk - 1) {
#pragma unroll
                    for (int x = 0; x < 32; x += 4) {
                        mx0 = fmaxf(mx0, __uint_as_float(v[x]));
                        mx1 = fmaxf(mx1, __uint_as_float(v[x + 1]));
                        mx2 = fmaxf(mx2, __uint_as_float(v[x + 2]));
                        mx3 = fmaxf(mx3, __uint_as_float(v[x + 3]));
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 32; ++x) {
                        if (x > lim) v[x] = __float_as_uint(-INFINITY);  // masked: exp2 -> +0
                        mx0 = fmaxf(mx0, __uint_as_float(v[x]));
                    }
                }
                float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
                mx = mx == -INFINITY ? mx : mx * scale_log2;  // scale > 0: max commutes with it
                bool resc = false;
                float alpha = 1.f;
                if (mx > m) {
                    if (m == -INFINITY) {
                        m = mx;  // first visible keys of the row: O row and l are still 0
                    } else if (mx > m + 8.f) {
                        alpha = ex2(m - mx);
                        m = mx;
                        resc = true;
#pragma unroll
                        for (int i = 0; i < 8; ++i) lp[i] *= alpha;
                    }
                }
                const float nb = m == -INFINITY ? 0.f : -m;
                uint32_t pk[16];
#pragma unroll
                for (int x = 0; x < 32; x += 2) {
                    // masked columns hold -inf: fma(-inf, scale, nb) = -inf and ex2(-inf) = +0
                    float a0, a1, p0, p1;
                    fma2(a0, a1, __uint_as_float(v[x]), __uint_as_float(v[x + 1]), scale_log2, scale_log2, nb, nb);
                    p0 = ex2(a0);
                    p1 = ex2(a1);
                    add2(lp[x & 7], lp[(x + 1) & 7], lp[x & 7], lp[(x + 1) & 7], p0, p1);
                    pk[x >> 1] = pack_bf16(p0, p1);
                }
                tmem_st16(tS, pk);  // P (bf16) over S columns [0, 16) of this buffer, already read
                if (j > 0 && __any_sync(0xffffffffu, resc)) {
                    // O may still be accumulating the previous pass: wait for that P.V (the only
                    // one that can be in flight -- the next one needs this pass's P)
                    mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int cc = 0; cc < 4; ++cc) {
                        uint32_t o[32];
                        tmem_ld32(tO + cc * 32, o);
#pragma unroll
                        for (int x = 0; x < 32; ++x) o[x] = __float_as_uint(__uint_as_float(o[x]) * alpha);
                        tmem_st32(tO + cc * 32, o);
                    }
                }
                tmem_st_wait();
            }
            if (trs) trace[8 + 12 * j] = clock64();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[b]);
        }
        if (np > 0 && warp_valid) {
            const float l = ((lp[0] + lp[1]) + (lp[2] + lp[3])) + ((lp[4] + lp[5]) + (lp[6] + lp[7]));
            mbar_wait(o_done, 0);
            tc_fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            bf16 *dst = out + ((size_t)(it.row0 + tok0 + (valid ? k : 0)) * H + kvh * G + r % G) * kHD;
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t o[32];
                tmem_ld32(tO + cc * 32, o);
                if (valid) {
#pragma unroll
                    for (int x = 0; x < 32; x += 8) {
                        uint4 w;
                        w.x = pack_bf16(__uint_as_float(o[x]) * inv, __uint_as_float(o[x + 1]) * inv);
                        w.y = pack_bf16(__uint_as_float(o[x + 2]) * inv, __uint_as_float(o[x + 3]) * inv);
                        w.z = pack_bf16(__uint_as_float(o[x + 4]) * inv, __uint_as_float(o[x + 5]) * inv);
                        w.w = pack_bf16(__uint_as_float(o[x + 6]) * inv, __uint_as_float(o[x + 7]) * inv);
                        *reinterpret_cast<uint4 *>(dst + cc * 32 + x) = w;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (ctat && threadIdx.x == 0) ctat[2] = (long long)globaltimer_ns();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

}  // namespace

int attn_tc_max_tokens(int G) { return 2 * (128 / G); }

long long *trace_buf() {
    static long long *p = nullptr;
    if (!p) {
        RS_CUDA(cudaMalloc(&p, 8 * (1 + 12 * kMaxPasses + 4 * 16384)));
        RS_CUDA(cudaMemset(p, 0, 8 * (1 + 12 * kMaxPasses + 4 * 16384)));
    }
    return p;
}

void k_attention_tc(const bf16 *q, const RowDesc *rows, const AttnItem *items, const AttnPlan &plan, int n_items,
                    const KvCache &kv, int layer, const TfShape &s, bf16 *out, cudaStream_t st, double flops,
                    double bytes) {
    if (n_items <= 0) return;
    ProfScope prof("attn", flops, bytes, st);
    if (s.hd != kHD) throw std::invalid_argument("attention: head_dim must be 128");
    if (s.H / s.KV > 128) throw std::invalid_argument("attention: GQA group too large");
    static const bool attr = [] {  // thread-safe one-time init (engine + learner threads)
        RS_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        return true;
    }();
    (void)attr;
    const int total_rows = kv.layers * kv.B * kv.KV * kv.max_ctx;
    const CUtensorMap tk = make_tma_map_bf16(kv.k, total_rows, kHD, kHD, kCk);
    const CUtensorMap tv = make_tma_map_bf16(kv.v, total_rows, kHD, kHD, kCk);
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(s.hd));
    launch_pdl(attn_tc_kernel, dim3(2 * n_items, s.KV), kThreads, kSmem, st, tk, tv, q, rows, items, plan, kv, layer,
               s.H, s.KV, scale_log2, out, tuning().attn_trace ? trace_buf() : (long long *)nullptr,
               tuning().attn_skip);
    if (tuning().attn_trace) {
        RS_CUDA(cudaStreamSynchronize(st));
        const int nct = 2 * n_items * s.KV;
        static std::vector<long long> host;
        host.assign(1 + 12 * kMaxPasses + 4 * (size_t)nct, 0);
        RS_CUDA(cudaMemcpy(host.data(), trace_buf(), host.size() * 8, cudaMemcpyDeviceToHost));
        RS_CUDA(cudaMemset(trace_buf(), 0, host.size() * 8));
        if (tuning().attn_trace == layer + 1 && n_items >= 32) {
            fprintf(stderr, "attn trace layer %d items %d (cycles from CTA start):\n", layer, n_items);
            for (int j = 0; j < 64; ++j) {
                const long long *h = host.data() + 1 + 12 * j;
                auto t = [&](int i) { return h[i] ? h[i] - host[0] : -1; };
                fprintf(stderr, "  pass %2d issueK %6lld issueV %6lld | landK %6lld landV %6lld P %6lld | sm %6lld..%6lld | "
                        "S %6lld..%6lld\n", j, t(0), t(1), t(2), t(3), t(4), t(6), t(7), t(10), t(11));
            }
            // per-CTA timeline (ns from the first CTA start): start, prologue, duration; CTAs that
            // exited early (no second M-tile) have no record
            const long long *c = host.data() + 1 + 12 * kMaxPasses;
            long long t0 = -1, tend = 0;
            std::vector<long long> st0, pro, dur;
            std::vector<int> per_sm(1024, 0);
            for (int i = 0; i < nct; ++i)
                if (c[4 * i]) t0 = t0 < 0 ? c[4 * i] : std::min(t0, c[4 * i]);
            for (int i = 0; i < nct; ++i) {
                if (!c[4 * i]) continue;
                st0.push_back(c[4 * i] - t0);
                pro.push_back(c[4 * i + 1] - c[4 * i]);
                dur.push_back(c[4 * i + 2] - c[4 * i]);
                tend = std::max(tend, c[4 * i + 2] - t0);
                per_sm[c[4 * i + 3] & 1023]++;
            }
            auto pct = [](std::vector<long long> v, double q) {
                std::sort(v.begin(), v.end());
                return v.empty() ? 0LL : v[(size_t)(q * (v.size() - 1))];
            };
            int sm2 = 0, sm1 = 0;
            for (int x : per_sm) sm2 += x >= 2, sm1 += x == 1;
            fprintf(stderr, "  CTAs %zu (of %d), SMs with 1 / >=2: %d / %d; span %lld ns; start p50/p90/max %lld/%lld/%lld; "
                    "prologue p50/max %lld/%lld; duration min/p50/p90/max %lld/%lld/%lld/%lld ns\n",
                    dur.size(), nct, sm1, sm2, tend, pct(st0, .5), pct(st0, .9), pct(st0, 1), pct(pro, .5), pct(pro, 1),
                    pct(dur, 0), pct(dur, .5), pct(dur, .9), pct(dur, 1));
        }
    }
    RS_LAUNCHED();
}

}  // namespace rs

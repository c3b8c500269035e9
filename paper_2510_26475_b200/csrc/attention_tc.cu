// attention_tc.cu -- tree-causal GQA attention of the TARGET on 5th-gen tensor cores (sm_100a).
//
// One CTA per work item = up to two 128-row M-tiles of one (sequence, kv head): row =
// token * G + head (T = 128 / G tokens per tile). Keys are visited in LOGICAL order in chunks
// of 128 positions; a pass = (chunk, key group). Chunks wholly below the tree start are shared
// by every token of the item (one K/V tile for both M-tiles); the chunks that reach into the
// tree are replayed once per group of tokens sharing a key mapping (the tokens of one draft
// chain, the root riding with chain 0), rows of other groups masked -- the tree-causal mask of
// SURVEY.md §8 A3. Every row therefore sees exactly the key sequence (chunk boundaries, column
// order, accumulation order) it would see decoded alone or prefilled, so its output is bitwise
// independent of the tree it sits in (tests/test_transformer_gpu.py).
//
// Warp roles (384 threads):
//   warps 2-3   producers of a 2-stage shared-memory K/V ring: a chunk is 2 x 2 TMA boxes of
//               128 keys x 64 dims (128B swizzle) when its keys are physically contiguous, or
//               cp.async rows (context + the chain's own slots) in the same swizzled layout for
//               tree passes; warp 2 also owns the TMEM allocation; warp 0 idles;
//   warp 1      one elected lane issues tcgen05.mma: S_i = Q_i K^T (SS, 128x128x128) into
//               TMEM and O_i += P_i V (TS: P read from TMEM where it overwrote S_i, V as an
//               MN-major smem operand), ping-ponging the two M-tiles so one tile's softmax
//               overlaps the other tile's MMAs;
//   warps 4-7 / 8-11  softmax of M-tile 0 / 1: one thread per row (its TMEM lane) reads the
//               row's 128 scores of S (tcgen05.ld), online softmax in the exp2 domain, writes P as
//               bf16 back into TMEM (tcgen05.st), rescales O in TMEM when the running max moves,
//               and finally writes O / l as bf16. One thread owns the whole row, so the row max
//               needs no cross-warp exchange (measured: the two-threads-per-row variant spent
//               ~340 of its ~1.9K cycles per pass in that exchange).
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512) columns.
#include <cstdio>
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
constexpr int kCk = kAttnChunk;                 // keys per chunk
constexpr int kStages = 2;
constexpr int kHalfBytes = 128 * 128;          // 128 rows x 64 bf16 (one 128B-swizzled box)
constexpr int kTileBytes = 2 * kHalfBytes;     // 128 rows x 128 dims
constexpr int kStageBytes = 2 * kTileBytes;    // K + V
constexpr int kQBytes = 2 * kTileBytes;        // two M-tiles
constexpr int kMaxPasses = kAttnMaxPasses;
constexpr int kMaxGroups = kAttnMaxGroups;
constexpr int kMaxTok = 256;
constexpr int kThreads = 384;  // 4 control warps + 2 x 4 softmax warps
constexpr uint32_t kIdescS = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescPV = kIdescS | (1u << 16);  // B (= V) is MN-major

using Pass = AttnPass;

struct Plan {
    int npasses, ngroups, T, ntok;
    int g_chain[kMaxGroups], g_maxpos[kMaxGroups];
    short tok_grp[kMaxTok];
    int tok_pos[kMaxTok];
    Pass pass[kMaxPasses];
};

constexpr int kBarBytes = 256;
constexpr int kSmem = 1024 + kQBytes + kStages * kStageBytes + kBarBytes + (int)sizeof(Plan);

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
// byte offset of (row r, 16-byte chunk c of 16) in a 128-row x 128-dim tile of two swizzled halves
__device__ __forceinline__ uint32_t swz_off(int r, int c) {
    return (uint32_t)((c >> 3) * kHalfBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, const bf16 *q,
                   const RowDesc *rows, const AttnItem *items, AttnPlan plan, KvCache kv, int layer, int H, int KV,
                   float scale_log2, bf16 *out, long long *trace) {
    // trace (diagnostics, CTA (0,0) only): [0] start, per pass j: [1+4j] fullK ok, [2+4j] p0 ok,
    // [3+4j] p1 ok (MMA thread), [4+4j] softmax tile 0 s_full ok
    const bool tr = trace && blockIdx.x == 0 && blockIdx.y == 0;
    if (tr && threadIdx.x == 0) trace[0] = clock64();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem;
    uint8_t *sKV = smem + kQBytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sKV + kStages * kStageBytes);
    // K and V halves of a stage fill and drain separately: S = Q K^T can start while V is in
    // flight, and K(j + 2) loads as soon as the S MMAs of pass j are done.
    uint64_t *fullK = bars, *fullV = bars + kStages, *emptyK = bars + 2 * kStages, *emptyV = bars + 3 * kStages;
    uint64_t *s_full = bars + 4 * kStages, *p_full = s_full + 2, *o_done = p_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_done + 1);
    Plan &pl = *reinterpret_cast<Plan *>(reinterpret_cast<uint8_t *>(bars) + kBarBytes);

    pdl_trigger();
    const AttnItem it = items[blockIdx.x];  // host-uploaded plan: independent of the previous kernel
    const int kvh = blockIdx.y;
    const int G = H / KV;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---- plan (host-built, tf_pair.cpp Batch::plan_tc) -> smem, by warp 0 --------------------
    if (warp == 0) {
        for (int j = lane; j < it.npass; j += 32) pl.pass[j] = plan.passes[it.pass0 + j];
        for (int g = lane; g < it.ngrp; g += 32) {
            const AttnGroup gr = plan.groups[it.grp0 + g];
            pl.g_chain[g] = gr.chain;
            pl.g_maxpos[g] = gr.maxpos;
        }
        for (int k = lane; k < it.nrows; k += 32) {
            pl.tok_pos[k] = rows[it.row0 + k].pos;
            pl.tok_grp[k] = plan.tok_grp[it.row0 + k];
        }
        if (lane == 0) {
            pl.npasses = it.npass;
            pl.ngroups = it.ngrp;
            pl.T = 128 / G;
            pl.ntok = it.nrows;
        }
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&fullK[s], 1);
            mbar_init(&fullV[s], 1);
            mbar_init(&emptyK[s], 1);
            mbar_init(&emptyV[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);  // the tile's four softmax warps
        }
        mbar_init(o_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    pdl_wait();  // Q and the K/V cache come from the previous kernel (RoPE / KV store)
    // ---- Q tiles -> smem (softmax warps: one row each, zero rows beyond the item) -------------
    if (warp >= 4) {
        const int T0 = 128 / G;
        const int tile = (warp - 4) >> 2, r = (warp & 3) * 32 + lane;
        const int k = tile * T0 + r / G;
        const bool valid = r < T0 * G && k < it.nrows;
        uint8_t *base = sQ + tile * kTileBytes;
        const bf16 *src = q + ((size_t)(it.row0 + k) * H + kvh * G + r % G) * kHD;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            int4 v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c)
                v[c] = valid ? *reinterpret_cast<const int4 *>(src + h * 64 + c * 8) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int c = 0; c < 8; ++c) *reinterpret_cast<int4 *>(base + swz_off(r, h * 8 + c)) = v[c];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const int T = 128 / G;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int np = pl.npasses;
    const size_t kvrow0 = (((size_t)layer * kv.B + it.seq) * kv.KV + kvh) * kv.max_ctx;

    if (warp == 2 || warp == 3) {
        // ---- producers: one ring, every pass in order (so each thread's parity waits never
        // alias); contiguous passes by TMA from one thread, tree passes whose keys are
        // remapped to a chain's slots by cp.async from all 64 threads in the swizzled layout.
        const int t = threadIdx.x - 64;  // 0..63
        for (int j = 0; j < np; ++j) {
            const Pass ps = pl.pass[j];
            const int s = j % kStages;
            const uint32_t par = ((j / kStages) & 1) ^ 1;
            uint8_t *dst = sKV + s * kStageBytes;
            if (!ps.manual) {
                const int y = (int)(kvrow0 + ps.chunk * kCk);
                mbar_wait(&emptyK[s], par);
                if (t == 0) {
                    if (tr) trace[9 + 12 * j] = clock64();
                    mbar_arrive_expect_tx(&fullK[s], kTileBytes);
                    tma_load_2d(dst, &tmK, &fullK[s], 0, y);
                    tma_load_2d(dst + kHalfBytes, &tmK, &fullK[s], 64, y);
                }
                mbar_wait(&emptyV[s], par);
                if (t == 0) {
                    if (tr) trace[10 + 12 * j] = clock64();
                    mbar_arrive_expect_tx(&fullV[s], kTileBytes);
                    tma_load_2d(dst + kTileBytes, &tmV, &fullV[s], 0, y);
                    tma_load_2d(dst + kTileBytes + kHalfBytes, &tmV, &fullV[s], 64, y);
                }
                continue;
            }
            mbar_wait(&emptyK[s], par);
            mbar_wait(&emptyV[s], par);
            const int ch = pl.g_chain[ps.grp], lim = pl.g_maxpos[ps.grp];
            for (int idx = t; idx < kCk * 16; idx += 64) {
                const int r = idx >> 4, c = idx & 15;
                const int p = ps.chunk * kCk + r;
                const uint32_t o = swz_off(r, c);
                if (p <= lim) {
                    const int phys = p < it.ltree ? p : it.tbase + ch * it.nstride + (p - it.ltree);
                    const size_t go = (kvrow0 + phys) * kHD + c * 8;
                    cp16(smem_u32(dst + o), kv.k + go);
                    cp16(smem_u32(dst + kTileBytes + o), kv.v + go);
                } else {
                    *reinterpret_cast<int4 *>(dst + o) = make_int4(0, 0, 0, 0);
                    *reinterpret_cast<int4 *>(dst + kTileBytes + o) = make_int4(0, 0, 0, 0);
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 1, 64;" ::: "memory");
            if (t == 0) {
                mbar_arrive(&fullK[s]);
                mbar_arrive(&fullV[s]);
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer ---------------------------------------------------------------------------
        if (lane == 0) {
            int pend[2] = {-1, -1};
            int pv_n[2] = {0, 0};
            uint8_t users[kMaxPasses];
            for (int j = 0; j < np; ++j) users[j] = (uint8_t)__popc(pl.pass[j].tiles);
            auto issue_pv = [&](int i) {
                const int jp = pend[i];
                mbar_wait(&fullV[jp % kStages], (jp / kStages) & 1);
                if (tr && i == 0) trace[11 + 12 * jp] = clock64();
                mbar_wait(&p_full[i], pv_n[i] & 1);
                if (tr) trace[2 + 12 * jp + i] = clock64();
                tc_fence_after();
                const uint8_t *v = sKV + (jp % kStages) * kStageBytes + kTileBytes;
                const uint32_t d_o = tmem + 256 + i * 128, a_p = tmem + i * 128;
#pragma unroll
                for (int k = 0; k < kCk / 16; ++k)
                    tc_mma_ts(d_o, a_p + k * 8, sw128_desc_mn(v + k * 2048, kHalfBytes), kIdescPV,
                              (pv_n[i] > 0 || k > 0) ? 1u : 0u);
                ++pv_n[i];
                pend[i] = -1;
                if (--users[jp] == 0) tc_commit(&emptyV[jp % kStages]);
            };
            for (int j = 0; j < np; ++j) {
                const Pass ps = pl.pass[j];
                // a pending P.V whose stage the producers need next must go first
                for (int i = 0; i < 2; ++i)
                    if (pend[i] >= 0 && pend[i] <= j - kStages) issue_pv(i);
                const int s = j % kStages;
                mbar_wait(&fullK[s], (j / kStages) & 1);
                if (tr) trace[1 + 12 * j] = clock64();
                tc_fence_after();
                const uint8_t *kt = sKV + s * kStageBytes;
                for (int i = 0; i < 2; ++i) {
                    if (!(ps.tiles & (1 << i))) continue;
                    if (pend[i] >= 0) issue_pv(i);
                    // Phase offset: tile 1's first scores wait for tile 0's first softmax, so the
                    // two softmax groups run half a period apart -- each overlaps the other
                    // tile's MMAs instead of both contending for the MUFU at once.
                    if (i == 1 && j == 0 && (ps.tiles & 1) && pv_n[1] == 0) mbar_wait(&p_full[0], 0);
                    const uint8_t *qt = sQ + i * kTileBytes;
                    const uint32_t d_s = tmem + i * 128;
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc_mma(d_s, sw128_desc(qt + h * kHalfBytes) + 2 * k, sw128_desc(kt + h * kHalfBytes) + 2 * k,
                                   kIdescS, (h | k) ? 1u : 0u);
                    tc_commit(&s_full[i]);
                    pend[i] = j;
                }
                tc_commit(&emptyK[s]);
            }
            for (int i = 0; i < 2; ++i)
                if (pend[i] >= 0) issue_pv(i);
            tc_commit(o_done);
        }
    } else if (warp >= 4) {
        // ---- softmax: one thread per row of M-tile `tile` ----------------------------------------
        // Per pass: one TMEM read of the row's 128 scores, the row max, p = 2^(s*scale - m) written
        // as bf16 over the consumed S columns (the 64-column halves [64h, 64h + 64) into S columns
        // [32h, 32h + 32)). The running max m only moves when the chunk max exceeds it by more
        // than 2^8 (so p <= 256): O in TMEM is then rescaled. Row sums are kept as 8 interleaved
        // partials per 64-column half. Every choice depends only on the row's own scores, so the
        // arithmetic is identical whatever item the row sits in.
        const int tile = (warp - 4) >> 2, qd = warp & 3;
        const int r = qd * 32 + lane;
        const int k = tile * T + r / G;
        const bool valid = r < T * G && k < pl.ntok;
        const bool warp_valid = __any_sync(0xffffffffu, valid);
        const int pos = valid ? pl.tok_pos[k] : -1;
        const int grp = valid ? pl.tok_grp[k] : -2;
        const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
        const uint32_t tS = tmem + lane_off + tile * 128, tO = tmem + lane_off + 256 + tile * 128;
        float m = -INFINITY;
        float lp[2][8];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < 8; ++i) lp[h][i] = 0.f;
        int n = 0;
        for (int j = 0; j < np; ++j) {
            const Pass ps = pl.pass[j];
            if (!(ps.tiles & (1 << tile))) continue;
            mbar_wait(&s_full[tile], n & 1);
            const bool trs = tr && tile == 0 && warp == 4 && lane == 0;
            if (trs) trace[4 + 12 * j] = clock64();
            tc_fence_after();
            const int c0 = ps.chunk * kCk;
            const bool mine = valid && (ps.grp < 0 || ps.grp == grp);
            const int lim = mine ? pos - c0 : -1;  // own columns x <= lim are visible
            if (warp_valid) {
                uint32_t v[128];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32_nw(tS + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
                tmem_ld_wait();
                float mxh[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int lh = lim - 64 * h;
                    float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
                    if (lh >= 63) {
#pragma unroll
                        for (int x = 0; x < 64; x += 4) {
                            mx0 = fmaxf(mx0, __uint_as_float(v[64 * h + x]));
                            mx1 = fmaxf(mx1, __uint_as_float(v[64 * h + x + 1]));
                            mx2 = fmaxf(mx2, __uint_as_float(v[64 * h + x + 2]));
                            mx3 = fmaxf(mx3, __uint_as_float(v[64 * h + x + 3]));
                        }
                    } else {
#pragma unroll
                        for (int x = 0; x < 64; ++x)
                            if (x <= lh) mx0 = fmaxf(mx0, __uint_as_float(v[64 * h + x]));
                    }
                    mxh[h] = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
                }
                float mx = fmaxf(mxh[0], mxh[1]);
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
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int i = 0; i < 8; ++i) lp[h][i] *= alpha;
                    }
                }
                const float nb = m == -INFINITY ? 0.f : -m;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int lh = lim - 64 * h;
                    const bool all = lh >= 63;
                    uint32_t pk[32];
#pragma unroll
                    for (int x = 0; x < 64; x += 2) {
                        float p0 = ex2(fmaf(__uint_as_float(v[64 * h + x]), scale_log2, nb));
                        float p1 = ex2(fmaf(__uint_as_float(v[64 * h + x + 1]), scale_log2, nb));
                        if (!all) {
                            p0 = x <= lh ? p0 : 0.f;
                            p1 = x + 1 <= lh ? p1 : 0.f;
                        }
                        lp[h][x & 7] += p0;
                        lp[h][(x + 1) & 7] += p1;
                        pk[x >> 1] = pack_bf16(p0, p1);
                    }
                    // P (bf16) of this half over S columns [32 h, 32 h + 32), already read
                    tmem_st16(tS + h * 32, *reinterpret_cast<uint32_t(*)[16]>(pk));
                    tmem_st16(tS + h * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(pk + 16));
                }
                if (n > 0 && __any_sync(0xffffffffu, resc)) {
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
            if (tr && tile == 0 && lane == 0) trace[5 + (warp - 4) + 12 * j] = clock64();  // this warp's P done
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[tile]);
            ++n;
        }
        if (n > 0 && warp_valid) {
            const float lh0 = ((lp[0][0] + lp[0][1]) + (lp[0][2] + lp[0][3])) + ((lp[0][4] + lp[0][5]) + (lp[0][6] + lp[0][7]));
            const float lh1 = ((lp[1][0] + lp[1][1]) + (lp[1][2] + lp[1][3])) + ((lp[1][4] + lp[1][5]) + (lp[1][6] + lp[1][7]));
            const float l = lh0 + lh1;
            mbar_wait(o_done, 0);
            tc_fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            bf16 *dst = out + ((size_t)(it.row0 + (valid ? k : 0)) * H + kvh * G + r % G) * kHD;
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
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

}  // namespace

int attn_tc_max_tokens(int G) { return 2 * (128 / G); }

void k_attention_tc(const bf16 *q, const RowDesc *rows, const AttnItem *items, const AttnPlan &plan, int n_items,
                    const KvCache &kv, int layer, const TfShape &s, bf16 *out, cudaStream_t st, double flops,
                    double bytes) {
    if (n_items <= 0) return;
    ProfScope prof("attn", flops, bytes, st);
    if (s.hd != kHD) throw std::invalid_argument("attention: head_dim must be 128");
    if (s.H / s.KV > 128) throw std::invalid_argument("attention: GQA group too large");
    static const bool attr = [] {  // thread-safe one-time init (engine + learner threads)
        static_assert(sizeof(Plan) + kBarBytes + 1024 + kQBytes + kStages * kStageBytes <= 232448, "smem");
        RS_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        return true;
    }();
    (void)attr;
    const int total_rows = kv.layers * kv.B * kv.KV * kv.max_ctx;
    const CUtensorMap tk = make_tma_map_bf16(kv.k, total_rows, kHD, kHD, kCk);
    const CUtensorMap tv = make_tma_map_bf16(kv.v, total_rows, kHD, kHD, kCk);
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(s.hd));
    static long long *trace = nullptr;
    if (tuning().attn_trace && !trace) RS_CUDA(cudaMalloc(&trace, 8 * (1 + 12 * kMaxPasses)));
    launch_pdl(attn_tc_kernel, dim3(n_items, s.KV), kThreads, kSmem, st, tk, tv, q, rows, items, plan, kv, layer,
               s.H, s.KV, scale_log2, out, tuning().attn_trace ? trace : nullptr);
    if (tuning().attn_trace) {
        RS_CUDA(cudaStreamSynchronize(st));
        static long long host[1 + 12 * kMaxPasses];
        RS_CUDA(cudaMemcpy(host, trace, sizeof(host), cudaMemcpyDeviceToHost));
        if (tuning().attn_trace == layer + 1 && n_items >= 32) {
            fprintf(stderr, "attn trace layer %d items %d:\n", layer, n_items);
            for (int j = 0; j < 24; ++j) {
                const long long *h = host + 1 + 12 * j;
                fprintf(stderr, "  pass %2d fullK %6lld p0 %6lld p1 %6lld sm0 %6lld | P done +%lld +%lld +%lld +%lld | "
                        "issueK %6lld issueV %6lld fullV %6lld\n",
                        j, h[0] - host[0], h[1] - host[0], h[2] - host[0], h[3] - host[0], h[4] - h[3], h[5] - h[3],
                        h[6] - h[3], h[7] - h[3], h[8] - host[0], h[9] - host[0], h[10] - host[0]);
            }
        }
    }
    RS_LAUNCHED();
}

}  // namespace rs

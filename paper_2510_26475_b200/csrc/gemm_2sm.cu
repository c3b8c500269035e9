// gemm_2sm.cu -- weight GEMMs on SM PAIRS (tcgen05.mma.cta_group::2), weights as the M operand.
//
//   C[T, N] = X[T, K] . W[N, K]^T     (X: T tokens of activations, W: N output features)
//
// computed as C^T = W . X^T: a CTA pair (thread-block cluster of 2) owns a 256-feature x BT-token
// tile. Each CTA stages its own 128 weight rows and HALF of the token rows (BT/2) per 64-wide
// k-block; the leader's single elected thread issues 128x... M=256 tcgen05.mma.cta_group::2 that
// read the weight halves and the token halves of BOTH CTAs, and each CTA's TMEM receives the
// fp32 accumulator of its own 128 features x BT tokens. Per SM and k-block this moves
// 16 KB + BT/2 x 128 B instead of 16 KB + BT x 128 B, and the feature dimension of every Qwen
// projection (QKV, O, gate/up, down, LM head) is a multiple of 256 while the token count (the
// verify tree: batch x (t n + 1)) is arbitrary -- no padded 128-row tiles.
//
// Roles per CTA (256 threads): warp 0 lane 0 = TMA producer (both CTAs; complete_tx lands on
// the LEADER's full barrier, the leader alone arms it with both CTAs' bytes), warp 1 lane 0 of
// the leader = MMA issuer (commits multicast to both CTAs' empty / accumulator-full barriers),
// warp 2 = TMEM allocator (cta_group::2, both CTAs), warps 4-7 = epilogue: thread = one feature
// row (TMEM lane), 32 tokens per tcgen05.ld, stores C[t][f] coalesced across the warp's lanes,
// then arrives (remotely for the peer) on the leader's accumulator-empty barrier.
// Epilogues: bias + bf16, scaled fp32 with a token row map (LM head), fp32 residual add
// (deterministic split-K order), SiLU(gate) * up with gate/up rows interleaved pairwise.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "gemm.h"
#include "launch.cuh"
#include "model.h"
#include "prof.h"
#include "tc.cuh"

namespace rs {

int gemm2_splits(const GemmArgs &g);

namespace {

constexpr int kBM = 128;  // weight rows per CTA (256 per pair)
constexpr int kBK = 64;
constexpr int kThr = 384;   // warps 0-3 control (TMA, MMA, TMEM), 4-11 epilogue
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quadrant, alternate 32-token chunks

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a local shared variable) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
// "accumulator drained": the epilogue's TMEM reads have completed (tcgen05.wait::ld) when it
// arrives, and the MMA warp only needs that, not the epilogue's global stores -- a release arrive
// would make every epilogue thread wait for its stores to reach the GPU (MEMBAR.ALL.GPU)
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// the exit barrier only protects the CTAs' shared memory / barriers / TMEM, not global data
__device__ __forceinline__ void cluster_sync_exit() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2sm(void *dst, const CUtensorMap *map, uint32_t bar_cluster, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// arrive on the barrier at the same offset in both CTAs of the pair once prior MMAs are done
__device__ __forceinline__ void tc_commit2_mc(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

template <int BT>
struct Cfg2 {
    static constexpr int kABytes = kBM * kBK * 2;          // own 128 weight rows
    static constexpr int kBBytes = (BT / 2) * kBK * 2;     // own half of the token rows
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStgBytes = 2 * 32 * 132 * 4;  // per epilogue group: 4 x 32 x 33 or 32 x 132 fp32
    // as many ring stages as the 227 KB opt-in shared memory leaves after the fixed parts (max 8)
    static constexpr int kFixed = 1024 + 256 + kStgBytes + 256 * 16 + 2048;  // + static smem / slack
    static constexpr int kStages = (232448 - kFixed) / kStageBytes > 8 ? 8 : (232448 - kFixed) / kStageBytes;
    static constexpr int kTmemCols = 2 * BT <= 128 ? 128 : 2 * BT <= 256 ? 256 : 512;
    static constexpr int kSmem = 1024 + kStages * kStageBytes + 256 + kStgBytes + 256 * 16;
    // kind::f16, bf16 x bf16 -> f32, both K-major, N = BT tokens, M = 256 features (pair)
    static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BT >> 3) << 17) |
                                       (static_cast<uint32_t>(256 >> 4) << 24);
    // dynamic + static (s_last) shared memory within the 227 KB opt-in limit, and the barrier
    // area (full/empty per stage, tfull/tempty x 2, the TMEM slot) within its 256 bytes
    static_assert(kSmem + 1024 <= 232448, "gemm2: shared memory over the 227 KB opt-in budget");
    static_assert((2 * kStages + 4) * 8 + 4 <= 256, "gemm2: barrier area overflow");
    static_assert(kStages >= 2, "gemm2: ring needs at least two stages");
};

// SiLU with the approximate division (MUFU.RCP + FMUL): the IEEE quotient's special-case check
// and slow path sat in every SwiGLU epilogue chunk; the output is rounded to bf16 anyway.
// g -> -inf: __expf(-g) = inf, __fdividef(g, inf) = -0.
__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Epilogue of one 32-token chunk of this warp's 32 feature rows f0w .. f0w + 31 (lane = row).
// The accumulator (thread = feature row, registers = tokens) is transposed through a
// 32 x 33 fp32 staging block so global memory is written token-row-wise with 16-byte vectors:
// C[t][f0w .. f0w + 31] is 128 B (fp32) / 64 B (bf16) / 32 B (SwiGLU, 16 outputs) contiguous.
// Residual rows of one 32-token chunk (same lane mapping as epi2_chunk), loaded ahead of the
// chunk that needs them so the L2 round trip overlaps the previous chunk's work.
__device__ __forceinline__ void resid_prefetch(const GemmEpi &ep, int f0w, int t0, int F, int T, float4 (&cur)[8]) {
    const int lane = threadIdx.x & 31, sub = lane >> 3, f = f0w + (lane & 7) * 4;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int t = t0 + i * 4 + sub;
        cur[i] = (t < T && f < F) ? __ldcg(reinterpret_cast<const float4 *>(static_cast<float *>(ep.out) +
                                                                             (size_t)t * ep.ldo + f))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

template <int EPI>
__device__ __forceinline__ void epi2_chunk(const GemmEpi &ep, uint32_t taddr, int f0w, int t0, int F, int T,
                                           float (*stg)[33], const float4 *pre = nullptr) {
    uint32_t v[32];
    tmem_ld32(taddr, v);
    const int lane = threadIdx.x & 31;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[j][lane] = __uint_as_float(v[j]);  // stg[token][feature]
    __syncwarp();
    if constexpr (EPI == kEpiF32 || EPI == kEpiResidual) {
        // 8 lanes x float4 per token row, 4 token rows per pass
        const int sub = lane >> 3, c4 = (lane & 7) * 4;
        const int f = f0w + c4;
        float4 cur[8];
        int rowo[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int j = i * 4 + sub, t = t0 + j;
            rowo[i] = -1;
            if (t < T && f < F) {
                rowo[i] = EPI == kEpiF32 ? (ep.row_map ? __ldg(ep.row_map + t) : t) : t;
                if (EPI == kEpiResidual && rowo[i] >= 0)
                    cur[i] = pre ? pre[i]
                                 : __ldcg(reinterpret_cast<const float4 *>(static_cast<float *>(ep.out) +
                                                                           (size_t)rowo[i] * ep.ldo + f));
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (rowo[i] < 0) continue;
            const int j = i * 4 + sub;
            float4 o = make_float4(stg[j][c4], stg[j][c4 + 1], stg[j][c4 + 2], stg[j][c4 + 3]);
            if (EPI == kEpiF32) {
                o.x *= ep.scale;
                o.y *= ep.scale;
                o.z *= ep.scale;
                o.w *= ep.scale;
            } else {
                o.x += cur[i].x;
                o.y += cur[i].y;
                o.z += cur[i].z;
                o.w += cur[i].w;
            }
            *reinterpret_cast<float4 *>(static_cast<float *>(ep.out) + (size_t)rowo[i] * ep.ldo + f) = o;
        }
    } else if constexpr (EPI == kEpiBF16) {
        // 4 lanes x 8 bf16 per token row, 8 token rows per pass
        const int sub = lane >> 2, c8 = (lane & 3) * 8;
        const int f = f0w + c8;
        __align__(16) __nv_bfloat162 bb[4];
        if (ep.bias && f < F) *reinterpret_cast<int4 *>(bb) = __ldg(reinterpret_cast<const int4 *>(
                                  static_cast<const __nv_bfloat16 *>(ep.bias) + f));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = i * 8 + sub, t = t0 + j;
            if (t >= T || f >= F) continue;
            __align__(16) __nv_bfloat162 h[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float a = stg[j][c8 + 2 * k], b = stg[j][c8 + 2 * k + 1];
                if (ep.bias) {
                    a += __low2float(bb[k]);
                    b += __high2float(bb[k]);
                }
                h[k] = __floats2bfloat162_rn(a, b);
            }
            *reinterpret_cast<int4 *>(static_cast<__nv_bfloat16 *>(ep.out) + (size_t)t * ep.ldo + f) =
                *reinterpret_cast<const int4 *>(h);
        }
    } else if constexpr (EPI == kEpiQKVRope) {
        // handled by epi2_qkv_rope (needs the whole 128-dim head of the CTA)
    } else {  // kEpiSwiGLU2: feature rows 2i / 2i + 1 = gate_i / up_i -> 16 outputs per token
        const int sub = lane >> 1, c16 = (lane & 1) * 16;  // 2 lanes x 8 outputs per token row
        const int fo = (f0w >> 1) + (c16 >> 1);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int j = i * 16 + sub, t = t0 + j;
            if (t >= T || 2 * fo >= F) continue;
            __align__(16) __nv_bfloat162 h[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float g0 = stg[j][c16 + 4 * k], u0 = stg[j][c16 + 4 * k + 1];
                const float g1 = stg[j][c16 + 4 * k + 2], u1 = stg[j][c16 + 4 * k + 3];
                h[k] = __floats2bfloat162_rn(silu(g0) * u0, silu(g1) * u1);
            }
            *reinterpret_cast<int4 *>(static_cast<__nv_bfloat16 *>(ep.out) + (size_t)t * ep.ldo + fo) =
                *reinterpret_cast<const int4 *>(h);
        }
    }
}

// QKV + bias + RoPE + K/V cache store for one 32-token chunk. The CTA's 128 features are one
// head (hd = 128): the four epilogue warps stage bf16(acc + bias) of all 128 dims x 32 tokens,
// then every thread rotates 8-dim vectors (i, i + 64 pairs, rotate-half, Qwen2) and stores 16 B
// into q [t][head] or the K / V cache slot of the token (RowDesc::seq / phys / pos). The bias
// value of the thread's dim is loaded once per tile and the cos / sin of the chunk were loaded
// during the previous chunk (rope_cs_load), so no global round trip sits on the chunk's path.
__device__ __forceinline__ void rope_cs_load(const QkvStore &s, const int4 *tok, int tbase, int t0, int T, int tid,
                                             float4 (&cs)[4][4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int vi = tid + 128 * k, j = vi >> 4, g = vi & 15;
        const int pos = t0 + j < T ? tok[t0 + j - tbase].x : 0;
        const float4 *src = reinterpret_cast<const float4 *>(s.rope + ((size_t)pos * 64 + ((8 * g) & 63)) * 2);
#pragma unroll
        for (int e = 0; e < 4; ++e) cs[k][e] = __ldg(src + e);
    }
}

__device__ __forceinline__ void epi2_qkv_rope(const GemmEpi &ep, uint32_t taddr, int head, int q_warp, int t0, int T,
                                              float (*stg)[132], const int4 *tok, int tbase, int bar,
                                              const float4 (&cs)[4][4], float b) {
    const int lane = threadIdx.x & 31;
    const int dim = q_warp * 32 + lane;
    const QkvStore &s = ep.qkv;
    const int tid = q_warp * 32 + lane;
    const bool is_q = head < s.H, is_k = !is_q && head < s.H + s.KV;
    uint32_t v[32];
    tmem_ld32(taddr, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[j][dim] = __bfloat162float(__float2bfloat16(__uint_as_float(v[j]) + b));
    asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int vi = tid + 128 * k, j = vi >> 4, g = vi & 15;  // token j, dims 8g .. 8g + 7
        const int t = t0 + j;
        if (t >= T) continue;
        const int4 r = tok[t - tbase];  // pos, seq, phys
        const int d0 = 8 * g;
        float o[8];
        if (is_q || is_k) {
            const int i0 = d0 & 63;
            const float *csf = reinterpret_cast<const float *>(cs[k]);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float c = csf[2 * e], sn = csf[2 * e + 1];
                const float x1 = stg[j][i0 + e], x2 = stg[j][i0 + 64 + e];
                o[e] = d0 < 64 ? x1 * c - x2 * sn : x2 * c + x1 * sn;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = stg[j][d0 + e];
        }
        __nv_bfloat16 *dst;
        if (is_q) {
            dst = static_cast<__nv_bfloat16 *>(s.q) + ((size_t)t * s.H + head) * 128;
        } else {
            const int kvh = is_k ? head - s.H : head - s.H - s.KV;
            const size_t off = ((((size_t)s.layer * s.B + r.y) * s.KV + kvh) * s.max_ctx + r.z) * 128;
            dst = static_cast<__nv_bfloat16 *>(is_k ? s.k : s.v) + off;
        }
        __align__(16) __nv_bfloat162 h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
        *reinterpret_cast<int4 *>(dst + d0) = *reinterpret_cast<const int4 *>(h);
    }
    asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");  // stg is reused by the next chunk
}

// F = features (rows of W), T = tokens (rows of X). Units = (feature pair-tile, token tile, split),
// token tiles fastest so the pairs that share a weight tile run together (one HBM read).
template <int BT, int EPI>
__global__ void __launch_bounds__(kThr, 1) __cluster_dims__(2, 1, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmEpi ep, int F,
                 int T, int K, int splits, int ngrp, int *sem, float *ws, long long *g2trace, int g2slot) {
    using C = Cfg2<BT>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // aligned by pointer arithmetic on the shared array (not through an integer), so the compiler
    // keeps the shared address space and emits STS / LDS instead of generic ST / LD
    uint8_t *smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint8_t *sA = smem;
    uint8_t *sB = smem + C::kStages * C::kABytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::kStages * C::kStageBytes);
    uint64_t *empty = full + C::kStages;
    uint64_t *tfull = empty + C::kStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    float(*stg_all)[33] = reinterpret_cast<float(*)[33]>(smem + C::kStages * C::kStageBytes + 256);
    int4 *tok_tab = reinterpret_cast<int4 *>(smem + C::kStages * C::kStageBytes + 256 + C::kStgBytes);  // [BT]

    __shared__ int s_last;  // split-K: this CTA holds the last partial of its tile
    pdl_trigger();
    if (g2trace && blockIdx.x == 0 && threadIdx.x == 0) g2trace[g2slot * 8 + 0] = clock64();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int num_f = (F + 2 * kBM - 1) / (2 * kBM), num_t = (T + BT - 1) / BT;
    const int num_k = (K + kBK - 1) / kBK;
    const int num_units = num_f * num_t * splits;
    auto unit_coords = [&](int unit, int &f0, int &t0, int &kb0, int &kb1) {
        const int split = unit % splits, tile = unit / splits;
        f0 = (tile / num_t) * 2 * kBM + rank * kBM;
        t0 = (tile % num_t) * BT;
        kb0 = split * num_k / splits;
        kb1 = (split + 1) * num_k / splits;
    };

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * 32 * kEpiWarps);  // both CTAs' epilogue threads
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::);
    }
    tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t lead_full = mapa(full, 0);  // full[0] of the leader; stage s at + 8 s
            // weights do not depend on the previous kernel: the first ring's worth of W k-blocks
            // goes out before the programmatic-dependency wait, the token rows after it
            int pre = 0;
            if (pair < num_units) {
                int f0, t0, kb0, kb1;
                unit_coords(pair, f0, t0, kb0, kb1);
                pre = min(C::kStages, kb1 - kb0);
                for (int i = 0; i < pre; ++i) {
                    if (leader) mbar_arrive_expect_tx(&full[i], 2 * C::kStageBytes);
                    tma_load_2sm(sA + i * C::kABytes, &tmW, lead_full + 8 * i, (kb0 + i) * kBK, f0);
                }
            }
            pdl_wait();
            if (g2trace && blockIdx.x == 0) g2trace[g2slot * 8 + 1] = clock64();
            int stage = 0;
            uint32_t phase = 0;
            int issued = 0;
            for (int unit = pair; unit < num_units; unit += npairs) {
                int f0, t0, kb0, kb1;
                unit_coords(unit, f0, t0, kb0, kb1);
                const int tb = t0 + (int)rank * (BT / 2);
                for (int kb = kb0; kb < kb1; ++kb, ++issued) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (issued >= pre) {
                        if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
                        tma_load_2sm(sA + stage * C::kABytes, &tmW, lead_full + 8 * stage, kb * kBK, f0);
                    }
                    tma_load_2sm(sB + stage * C::kBBytes, &tmX, lead_full + 8 * stage, kb * kBK, tb);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int unit = pair; unit < num_units; unit += npairs, ++it) {
                const int acc = it & 1;
                int f0, t0, kb0, kb1;
                unit_coords(unit, f0, t0, kb0, kb1);
                mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BT;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    if (g2trace && blockIdx.x == 0 && it == 0 && stage == 0 && phase == 0) g2trace[g2slot * 8 + 2] = clock64();
                    tc_fence_after();
                    const uint64_t ad = sw128_desc(sA + stage * C::kABytes);
                    const uint64_t bd = sw128_desc(sB + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        tc_mma2(tmem_d, ad + 2 * k, bd + 2 * k, C::kIdesc, (kb != kb0) || k != 0);
                    tc_commit2_mc(&empty[stage]);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit2_mc(&tfull[acc]);
                if (g2trace && blockIdx.x == 0 && it == 0) g2trace[g2slot * 8 + 3] = clock64();
            }
        }
    }
    // Single-wave launches (ngrp == 3: one unit per pair, no split-K) give the accumulator to a third
    // epilogue group: warps 0-3, idle once the last k-block is issued. Their staging buffer is the
    // first ring stages, free once the accumulator is complete (every TMA load was consumed).
    __syncwarp();
    if (warp >= 4 || (ngrp == 3 && pair < num_units)) {
        pdl_wait();
        const int q = warp & 3;                          // TMEM lane quadrant
        const int grp = warp >= 4 ? (warp - 4) >> 2 : 2;  // chunks grp, grp + ngrp, ...
        const int ebar = grp < 2 ? 2 + grp : 5;          // named barrier of the group (QKV epilogue)
        float(*stg_grp)[33] = grp < 2 ? stg_all + grp * 4 * 32 : reinterpret_cast<float(*)[33]>(sA);
        const uint32_t lead_tempty = mapa(tempty, 0);
        int it = 0;
        for (int unit = pair; unit < num_units; unit += npairs, ++it) {
            int f0, t0, kb0, kb1;
            unit_coords(unit, f0, t0, kb0, kb1);
            const int split = unit % splits, tile = unit / splits;
            const int acc = it & 1;
            if constexpr (EPI == kEpiQKVRope) {
                // (pos, seq, phys) of the tile's tokens, staged while the MMAs still run
                const RowDesc *rws = static_cast<const RowDesc *>(ep.qkv.rows);
                if (grp < 2) {
                    asm volatile("bar.sync 4, 256;" ::: "memory");  // previous tile done with the table
                    for (int i = threadIdx.x - 128; i < BT; i += 256)
                        if (t0 + i < T) {
                            const RowDesc r = rws[t0 + i];
                            tok_tab[i] = make_int4(r.pos, r.seq, r.phys, 0);
                        }
                    asm volatile("bar.sync 4, 256;" ::: "memory");
                    if (ngrp == 3) asm volatile("bar.arrive 6, 384;" ::: "memory");
                } else {
                    asm volatile("bar.sync 6, 384;" ::: "memory");  // the table is staged
                }
            }
            // the epilogue's first global inputs do not depend on the MMAs: in flight before the
            // accumulator is ready (the first residual rows; the QKV bias and first cos / sin)
            float4 cur[2][8];
            float4 cs[4][4];
            float qb = 0.f;
            if constexpr (EPI == kEpiResidual) {
                if (splits == 1 && grp < BT / 32) resid_prefetch(ep, f0 + q * 32, t0 + grp * 32, F, T, cur[0]);
            } else if constexpr (EPI == kEpiQKVRope) {
                const int tid = q * 32 + lane;
                qb = __bfloat162float(static_cast<const __nv_bfloat16 *>(ep.bias)[f0 + tid]);
                if (f0 / 128 < ep.qkv.H + ep.qkv.KV && grp < BT / 32)
                    rope_cs_load(ep.qkv, tok_tab, t0, t0 + grp * 32, T, tid, cs);
            }
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            if (g2trace && blockIdx.x == 0 && threadIdx.x == 128 && it == 0) g2trace[g2slot * 8 + 4] = clock64();
            tc_fence_after();
            const uint32_t tb = tmem_base + acc * BT + (static_cast<uint32_t>(q * 32) << 16);
            if (EPI == kEpiResidual && splits > 1) {
                // Split-K without hand-offs: every split parks its fp32 partial (this CTA's 128
                // features x BT tokens, token-major) in the workspace; the split that arrives last
                // sums ALL partials in split order -- the same order whichever split is last -- back
                // into its accumulator and runs the one residual epilogue.
                const int slot = tile * 2 + (int)rank;
                float *mine = ws + ((size_t)slot * splits + split) * (128 * BT);
                const int f = q * 32 + lane;
                // feature-major: thread f owns ws[f][0 .. BT), 16-byte stores / loads
                float4 *mrow = reinterpret_cast<float4 *>(mine + (size_t)f * BT);
#pragma unroll 1
                for (int c = grp; c < BT / 32; c += 2) {
                    uint32_t v[32];
                    tmem_ld32(tb + c * 32, v);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        __stcg(mrow + c * 8 + j, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                             __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
                }
                __threadfence();
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (warp == 4 && lane == 0) s_last = atomicAdd(sem + slot, 1) == splits - 1;
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (!s_last) {
                    tc_fence_before();
                    if (unit + 2 * npairs < num_units) mbar_arrive_remote_relaxed(lead_tempty + 8 * acc);
                    continue;
                }
                __threadfence();
                const float4 *base = reinterpret_cast<const float4 *>(ws + (size_t)slot * splits * (128 * BT) + (size_t)f * BT);
                constexpr int kSplitStride = 128 * BT / 4;  // float4s between consecutive splits
#pragma unroll 1
                for (int c = grp; c < BT / 32; c += 2) {
                    float4 a[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) a[j] = __ldcg(base + c * 8 + j);
#pragma unroll 1
                    for (int sp = 1; sp < splits; ++sp) {
                        float4 b[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) b[j] = __ldcg(base + (size_t)sp * kSplitStride + c * 8 + j);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            a[j].x += b[j].x;
                            a[j].y += b[j].y;
                            a[j].z += b[j].z;
                            a[j].w += b[j].w;
                        }
                    }
                    uint32_t v[32];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        v[4 * j] = __float_as_uint(a[j].x);
                        v[4 * j + 1] = __float_as_uint(a[j].y);
                        v[4 * j + 2] = __float_as_uint(a[j].z);
                        v[4 * j + 3] = __float_as_uint(a[j].w);
                    }
                    tmem_st32(tb + c * 32, v);
                }
                tmem_st_wait();
                tc_fence_before();
                if (warp == 4 && lane == 0) sem[slot] = 0;  // ready for the next launch
                tc_fence_after();
            }
            if constexpr (EPI == kEpiQKVRope) {
                const int head = f0 / 128, tid = q * 32 + lane;
                const bool rope = head < ep.qkv.H + ep.qkv.KV;  // q and k heads rotate, v heads do not
                const float b = qb;
#pragma unroll 1
                for (int c = grp; c < BT / 32; c += ngrp) {
                    epi2_qkv_rope(ep, tb + c * 32, head, q, t0 + c * 32, T, reinterpret_cast<float(*)[132]>(stg_grp),
                                  tok_tab, t0, ebar, cs, b);
                    // the next chunk's cos / sin, in flight during its TMEM read and staging
                    if (rope && c + ngrp < BT / 32) rope_cs_load(ep.qkv, tok_tab, t0, t0 + (c + ngrp) * 32, T, tid, cs);
                }
            } else if constexpr (EPI == kEpiResidual) {
                // software-pipelined: chunk c + 1's residual rows are in flight while chunk c is done
                // (the first chunk's were issued before the accumulator wait; after a split-K
                // reduction they are read now, the other splits having updated nothing)
                if (splits > 1 && grp < BT / 32) resid_prefetch(ep, f0 + q * 32, t0 + grp * 32, F, T, cur[0]);
                // (the loop counter stays compile-time so the register double buffer does too)
#pragma unroll
                for (int i = 0; i < (BT / 32 + 1) / 2; ++i) {
                    const int c = grp + i * ngrp;
                    if (c >= BT / 32) break;
                    if (c + ngrp < BT / 32) resid_prefetch(ep, f0 + q * 32, t0 + (c + ngrp) * 32, F, T, cur[(i + 1) & 1]);
                    epi2_chunk<EPI>(ep, tb + c * 32, f0 + q * 32, t0 + c * 32, F, T, stg_grp + q * 32, cur[i & 1]);
                }
            } else {
#pragma unroll 1
                for (int c = grp; c < BT / 32; c += ngrp)
                    epi2_chunk<EPI>(ep, tb + c * 32, f0 + q * 32, t0 + c * 32, F, T, stg_grp + q * 32);
            }
            tc_fence_before();
            // the MMA warp waits for this accumulator again only if the pair has a unit two ahead
            // (the third group only runs single-unit launches)
            if (grp < 2 && unit + 2 * npairs < num_units) mbar_arrive_remote_relaxed(lead_tempty + 8 * acc);
            if (g2trace && blockIdx.x == 0 && threadIdx.x == 128 && it == 0) g2trace[g2slot * 8 + 5] = clock64();
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_exit();  // no CTA leaves while its peer may still signal its barriers
    if (g2trace && blockIdx.x == 0 && threadIdx.x == 128) g2trace[g2slot * 8 + 6] = clock64();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::kTmemCols));
    }
}

int num_sms2() {
    static const int n = [] {
        int dev = 0, v = 0;
        RS_CUDA(cudaGetDevice(&dev));
        RS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

template <int BT, int EPI>
void launch2(const GemmArgs &g, cudaStream_t st) {
    using C = Cfg2<BT>;
    static const bool attr = [] {  // thread-safe one-time init (engine + learner threads)
        RS_CUDA(cudaFuncSetAttribute(gemm2_kernel<BT, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        return true;
    }();
    (void)attr;
    const int F = g.N, T = g.M;
    const CUtensorMap tw = make_tma_map_bf16(g.B, F, g.K, g.ldb, kBM);
    const CUtensorMap tx = make_tma_map_bf16(g.A, T, g.K, g.lda, BT / 2);
    const int tiles = ((F + 2 * kBM - 1) / (2 * kBM)) * ((T + BT - 1) / BT);
    const int num_k = (g.K + kBK - 1) / kBK;
    const int splits = EPI == kEpiResidual ? std::max(1, std::min(gemm2_splits(g), num_k)) : 1;
    int *sem = nullptr;
    float *ws = nullptr;
    if (splits > 1) {
        // per host thread (engine / learner streams never share them): arrival counters, zero
        // between launches (the last split resets its own), and the partial-tile workspace
        static thread_local int *sems = nullptr;
        static thread_local int sems_n = 0;
        static thread_local float *wsb = nullptr;
        static thread_local size_t ws_n = 0;
        if (sems_n < 2 * tiles) {
            if (sems) cudaFree(sems);
            sems_n = std::max(2 * tiles, 8192);
            RS_CUDA(cudaMalloc(&sems, (size_t)sems_n * sizeof(int)));
            RS_CUDA(cudaMemsetAsync(sems, 0, (size_t)sems_n * sizeof(int), st));
        }
        const size_t need = (size_t)2 * tiles * splits * 128 * BT;
        if (ws_n < need) {
            if (wsb) cudaFree(wsb);
            ws_n = need;
            RS_CUDA(cudaMalloc(&wsb, ws_n * sizeof(float)));
        }
        sem = sems;
        ws = wsb;
    }
    const int pairs = std::min(tiles * splits, num_sms2() / 2);
    const int ngrp = tuning().epi3 >= 0 && splits == 1 && tiles <= pairs ? 3 : 2;
    // diagnostics (RS_TUNE gemm_trace=1): per launch of CTA 0: start, after the dependency wait,
    // first full stage, last MMA commit of tile 0, epilogue start / end of tile 0, exit
    static long long *tr = nullptr;
    static int slot = 0;
    if (tuning().gemm_trace && !tr) RS_CUDA(cudaMalloc(&tr, 8 * 8 * 4096));
    launch_pdl(gemm2_kernel<BT, EPI>, dim3(2 * pairs), kThr, C::kSmem, st, tw, tx, g.epi, F, T, g.K, splits, ngrp, sem, ws,
               tuning().gemm_trace ? tr : (long long *)nullptr, slot);
    if (tuning().gemm_trace) {
        RS_CUDA(cudaStreamSynchronize(st));
        long long h[8];
        RS_CUDA(cudaMemcpy(h, tr + slot * 8, sizeof(h), cudaMemcpyDeviceToHost));
        if (slot < 4096 && F < 20000 && T > 1000)
            fprintf(stderr, "gemm2 F=%d T=%d K=%d BT=%d epi=%d: wait %lld full0 %lld mma_done %lld epi %lld..%lld exit %lld\n",
                    F, T, g.K, BT, EPI, h[1] - h[0], h[2] - h[0], h[3] - h[0], h[4] - h[0], h[5] - h[0], h[6] - h[0]);
        slot = (slot + 1) % 4096;
    }
    RS_LAUNCHED();
}

}  // namespace

bool gemm2_supported(const GemmArgs &g) {
    return g.K % 8 == 0 && g.lda % 8 == 0 && g.ldb % 8 == 0 && g.epi.stats == nullptr && g.M > 0 && g.N > 0 &&
           g.epi.kind != kEpiSwiGLU;
}

// Token tile: the BT of {256 .. 64} with the least modelled time for the unit count of one
// (features, tokens, splits) problem -- waves of SM pairs x k-blocks per unit x cycles per
// k-block, where a k-block costs max(tensor time, per-SM operand traffic at ~58 B/clk) -- plus
// a fixed charge per extra split. The result never changes a token's arithmetic (token-tile
// invariance), only the schedule.
int gemm2_pick_bt(int F, int T, int K, int splits, int sms) {
    const int pairs = sms / 2, nf = (F + 255) / 256, nk = (K + 63) / 64;
    double best = 1e30;
    int bt = 256;
    for (int cand : {256, 224, 192, 160, 128, 96, 64}) {
        const double units = (double)nf * ((T + cand - 1) / cand) * splits;
        const double waves = std::ceil(units / pairs);
        const double per_kb = std::max(2.12 * cand, (16384.0 + 64.0 * cand) / 58.0);
        const double cost = waves * std::ceil((double)nk / splits) * per_kb + (splits - 1) * 2000.0;
        if (cost < best * 0.999) {
            best = cost;
            bt = cand;
        }
    }
    return bt;
}

// Split-K for the residual epilogue is a function of (F, K) only -- never of the token count --
// so a token's partial-sum order, and with it its bits, does not depend on the batch it is in.
int gemm2_splits(const GemmArgs &g) {
    if (g.epi.kind != kEpiResidual) return 1;
    if (g.splits > 0) return g.splits;
    // measured on B200 (down projection, K = 11008, 1344 tokens): 3 splits at BT 224 cost more
    // (three read-modify-write passes over the fp32 residual + ordered hand-offs) than one split
    // at BT 160 (8.94 vs 8.45 ms/step of verify GEMMs), so the automatic choice is one split
    return 1;
}

void gemm2_bf16(const GemmArgs &g, cudaStream_t st) {
    const int splits = gemm2_splits(g);
    const int bt = g.block_n ? g.block_n : gemm2_pick_bt(g.N, g.M, g.K, splits, num_sms2());
    auto by_bt = [&](auto tag) {
        constexpr int E = decltype(tag)::value;
        switch (bt) {
            case 64: launch2<64, E>(g, st); break;
            case 96: launch2<96, E>(g, st); break;
            case 128: launch2<128, E>(g, st); break;
            case 160: launch2<160, E>(g, st); break;
            case 192: launch2<192, E>(g, st); break;
            case 224: launch2<224, E>(g, st); break;
            case 256: launch2<256, E>(g, st); break;
            default: throw std::invalid_argument("gemm2: token tile must be 64..256 in steps of 32");
        }
    };
    switch (g.epi.kind) {
        case kEpiBF16: by_bt(std::integral_constant<int, kEpiBF16>{}); break;
        case kEpiF32: by_bt(std::integral_constant<int, kEpiF32>{}); break;
        case kEpiResidual: by_bt(std::integral_constant<int, kEpiResidual>{}); break;
        case kEpiSwiGLU2: by_bt(std::integral_constant<int, kEpiSwiGLU2>{}); break;
        case kEpiQKVRope:
            if (g.N % 128 || !g.epi.bias) throw std::invalid_argument("gemm2: QKV+RoPE needs 128-dim heads and a bias");
            by_bt(std::integral_constant<int, kEpiQKVRope>{});
            break;
        default: throw std::invalid_argument("gemm2: unsupported epilogue");
    }
}

}  // namespace rs

// gemm_sm100.cu -- persistent warp-specialised bf16 GEMM on 5th-gen tensor cores.
//
//   C[M, N] = A[M, K] . B[N, K]^T      (A activations, B weights; both K-major bf16)
//
// One CTA per SM loops over 128 x BN output tiles (M fastest, so co-resident CTAs share the
// weight tile in L2). Warp 0 streams A/B k-blocks (64 wide, 128B-swizzled) into a STAGES-deep
// shared-memory ring with TMA; one elected lane of warp 1 issues tcgen05.mma (kind::f16,
// 128 x BN x 16, fp32 accumulation in TMEM) and commits to the ring's empty barriers; two
// TMEM accumulators (2 x BN columns) let warps 4-7 drain tile i (tcgen05.ld 32x32b) while
// tile i+1 accumulates. Epilogues are fused: bias + bf16 store, scaled fp32 store (LM head
// logits), fp32 residual add, and SiLU(gate) * up for the interleaved gate/up projection.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "gemm.h"
#include "launch.cuh"
#include "tc.cuh"
#include "prof.h"

namespace rs {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;

template <int BN>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
    static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    static constexpr int kSmem = 1024 + kStages * kStageBytes + 256;
    static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                       (static_cast<uint32_t>(BM >> 4) << 24);
};

__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }  // as gemm_2sm.cu

// Epilogue for one thread = one output row, 32 consecutive accumulator columns.
template <int EPI, int BN>
__device__ __forceinline__ void epilogue_chunk(const GemmEpi &ep, uint32_t tbase, int row, int col0, int chunk, int M,
                                               int N, double &rm, double &rs) {
    uint32_t v[32];
    if constexpr (EPI == kEpiSwiGLU) {
        // accumulator columns [0, BN/2) are gate, [BN/2, BN) are up, for BN/2 outputs
        uint32_t u[32];
        tmem_ld32(tbase + chunk * 32, v);
        tmem_ld32(tbase + BN / 2 + chunk * 32, u);
        if (row >= M) return;
        const int n0 = col0 / 2 + chunk * 32;  // output column
        const int Nout = N / 2;
        __nv_bfloat16 *out = static_cast<__nv_bfloat16 *>(ep.out) + static_cast<size_t>(row) * ep.ldo + n0;
        if (n0 + 32 <= Nout) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
                __align__(16) __nv_bfloat162 h[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float a = silu(__uint_as_float(v[j + 2 * k])) * __uint_as_float(u[j + 2 * k]);
                    const float b = silu(__uint_as_float(v[j + 2 * k + 1])) * __uint_as_float(u[j + 2 * k + 1]);
                    h[k] = __floats2bfloat162_rn(a, b);
                }
                *reinterpret_cast<int4 *>(out + j) = *reinterpret_cast<int4 *>(h);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (n0 + j < Nout) out[j] = __float2bfloat16(silu(__uint_as_float(v[j])) * __uint_as_float(u[j]));
        }
        return;
    } else if constexpr (EPI == kEpiSwiGLU2) {
        // pairwise interleave: accumulator columns 2i / 2i + 1 are gate_i / up_i
        tmem_ld32(tbase + chunk * 32, v);
        if (row >= M) return;
        const int n0 = col0 / 2 + chunk * 16;  // output column
        const int Nout = N / 2;
        __nv_bfloat16 *out = static_cast<__nv_bfloat16 *>(ep.out) + static_cast<size_t>(row) * ep.ldo + n0;
        if (n0 + 16 <= Nout) {
            __align__(16) __nv_bfloat162 h[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                h[k] = __floats2bfloat162_rn(silu(__uint_as_float(v[4 * k])) * __uint_as_float(v[4 * k + 1]),
                                             silu(__uint_as_float(v[4 * k + 2])) * __uint_as_float(v[4 * k + 3]));
            reinterpret_cast<int4 *>(out)[0] = reinterpret_cast<const int4 *>(h)[0];
            reinterpret_cast<int4 *>(out)[1] = reinterpret_cast<const int4 *>(h)[1];
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (n0 + j < Nout)
                    out[j] = __float2bfloat16(silu(__uint_as_float(v[2 * j])) * __uint_as_float(v[2 * j + 1]));
        }
        return;
    } else {
        tmem_ld32(tbase + chunk * 32, v);
        if (row >= M) return;
        const int n0 = col0 + chunk * 32;
        if constexpr (EPI == kEpiBF16) {
            __nv_bfloat16 *out = static_cast<__nv_bfloat16 *>(ep.out) + static_cast<size_t>(row) * ep.ldo + n0;
            const __nv_bfloat16 *bias = static_cast<const __nv_bfloat16 *>(ep.bias);
            if (n0 + 32 <= N) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    __align__(16) __nv_bfloat162 h[4];
                    __align__(16) __nv_bfloat162 bb[4];
                    if (bias) *reinterpret_cast<int4 *>(bb) = __ldg(reinterpret_cast<const int4 *>(bias + n0 + j));
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        float a = __uint_as_float(v[j + 2 * k]), b = __uint_as_float(v[j + 2 * k + 1]);
                        if (bias) {
                            a += __low2float(bb[k]);
                            b += __high2float(bb[k]);
                        }
                        h[k] = __floats2bfloat162_rn(a, b);
                    }
                    *reinterpret_cast<int4 *>(out + j) = *reinterpret_cast<int4 *>(h);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (n0 + j >= N) continue;
                    float a = __uint_as_float(v[j]);
                    if (bias) a += __bfloat162float(bias[n0 + j]);
                    out[j] = __float2bfloat16(a);
                }
            }
        } else if constexpr (EPI == kEpiF32) {
            const int orow = ep.row_map ? ep.row_map[row] : row;
            if (orow < 0) return;
            float *out = static_cast<float *>(ep.out) + static_cast<size_t>(orow) * ep.ldo + n0;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * ep.scale);
            if (n0 + 32 <= N) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4 *>(out + j) = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                                      __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (n0 + j < N) out[j] = __uint_as_float(v[j]);
            }
            if (ep.stats) {  // running fp32 max of the tile's columns except the global last (EOS)
                float cm = -INFINITY;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (n0 + j < N - 1) cm = fmaxf(cm, __uint_as_float(v[j]));
                rm = fmax(rm, (double)cm);
            }
        } else {  // kEpiResidual: out (fp32) += acc (L2-coherent loads: split-K partials of other SMs)
            float *out = static_cast<float *>(ep.out) + static_cast<size_t>(row) * ep.ldo + n0;
            if (n0 + 32 <= N) {
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    float4 f = __ldcg(reinterpret_cast<const float4 *>(out + j));
                    f.x += __uint_as_float(v[j]);
                    f.y += __uint_as_float(v[j + 1]);
                    f.z += __uint_as_float(v[j + 2]);
                    f.w += __uint_as_float(v[j + 3]);
                    *reinterpret_cast<float4 *>(out + j) = f;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (n0 + j < N) out[j] = __ldcg(out + j) + __uint_as_float(v[j]);
            }
        }
    }
}

// Second epilogue pass of the LM head (kEpiF32 with stats, BN = 256 = one stats tile): the
// tile's fp64 softmax partials in EXACTLY tilestat.cuh's order -- "lane" l of the canonical
// warp owns columns l + 32 j, partials summed in j order, then the xor-butterfly -- so a row's
// statistics are bitwise those of the stand-alone row-stats kernel. The accumulator is
// re-read from TMEM (and re-scaled) instead of being held in registers.
__device__ __forceinline__ void stats_pass(const GemmEpi &ep, uint32_t tb, int row, int n0, int M, int N, float mx) {
    const bool live = mx != -INFINITY;
    const bool unit = ep.tau == 1.0;
    const double m = !live ? -INFINITY : unit ? (double)mx : (double)mx / ep.tau;
    double acc[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) acc[l] = 0.0;
#pragma unroll 1
    for (int c = 0; c < 8; ++c) {
        uint32_t v[32];
        tmem_ld32(tb + c * 32, v);  // warp-collective: every lane, live or not
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            const float f = __uint_as_float(v[l]) * ep.scale;
            if (live && n0 + c * 32 + l < N - 1 && f != -INFINITY) {
                const double y = unit ? (double)f : (double)f / ep.tau;
                acc[l] += exp(y - m);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int l = 0; l < o; ++l) acc[l] = acc[l] + acc[l + o];
    if (row < M) {
        const int orow = ep.row_map ? ep.row_map[row] : row;
        if (orow >= 0) {
            const int ntiles = (N + 255) / 256;
            double *st = ep.stats + ((size_t)orow * ntiles + n0 / 256) * 2;
            st[0] = m;
            st[1] = live ? acc[0] : 0.0;
        }
    }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmEpi ep, int M,
                int N, int K, int splits, int *sem) {
    using C = Cfg<BN>;
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

    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
    const int num_tiles = num_m * num_n;
    const int num_k = (K + BK - 1) / BK;
    // work unit = (tile, K split); splits of one tile are adjacent units, K ranges balanced
    const int num_units = num_tiles * splits;
    auto krange = [&](int s, int &kb0, int &kb1) {
        kb0 = s * num_k / splits;
        kb1 = (s + 1) * num_k / splits;
    };

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // The weights (B) do not depend on the previous kernel: the first ring's worth of B
            // k-blocks is requested before the programmatic-dependency wait, so the HBM latency
            // of the weight stream overlaps the previous kernel's tail. A (activations) follows.
            int pre = 0;
            if (blockIdx.x < num_units) {
                const int tile = blockIdx.x / splits;
                const int n0 = (tile / num_m) * BN;
                int kb0, kb1;
                krange(blockIdx.x % splits, kb0, kb1);
                pre = min(C::kStages, kb1 - kb0);
                for (int i = 0; i < pre; ++i) {
                    mbar_arrive_expect_tx(&full[i], C::kStageBytes);
                    tma_load_2d(sB + i * C::kBBytes, &tmB, &full[i], (kb0 + i) * BK, n0);
                }
            }
            pdl_wait();  // activations / residual of the previous kernel
            int stage = 0;
            uint32_t phase = 0;
            int issued = 0;
            for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
                const int tile = unit / splits;
                const int m0 = (tile % num_m) * BM, n0 = (tile / num_m) * BN;
                int kb0, kb1;
                krange(unit % splits, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb, ++issued) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (issued >= pre) {
                        mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        tma_load_2d(sB + stage * C::kBBytes, &tmB, &full[stage], kb * BK, n0);
                    }
                    tma_load_2d(sA + stage * C::kABytes, &tmA, &full[stage], kb * BK, m0);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                int kb0, kb1;
                krange(unit % splits, kb0, kb1);
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = sw128_desc(sA + stage * C::kABytes);
                    const uint64_t bd = sw128_desc(sB + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)  // +32 bytes per 16-wide K step inside the swizzle atom
                        tc_mma(tmem_d, ad + 2 * k, bd + 2 * k, C::kIdesc, (kb != kb0) || k != 0);
                    tc_commit(&empty[stage]);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        pdl_wait();  // outputs / residual / bias reads happen after the previous kernel
        const int q = warp - 4;  // TMEM lane quadrant == warp % 4
        int it = 0;
        for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++it) {
            const int tile = unit / splits, split = unit % splits;
            const int m0 = (tile % num_m) * BM, n0 = (tile / num_m) * BN;
            const int acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            if (EPI == kEpiResidual && splits > 1) {
                // deterministic split-K: partials are added in split order (each split's
                // read-modify-write waits for its predecessor), so a row's result does not
                // depend on which SM ran which split -- nor on M.
                int v;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(sem + tile) : "memory");
                    if (v < split) __nanosleep(32);
                } while (v < split);
            }
            const uint32_t tb = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
            const int row = m0 + q * 32 + lane;
            constexpr int kChunks = (EPI == kEpiSwiGLU ? BN / 2 : BN) / 32;
            double rm = -INFINITY, rs = 0.0;
#pragma unroll 1
            for (int c = 0; c < kChunks; ++c) epilogue_chunk<EPI, BN>(ep, tb, row, n0, c, M, N, rm, rs);
            if constexpr (EPI == kEpiF32 && BN == 256) {
                // the tile max is warp-uniform only per row; every lane joins the TMEM loads
                if (ep.stats) stats_pass(ep, tb, row, n0, M, N, (float)rm);
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            if (EPI == kEpiResidual && splits > 1) {
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");  // all 4 epilogue warps wrote their rows
                if (q == 0 && lane == 0)
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sem + tile), "r"(split + 1) : "memory");
            }
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::kTmemCols));
    }
}

// ---- host: tensor maps ------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap make_map(const void *base, int rows, int cols, int ld, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

}  // namespace

CUtensorMap make_tma_map_bf16(const void *base, int rows, int cols, int ld, int box_rows) {
    return make_map(base, rows, cols, ld, box_rows);
}

namespace {

int num_sms() {
    static const int n = [] {
        int dev = 0, v = 0;
        RS_CUDA(cudaGetDevice(&dev));
        RS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

template <int BN, int EPI>
void launch(const GemmArgs &g, cudaStream_t st) {
    using C = Cfg<BN>;
    static const bool attr = [] {  // thread-safe one-time init (engine + learner threads)
        RS_CUDA(cudaFuncSetAttribute(gemm_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        return true;
    }();
    (void)attr;
    const CUtensorMap ta = make_map(g.A, g.M, g.K, g.lda, BM);
    const CUtensorMap tb = make_map(g.B, g.N, g.K, g.ldb, BN);
    const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
    const int num_k = (g.K + BK - 1) / BK;
    int splits = EPI == kEpiResidual ? std::max(1, std::min(g.splits, num_k)) : 1;
    int *sem = nullptr;
    if (splits > 1) {
        // per-tile split counters, zeroed before every launch (grid <= #SMs, all CTAs resident)
        static thread_local int *sems = nullptr;
        static thread_local int sems_n = 0;
        if (sems_n < tiles) {
            if (sems) cudaFree(sems);
            sems_n = std::max(tiles, 4096);
            RS_CUDA(cudaMalloc(&sems, (size_t)sems_n * sizeof(int)));
        }
        RS_CUDA(cudaMemsetAsync(sems, 0, (size_t)tiles * sizeof(int), st));
        sem = sems;
    }
    const int grid = std::min(tiles * splits, num_sms());
    launch_pdl(gemm_kernel<BN, EPI>, grid, kThreads, C::kSmem, st, ta, tb, g.epi, g.M, g.N, g.K, splits, sem);
    RS_LAUNCHED();
}

}  // namespace

void gemm_bf16(const GemmArgs &g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return;
    if (g.epi.kind == kEpiQKVRope && (tuning().gemm2 < 0 || g.force_1sm || !gemm2_supported(g)))
        throw std::invalid_argument("gemm_bf16: the fused QKV+RoPE epilogue runs on the SM-pair kernel only");
    if (tuning().gemm2 >= 0 && !g.force_1sm && gemm2_supported(g)) {
        const double out_el = g.epi.kind == kEpiSwiGLU2 ? 0.5 * g.M * g.N : (double)g.M * g.N;
        const double out_b = g.epi.kind == kEpiBF16 || g.epi.kind == kEpiSwiGLU2 ? 2.0 : g.epi.kind == kEpiF32 ? 4.0 : 8.0;
        ProfScope prof("gemm", 2.0 * g.M * g.N * g.K, 2.0 * ((double)g.M * g.K + (double)g.N * g.K) + out_el * out_b, st);
        gemm2_bf16(g, st);
        return;
    }
    if (g.K % 8 || g.lda % 8 || g.ldb % 8) throw std::invalid_argument("gemm_bf16: K and leading dims must be multiples of 8");
    if (g.epi.kind == kEpiSwiGLU && (g.N % 256)) throw std::invalid_argument("gemm_bf16: SwiGLU needs N % 256 == 0");
    int bn = g.block_n;
    if (!bn) {
        // tile width that best fills the SMs: wave count x per-tile time (proportional to BN)
        const int tm = (g.M + BM - 1) / BM;
        double best = 1e30;
        bn = 256;
        for (int cand : {256, 224, 192, 160, 128}) {
            const int tiles = tm * ((g.N + cand - 1) / cand);
            const double cost = (double)((tiles + num_sms() - 1) / num_sms()) * cand * (cand < 256 ? 1.02 : 1.0);
            if (cost < best) {
                best = cost;
                bn = cand;
            }
        }
    }
    if (g.epi.kind == kEpiSwiGLU || g.epi.stats) bn = 256;
    if (g.epi.kind == kEpiSwiGLU2 && (g.N % 2)) throw std::invalid_argument("gemm_bf16: SwiGLU needs an even N");
    const double out_el = g.epi.kind == kEpiSwiGLU || g.epi.kind == kEpiSwiGLU2 ? 0.5 * g.M * g.N : (double)g.M * g.N;
    const double out_b = g.epi.kind == kEpiBF16 || g.epi.kind == kEpiSwiGLU || g.epi.kind == kEpiSwiGLU2 ? 2.0
                         : g.epi.kind == kEpiF32                                                        ? 4.0
                                                                                                        : 8.0;
    ProfScope prof("gemm", 2.0 * g.M * g.N * g.K, 2.0 * ((double)g.M * g.K + (double)g.N * g.K) + out_el * out_b, st);
    auto by_bn = [&](auto epi_tag) {
        constexpr int E = decltype(epi_tag)::value;
        switch (bn) {
            case 128: launch<128, E>(g, st); break;
            case 160: launch<160, E>(g, st); break;
            case 192: launch<192, E>(g, st); break;
            case 224: launch<224, E>(g, st); break;
            case 256: launch<256, E>(g, st); break;
            default: throw std::invalid_argument("gemm_bf16: block_n must be 128/160/192/224/256");
        }
    };
    switch (g.epi.kind) {
        case kEpiBF16: by_bn(std::integral_constant<int, kEpiBF16>{}); break;
        case kEpiF32: by_bn(std::integral_constant<int, kEpiF32>{}); break;
        case kEpiResidual: by_bn(std::integral_constant<int, kEpiResidual>{}); break;
        case kEpiSwiGLU: launch<256, kEpiSwiGLU>(g, st); break;
        case kEpiSwiGLU2: by_bn(std::integral_constant<int, kEpiSwiGLU2>{}); break;
        default: throw std::invalid_argument("gemm_bf16: unknown epilogue");
    }
}

}  // namespace rs

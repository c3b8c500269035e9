// kv_stream_bench.cu -- how fast can one CTA per (sequence, kv head) stream its K/V cache span
// into shared memory? Isolates the memory side of attention_tc.cu at the benchmarked geometry
// (cfg2: 64 sequences x 2 kv heads, 1728 keys of 256 B per span; 14B-8K: 32 x 8, 8256 keys).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/kv_stream_bench tools/kv_stream_bench.cu -lcuda
//   tools/kv_stream_bench items keys depthK depthV mode [delay_cycles]
// mode 0: 2D TMA, two 128 B x 64-row boxes per 16 KB stage (attention_tc.cu today)
// mode 1: 3D TMA, one {64 dims, 64 rows, 2 halves} box per stage (same smem layout)
// mode 2: 1D bulk copy (cp.async.bulk) of the contiguous 16 KB per stage (unswizzled)
// mode 3: plain coalesced 16-byte loads by 256 threads (no smem), the LDG reference
// hog (arg 8): 4 extra warps run alongside the stream: 1 tcgen05.ld loop (TMEM reads), 2 ld.shared
// loop, 3 ex2 loop, 4 tcgen05.st loop, 5 tcgen05.mma SS loop (M128 N64 K16 from smem), 6 tcgen05.mma TS loop,
// 7 SS loop with N=128
// mode 4: mode 0 plus an L2 prefetch (cp.async.bulk.prefetch.L2) of the 16 KB block `pf` passes ahead
//   tools/kv_stream_bench items keys depthK depthV mode delay pf
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e = (x);                                                                       \
        if (e != cudaSuccess) {                                                                    \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                            \
            exit(1);                                                                               \
        }                                                                                          \
    } while (0)

constexpr int kStage = 16384;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                     su32(b)),
                 "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

__global__ void __launch_bounds__(256, 1) tma_stream(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                                                    const uint8_t *gk, const uint8_t *gv, int keys, int max_ctx, int dk,
                                                    int dv, int mode, int delay, int pf, int hog, unsigned long long *sink) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *rk = sm, *rv = sm + dk * kStage;
    uint64_t *bars = (uint64_t *)(rv + dv * kStage);
    uint64_t *fk = bars, *ek = bars + 8, *fv = bars + 16, *ev = bars + 24;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) {
            mb_init(&fk[i], 1);
            mb_init(&ek[i], 1);
            mb_init(&fv[i], 1);
            mb_init(&ev[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __shared__ uint32_t tslot;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int np = keys / 64;
    const int row0 = blockIdx.x * max_ctx;
    if ((warp == 0 || warp == 1) && lane == 0) {
        const bool isK = warp == 0;
        const int depth = isK ? dk : dv;
        uint8_t *ring = isK ? rk : rv;
        uint64_t *full = isK ? fk : fv, *empty = isK ? ek : ev;
        const CUtensorMap *tm = isK ? &tk : &tv;
        const uint8_t *g = isK ? gk : gv;
        for (int j = 0, s = 0, ph = 1; j < np; ++j) {
            mb_wait(&empty[s], ph);
            uint8_t *dst = ring + s * kStage;
            mb_expect(&full[s], kStage);
            const int y = row0 + j * 64;
            if (mode == 4 && j + pf < np) {
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g + (size_t)(y + pf * 64) * 256), "r"(kStage)
                             : "memory");
            }
            if (j == 0 && mode == 4) {
                for (int i = 1; i < pf && i < np; ++i)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g + (size_t)(y + i * 64) * 256), "r"(kStage)
                                 : "memory");
            }
            if (mode == 0 || mode == 4) {
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                                 su32(dst)),
                             "l"(tm), "r"(su32(&full[s])), "r"(0), "r"(y)
                             : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                                 su32(dst + 8192)),
                             "l"(tm), "r"(su32(&full[s])), "r"(64), "r"(y)
                             : "memory");
            } else if (mode == 1) {
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                                 su32(dst)),
                             "l"(tm), "r"(su32(&full[s])), "r"(0), "r"(y), "r"(0)
                             : "memory");
            } else {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                             "l"(g + (size_t)y * 256), "r"(kStage), "r"(su32(&full[s]))
                             : "memory");
            }
            if (++s == depth) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 2 && lane == 0) {
        // consumer: K(j) then V(j), an optional busy delay per pass (the compute)
        unsigned long long acc = 0;
        for (int j = 0; j < np; ++j) {
            mb_wait(&fk[j % dk], (j / dk) & 1);
            acc += rk[(j % dk) * kStage + 64];
            mb_arrive(&ek[j % dk]);
            if (delay) {
                const long long t0 = clock64();
                while (clock64() - t0 < delay) {
                }
            }
            mb_wait(&fv[j % dv], (j / dv) & 1);
            acc += rv[(j % dv) * kStage + 64];
            mb_arrive(&ev[j % dv]);
        }
        if (acc == 12345) sink[0] = acc;
        done = 1;
    } else if (warp == 4 && hog >= 5) {
        // one elected thread keeps the tensor core busy reading shared memory (the last ring stage)
        if (lane == 0) {
            __shared__ __align__(8) uint64_t mmab;
            mb_init(&mmab, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const uint8_t *op = rv + (dv - 1) * kStage;
            auto desc = [](const void *p) {
                uint64_t d = (uint64_t)((su32(p) & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
                return d;
            };
            const uint32_t n = hog == 7 ? 128 : 64;
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
            uint32_t ph = 0;
            while (!done) {
                for (int i = 0; i < 8; ++i) {
                    if (hog == 6)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tslot + 256),
                                     "r"(tslot + 128 + i * 8), "l"(desc(op) + 2 * (i & 3)), "r"(idesc), "r"(i));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tslot + 256),
                                     "l"(desc(op) + 2 * (i & 3)), "l"(desc(op + 8192) + 2 * (i & 3)), "r"(idesc), "r"(i));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mmab)) : "memory");
                mb_wait(&mmab, ph);
                ph ^= 1;
            }
        }
    } else if (warp >= 4 && hog && hog < 5) {
        const uint32_t t = tslot + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t x = lane, acc = 0;
        float f = lane * 0.001f;
        while (!done) {
            if (hog == 1) {
                uint32_t v[32];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                             : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                             : "r"(t + (x & 7) * 32));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 32; ++i) acc += v[i];
            } else if (hog == 2) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    uint32_t a0, a1, a2, a3;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                                 : "r"(su32(rk + ((x * 16 + i * 512) & 8191))));
                    acc += a0 ^ a3;
                }
            } else if (hog == 3) {
#pragma unroll
                for (int i = 0; i < 64; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f));
            } else {
                uint32_t v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = x + i;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                             ::"r"(t + (x & 7) * 32), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            ++x;
        }
        if (acc == 12345 || f == 1.2345f) sink[0] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(512));
}

__global__ void __launch_bounds__(256) ldg_stream(const int4 *gk, const int4 *gv, int keys, int max_ctx,
                                                  unsigned long long *sink) {
    const size_t base = (size_t)blockIdx.x * max_ctx * 16;  // int4 per row: 16
    const int n = keys * 16;
    int acc = 0;
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += 256) {
        const int4 a = __ldcs(gk + base + i), b = __ldcs(gv + base + i);
        acc ^= a.x ^ a.w ^ b.y ^ b.z;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
    const int items = argc > 1 ? atoi(argv[1]) : 128;
    const int keys = argc > 2 ? atoi(argv[2]) : 1728;
    const int dk = argc > 3 ? atoi(argv[3]) : 5;
    const int dv = argc > 4 ? atoi(argv[4]) : 4;
    const int mode = argc > 5 ? atoi(argv[5]) : 0;
    const int delay = argc > 6 ? atoi(argv[6]) : 0;
    const int pf = argc > 7 ? atoi(argv[7]) : 8;
    const int hog = argc > 8 ? atoi(argv[8]) : 0;
    const int max_ctx = keys + 192;
    const size_t bytes = (size_t)items * max_ctx * 256;
    uint8_t *k, *v;
    unsigned long long *sink;
    CK(cudaMalloc(&k, bytes));
    CK(cudaMalloc(&v, bytes));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(k, 1, bytes));
    CK(cudaMemset(v, 2, bytes));
    uint8_t *flush;
    const size_t fbytes = 512ull << 20;
    CK(cudaMalloc(&flush, fbytes));
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    EncodeFn enc = (EncodeFn)p;
    CUtensorMap tk, tv;
    const size_t rows = (size_t)items * max_ctx;
    for (int w = 0; w < 2; ++w) {
        CUtensorMap *m = w ? &tv : &tk;
        void *base = w ? v : k;
        CUresult r;
        if (mode == 1) {
            const cuuint64_t dims[3] = {64, rows, 2};
            const cuuint64_t strides[2] = {256, 128};
            const cuuint32_t box[3] = {64, 64, 2};
            const cuuint32_t es[3] = {1, 1, 1};
            r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            const cuuint64_t dims[2] = {128, rows};
            const cuuint64_t strides[1] = {256};
            const cuuint32_t box[2] = {64, 64};
            const cuuint32_t es[2] = {1, 1};
            r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            return 1;
        }
    }
    const int smem = 1024 + (dk + dv) * kStage + 256;
    CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f, tot = 0;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
        CK(cudaMemsetAsync(flush, r, fbytes));  // evict the spans from L2
        CK(cudaEventRecord(e0));
        if (mode == 3)
            ldg_stream<<<items, 256>>>((const int4 *)k, (const int4 *)v, keys, max_ctx, sink);
        else
            tma_stream<<<items, 256, smem>>>(tk, tv, k, v, keys, max_ctx, dk, dv, mode, delay, pf, hog, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (r >= 2) {
            best = ms < best ? ms : best;
            tot += ms;
        }
    }
    const double moved = 2.0 * items * (double)keys * 256;
    printf("hog %d items %4d keys %5d depth K%d V%d mode %d pf %2d delay %5d: best %8.2f us  mean %8.2f us  %7.1f GB/s (best)\n", hog,
           items, keys, dk, dv, mode, pf, delay, best * 1e3, tot / reps * 1e3, moved / (best * 1e-3) / 1e9);
    return 0;
}

// mma_issue_bench.cu -- issue cost and execution time of back-to-back tcgen05.mma (kind::f16,
// cta_group::1, M = 128) from one thread, by N and operand source (SS: A and B in shared memory,
// TS: A in tensor memory). One CTA; clock64 around the issue loop and until the commit lands.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mma_issue_bench tools/mma_issue_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool TS>
__global__ void bench(int n_mma, uint32_t N, long long *out, int issuers) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(gridDim.x > 1 ? 256 : 512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(issuers));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp >= 1 && warp <= issuers && lane == 0) {
        const uint32_t t = tslot;
        const uint32_t dcol = N > 128 ? 256 : 128;
        auto desc = [](const void *p) {
            return (uint64_t)((su32(p) & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
                   (2ull << 61);
        };
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t da = desc(sm), db = desc(sm + 32768);
        const long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i) {
            if (TS)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(
                                 t + dcol),
                             "r"(t + (i & 7) * 8), "l"(db + 2 * (i & 3)), "r"(idesc), "r"(i & 7));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                                 t + dcol),
                             "l"(da + 2 * (i & 3)), "l"(db + 2 * (i & 3)), "r"(idesc), "r"(i & 7));
        }
        const long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                         su32(&bar))
                     : "memory");
        const long long t2 = clock64();
        if (blockIdx.x == 0 && warp == 1) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(gridDim.x > 1 ? 256 : 512));
}

int main(int argc, char **argv) {
    const int issuers = argc > 1 ? atoi(argv[1]) : 1, ctas = argc > 2 ? atoi(argv[2]) : 1;
    long long *d, h[2];
    cudaMalloc(&d, 16);
    const int smem = 65536 + 1024;  // two CTAs per SM fit
    cudaFuncSetAttribute(bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int ts = 0; ts < 2; ++ts)
        for (uint32_t N : {32u, 64u, 128u, 256u})
            if (ctas == 1 || N <= 128)
            for (int n : {8, 64, 512}) {
                for (int rep = 0; rep < 2; ++rep) {
                    if (ts)
                        bench<true><<<ctas, 128, smem>>>(n, N, d, issuers);
                    else
                        bench<false><<<ctas, 128, smem>>>(n, N, d, issuers);
                    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                }
                const cudaError_t e = cudaGetLastError();
                printf("issuers %d ctas %d %s N=%3u n=%4d: issue %7.1f cyc/mma, complete %7.1f cyc/mma (floor %u) %s\n", issuers, ctas, ts ? "TS" : "SS", N, n,
                       (double)h[0] / n, (double)h[1] / n, 128 * N / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}

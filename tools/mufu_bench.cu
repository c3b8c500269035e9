// mufu_bench.cu -- per-SM throughput of MUFU.EX2, FFMA2 and the packed-pair polynomial exp2
// (the attention softmax's candidate exponentials), one CTA per SM, W warps per CTA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mufu_bench tools/mufu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <int MODE>
__global__ void k(float *out, int iters, float s) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = -(float)(threadIdx.x + i) * 1e-3f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = ex2(a[i]) * s - 1.0f;       // MUFU + FFMA
            else if (MODE == 1) a[i] = fmaf(a[i], s, -1.0f);  // FFMA only
            else {                                            // ex2.approx.f16x2: two results per op
                uint32_t h = __float_as_uint(a[i]), r;
                asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h));
                a[i] = __uint_as_float(r ^ 0x80008000u);
            }
        }
    }
    long long t1 = clock64();
    float acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += a[i];
    if (acc == 12345.f) out[0] = acc;
    if (threadIdx.x == 0) out[1 + blockIdx.x] = (float)(t1 - t0);
}
int main() {
    float *o;
    cudaMalloc(&o, 4096 * 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode = 0; mode < 3; ++mode)
        for (int warps : {4, 8, 16, 32}) {
            const int iters = 4096;
            if (mode == 0) k<0><<<sms, warps * 32>>>(o, iters, 0.5f);
            else if (mode == 1) k<1><<<sms, warps * 32>>>(o, iters, 0.5f);
            else k<2><<<sms, warps * 32>>>(o, iters, 0.5f);
            cudaDeviceSynchronize();
            float cyc;
            cudaMemcpy(&cyc, o + 1, 4, cudaMemcpyDeviceToHost);
            const double ops = (double)warps * 32 * iters * 8;
            printf("mode %s warps/SM %2d: %.2f ops/clk/SM\n", mode == 0 ? "ex2+ffma" : mode == 1 ? "ffma    " : "ex2.f16x2 (ops = pairs)", warps, ops / cyc);
        }
    return 0;
}

// common.cuh -- shared device helpers for the respec_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace rs {

// Error taxonomy mirrors the reference's exception classes (SURVEY.md §8 B "Errors").
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

void note_launch();  // counts kernel launches (rs_launch_count)
void note_copy(bool h2d, size_t bytes);  // host<->device traffic accounting (rs_step_info)
int64_t copy_bytes(bool h2d);
void reset_copy_bytes();

#define RS_CUDA(call)                                                                              \
    do {                                                                                           \
        cudaError_t e__ = (call);                                                                  \
        if (e__ != cudaSuccess)                                                                    \
            throw ::rs::CudaError(std::string(#call) + ": " + cudaGetErrorString(e__) + " @ " +   \
                                  __FILE__ + ":" + std::to_string(__LINE__));                      \
    } while (0)

#define RS_LAUNCHED()                                                                              \
    do {                                                                                           \
        ::rs::note_launch();                                                                       \
        cudaError_t e__ = cudaGetLastError();                                                      \
        if (e__ != cudaSuccess)                                                                    \
            throw ::rs::CudaError(std::string("kernel launch: ") + cudaGetErrorString(e__) +      \
                                  " @ " + __FILE__ + ":" + std::to_string(__LINE__));              \
    } while (0)

// Device-side error codes, surfaced by the host engine as the reference's messages.
enum DevErr : int {
    kErrNone = 0,
    kErrAcceptQ = 1,       // "accept_prob: drafted token must have q > 0"
    kErrAcceptRange = 2,   // "accept_prob: probabilities out of range"
    kErrResidual = 3,      // "residual_dist: degenerate residual (p == q)"
    kErrAllZero = 4,       // "sample_from: all-zero distribution"
    kErrRowIndex = 5,      // "row_index: token out of vocabulary"
    kErrCapacity = 6,      // context exceeds the engine's KV / token capacity
};
const char *dev_err_message(int code);

// Process-wide tuning knobs set through rs_set_tuning (0 = automatic).
struct Tuning {
    int accept_cluster = 0;  // CTAs per sequence in the fused acceptance kernel: 0 auto, 1/2/4/8 forced
    int lazy_lm = 0;         // lazy verify LM head (root rows, then the selected chains): 0 on, -1 off
    int epi3 = 0;            // single-wave SM-pair GEMMs: third epilogue group on the producer / MMA warps: 0 on, -1 off
    int accept_minb = 4;     // acceptance kernel register budget for 256-thread CTAs: resident CTAs per SM (1, 3 or 4)
    int fused_stats = 0;     // drafter LM-head stats: 1 fused GEMM epilogue; 0 / -1 separate row-stats kernel
    int attn_trace = 0;      // diagnostics: layer + 1 whose attention pass timeline is printed
    int attn_skip = 0;       // diagnostics (wrong results): bit 0 softmax math, bit 1 score MMAs, bit 2 P.V MMAs, bit 3 exps, bit 4 S loads
    int pdl = 0;             // programmatic dependent launch on the forward path: 0 / 1 on, -1 off
    int gemm2 = 0;           // weight GEMMs on SM pairs (gemm_2sm.cu): 0 / 1 on, -1 single-SM kernel
    int gemm_trace = 0;      // diagnostics: per-launch timeline of the SM-pair GEMM (CTA 0)
    int kd_rows = 0;         // tests: cap on KD rows per group in rs_engine_kd_grad (0 = workspace size)
};
Tuning &tuning();

#ifdef __CUDACC__
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide reductions; `red` must hold >= 32 doubles of shared memory. All threads get
// the result. Safe to call back-to-back (leading __syncthreads protects `red`).
__device__ __forceinline__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    v = lane < nw ? red[lane] : 0.0;
    return warp_sum(v);
}
__device__ __forceinline__ double block_max(double v, double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    v = lane < nw ? red[lane] : -INFINITY;
    return warp_max(v);
}
// Min / max of an integer key (ties resolved by the caller's encoding).
__device__ __forceinline__ long long block_min_ll(long long v, long long *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    v = lane < nw ? red[lane] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ long long block_max_ll(long long v, long long *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    v = lane < nw ? red[lane] : LLONG_MIN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// Exclusive scan of one double per thread (block-wide). `red` >= 32 doubles.
__device__ __forceinline__ double block_exclusive_scan(double v, double *red, double *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    double x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) red[wid] = x;
    __syncthreads();
    if (wid == 0) {
        double w = lane < nw ? red[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            double y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) red[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const double warp_prefix = wid > 0 ? red[wid - 1] : 0.0;
    if (total) *total = red[nw - 1];
    return warp_prefix + x - v;
}
#endif

}  // namespace rs

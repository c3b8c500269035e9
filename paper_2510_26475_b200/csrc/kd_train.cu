// kd_train.cu -- element-wise and reduction kernels of the whole-drafter KD backward pass
// (kd_update, learner.cpp:62-82 / :146-151: the reference's gradient moves EVERY drafter
// parameter). The contractions of the backward pass -- weight gradients dW = dY^T X, input
// gradients dX = dY W, and the attention backward's S = Q K^T, dP = dO V^T, dV = P^T dO,
// dK = dS^T Q, dQ = dS K -- run on the tcgen05 GEMMs (gemm_2sm.cu); these kernels do the rest:
// RMSNorm / SwiGLU / RoPE backward, the causal softmax backward, column sums for gains and the
// QKV bias, casts, and the fp32 SGD step of the norm gains. Every reduction runs in a fixed
// order, so a gradient is bitwise reproducible (async == sync learner updates).
#include <algorithm>
#include <cuda_bf16.h>

#include "common.cuh"
#include "kd.h"

namespace rs {

using bf16 = __nv_bfloat16;

namespace {

__device__ __forceinline__ float block_sum(float v, float *red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float t = 0.f;
    for (int i = 0; i < nw; ++i) t += red[i];  // fixed order
    return t;
}

// y = x * r * g, r = rsqrt(mean(x^2) + eps):
//   dx = base + r * g * dy - x * r^3 * (sum_k g_k dy_k x_k) / d,   gterm = dy * x * r
__global__ void __launch_bounds__(256) rms_bwd_kernel(const float *x, int ldx, const float *g, const float *dy,
                                                      int lddy, int d, float eps, const float *base, int ldb,
                                                      float *dx, int lddx, float *gterm, int ldg) {
    __shared__ float red[8];
    const int m = blockIdx.x;
    const float *xr = x + (size_t)m * ldx, *dr = dy + (size_t)m * lddy;
    float ss = 0.f, dot = 0.f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const float xv = xr[c];
        ss += xv * xv;
        dot += g[c] * dr[c] * xv;
    }
    ss = block_sum(ss, red);
    dot = block_sum(dot, red);
    const float r = rsqrtf(ss / (float)d + eps);
    const float k = r * r * r * dot / (float)d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const float xv = xr[c], dv = dr[c];
        if (dx) dx[(size_t)m * lddx + c] = (base ? base[(size_t)m * ldb + c] : 0.f) + r * g[c] * dv - xv * k;
        if (gterm) gterm[(size_t)m * ldg + c] = dv * xv * r;
    }
}

// partial[chunk][c] = sum of rows [chunk * rows_per, ...) of column c, in row order
__global__ void colsum_partial_kernel(const float *in, int ld, int M, int C, int rows_per, float *partial) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int chunk = blockIdx.y;
    if (c >= C) return;
    const int r0 = chunk * rows_per, r1 = min(M, r0 + rows_per);
    float s = 0.f;
    for (int r = r0; r < r1; ++r) s += in[(size_t)r * ld + c];
    partial[(size_t)chunk * C + c] = s;
}
__global__ void colsum_final_kernel(const float *partial, int chunks, int C, float *out, int accumulate) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    float s = 0.f;
    for (int k = 0; k < chunks; ++k) s += partial[(size_t)k * C + c];
    out[c] = accumulate ? out[c] + s : s;
}

// gate/up interleaved pairwise (row 2i gate_i, 2i+1 up_i; the model layout):
//   h = silu(g) * u  ->  dg = dh * u * sig * (1 + g (1 - sig)),  du = dh * silu(g)
__global__ void swiglu_bwd_kernel(const bf16 *gu, int ldgu, const float *dh, int lddh, int M, int F, bf16 *dgu,
                                  int lddgu) {
    const size_t n = (size_t)M * F;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int m = (int)(i / F), f = (int)(i % F);
        const __nv_bfloat162 p = *reinterpret_cast<const __nv_bfloat162 *>(gu + (size_t)m * ldgu + 2 * f);
        const float g = __bfloat162float(p.x), u = __bfloat162float(p.y);
        const float sig = 1.f / (1.f + __expf(-g));
        const float d = dh[(size_t)m * lddh + f];
        __nv_bfloat162 o;
        o.x = __float2bfloat16(d * u * sig * (1.f + g * (1.f - sig)));
        o.y = __float2bfloat16(d * g * sig);
        *reinterpret_cast<__nv_bfloat162 *>(dgu + (size_t)m * lddgu + 2 * f) = o;
    }
}

// RoPE backward in place: forward (x1, x2) -> (x1 c - x2 s, x2 c + x1 s) on pairs (i, i + hd/2)
// with the table of model.cu (rope_table_kernel); backward rotates by -angle.
__global__ void rope_bwd_kernel(float *x, int ldx, int heads, int hd, const int *pos, const float *rope) {
    const int m = blockIdx.x, half = hd / 2;
    const float *cs = rope + (size_t)pos[m] * half * 2;
    float *row = x + (size_t)m * ldx;
    for (int idx = threadIdx.x; idx < heads * half; idx += blockDim.x) {
        const int h = idx / half, i = idx % half;
        float *p = row + h * hd;
        const float c = cs[2 * i], s = cs[2 * i + 1];
        const float d1 = p[i], d2 = p[i + half];
        p[i] = d1 * c + d2 * s;
        p[i + half] = d2 * c - d1 * s;
    }
}

// Causal softmax backward of one query row i (keys 0..i of the same sequence):
//   P = softmax(S * scale), D = sum_j P dP, dS = P (dP - D) * scale (w.r.t. the raw scores)
// P and dS are written in bf16 over [0, ldo) with zeros past the row's keys.
// Row i of a stack of query heads, each T causal rows: row i attends keys 0 .. i % T.
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const float *S, const float *dP, int lds, int T, float scale,
                                                          bf16 *P, bf16 *dS, int ldo) {
    __shared__ float red[8];
    const int i = blockIdx.x;
    const float *s = S + (size_t)i * lds, *dp = dP + (size_t)i * lds;
    const int n = i % T + 1;
    float mx = -INFINITY;
    for (int j = threadIdx.x; j < n; j += blockDim.x) mx = fmaxf(mx, s[j] * scale);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    {
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) red[w] = mx;
        __syncthreads();
        mx = -INFINITY;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) mx = fmaxf(mx, red[k]);
    }
    float l = 0.f;
    for (int j = threadIdx.x; j < n; j += blockDim.x) l += __expf(s[j] * scale - mx);
    l = block_sum(l, red);
    const float inv = 1.f / l;
    float dsum = 0.f;
    for (int j = threadIdx.x; j < n; j += blockDim.x) dsum += __expf(s[j] * scale - mx) * inv * dp[j];
    dsum = block_sum(dsum, red);
    bf16 *po = P + (size_t)i * ldo, *dso = dS + (size_t)i * ldo;
    for (int j = threadIdx.x; j < ldo; j += blockDim.x) {
        float p = 0.f, d = 0.f;
        if (j < n) {
            p = __expf(s[j] * scale - mx) * inv;
            d = p * (dp[j] - dsum) * scale;
        }
        po[j] = __float2bfloat16(p);
        dso[j] = __float2bfloat16(d);
    }
}

// out[(k T + t) hd + c] = in[t ldi + k hd + c]: the heads of one GQA group stacked row-wise
// (16-byte vectors; hd % 8 == 0).
__global__ void stack_heads_kernel(const bf16 *in, int ldi, int T, int heads, int hd, bf16 *out) {
    const int v = hd / 8;
    const size_t n = (size_t)heads * T * v;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % v) * 8;
        const size_t r = i / v;
        const int k = (int)(r / T), t = (int)(r % T);
        *reinterpret_cast<int4 *>(out + r * hd + c) =
            *reinterpret_cast<const int4 *>(in + (size_t)t * ldi + (size_t)k * hd + c);
    }
}

// out[t ldo + k hd + c] = in[(k T + t) hd + c] (fp32, the inverse of stack_heads)
__global__ void unstack_heads_kernel(const float *in, int T, int heads, int hd, float *out, int ldo) {
    const int v = hd / 4;
    const size_t n = (size_t)heads * T * v;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % v) * 4;
        const size_t r = i / v;
        const int k = (int)(r / T), t = (int)(r % T);
        *reinterpret_cast<float4 *>(out + (size_t)t * ldo + (size_t)k * hd + c) =
            *reinterpret_cast<const float4 *>(in + r * hd + c);
    }
}

__global__ void cast_bf16_kernel(const float *in, int ldi, int M, int C, bf16 *out, int ldo) {
    const size_t n = (size_t)M * C;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int m = (int)(i / C), c = (int)(i % C);
        out[(size_t)m * ldo + c] = __float2bfloat16(in[(size_t)m * ldi + c]);
    }
}

__global__ void sgd_f32_kernel(const float *w, const float *g, float scale, size_t n, float *out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = __fadd_rn(w[i], __fmul_rn(scale, g[i]));  // no FMA contraction: w + scale * g as written
}

int grid_for(size_t n) { return (int)std::min<size_t>(2368, (n + 255) / 256); }

}  // namespace

void rms_bwd(const float *x, int ldx, const float *g, const float *dy, int lddy, int M, int d, float eps,
             const float *base, int ldb, float *dx, int lddx, float *gterm, int ldg, cudaStream_t st) {
    if (M <= 0) return;
    rms_bwd_kernel<<<M, 256, 0, st>>>(x, ldx, g, dy, lddy, d, eps, base, ldb, dx, lddx, gterm, ldg);
    RS_LAUNCHED();
}

void colsum_f32(const float *in, int ld, int M, int C, float *out, bool accumulate, float *partial, int max_chunks,
                cudaStream_t st) {
    if (C <= 0) return;
    const int chunks = std::max(1, std::min(max_chunks, (M + 63) / 64));
    const int rows_per = (M + chunks - 1) / chunks;
    if (M > 0) {
        colsum_partial_kernel<<<dim3((C + 255) / 256, chunks), 256, 0, st>>>(in, ld, M, C, rows_per, partial);
        RS_LAUNCHED();
    }
    colsum_final_kernel<<<(C + 255) / 256, 256, 0, st>>>(partial, M > 0 ? chunks : 0, C, out, accumulate ? 1 : 0);
    RS_LAUNCHED();
}

void swiglu_bwd(const bf16 *gu, int ldgu, const float *dh, int lddh, int M, int F, bf16 *dgu, int lddgu,
                cudaStream_t st) {
    if (M <= 0) return;
    swiglu_bwd_kernel<<<grid_for((size_t)M * F), 256, 0, st>>>(gu, ldgu, dh, lddh, M, F, dgu, lddgu);
    RS_LAUNCHED();
}

void rope_bwd(float *x, int ldx, int M, int heads, int hd, const int *pos, const float *rope, cudaStream_t st) {
    if (M <= 0) return;
    rope_bwd_kernel<<<M, 256, 0, st>>>(x, ldx, heads, hd, pos, rope);
    RS_LAUNCHED();
}

void softmax_bwd(const float *S, const float *dP, int lds, int rows, int T, float scale, bf16 *P, bf16 *dS, int ldo,
                 cudaStream_t st) {
    if (rows <= 0 || T <= 0) return;
    softmax_bwd_kernel<<<rows, 256, 0, st>>>(S, dP, lds, T, scale, P, dS, ldo);
    RS_LAUNCHED();
}

void stack_heads(const bf16 *in, int ldi, int T, int heads, int hd, bf16 *out, cudaStream_t st) {
    if (T <= 0 || heads <= 0) return;
    stack_heads_kernel<<<grid_for((size_t)heads * T * (hd / 8)), 256, 0, st>>>(in, ldi, T, heads, hd, out);
    RS_LAUNCHED();
}

void unstack_heads(const float *in, int T, int heads, int hd, float *out, int ldo, cudaStream_t st) {
    if (T <= 0 || heads <= 0) return;
    unstack_heads_kernel<<<grid_for((size_t)heads * T * (hd / 4)), 256, 0, st>>>(in, T, heads, hd, out, ldo);
    RS_LAUNCHED();
}

void cast_bf16(const float *in, int ldi, int M, int C, bf16 *out, int ldo, cudaStream_t st) {
    if (M <= 0 || C <= 0) return;
    cast_bf16_kernel<<<grid_for((size_t)M * C), 256, 0, st>>>(in, ldi, M, C, out, ldo);
    RS_LAUNCHED();
}

void sgd_f32(const float *w, const float *g, float scale, size_t n, float *out, cudaStream_t st) {
    if (!n) return;
    sgd_f32_kernel<<<grid_for(n), 256, 0, st>>>(w, g, scale, n, out);
    RS_LAUNCHED();
}

}  // namespace rs

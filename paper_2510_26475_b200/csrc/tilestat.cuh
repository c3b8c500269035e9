// tilestat.cuh -- the ONE definition of a logit tile's softmax partials, shared by the
// full-chip row-stats kernel (rowstats.cu) and the acceptance kernel's on-demand stats
// (sd_kernels.cu), so a row's (max, sum exp) is bitwise the same whichever computes it.
//
// Tile t covers columns [256 t, min(256 t + 256, V - 1)) -- the EOS column V-1 is excluded,
// its bias is request-specific and folded in by the consumer. One warp per tile: lane l owns
// columns 256 t + l + 32 j (j = 0..7); the max is taken on the fp32 logits (exact: the fp64
// image of the fp32 maximum), the sum in fp64 with the same exp() the consumers use, lane
// partials in j order, then the xor-butterfly warp sum.
#pragma once
#include "common.cuh"

namespace rs {

__device__ __forceinline__ void tile_stat(const float *z, int V, int t, double tau, int lane, double &m, double &s) {
    const int lo = t * 256, hi = min(lo + 256, V - 1);
    float v[8];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int x = lo + lane + 32 * j;
        v[j] = x < hi ? z[x] : -INFINITY;
        mx = fmaxf(mx, v[j]);
    }
    mx = warp_maxf(mx);
    m = -INFINITY;
    s = 0.0;
    if (mx != -INFINITY) {
        m = tau == 1.0 ? (double)mx : (double)mx / tau;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (v[j] == -INFINITY) continue;
            const double y = tau == 1.0 ? (double)v[j] : (double)v[j] / tau;
            s += exp(y - m);
        }
        s = warp_sum(s);
    }
}

}  // namespace rs

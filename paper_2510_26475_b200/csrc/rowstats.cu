// rowstats.cu -- exact (fp64) softmax tile partials of logit rows, at full-chip parallelism.
//
// For every selected row and every 256-column tile: m_t = max(z/tau) over the tile (EOS column
// V-1 excluded -- its bias is request-specific and folded in by the consumer) and
// s_t = sum exp(z/tau - m_t) in fp64. One warp per tile: the max is taken on the fp32 logits
// (exact: the fp64 image of the fp32 maximum), the sum in fp64 with the same exp() the
// consumers use. The row's normaliser is then a ~600-term combine and an inverse-CDF draw a
// tile-prefix walk (sd_kernels.cu), instead of full 152K-element fp64 passes on one SM.
#include "common.cuh"
#include "launch.cuh"
#include "prof.h"
#include "sd.h"
#include "tilestat.cuh"

namespace rs {

namespace {

__global__ void __launch_bounds__(256) row_stats_kernel(const float *rows, const int32_t *row_ids, int nrows, int V,
                                                        double tau, double *stats) {
    pdl_trigger();
    pdl_wait();
    const int ntiles = (V + 255) / 256;
    const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= (long long)nrows * ntiles) return;
    const int k = static_cast<int>(gw / ntiles), t = static_cast<int>(gw % ntiles);
    const int row = row_ids ? row_ids[k] : k;
    if (row < 0) return;
    double m, s;
    tile_stat(rows + (size_t)row * V, V, t, tau, lane, m, s);
    if (lane == 0) {
        double *o = stats + ((size_t)row * ntiles + t) * 2;
        o[0] = m;
        o[1] = s;
    }
}

}  // namespace

void row_stats(const float *rows, const int32_t *row_ids, int nrows, int V, double tau, double *stats,
               cudaStream_t st) {
    if (nrows <= 0) return;
    const long long warps = (long long)nrows * ((V + 255) / 256);
    ProfScope prof("rowstats", 0, (double)nrows * V * 4.0, st);
    launch_pdl(row_stats_kernel, (unsigned)((warps + 7) / 8), 256, 0, st, rows, row_ids, nrows, V, tau, stats);
    RS_LAUNCHED();
}

}  // namespace rs

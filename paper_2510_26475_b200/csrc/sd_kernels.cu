// sd_kernels.cu -- model-agnostic speculative-decoding kernels (sm_100a).
//
// K3 "fused softmax + acceptance": one CTA per active sequence walks the reference's
// acceptance algorithm (specdec.cpp:197-267) over the logit rows the model forwards produced.
// All probability arithmetic is fp64 with exactly the reference's formula
// p = exp(z/tau - max) / sum (model.cpp:53-68); only summation ORDER differs (ulp-level, a
// token can flip only if a uniform lands within ~1e-16 of a CDF boundary).
//
// Softmax statistics are hierarchical. Rows produced by the LM-head GEMM arrive with
// per-256-column tile partials (max, sum exp) computed in the GEMM epilogue, so a row's
// normaliser costs ~600 fp64 terms instead of a 152K-element pass, and an inverse-CDF draw
// (model.cpp:23-40) is a warp prefix over tile masses followed by a warp scan inside the one
// tile that brackets the uniform. Residual distributions max(0, p - q) / Z (specdec.cpp:35-52)
// need one CTA-wide pass that yields Z and the tile masses together. Rows without GEMM
// statistics (the fp64 tabular parity path) compute the same quantities in-kernel.
//
// The drafting sampler draws each chain's tokens with the request's own draft stream at the
// offsets the reference's sequential loop would use (specdec.cpp:177-192); chains are drafted
// level-synchronously and an EOS-shortened chain triggers a redraft pass with corrected
// offsets (sd_redraft_check), so the stream order is preserved exactly.
#include <cfloat>
#include <climits>

#include <cooperative_groups.h>

#include "common.cuh"
#include "prof.h"
#include "launch.cuh"
#include "sd.h"
#include "tilestat.cuh"

namespace rs {

namespace {

constexpr int kTileW = 256;     // = the LM-head GEMM's BLOCK_N
constexpr int kMaxTiles = 2048; // V <= 524288
constexpr int kMaxCand = 16;
constexpr int kMaxCluster = 8;

namespace cg = cooperative_groups;

// A sequence's acceptance runs on a thread-block CLUSTER of `size` CTAs (1 when the batch
// alone fills the chip). Every CTA walks the same control flow on the same data; the only
// split work is the full-vocabulary passes (residual tile sums, argmax, full-row records),
// whose tile partials are exchanged through distributed shared memory. Tile t is always
// summed by one warp in the same lane order, so results are bitwise independent of `size`.
struct Cl {
    unsigned rank, size;
    __device__ __forceinline__ bool lead() const { return rank == 0 && threadIdx.x == 0; }
};
__device__ __forceinline__ void cl_sync(const Cl &cl) {
    if (cl.size > 1) cg::this_cluster().sync();
    else __syncthreads();
}
// Combine one (value, key) pair per CTA across the cluster: max value, then min key.
__device__ void cl_maxkey(const Cl &cl, double &best, long long &key, double *slot_v, long long *slot_k) {
    if (cl.size == 1) return;
    if (threadIdx.x == 0) {
        *slot_v = best;
        *slot_k = key;
    }
    cl_sync(cl);
    auto cluster = cg::this_cluster();
    double b = -INFINITY;
    long long k = LLONG_MAX;
    for (unsigned r = 0; r < cl.size; ++r) {
        const double v = *cluster.map_shared_rank(slot_v, r);
        const long long kk = *cluster.map_shared_rank(slot_k, r);
        if (v > b || (v == b && kk < k)) {
            b = v;
            k = kk;
        }
    }
    best = b;
    key = k;
    cl_sync(cl);
}

template <class T>
struct RowRef {
    const T *z;
    int V;
    double bias;
    double tau;
    const double *gst;  // GEMM tile partials (max, sum) of z/tau excluding column V-1, or null
    // z'/tau with the EOS bias added to the last logit before the temperature division
    // (model.cpp:137-138, :58-61); tau == 1 skips the (exact anyway) division.
    __device__ __forceinline__ double v(int x) const {
        double y = static_cast<double>(__ldg(z + x));  // rows are read-only here: loads may run ahead of stores
        if (x == V - 1) y += bias;
        return tau == 1.0 ? y : y / tau;
    }
};

struct Stats {
    double m, S, inv;  // inv = 1 / S (multiply instead of a per-element fp64 divide)
};

__device__ __forceinline__ int ntiles_of(int V) { return (V + kTileW - 1) / kTileW; }
__device__ __forceinline__ int tile_lo(int t) { return t * kTileW; }
__device__ __forceinline__ int tile_hi(int t, int V) { return min((t + 1) * kTileW, V - 1); }  // EOS excluded

template <class T>
__device__ Stats row_stats(const RowRef<T> &r, double *red) {
    if (r.gst) {
        const int nt = ntiles_of(r.V);
        double m = -INFINITY;
        for (int t = threadIdx.x; t < nt; t += blockDim.x) m = fmax(m, __ldcg(r.gst + 2 * t));
        const double ve = r.v(r.V - 1);
        m = fmax(block_max(m, red), ve);
        double s = 0.0;
        for (int t = threadIdx.x; t < nt; t += blockDim.x) {
            const double st = __ldcg(r.gst + 2 * t + 1);
            if (st > 0.0) s += st * exp(__ldcg(r.gst + 2 * t) - m);
        }
        s = block_sum(s, red) + exp(ve - m);
        return {m, s, 1.0 / s};
    }
    double m = -INFINITY;
    for (int x = threadIdx.x; x < r.V; x += blockDim.x) m = fmax(m, r.v(x));
    m = block_max(m, red);
    double s = 0.0;
    for (int x = threadIdx.x; x < r.V; x += blockDim.x) s += exp(r.v(x) - m);
    s = block_sum(s, red);
    return {m, s, 1.0 / s};
}

template <class T>
__device__ __forceinline__ double prob(const RowRef<T> &r, const Stats &s, int x) {
    return exp(r.v(x) - s.m) * s.inv;
}

// L1 prefetch of a logit element's line: issued a tile-pair ahead in the full-vocabulary passes
// so the loads of the next tiles are in flight while this pair's fp64 exps run (the passes are
// otherwise bound by load latency -- long-scoreboard stalls on the fp32 -> fp64 converts).
__device__ __forceinline__ void pf_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
struct NoPrefetch {
    __device__ __forceinline__ void operator()(int) const {}
};

template <class T>
struct ProbFn {
    RowRef<T> r;
    Stats s;
    __device__ __forceinline__ double operator()(int x) const { return prob(r, s, x); }
    __device__ __forceinline__ void pf(int x) const { pf_l1(r.z + x); }
};

// p_cur after k sibling rejections: r_j = max(0, r_{j-1} - q1) / Z_j (specdec.cpp:209 -> :35-52)
template <class T>
struct PCurFn {
    RowRef<T> p;
    Stats sp;
    RowRef<T> q;
    Stats sq;
    const double *Z;
    int k;
    __device__ __forceinline__ double operator()(int x) const {
        double r = prob(p, sp, x);
        if (k > 0) {
            const double qq = prob(q, sq, x);
            for (int j = 0; j < k; ++j) r = fmax(0.0, r - qq) * Z[j];  // Z holds 1 / Z_j
        }
        return r;
    }
    __device__ __forceinline__ void pf(int x) const {
        pf_l1(p.z + x);
        if (k > 0) pf_l1(q.z + x);
    }
};

// Contiguous tile range of cluster rank c: [c * nt / C, (c + 1) * nt / C).
__device__ __forceinline__ int cl_tile0(const Cl &cl, unsigned c, int nt) { return (int)((long)c * nt / cl.size); }
__device__ __forceinline__ unsigned cl_owner(const Cl &cl, int t, int nt) {
    unsigned c = 0;
    while (c + 1 < cl.size && cl_tile0(cl, c + 1, nt) <= t) ++c;
    return c;
}

// Warm L2 with this CTA's share of a logit row (TMA bulk prefetch, 16 B granules).
__device__ __forceinline__ void l2_prefetch_share(const void *row, size_t bytes, const Cl &cl) {
    if (threadIdx.x >= 32 || bytes < 65536 || (reinterpret_cast<uintptr_t>(row) & 15)) return;
    const size_t per = ((bytes + cl.size - 1) / cl.size + 15) & ~size_t(15);
    const size_t b0 = per * cl.rank;
    if (b0 >= bytes) return;
    const size_t n = (bytes - b0 < per ? bytes - b0 : per) & ~size_t(15);
    const char *p = static_cast<const char *>(row) + b0;
    constexpr size_t kChunk = 32768;
    for (size_t off = (size_t)threadIdx.x * kChunk; off < n; off += 32 * kChunk) {
        const uint32_t len = (uint32_t)(n - off < kChunk ? n - off : kChunk);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(len) : "memory");
    }
}

// Gather the other ranks' tile values into every CTA's `mass`, then the total.
__device__ double gather_masses(int nt, double *mass, double *red, const Cl &cl) {
    if (cl.size > 1) __threadfence();  // tile functors may have written global scratch read by peers
    cl_sync(cl);
    if (cl.size > 1) {
        auto cluster = cg::this_cluster();
        for (int t = threadIdx.x; t <= nt; t += blockDim.x) {
            const unsigned own = t == nt ? 0u : cl_owner(cl, t, nt);
            if (own != cl.rank) mass[t] = *cluster.map_shared_rank(mass + t, own);
        }
        cl_sync(cl);  // peers have read our tiles before anyone overwrites `mass` again
    }
    double s = 0.0;
    for (int t = threadIdx.x; t <= nt; t += blockDim.x) s += mass[t];
    return block_sum(s, red);
}

// Per-tile sums of f over the tile partition (tiles over [0, V-1) plus the EOS pseudo-tile at
// index nt) into `mass`; returns the total. One warp per tile, lane l summing columns
// l + 32 j in j order, then the warp butterfly -- whichever warp / CTA owns the tile. Each CTA
// of the cluster takes a contiguous tile range; a warp handles two tiles per iteration with
// all 16 column values fetched before any is summed (memory-level parallelism).
template <class F, class P>
__device__ double tile_sums(const F &f, const P &pf, int V, double *mass, double *red, const Cl &cl) {
    const int nt = ntiles_of(V);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int t0 = cl_tile0(cl, cl.rank, nt), t1 = cl_tile0(cl, cl.rank + 1, nt);
    auto touch = [&](int tt) {
        if (tt >= t1) return;
        const int hi = tile_hi(tt, V);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int x = tile_lo(tt) + lane + 32 * j;
            if (x < hi) pf(x);
        }
    };
    touch(t0 + w);
    touch(t0 + w + nw);
    for (int t = t0 + w; t < t1; t += 2 * nw) {
        const int u = t + nw;
        touch(t + 2 * nw);
        touch(u + 2 * nw);
        const int hi = tile_hi(t, V), hu = u < t1 ? tile_hi(u, V) : 0;
        double va[8], vb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int x = tile_lo(t) + lane + 32 * j;
            va[j] = x < hi ? f(x) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int x = tile_lo(u) + lane + 32 * j;
            vb[j] = x < hu ? f(x) : 0.0;
        }
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            sa += va[j];
            sb += vb[j];
        }
        sa = warp_sum(sa);
        sb = warp_sum(sb);
        if (lane == 0) {
            mass[t] = sa;
            if (u < t1) mass[u] = sb;
        }
    }
    if (cl.rank == 0 && threadIdx.x == 0) mass[nt] = f(V - 1);
    return gather_masses(nt, mass, red, cl);
}
template <class F>
__device__ __forceinline__ double tile_sums(const F &f, int V, double *mass, double *red, const Cl &cl) {
    return tile_sums(f, NoPrefetch{}, V, mass, red, cl);
}

// Tile masses of a probability row straight from the GEMM partials.
template <class T>
__device__ void gemm_masses(const RowRef<T> &r, const Stats &st, double *mass) {
    const int nt = ntiles_of(r.V);
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        const double s = __ldcg(r.gst + 2 * t + 1);
        mass[t] = s > 0.0 ? s * exp(__ldcg(r.gst + 2 * t) - st.m) * st.inv : 0.0;
    }
    if (threadIdx.x == 0) mass[nt] = exp(r.v(r.V - 1) - st.m) * st.inv;
    __syncthreads();
}

struct CdfScratch {
    int cand_t[kMaxCand];
    double cand_c[kMaxCand];
    int ncand;
    int result;
};

// Inverse-CDF draw (model.cpp:23-40): first x with u < cum(x); on rounding slack the last x
// with nonzero mass. masses[t] * scale = mass of tile t; the tile whose cumulative range
// brackets u (within 1e-10) is rescanned element by element by warp 0.
template <class F>
__device__ int inv_cdf(const F &f, int V, const double *mass, double scale, double u, CdfScratch &cs,
                       long long *redl, int *err) {
    const int nt = ntiles_of(V);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        cs.ncand = 0;
        cs.result = -1;
    }
    __syncthreads();
    if (w == 0) {
        const int per = (nt + 1 + 31) / 32;
        const int t0 = min(lane * per, nt + 1), t1 = min(t0 + per, nt + 1);
        double ls = 0.0;
        for (int t = t0; t < t1; ++t) ls += mass[t] * scale;
        double incl = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        double c = incl - ls;
        for (int t = t0; t < t1; ++t) {
            const double wt = mass[t] * scale;
            if (u >= c - 1e-10 && u < c + wt + 1e-10) {
                const int k = atomicAdd(&cs.ncand, 1);
                if (k < kMaxCand) {
                    cs.cand_t[k] = t;
                    cs.cand_c[k] = c;
                }
            }
            c += wt;
        }
        __syncwarp();
        const int nc = min(cs.ncand, kMaxCand);
        if (lane == 0) {  // candidates in increasing tile order
            for (int i = 1; i < nc; ++i)
                for (int j = i; j > 0 && cs.cand_t[j - 1] > cs.cand_t[j]; --j) {
                    const int tt = cs.cand_t[j];
                    cs.cand_t[j] = cs.cand_t[j - 1];
                    cs.cand_t[j - 1] = tt;
                    const double cc = cs.cand_c[j];
                    cs.cand_c[j] = cs.cand_c[j - 1];
                    cs.cand_c[j - 1] = cc;
                }
        }
        __syncwarp();
        int found = -1;  // warp-uniform
        for (int k = 0; k < nc && found < 0; ++k) {
            const int t = cs.cand_t[k];
            const double c0 = cs.cand_c[k];
            if (t == nt) {  // EOS pseudo-tile
                if (u < c0 + f(V - 1)) found = V - 1;
            } else {
                const int lo = tile_lo(t) + lane * 8, hi = tile_hi(t, V);
                double vals[8];
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    vals[k] = lo + k < hi ? f(lo + k) : 0.0;
                    s += vals[k];
                }
                double in2 = s;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, in2, o);
                    if (lane >= o) in2 += y;
                }
                double cum = c0 + (in2 - s);
                int mine = -1;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (lo + k >= hi) break;
                    cum += vals[k];
                    if (mine < 0 && u < cum) mine = lo + k;
                }
                const unsigned b = __ballot_sync(0xffffffffu, mine >= 0);
                if (b) found = __shfl_sync(0xffffffffu, mine, __ffs(b) - 1);
            }
        }
        if (lane == 0) cs.result = found;
    }
    __syncthreads();
    int res = cs.result;
    if (res >= 0 && res < V) return res;
    // rounding slack at the top of the CDF: the last token with nonzero mass
    long long last = -1;
    for (int x = V - 1 - (int)threadIdx.x; x >= 0 && last < 0; x -= blockDim.x)
        if (f(x) > 0.0) last = x;
    last = block_max_ll(last, redl);
    if (last < 0) {
        if (threadIdx.x == 0) atomicCAS(err, 0, kErrAllZero);
        return 0;
    }
    return static_cast<int>(last);
}

// Argmax of p with lowest-index tie break. For fp32 rows p is strictly monotone in the logit
// (distinct fp32 logits give distinct fp64 probabilities), so the GEMM tile maxima locate
// the winner; fp64 rows (tabular parity path) compare the probabilities themselves.
template <class T>
__device__ int row_argmax(const RowRef<T> &r, const Stats &st, double *red, long long *redl, const int *excl,
                          int n_excl, const Cl &cl, double *slot_v, long long *slot_k) {
    double best = -1.0;
    int bi = INT_MAX;
    for (int x = cl.rank * blockDim.x + threadIdx.x; x < r.V; x += cl.size * blockDim.x) {
        bool skip = false;
        for (int e = 0; e < n_excl; ++e) skip |= excl[e] == x;
        if (skip) continue;
        const double p = sizeof(T) == 4 ? r.v(x) : prob(r, st, x);
        if (p > best || bi == INT_MAX) {
            best = p;
            bi = x;
        }
    }
    double m = block_max(bi == INT_MAX ? -INFINITY : best, red);
    long long key = (bi != INT_MAX && best == m) ? bi : LLONG_MAX;
    key = block_min_ll(key, redl);
    cl_maxkey(cl, m, key, slot_v, slot_k);
    return static_cast<int>(key);
}

struct Seq {
    int r;  // request id
    int a;  // active slot
    int len;
    int plen;
    int maxlen;
    double bias;
};

__device__ __forceinline__ double u_of(const MtStream &ms, int k) { return to_unit_double(ms.out[ms.pos + k]); }

// Append one emitted token with its StepRecord (specdec.cpp:62-74, :276-283).
template <class T>
__device__ void emit(const SdDev &d, Seq &q, int tok, const RowRef<T> &row, const Stats &st, bool drafted,
                     double logq, bool &ended, const Cl &cl) {
    const int gen = q.len - q.plen;
    if (cl.lead()) {
        if (q.len < d.tok_cap && gen < d.steps_cap) {
            d.tok[(size_t)q.r * d.tok_cap + q.len] = tok;
            const size_t si = (size_t)q.r * d.steps_cap + gen;
            d.st_tok[si] = tok;
            d.st_logp[si] = log(prob(row, st, tok));
            d.st_drafted[si] = drafted ? 1 : 0;
            d.st_logq[si] = drafted ? logq : 0.0;
        } else {
            atomicCAS(d.err, 0, kErrCapacity);
        }
    }
    if (d.st_full && gen < d.steps_cap) {
        double *dst = d.st_full + ((size_t)q.r * d.steps_cap + gen) * d.V;
        for (int x = cl.rank * blockDim.x + threadIdx.x; x < d.V; x += cl.size * blockDim.x)
            dst[x] = log(prob(row, st, x));
    }
    q.len += 1;
    if (tok == d.eos) ended = true;
}

template <class T>
__device__ __forceinline__ RowRef<T> prow(const SdDev &d, const Seq &q, int slot) {
    const size_t row = (size_t)q.a * d.slots + slot;
    return RowRef<T>{static_cast<const T *>(d.P) + row * d.V, d.V, q.bias, d.tau_p,
                     d.Pst ? d.Pst + row * d.ntiles * 2 : nullptr};
}
template <class T>
__device__ __forceinline__ RowRef<T> qrow(const SdDev &d, const Seq &q, int slot) {
    const size_t row = (size_t)q.a * d.slots + slot;
    return RowRef<T>{static_cast<const T *>(d.Q) + row * d.V, d.V, q.bias, d.tau_q,
                     d.Qst ? d.Qst + row * d.ntiles * 2 : nullptr};
}

// Target rows without precomputed statistics (SdDev::lazy_pst): the acceptance kernel fills a
// row's tile partials the first time it touches the row -- typically 2-3 of the 1 + t*n
// verified rows per sequence -- split over the cluster's warps, with the same tile_stat the
// full-chip row-stats kernel uses.
template <class T>
__device__ RowRef<T> prow_ready(const SdDev &d, const Seq &q, int slot, const Cl &cl) {
    RowRef<T> r = prow<T>(d, q, slot);
    if constexpr (sizeof(T) == 4) {
        if (d.lazy_pst && r.gst) {
            double *g = const_cast<double *>(r.gst);
            const int nt = ntiles_of(r.V), lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            const int t1 = cl_tile0(cl, cl.rank + 1, nt);
            const float *zf = reinterpret_cast<const float *>(r.z);
            auto touch = [&](int tt) {
                if (tt >= t1) return;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (tile_lo(tt) + lane + 32 * j < tile_hi(tt, r.V)) pf_l1(zf + tile_lo(tt) + lane + 32 * j);
            };
            for (int t = cl_tile0(cl, cl.rank, nt) + (threadIdx.x >> 5); t < t1; t += nw) {
                touch(t + nw);
                double m, s;
                tile_stat(reinterpret_cast<const float *>(r.z), r.V, t, r.tau, lane, m, s);
                if (lane == 0) {
                    g[2 * t] = m;
                    g[2 * t + 1] = s;
                }
            }
            __threadfence();
            cl_sync(cl);
        }
    }
    return r;
}

// Draw from a plain probability row (masses from the GEMM partials when present).
template <class T>
__device__ int sample_row(const RowRef<T> &r, const Stats &st, double u, double *mass, CdfScratch &cs, double *red,
                          long long *redl, int *err, const Cl &cl) {
    const ProbFn<T> f{r, st};
    if (r.gst) {
        gemm_masses(r, st, mass);
        return inv_cdf(f, r.V, mass, 1.0, u, cs, redl, err);
    }
    tile_sums(f, [&](int x) { f.pf(x); }, r.V, mass, red, cl);
    return inv_cdf(f, r.V, mass, 1.0, u, cs, redl, err);
}

__global__ void cycle_begin_kernel(SdDev d) {
    pdl_trigger();
    pdl_wait();
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= d.nact) return;
    const int r = d.active[a];
    d.d_used[r] = 0;
    d.a_used[r] = 0;
    d.cont[r] = 1;
    d.ended[r] = 0;
    d.accept_len[r] = 0;
    d.drafted[r] = 0;
    d.emitted[r] = 0;
    d.n_rounds[r] = 0;
}

// specdec.cpp:165-171: remaining = max_emit - |accepted|; < 2 -> no drafting this round.
__global__ void round_setup_kernel(SdDev d, int round) {
    pdl_trigger();
    pdl_wait();
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= d.nact) return;
    const int r = d.active[a];
    int ne = -1;
    if (d.cont[r]) {
        const int gen = d.len[r] - d.prompt_len[r];
        const int rem = d.max_len[r] - gen;
        ne = rem < 2 ? (round == 0 ? 0 : -1) : min(d.n, rem - 1);
    }
    d.n_eff[r] = ne;
    d.rsel[r] = -1;
    d.racc[r] = 0;
    for (int i = 0; i < d.t; ++i) {
        const size_t ci = (size_t)r * d.t_max + i;
        d.chain_len[ci] = 0;
        d.chain_stop[ci] = 0;
        d.chain_off[ci] = d.d_used[r] + i * max(ne, 0);  // provisional: no EOS truncation
    }
}

template <class T>
__global__ void __launch_bounds__(512) draft_sample_kernel(SdDev d, int depth) {
    pdl_trigger();
    pdl_wait();
    __shared__ double red[32];
    __shared__ long long redl[32];
    __shared__ int picked[kMaxBranch];
    __shared__ double mass[kMaxTiles + 1];
    __shared__ CdfScratch cs;
    __shared__ double slot_v;
    __shared__ long long slot_k;
    const Cl cl{0u, 1u};
    const int a = blockIdx.x;
    const int r = d.active[a];
    const int ne = d.n_eff[r];
    if (depth >= ne) return;  // also covers ne <= 0
    Seq q{r, a, d.len[r], d.prompt_len[r], d.max_len[r], d.eos_bias[r]};
    const MtStream &D = d.rng[2 * r];
    const bool greedy = d.verify_mode == 1;
    if (depth == 0) {
        if (d.chain_len[(size_t)r * d.t_max] != 0) return;  // already drafted (redraft pass)
        const RowRef<T> row = qrow<T>(d, q, 0);
        const Stats st = row_stats(row, red);
        if (!greedy) {
            if (row.gst) gemm_masses(row, st, mass);
            else {
                const ProbFn<T> pfn{row, st};
                tile_sums(pfn, [&](int x) { pfn.pf(x); }, row.V, mass, red, cl);
            }
        }
        for (int i = 0; i < d.t; ++i) {
            int c;
            if (greedy) {
                c = row_argmax(row, st, red, redl, picked, i, cl, &slot_v, &slot_k);
            } else {
                const double u = u_of(D, d.chain_off[(size_t)r * d.t_max + i]);
                c = inv_cdf(ProbFn<T>{row, st}, d.V, mass, 1.0, u, cs, redl, d.err);
            }
            if (threadIdx.x == 0) {
                picked[i] = c;
                const size_t ci = (size_t)r * d.t_max + i;
                d.chain_tok[ci * d.n_max + 0] = c;
                d.chain_len[ci] = 1;
                d.chain_stop[ci] = c == d.eos;
            }
            __syncthreads();
        }
        return;
    }
    const int i = blockIdx.y;
    const size_t ci = (size_t)r * d.t_max + i;
    if (d.chain_stop[ci] || d.chain_len[ci] != depth) return;
    const RowRef<T> row = qrow<T>(d, q, 1 + i * d.n + depth);
    const Stats st = row_stats(row, red);
    int c;
    if (greedy) c = row_argmax(row, st, red, redl, picked, 0, cl, &slot_v, &slot_k);
    else c = sample_row(row, st, u_of(D, d.chain_off[ci] + depth), mass, cs, red, redl, d.err, cl);
    if (threadIdx.x == 0) {
        d.chain_tok[ci * d.n_max + depth] = c;
        d.chain_len[ci] = depth + 1;
        d.chain_stop[ci] = c == d.eos;
    }
}

// Offsets must equal the reference's sequential consumption: chain i starts after the
// draws of chains 0..i-1 (specdec.cpp:177-192). Any mismatch -> fix + request a redraft.
__global__ void redraft_check_kernel(SdDev d) {
    pdl_trigger();
    pdl_wait();
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= d.nact) return;
    const int r = d.active[a];
    if (d.n_eff[r] <= 0 || d.verify_mode == 1) return;
    int off = d.d_used[r];
    bool bad = false;
    for (int i = 0; i < d.t; ++i) {
        const size_t ci = (size_t)r * d.t_max + i;
        if (d.chain_off[ci] != off) bad = true;
        off += d.chain_len[ci];
    }
    if (!bad) return;
    off = d.d_used[r];
    for (int i = 0; i < d.t; ++i) {
        const size_t ci = (size_t)r * d.t_max + i;
        const int li = d.chain_len[ci];
        d.chain_off[ci] = off;
        off += li;
        d.chain_len[ci] = 0;
        d.chain_stop[ci] = 0;
    }
    atomicExch(d.flag, 1);
}

// MB = minimum resident CTAs per SM the register budget is sized for: 1 (up to 512 threads) or,
// for the 256-thread clusters of large vocabularies, 3 / 4 (a wave holds more sequences' clusters)
template <class T, int MB>
__global__ void __launch_bounds__(MB == 1 ? 512 : 256, MB) accept_kernel(SdDev d, int round, int naive, int stage) {
    pdl_trigger();
    pdl_wait();
    // an EOS-shortened chain shifted the draft-stream offsets of later chains: this optimistic
    // pass is void (no state change); the host redrafts with the corrected offsets and reruns
    if (*d.flag) return;
    __shared__ double red[32];
    __shared__ long long redl[32];
    __shared__ double Z[kMaxBranch];
    __shared__ double mass[kMaxTiles + 1];
    __shared__ CdfScratch cs;
    __shared__ double slot_v;
    __shared__ long long slot_k;
    const Cl cl{cg::this_cluster().block_rank(), cg::this_cluster().num_blocks()};
    const int a = blockIdx.x / cl.size;
    const int r = d.active[a];
    Seq q{r, a, d.len[r], d.prompt_len[r], d.max_len[r], d.eos_bias[r]};
    const bool greedy = d.verify_mode == 1;
    const MtStream &A = d.rng[2 * r + 1];
    const MtStream &D = d.rng[2 * r];
    bool ended = false;
    int emitted = 0;

    // stage 0: the whole acceptance; 1 / 2: split around the LM head of the selected chains (lazy
    // verify LM head): stage 1 runs the branch point on the root rows and, when a chain is
    // selected, parks (sel, acur, alen, alen0, emitted, len) in d.stg; stage 2 verifies that chain
    if (naive && stage == 2) return;
    if (naive) {
        // Non-spec step (server.cpp:328-347): one target sample on the DRAFT stream.
        const RowRef<T> p = prow_ready<T>(d, q, 0, cl);
        const Stats sp = row_stats(p, red);
        int x;
        if (greedy) x = row_argmax(p, sp, red, redl, nullptr, 0, cl, &slot_v, &slot_k);
        else x = sample_row(p, sp, u_of(D, d.d_used[r]), mass, cs, red, redl, d.err, cl);
        emit(d, q, x, p, sp, false, 0.0, ended, cl);
        if (cl.lead()) {
            if (!greedy) d.d_used[r] += 1;
            d.len[r] = q.len;
            d.emitted[r] += 1;
            d.ended[r] = ended;
            d.cont[r] = 0;
        }
        return;
    }

    const int ne = d.n_eff[r];
    if (ne < 0) return;
    if (stage == 2 && d.stg[(size_t)r * 6] < 0) return;  // the cycle ended in stage 1
    if (stage == 1 && cl.lead()) d.stg[(size_t)r * 6] = -1;
    int acur = d.a_used[r];
    int alen = d.accept_len[r];
    int alen0 = alen;
    int sel_out = -1;
    int cont = 0;
    const int t = d.t, n = d.n;
    const int *ctok = d.chain_tok + (size_t)r * d.t_max * d.n_max;
    const int *clen = d.chain_len + (size_t)r * d.t_max;

    if (ne == 0) {
        // max_emit == 1: no round runs, the single token is the bonus from the target on the
        // ACCEPT stream (specdec.cpp:256-266; SURVEY App. A "Engine != generate()").
        const RowRef<T> p = prow_ready<T>(d, q, 0, cl);
        const Stats sp = row_stats(p, red);
        const int x = greedy ? row_argmax(p, sp, red, redl, nullptr, 0, cl, &slot_v, &slot_k)
                             : sample_row(p, sp, u_of(A, acur++), mass, cs, red, redl, d.err, cl);
        emit(d, q, x, p, sp, false, 0.0, ended, cl);
        ++emitted;
        if (cl.lead()) {
            int *rc = d.round_cost + ((size_t)r * kMaxRounds + 0) * 3;
            rc[0] = 0;
            rc[1] = 0;
            rc[2] = 1;
            d.n_rounds[r] = 1;
        }
        goto done;
    }

    {
      int sel = -1;
      if (stage == 2) {
        const int32_t *sv = d.stg + (size_t)r * 6;
        sel = sv[0];
        acur = sv[1];
        alen = sv[2];
        alen0 = sv[3];
        emitted = sv[4];
        q.len = sv[5];
      } else {
        // RoundCost{longest, t, tree_tokens + 1} (specdec.cpp:195)
        int longest = 0, tree = 0;
        for (int i = 0; i < t; ++i) {
            longest = max(longest, clen[i]);
            tree += clen[i];
        }
        if (cl.lead()) {
            int *rc = d.round_cost + ((size_t)r * kMaxRounds + round) * 3;
            rc[0] = longest;
            rc[1] = t;
            rc[2] = tree + 1;
            d.n_rounds[r] = round + 1;
            d.drafted[r] = 1;
            d.d_used[r] += tree;
        }

        {
            const size_t rb = (size_t)d.V * sizeof(T);
            l2_prefetch_share(prow<T>(d, q, 0).z, rb, cl);
            l2_prefetch_share(qrow<T>(d, q, 0).z, rb, cl);
        }
        const RowRef<T> p1 = prow_ready<T>(d, q, 0, cl);
        const RowRef<T> q1 = qrow<T>(d, q, 0);
        const Stats s1 = row_stats(p1, red);
        const Stats t1 = row_stats(q1, red);
        if (greedy) {
            const int a1 = row_argmax(p1, s1, red, redl, nullptr, 0, cl, &slot_v, &slot_k);
            for (int i = 0; i < t && sel < 0; ++i)
                if (ctok[(size_t)i * d.n_max] == a1) sel = i;
            if (sel < 0) {
                emit(d, q, a1, p1, s1, false, 0.0, ended, cl);
                ++emitted;
                goto done;
            }
        } else {
            // Branch point: recursive rejection over the t siblings (specdec.cpp:197-217).
            int k = 0;
            double zlast = 1.0;
            double *cache = d.pq_cache && t > 1 ? d.pq_cache + (size_t)a * 2 * d.V : nullptr;
            for (int i = 0; i < t; ++i) {
                const int cand = ctok[(size_t)i * d.n_max];
                PCurFn<T> pc{p1, s1, q1, t1, Z, k};
                const double pv = pc(cand), qv = prob(q1, t1, cand);
                const double acc = fmin(1.0, pv / qv);
                if (u_of(A, acur++) < acc) {
                    sel = i;
                    break;
                }
                // residual normaliser and its tile masses in one pass
                // The first residual pass caches p1(x), q1(x) in fp64 (the same bits prob()
                // returns); later sibling passes stream them instead of redoing two fp64 exps.
                // With the cache, cache[x] holds p_k(x) -- the residual after k rejections,
                // memoised pass by pass: one step of the recursion per pass instead of k, the
                // same operations in the same order as the loop (so the same bits).
                auto res_k = [&](int x) {
                    double rr, qq;
                    if (k == 0 || !cache) {
                        rr = prob(p1, s1, x);
                        qq = prob(q1, t1, x);
                        if (cache) {
                            cache[x] = rr;
                            cache[d.V + x] = qq;
                        } else {
                            for (int j = 0; j < k; ++j) rr = fmax(0.0, rr - qq) * Z[j];
                        }
                    } else {
                        qq = __ldcg(cache + d.V + x);
                        rr = fmax(0.0, __ldcg(cache + x) - qq) * Z[k - 1];
                        cache[x] = rr;
                    }
                    return fmax(0.0, rr - qq);
                };
                auto res_pf = [&](int x) {
                    if (k == 0 || !cache) {
                        pf_l1(p1.z + x);
                        pf_l1(q1.z + x);
                    }
                };
                const double z = tile_sums(res_k, res_pf, d.V, mass, red, cl);
                if (z <= 1e-12 && cl.lead()) atomicCAS(d.err, 0, kErrResidual);
                if (threadIdx.x == 0) Z[k] = 1.0 / z;
                __syncthreads();
                zlast = z;
                ++k;
            }
            if (sel < 0) {
                // all siblings rejected: draw from the final residual (masses of the last pass / Z_k)
                const PCurFn<T> fk{p1, s1, q1, t1, Z, k};
                const int x = inv_cdf(fk, d.V, mass, 1.0 / zlast, u_of(A, acur++), cs, redl, d.err);
                emit(d, q, x, p1, s1, false, 0.0, ended, cl);  // StepRecord keeps p1 (specdec.cpp:214)
                ++emitted;
                goto done;
            }
        }
        emit(d, q, ctok[(size_t)sel * d.n_max], p1, s1, true, log(prob(q1, t1, ctok[(size_t)sel * d.n_max])), ended, cl);
        ++emitted;
        ++alen;
        sel_out = sel;
        if (ended) goto done;
        if (stage == 1) {
            if (cl.lead()) {
                int32_t *sv = d.stg + (size_t)r * 6;
                sv[0] = sel;
                sv[1] = acur;
                sv[2] = alen;
                sv[3] = alen0;
                sv[4] = emitted;
                sv[5] = q.len;
            }
            return;
        }
      }
        sel_out = sel;
        const int *chain = ctok + (size_t)sel * d.n_max;
        const int L = clen[sel];
        // Chain-style verification of the selected chain (specdec.cpp:226-245).
        for (int pos = 1; pos < L; ++pos) {
            {  // this position's pair and the next target row (next position or bonus)
                const size_t rb = (size_t)d.V * sizeof(T);
                if (pos == 1) {
                    l2_prefetch_share(prow<T>(d, q, 1 + sel * n).z, rb, cl);
                    l2_prefetch_share(qrow<T>(d, q, 1 + sel * n + 1).z, rb, cl);
                }
                l2_prefetch_share(prow<T>(d, q, 1 + sel * n + pos).z, rb, cl);
                if (pos + 1 < L) l2_prefetch_share(qrow<T>(d, q, 1 + sel * n + pos + 1).z, rb, cl);
            }
            const RowRef<T> pd = prow_ready<T>(d, q, 1 + sel * n + pos - 1, cl);
            const RowRef<T> qd = qrow<T>(d, q, 1 + sel * n + pos);
            const Stats sp = row_stats(pd, red);
            const Stats sq = row_stats(qd, red);
            const int dt = chain[pos];
            bool ok;
            int repl = -1;
            const double qv = prob(qd, sq, dt);
            if (greedy) {
                repl = row_argmax(pd, sp, red, redl, nullptr, 0, cl, &slot_v, &slot_k);
                ok = dt == repl;
            } else {
                const double pv = prob(pd, sp, dt);
                if (!(qv > 0.0) && threadIdx.x == 0) atomicCAS(d.err, 0, kErrAcceptQ);
                if ((pv < 0.0 || pv > 1.0 || qv > 1.0) && threadIdx.x == 0) atomicCAS(d.err, 0, kErrAcceptRange);
                ok = u_of(A, acur++) < fmin(1.0, pv / qv);
            }
            if (ok) {
                emit(d, q, dt, pd, sp, true, log(qv), ended, cl);
                ++emitted;
                ++alen;
                if (ended) goto done;
            } else {
                int x = repl;
                if (!greedy) {
                    auto res = [&](int y) { return fmax(0.0, prob(pd, sp, y) - prob(qd, sq, y)); };
                    const double z = tile_sums(res, [&](int y) { pf_l1(pd.z + y); pf_l1(qd.z + y); }, d.V, mass, red, cl);
                    if (z <= 1e-12 && cl.lead()) atomicCAS(d.err, 0, kErrResidual);
                    const double zi = 1.0 / z;
                    auto rn = [&](int y) { return fmax(0.0, prob(pd, sp, y) - prob(qd, sq, y)) * zi; };
                    x = inv_cdf(rn, d.V, mass, 1.0 / z, u_of(A, acur++), cs, redl, d.err);
                }
                emit(d, q, x, pd, sp, false, 0.0, ended, cl);
                ++emitted;
                goto done;
            }
        }
        // Full acceptance: next round, or the bonus from the target (specdec.cpp:165-169, :256-267).
        const int rem_after = q.maxlen - (q.len - q.plen);
        if (round + 1 < d.s && rem_after >= 2) {
            cont = 1;
        } else {
            const RowRef<T> pb = prow_ready<T>(d, q, 1 + sel * n + L - 1, cl);
            const Stats sb = row_stats(pb, red);
            const int x = greedy ? row_argmax(pb, sb, red, redl, nullptr, 0, cl, &slot_v, &slot_k)
                                 : sample_row(pb, sb, u_of(A, acur++), mass, cs, red, redl, d.err, cl);
            emit(d, q, x, pb, sb, false, 0.0, ended, cl);
            ++emitted;
        }
    }
done:
    if (cl.lead()) {
        d.len[r] = q.len;
        d.a_used[r] = acur;
        d.accept_len[r] = alen;
        d.emitted[r] += emitted;
        d.ended[r] = ended;
        d.cont[r] = cont && !ended;
        d.rsel[r] = sel_out;
        d.racc[r] = alen - alen0;
    }
}

__global__ void cycle_end_kernel(SdDev d, int naive) {
    pdl_trigger();
    pdl_wait();
    if (*d.flag) return;  // void optimistic pass (see accept_kernel)
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= d.nact) return;
    const int r = d.active[a];
    const int gen = d.len[r] - d.prompt_len[r];
    const int done = d.ended[r] || gen >= d.max_len[r];
    d.done[r] = done;
    d.rng[2 * r].pos += d.d_used[r];
    d.rng[2 * r + 1].pos += d.a_used[r];
    int *s = d.summary + (size_t)a * (kSummaryFixed + 3 * kMaxRounds);
    s[0] = done;
    s[1] = d.emitted[r];
    s[2] = naive ? 0 : d.accept_len[r];
    s[3] = naive ? 0 : d.drafted[r];
    s[4] = naive ? 0 : d.n_rounds[r];
    s[5] = d.len[r];
    if (!naive)
        for (int k = 0; k < 3 * d.n_rounds[r]; ++k) s[kSummaryFixed + k] = d.round_cost[(size_t)r * kMaxRounds * 3 + k];
    if (d.newtok) {
        const int e = min(d.emitted[r], d.newtok_cap), l = d.len[r];
        for (int k = 0; k < e; ++k) d.newtok[(size_t)a * d.newtok_cap + k] = d.tok[(size_t)r * d.tok_cap + l - e + k];
    }
}

// ---- tabular model rows ------------------------------------------------------------------
// row index from the last `order` tokens of tok[r][0..len) ++ ext[0..e) (model.cpp:113-130)
__device__ long long tab_row_index(const SdDev &d, const TabDev &m, int r, int len, const int *ext, int e) {
    long long idx = 0;
    for (int i = 0; i < m.order; ++i) {
        const int p = len + e - (m.order - i);
        int tok = 0;
        if (p >= 0) tok = p < len ? d.tok[(size_t)r * d.tok_cap + p] : ext[p - len];
        if (tok < 0 || tok >= m.V) return -1;
        idx = idx * m.V + tok;
    }
    return idx;
}

__global__ void tab_rows_kernel(SdDev d, TabDev m, int depth, int verify, int naive) {
    pdl_trigger();
    pdl_wait();
    // blockIdx.x = active slot, blockIdx.y = tree slot
    const int a = blockIdx.x, slot = blockIdx.y;
    const int r = d.active[a];
    const int ne = naive ? 0 : d.n_eff[r];
    if (!naive && ne < 0) return;
    const int len = d.len[r];
    const int *ext = nullptr;
    int e = 0;
    double *dst;
    if (verify) {
        if (slot > 0) {
            const int i = (slot - 1) / d.n, j = (slot - 1) % d.n;
            if (i >= d.t || j >= d.chain_len[(size_t)r * d.t_max + i]) return;
            ext = d.chain_tok + ((size_t)r * d.t_max + i) * d.n_max;
            e = j + 1;
        }
        dst = const_cast<double *>(static_cast<const double *>(d.P)) + ((size_t)a * d.slots + slot) * d.V;
    } else {
        if (depth >= ne) return;
        if (depth == 0) {
            if (slot != 0) return;
        } else {
            const int i = slot;
            if (i >= d.t) return;
            const size_t ci = (size_t)r * d.t_max + i;
            if (d.chain_stop[ci] || d.chain_len[ci] != depth) return;
            ext = d.chain_tok + ci * d.n_max;
            e = depth;
        }
        const int qslot = depth == 0 ? 0 : 1 + slot * d.n + depth;
        dst = const_cast<double *>(static_cast<const double *>(d.Q)) + ((size_t)a * d.slots + qslot) * d.V;
    }
    const long long row = tab_row_index(d, m, r, len, ext, e);
    if (row < 0) {
        if (threadIdx.x == 0) atomicCAS(d.err, 0, kErrRowIndex);
        return;
    }
    const double *src = m.table + row * m.V;
    for (int x = threadIdx.x; x < m.V; x += blockDim.x) dst[x] = src[x];
}

inline int sd_threads(int V, bool) { return V <= 256 ? 32 : V <= 4096 ? 256 : 512; }

}  // namespace

void sd_cycle_begin(const SdDev &d, cudaStream_t st) {
    if (d.nact <= 0) return;
    launch_pdl(cycle_begin_kernel, (d.nact + 127) / 128, 128, 0, st, d);
    RS_LAUNCHED();
}

void sd_round_setup(const SdDev &d, int round, cudaStream_t st) {
    if (d.nact <= 0) return;
    launch_pdl(round_setup_kernel, (d.nact + 127) / 128, 128, 0, st, d, round);
    RS_LAUNCHED();
}

void sd_draft_sample(const SdDev &d, int depth, RowType rt, cudaStream_t st) {
    if (d.nact <= 0) return;
    if ((d.V + kTileW - 1) / kTileW > kMaxTiles) throw std::invalid_argument("vocabulary too large for the sampler");
    dim3 grid(d.nact, depth == 0 ? 1 : d.t);
    const int th = std::min(512, sd_threads(d.V, d.Qst != nullptr));
    const double es = rt == RowType::F64 ? 8.0 : 4.0;
    ProfScope prof("sample", 0, (double)d.nact * (depth == 0 ? 1 : d.t) * d.V * es, st);
    if (rt == RowType::F64) launch_pdl(draft_sample_kernel<double>, grid, th, 0, st, d, depth);
    else launch_pdl(draft_sample_kernel<float>, grid, th, 0, st, d, depth);
    RS_LAUNCHED();
}

void sd_redraft_check(const SdDev &d, cudaStream_t st) {
    if (d.nact <= 0) return;
    launch_pdl(redraft_check_kernel, (d.nact + 127) / 128, 128, 0, st, d);
    RS_LAUNCHED();
}

void sd_accept(const SdDev &d, int round, bool naive, RowType rt, cudaStream_t st, int stage) {
    if (d.nact <= 0) return;
    const int th = sd_threads(d.V, false);
    // algorithmic bytes: every target row of the round plus every drafter row
    const double es = rt == RowType::F64 ? 8.0 : 4.0;
    ProfScope prof("accept", 0, (double)d.nact * (naive ? 1 : 2 * d.slots - 1) * d.V * es, st);
    // Register budget: 256-thread CTAs compiled for 4 resident per SM (64 registers, some spills)
    // -- measured at cfg2 (batch 64, V = 152K): 0.569 ms vs 0.657 at 2 per SM (128 registers) and
    // 0.625 at 3: a wave holds every sequence's cluster. Results are bitwise the same.
    // Large vocabularies: a cluster of up to 8 CTAs per sequence -- the residual passes are fp64 /
    // load-latency bound, so more CTAs in flight win even past one resident wave. Measured (cfg2,
    // V = 152K): batch 32 / 64 -> 8 CTAs (0.39 / 0.62 ms vs 0.57 / 0.68 at 4); batch 256 -> 4
    // (2.25 ms vs 2.39 at 2, 2.88 at 1). Results are bitwise independent of the cluster size.
    unsigned C = 1;
    int threads = th;
    if (d.V > 4096) {
        threads = 256;
        static const int sms = [] {  // of the current device, queried once (hot path)
            int dev = 0, v = 148;
            RS_CUDA(cudaGetDevice(&dev));
            RS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
            return v;
        }();
        while (C < kMaxCluster && (long)d.nact * C * 2 <= 8L * sms) C *= 2;
    }
    if (tuning().accept_cluster > 0) {
        C = static_cast<unsigned>(tuning().accept_cluster);
        threads = std::min(th, 256);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(d.nact * C);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = tuning().pdl >= 0 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const int nv = naive ? 1 : 0;
    const int mb = threads == 256 ? tuning().accept_minb : 1;
    if (rt == RowType::F64) {
        if (mb == 4) RS_CUDA(cudaLaunchKernelEx(&cfg, accept_kernel<double, 4>, d, round, nv, stage));
        else if (mb == 3) RS_CUDA(cudaLaunchKernelEx(&cfg, accept_kernel<double, 3>, d, round, nv, stage));
        else RS_CUDA(cudaLaunchKernelEx(&cfg, accept_kernel<double, 1>, d, round, nv, stage));
    } else {
        if (mb == 4) RS_CUDA(cudaLaunchKernelEx(&cfg, accept_kernel<float, 4>, d, round, nv, stage));
        else if (mb == 3) RS_CUDA(cudaLaunchKernelEx(&cfg, accept_kernel<float, 3>, d, round, nv, stage));
        else RS_CUDA(cudaLaunchKernelEx(&cfg, accept_kernel<float, 1>, d, round, nv, stage));
    }
    RS_LAUNCHED();
}

void sd_cycle_end(const SdDev &d, bool naive, cudaStream_t st) {
    if (d.nact <= 0) return;
    launch_pdl(cycle_end_kernel, (d.nact + 127) / 128, 128, 0, st, d, naive ? 1 : 0);
    RS_LAUNCHED();
}

void tab_draft_rows(const SdDev &d, const TabDev &m, int depth, cudaStream_t st) {
    if (d.nact <= 0) return;
    dim3 grid(d.nact, depth == 0 ? 1 : d.t);
    launch_pdl(tab_rows_kernel, grid, 32, 0, st, d, m, depth, 0, 0);
    RS_LAUNCHED();
}

void tab_verify_rows(const SdDev &d, const TabDev &m, bool naive, cudaStream_t st) {
    if (d.nact <= 0) return;
    dim3 grid(d.nact, naive ? 1 : d.slots);
    launch_pdl(tab_rows_kernel, grid, 32, 0, st, d, m, 0, 1, naive ? 1 : 0);
    RS_LAUNCHED();
}

}  // namespace rs

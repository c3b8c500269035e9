// kd.cu -- K5: reward-weighted KL distillation loss + analytic gradient (learner.cpp:33-82).
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <stdexcept>

#include "common.cuh"
#include "kd.h"
#include "prof.h"

namespace rs {

using bf16 = __nv_bfloat16;

double kd_weight(double r, const std::vector<double> &br, const rs_kd_policy &p) {
    switch (p.mode) {
        case 1: return 1.0;  // Uniform
        case 2: throw std::logic_error("kd_weight: frozen drafter takes no updates");
        case 0: break;
        default: throw std::invalid_argument("kd_weight: unknown weight mode");
    }
    if (br.empty()) throw std::invalid_argument("kd_weight: empty batch");
    const double mean = std::accumulate(br.begin(), br.end(), 0.0) / static_cast<double>(br.size());
    const double w = r / std::max(1e-6, mean);
    return std::clamp(w, p.clip_lo, p.clip_hi);
}

namespace {

struct Job {
    int seq_off;   // offset of the sample's token sequence (prompt + response)
    int ctx_len;   // context length for this position
    int lp_off;    // row offset (in units of V) into the target logprob rows
    int sample;    // selected-sample index
    double bias;
};

// Per position: drafter row stats (max, sum) and sum_x p(x) (lp(x) - log q(x)) (learner.cpp:33-54).
__global__ void __launch_bounds__(1024, 1) kd_job_kernel(const double *table, int order, int V, double tau, const int *tokens, const Job *jobs,
                              const double *lp, double *job_m, double *job_s, double *job_kl, long long *job_row) {
    __shared__ double red[32];
    const Job jb = jobs[blockIdx.x];
    long long row = 0;
    for (int i = 0; i < order; ++i) {  // row_index, model.cpp:113-130
        const int p = jb.ctx_len - (order - i);
        const int tok = p >= 0 ? tokens[jb.seq_off + p] : 0;
        row = row * V + tok;
    }
    const double *z = table + row * V;
    auto zv = [&](int x) { double y = z[x]; if (x == V - 1) y += jb.bias; return y / tau; };
    double m = -INFINITY;
    for (int x = threadIdx.x; x < V; x += blockDim.x) m = fmax(m, zv(x));
    m = block_max(m, red);
    double s = 0.0;
    for (int x = threadIdx.x; x < V; x += blockDim.x) s += exp(zv(x) - m);
    s = block_sum(s, red);
    double kl = 0.0;
    const double *l = lp ? lp + (size_t)jb.lp_off * V : nullptr;
    for (int x = threadIdx.x; l && x < V; x += blockDim.x) {
        if (isinf(l[x])) continue;  // p = 0 contributes nothing
        const double logq = log(exp(zv(x) - m) / s);
        kl += exp(l[x]) * (l[x] - logq);
    }
    kl = block_sum(kl, red);
    if (threadIdx.x == 0) {
        job_m[blockIdx.x] = m;
        job_s[blockIdx.x] = s;
        job_kl[blockIdx.x] = kl;
        job_row[blockIdx.x] = row;
    }
}

// One block per touched table row: grad(x) = sum over that row's jobs, in the reference's
// order (sample, then position), of w * (q(x) - p(x)) / tau; new = old + grad * (-lr)
// (learner.cpp:62-82, :146-151, model.cpp:161-170).
__global__ void __launch_bounds__(1024, 1) kd_row_kernel(const double *table, double *out, int V, double tau, const Job *jobs,
                              const int *row_jobs, const int *row_ptr, const long long *rows, const double *lp,
                              const double *job_m, const double *job_s, const double *w, double neg_lr,
                              int grad_only, const int *tokens) {
    const long long row = rows[blockIdx.x];
    const double inv_tau = 1.0 / tau;
    for (int x = threadIdx.x; x < V; x += blockDim.x) {
        double g = 0.0;
        for (int k = row_ptr[blockIdx.x]; k < row_ptr[blockIdx.x + 1]; ++k) {
            const int j = row_jobs[k];
            const Job jb = jobs[j];
            double y = table[row * V + x];
            if (x == V - 1) y += jb.bias;
            const double q = exp(y / tau - job_m[j]) / job_s[j];
            if (tokens) {  // policy gradient: A * (onehot(y_t) - pi) / tau, in rl.cpp:66-72's order
                g -= w[jb.sample] * q * inv_tau;
                if (x == tokens[jb.seq_off + jb.ctx_len]) g += w[jb.sample] * inv_tau;
                continue;
            }
            const double l = lp[(size_t)jb.lp_off * V + x];
            const double p = isinf(l) ? 0.0 : exp(l);
            g += w[jb.sample] * (q - p) * inv_tau;
        }
        out[row * V + x] = grad_only ? g : table[row * V + x] + g * neg_lr;
    }
}

// K5 for transformer-sized rows.
__global__ void __launch_bounds__(1024, 1) kd_rows_kernel(const float *trow, const float *drow, const double *w, const double *bias, int V,
                               double tau_p, double tau_q, double *loss, float *dz) {
    __shared__ double red[32];
    const int i = blockIdx.x;
    const float *zt = trow + (size_t)i * V;
    const float *zd = drow + (size_t)i * V;
    const double b = bias ? bias[i] : 0.0;
    auto vt = [&](int x) { double y = zt[x]; if (x == V - 1) y += b; return y / tau_p; };
    auto vd = [&](int x) { double y = zd[x]; if (x == V - 1) y += b; return y / tau_q; };
    double mt = -INFINITY, md = -INFINITY;
    for (int x = threadIdx.x; x < V; x += blockDim.x) {
        mt = fmax(mt, vt(x));
        md = fmax(md, vd(x));
    }
    mt = block_max(mt, red);
    md = block_max(md, red);
    double st = 0.0, sd = 0.0;
    for (int x = threadIdx.x; x < V; x += blockDim.x) {
        st += exp(vt(x) - mt);
        sd += exp(vd(x) - md);
    }
    st = block_sum(st, red);
    sd = block_sum(sd, red);
    const double lst = log(st), lsd = log(sd);
    const double wi = w[i];
    double kl = 0.0;
    for (int x = threadIdx.x; x < V; x += blockDim.x) {
        const double lp = vt(x) - mt - lst, lq = vd(x) - md - lsd;
        const double p = exp(lp), q = exp(lq);
        if (p > 0.0) kl += p * (lp - lq);
        dz[(size_t)i * V + x] = static_cast<float>(wi * (q - p) / tau_q);
    }
    kl = block_sum(kl, red);
    if (threadIdx.x == 0) loss[i] = wi * kl;
}

// ---- K5 at full-chip parallelism (transformer KD) ------------------------------------------
// Softmax tile partials of the target (P) and drafter (Q) rows in one pass: per row and 256-column
// tile (EOS column V-1 excluded, kd_lse_kernel folds it in with the row's bias) m = max(z / tau)
// and s = sum exp(z / tau - m). Same layout as row_stats (rowstats.cu), but the exponentials run in
// fp32: KD's p~ and q only feed a bf16 dZ and a fp64-accumulated loss, so the fp64 exp that the
// acceptance path needs for bitwise parity would only make this pass fp64-pipe bound.
__global__ void __launch_bounds__(256) kd_tile_stats_kernel(const float *P, const float *Q, int R, int V, float inv_p,
                                                            float inv_q, double *stP, double *stQ) {
    const int nt = (V + 255) / 256;
    const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= (long long)R * nt) return;
    const int r = static_cast<int>(gw / nt), t = static_cast<int>(gw % nt);
    const int lo = t * 256, hi = min(lo + 256, V - 1);
    const float *zp = P + (size_t)r * V, *zq = Q + (size_t)r * V;
    float vp[8], vq[8], mp = -INFINITY, mq = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int x = lo + lane + 32 * j;
        vp[j] = x < hi ? zp[x] * inv_p : -INFINITY;
        vq[j] = x < hi ? zq[x] * inv_q : -INFINITY;
        mp = fmaxf(mp, vp[j]);
        mq = fmaxf(mq, vq[j]);
    }
    mp = warp_maxf(mp);
    mq = warp_maxf(mq);
    float sp = 0.f, sq = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (vp[j] != -INFINITY) sp += expf(vp[j] - mp);
        if (vq[j] != -INFINITY) sq += expf(vq[j] - mq);
    }
    const double Sp = warp_sum((double)sp), Sq = warp_sum((double)sq);
    if (lane == 0) {
        double *op = stP + ((size_t)r * nt + t) * 2, *oq = stQ + ((size_t)r * nt + t) * 2;
        op[0] = mp == -INFINITY ? -INFINITY : (double)mp;
        op[1] = mp == -INFINITY ? 0.0 : Sp;
        oq[0] = mq == -INFINITY ? -INFINITY : (double)mq;
        oq[1] = mq == -INFINITY ? 0.0 : Sq;
    }
}

// Row log-normaliser log sum_x exp(z'/tau) of fp32 logit rows from their 256-column tile
// partials (rowstats.cu; EOS column excluded) plus the EOS column with the row's bias.
__global__ void kd_lse_kernel(const float *rows, const double *st, int nrows, int V, double tau, const double *bias,
                              double *lse) {
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= nrows) return;
    const int nt = (V + 255) / 256;
    const double *s = st + (size_t)r * nt * 2;
    const double ve = ((double)rows[(size_t)r * V + V - 1] + bias[r]) / tau;
    double m = ve;
    for (int t = lane; t < nt; t += 32) m = fmax(m, s[2 * t]);
    m = warp_max(m);
    double S = 0.0;
    for (int t = lane; t < nt; t += 32)
        if (s[2 * t + 1] > 0.0) S += s[2 * t + 1] * exp(s[2 * t] - m);
    S = warp_sum(S) + exp(ve - m);
    if (lane == 0) lse[r] = m + log(S);
}

// Per element of a 64-row x 256-column tile: p~ = softmax(target / tau_p), q = softmax(drafter /
// tau_q) (EOS bias on both, model.cpp:137-138), KL term p~ (log p~ - log q) (p~ > 0 only,
// learner.cpp:44-50) and dZ = w (q - p~) / tau_q (learner.cpp:75) times the LM-head output
// scale -- written TRANSPOSED ([V][ldt] bf16) so it is the K-major A operand of the
// dW = dZ^T . h GEMM. One warp per row, lane l on columns l + 32 j; KL partials per (row, tile).
// UnitTau (tau_p == tau_q == 1, the KD default): the three fp64 divisions per element are
// skipped -- x / 1.0 == x exactly, so the outputs are bitwise those of the general path.
template <bool UnitTau>
__global__ void __launch_bounds__(256, 4) kd_elem_kernel(const float *P, const float *Q, const double *lseP,
                                                      const double *lseQ, const double *w, const double *bias, int R,
                                                      int V, double tau_p, double tau_q, float zscale, bf16 *dzT,
                                                      int ldt, double *kl_part) {
    __shared__ __align__(16) bf16 tile[64][256 + 8];
    const int t = blockIdx.x, r0 = blockIdx.y * 64;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = gridDim.x;
    for (int rr = warp; rr < 64; rr += 8) {
        const int r = r0 + rr;
        double kl = 0.0;
        if (r < R) {
            const float *zp = P + (size_t)r * V, *zq = Q + (size_t)r * V;
            const double b = bias[r], lp0 = lseP[r], lq0 = lseQ[r], wr = w[r];
            float fp[8], fq[8];  // all 16 loads of the row issued before any math
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int x = t * 256 + lane + 32 * j;
                fp[j] = x < V ? __ldcs(zp + x) : 0.f;
                fq[j] = x < V ? __ldcs(zq + x) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = lane + 32 * j, x = t * 256 + c;
                float dz = 0.f;
                if (x < V) {
                    double vp = fp[j], vq = fq[j];
                    if (x == V - 1) {
                        vp += b;
                        vq += b;
                    }
                    const double lp = (UnitTau ? vp : vp / tau_p) - lp0, lq = (UnitTau ? vq : vq / tau_q) - lq0;
                    // fp32 exponentials: dZ is rounded to bf16 for the GEMM (rel. 4e-3) and a KL
                    // term's relative error stays ~1e-7, so fp64 exp bought nothing here but
                    // made the kernel fp64-pipe bound (0.5 ms vs ~0.12 ms of HBM per 487 rows)
                    const float p = expf((float)lp), q = expf((float)lq);
                    if (p > 0.f) kl += (double)p * (lp - lq);
                    const float g = (float)wr * (q - p);
                    dz = (UnitTau ? g : g / (float)tau_q) * zscale;
                }
                tile[rr][c] = __float2bfloat16(dz);
            }
        } else {
            for (int j = 0; j < 8; ++j) tile[rr][lane + 32 * j] = __float2bfloat16(0.f);
        }
        kl = warp_sum(kl);
        if (lane == 0 && r < R) kl_part[(size_t)r * nt + t] = kl;
    }
    __syncthreads();
    // transposed store: column c of the tile -> dzT[x][r0 .. r0 + 63] (128 contiguous bytes)
    const int c = threadIdx.x, x = t * 256 + c;
    if (x < V && r0 + 64 <= ldt) {
        bf16 *dst = dzT + (size_t)x * ldt + r0;
#pragma unroll
        for (int k = 0; k < 64; k += 8) {
            __align__(16) bf16 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = tile[k + i][c];
            *reinterpret_cast<int4 *>(dst + k) = *reinterpret_cast<const int4 *>(v);
        }
    }
}

// loss_r = w_r * sum_t kl_part[r][t] (fixed order: lane-strided partials, warp butterfly)
__global__ void kd_rowloss_kernel(const double *kl_part, int R, int nt, const double *w, double *loss) {
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= R) return;
    double s = 0.0;
    for (int t = lane; t < nt; t += 32) s += kl_part[(size_t)r * nt + t];
    s = warp_sum(s);
    if (lane == 0) loss[r] = w[r] * s;
}

// out[c][r] = in[r][c] for r < R, 0 for R <= r < ldo (bf16, 32 x 32 tiles)
__global__ void transpose_pad_kernel(const bf16 *in, int ldi, int R, int C, bf16 *out, int ldo) {
    __shared__ bf16 t[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int r = r0 + k, c = c0 + tx;
        t[k][tx] = (r < R && c < C) ? in[(size_t)r * ldi + c] : __float2bfloat16(0.f);
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int c = c0 + k, r = r0 + tx;
        if (c < C && r < ldo) out[(size_t)c * ldo + r] = t[tx][k];
    }
}

// w_new = bf16(w + scale * g)
__global__ void sgd_bf16_kernel(const bf16 *w, const float *g, float scale, size_t n, bf16 *out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = __float2bfloat16(__bfloat162float(w[i]) + scale * g[i]);
}

}  // namespace

void kd_tile_stats(const float *P, const float *Q, int R, int V, double tau_p, double tau_q, double *stP, double *stQ,
                   cudaStream_t st) {
    if (R <= 0) return;
    const long long warps = (long long)R * ((V + 255) / 256);
    kd_tile_stats_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(P, Q, R, V, (float)(1.0 / tau_p),
                                                                      (float)(1.0 / tau_q), stP, stQ);
    RS_LAUNCHED();
}

void kd_rows_lse(const float *rows, const double *stats, int nrows, int V, double tau, const double *bias, double *lse,
                 cudaStream_t st) {
    if (nrows <= 0) return;
    kd_lse_kernel<<<(nrows + 7) / 8, 256, 0, st>>>(rows, stats, nrows, V, tau, bias, lse);
    RS_LAUNCHED();
}

void kd_rows_elem(const float *P, const float *Q, const double *lseP, const double *lseQ, const double *w,
                  const double *bias, int R, int V, double tau_p, double tau_q, float zscale, bf16 *dzT, int ldt,
                  double *kl_part, double *loss, cudaStream_t st) {
    if (R <= 0) return;
    const int nt = (V + 255) / 256;
    ProfScope prof("kd", 0, (double)R * V * (4.0 + 4.0 + 2.0), st);
    auto kern = tau_p == 1.0 && tau_q == 1.0 ? kd_elem_kernel<true> : kd_elem_kernel<false>;
    kern<<<dim3(nt, (R + 63) / 64), 256, 0, st>>>(P, Q, lseP, lseQ, w, bias, R, V, tau_p, tau_q, zscale, dzT, ldt,
                                                  kl_part);
    RS_LAUNCHED();
    kd_rowloss_kernel<<<(R + 7) / 8, 256, 0, st>>>(kl_part, R, nt, w, loss);
    RS_LAUNCHED();
}

void transpose_pad_bf16(const bf16 *in, int ldi, int R, int C, bf16 *out, int ldo, cudaStream_t st) {
    if (C <= 0 || ldo <= 0) return;
    transpose_pad_kernel<<<dim3((C + 31) / 32, (ldo + 31) / 32), 256, 0, st>>>(in, ldi, R, C, out, ldo);
    RS_LAUNCHED();
}

void sgd_bf16(const bf16 *w, const float *g, float scale, size_t n, bf16 *out, cudaStream_t st) {
    if (!n) return;
    sgd_bf16_kernel<<<1184, 256, 0, st>>>(w, g, scale, n, out);
    RS_LAUNCHED();
}

void kd_rows_loss_grad(const float *target_rows, const float *drafter_rows, const double *weights,
                       const double *eos_bias, int rows, int V, double tau_p, double tau_q, double *loss_out,
                       float *dz_out, cudaStream_t st) {
    if (rows <= 0) return;
    kd_rows_kernel<<<rows, V <= 4096 ? 256 : 1024, 0, st>>>(target_rows, drafter_rows, weights, eos_bias, V, tau_p,
                                                             tau_q, loss_out, dz_out);
    RS_LAUNCHED();
}

std::vector<int> kd_select(int n, int interval, uint64_t *sel_state) {
    // learner.cpp:107-121: partial Fisher-Yates with selection_rng() % (n - i)
    if (interval < 1) throw std::invalid_argument("kd_update: interval must be >= 1");
    HostMt rng;
    std::copy(sel_state, sel_state + kMtN, rng.mt);
    rng.idx = static_cast<int>(sel_state[kMtN]);
    const size_t N = static_cast<size_t>(std::max(n, 0));
    const size_t take = (N + static_cast<size_t>(interval) - 1) / static_cast<size_t>(interval);
    std::vector<size_t> idx(N);
    std::iota(idx.begin(), idx.end(), size_t{0});
    for (size_t i = 0; i < take; ++i) {
        const size_t j = i + static_cast<size_t>(rng.next() % (N - i));
        std::swap(idx[i], idx[j]);
    }
    std::copy(rng.mt, rng.mt + kMtN, sel_state);
    sel_state[kMtN] = static_cast<uint64_t>(rng.idx);
    return std::vector<int>(idx.begin(), idx.begin() + static_cast<long>(take));
}

// Device K5 over the given (sample, weight) list: per-row gradient accumulated in the list's
// order (learner.cpp:62-82). grad_only: out = grad (rows untouched by any sample = 0);
// else out = table + grad * scale (the SGD step, model.cpp:161-170). Returns sum_i w_i KL_i.
double kd_core(rs_ctx *ctx, const TabularModel *drafter, const std::vector<const rs_kd_sample *> &sel,
               const std::vector<double> &w, double *out_dev, bool grad_only, double scale, bool policy) {
    const int V = drafter->vocab;
    cudaStream_t st = ctx->stream;
    std::vector<int32_t> tokens;
    std::vector<double> lp;
    std::vector<Job> jobs;
    std::vector<std::vector<int>> per_sample(sel.size());
    for (size_t i = 0; i < sel.size(); ++i) {
        const rs_kd_sample &s = *sel[i];
        const int seq_off = static_cast<int>(tokens.size());
        tokens.insert(tokens.end(), s.prompt, s.prompt + s.prompt_len);
        tokens.insert(tokens.end(), s.response, s.response + s.response_len);
        for (int t = 0; t < s.response_len; ++t) {
            const int lp_off = static_cast<int>(lp.size() / V);
            if (!policy) {
                if (!s.target_logprobs) throw std::invalid_argument("kd_loss: target log-probabilities required");
                lp.insert(lp.end(), s.target_logprobs + (size_t)t * V, s.target_logprobs + (size_t)(t + 1) * V);
            }
            per_sample[i].push_back(static_cast<int>(jobs.size()));
            jobs.push_back(Job{seq_off, s.prompt_len + t, lp_off, static_cast<int>(i), s.eos_bias});
        }
    }
    for (int v : tokens)
        if (v < 0 || v >= V) throw std::invalid_argument("row_index: token out of vocabulary");
    const size_t cells = drafter->host.size();
    if (grad_only) RS_CUDA(cudaMemsetAsync(out_dev, 0, cells * 8, st));
    else RS_CUDA(cudaMemcpyAsync(out_dev, drafter->table.p, cells * 8, cudaMemcpyDeviceToDevice, st));
    const int J = static_cast<int>(jobs.size());
    if (J == 0) {
        RS_CUDA(cudaStreamSynchronize(st));
        return 0.0;
    }
    std::vector<double> kl(J);
    std::vector<long long> rows(J);
    DBuf<int32_t> d_tok(tokens.size());
    DBuf<double> d_lp(std::max<size_t>(lp.size(), 1)), d_m(J), d_s(J), d_kl(J), d_w(std::max<size_t>(w.size(), 1));
    DBuf<Job> d_jobs(J);
    DBuf<long long> d_row(J);
    RS_CUDA(cudaMemcpyAsync(d_tok.p, tokens.data(), tokens.size() * 4, cudaMemcpyHostToDevice, st));
    RS_CUDA(cudaMemcpyAsync(d_lp.p, lp.data(), lp.size() * 8, cudaMemcpyHostToDevice, st));
    RS_CUDA(cudaMemcpyAsync(d_jobs.p, jobs.data(), J * sizeof(Job), cudaMemcpyHostToDevice, st));
    RS_CUDA(cudaMemcpyAsync(d_w.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice, st));
    const int th = V <= 256 ? 32 : V <= 4096 ? 256 : 1024;
    kd_job_kernel<<<J, th, 0, st>>>(drafter->table.p, drafter->order, V, drafter->temperature, d_tok.p, d_jobs.p,
                                    policy ? nullptr : d_lp.p, d_m.p, d_s.p, d_kl.p, d_row.p);
    RS_LAUNCHED();
    RS_CUDA(cudaMemcpyAsync(kl.data(), d_kl.p, J * 8, cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaMemcpyAsync(rows.data(), d_row.p, J * 8, cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    // group jobs by row, keeping job order (= sample order, then position)
    std::map<long long, std::vector<int>> by_row;
    for (int j = 0; j < J; ++j) by_row[rows[j]].push_back(j);
    std::vector<int> row_jobs, row_ptr{0};
    std::vector<long long> urows;
    for (auto &[r, js] : by_row) {
        urows.push_back(r);
        row_jobs.insert(row_jobs.end(), js.begin(), js.end());
        row_ptr.push_back(static_cast<int>(row_jobs.size()));
    }
    DBuf<int32_t> d_rj(row_jobs.size()), d_rp(row_ptr.size());
    DBuf<long long> d_ur(urows.size());
    RS_CUDA(cudaMemcpyAsync(d_rj.p, row_jobs.data(), row_jobs.size() * 4, cudaMemcpyHostToDevice, st));
    RS_CUDA(cudaMemcpyAsync(d_rp.p, row_ptr.data(), row_ptr.size() * 4, cudaMemcpyHostToDevice, st));
    RS_CUDA(cudaMemcpyAsync(d_ur.p, urows.data(), urows.size() * 8, cudaMemcpyHostToDevice, st));
    kd_row_kernel<<<(int)urows.size(), th, 0, st>>>(drafter->table.p, out_dev, V, drafter->temperature, d_jobs.p,
                                                    d_rj.p, d_rp.p, d_ur.p, d_lp.p, d_m.p, d_s.p, d_w.p, scale,
                                                    grad_only ? 1 : 0, policy ? d_tok.p : nullptr);
    RS_LAUNCHED();
    RS_CUDA(cudaStreamSynchronize(st));
    // loss on the pre-update drafter: sum_i w_i * sum_t KL_t (learner.cpp:142-145)
    double loss = 0.0;
    for (size_t i = 0; i < sel.size(); ++i) {
        double total = 0.0;
        for (int j : per_sample[i]) total += kl[j];
        loss += w[i] * total;
    }
    return loss;
}

void kd_update_tabular(rs_ctx *ctx, const TabularModel *drafter, const rs_kd_sample *buf, int n,
                       const rs_kd_policy &policy, uint64_t *sel_state, double cost, rs_model **out_model,
                       rs_kd_result *out) {
    if (policy.mode == 2) throw std::logic_error("kd_update: frozen drafter takes no updates");
    if (policy.interval < 1) throw std::invalid_argument("kd_update: interval must be >= 1");
    const int V = drafter->vocab;
    auto copy_model = [&](bool bump) {
        auto m = std::make_unique<TabularModel>();
        m->ctx = ctx;
        m->vocab = V;
        m->order = drafter->order;
        m->rows = drafter->rows;
        m->temperature = drafter->temperature;
        m->version = drafter->version + (bump ? 1 : 0);
        m->host = drafter->host;
        m->table.alloc(m->host.size());
        return m;
    };
    rs_kd_result res{};
    if (n <= 0) {  // empty buffer: no-op (learner.cpp:103-105)
        auto m = copy_model(false);
        RS_CUDA(cudaMemcpy(m->table.p, drafter->table.p, m->host.size() * 8, cudaMemcpyDeviceToDevice));
        *out_model = m.release();
        if (out) *out = res;
        return;
    }
    const std::vector<int> idx = kd_select(n, policy.interval, sel_state);
    const size_t take = idx.size();
    std::vector<double> br(take), w(take);
    for (size_t i = 0; i < take; ++i) br[i] = buf[idx[i]].reward;
    double wsum = 0, wmin = 0, wmax = 0;
    size_t distilled = 0;
    std::vector<const rs_kd_sample *> sel(take);
    for (size_t i = 0; i < take; ++i) {
        sel[i] = &buf[idx[i]];
        w[i] = kd_weight(sel[i]->reward, br, policy);
        wsum += w[i];
        wmin = i == 0 ? w[i] : std::min(wmin, w[i]);
        wmax = i == 0 ? w[i] : std::max(wmax, w[i]);
        distilled += static_cast<size_t>(sel[i]->response_len);
    }
    auto m = copy_model(true);
    const double loss = kd_core(ctx, drafter, sel, w, m->table.p, false, -policy.lr);
    RS_CUDA(cudaMemcpy(m->host.data(), m->table.p, m->host.size() * 8, cudaMemcpyDeviceToHost));
    res.updated = 1;
    res.samples_used = static_cast<int>(take);
    res.loss = loss;
    res.weight_mean = wsum / static_cast<double>(take);
    res.weight_min = wmin;
    res.weight_max = wmax;
    res.sim_time = cost * static_cast<double>(distilled);
    *out_model = m.release();
    if (out) *out = res;
}

namespace {
// Deterministic sum of squares: a fixed grid of CTAs each reduces a fixed strided slice, then
// one CTA adds the partials in index order (same bits run to run, independent of timing).
constexpr int kL2Blocks = 1184;
__global__ void __launch_bounds__(256) sumsq_partial_kernel(const bf16 *w, size_t n, double *part) {
    __shared__ double red[32];
    double s = 0.0;
    const size_t n8 = n / 8;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 u = *reinterpret_cast<const uint4 *>(w + i * 8);
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(h[j]);
            s += (double)f.x * f.x;
            s += (double)f.y * f.y;
        }
    }
    if (blockIdx.x == 0)
        for (size_t i = n8 * 8 + threadIdx.x; i < n; i += blockDim.x) {
            const double v = __bfloat162float(w[i]);
            s += v * v;
        }
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void __launch_bounds__(256) sumsq_final_kernel(const double *part, int n, double *out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}
}  // namespace

double weights_l2_bf16(const bf16 *w, size_t n, cudaStream_t st) {
    DBuf<double> part(kL2Blocks + 1);
    sumsq_partial_kernel<<<kL2Blocks, 256, 0, st>>>(w, n, part.p);
    RS_LAUNCHED();
    sumsq_final_kernel<<<1, 256, 0, st>>>(part.p, kL2Blocks, part.p + kL2Blocks);
    RS_LAUNCHED();
    double h = 0.0;
    RS_CUDA(cudaMemcpyAsync(&h, part.p + kL2Blocks, sizeof(double), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(h);
}

}  // namespace rs

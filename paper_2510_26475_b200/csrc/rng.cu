// rng.cu -- device mt19937_64 (one warp per stream for the twist).
#include "common.cuh"
#include "rng.cuh"

namespace rs {

namespace {

constexpr int kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x7FFFFFFFULL;

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t x = (a & kUpper) | (b & kLower);
    return c ^ (x >> 1) ^ ((x & 1ULL) ? kMtA : 0ULL);
}

// One warp twists state `mt` in place and writes the 312 tempered outputs to `out`.
__device__ void warp_twist(uint64_t *mt, uint64_t *out, uint64_t *scratch) {
    const int lane = threadIdx.x & 31;
    // new[i] for i < 156 depends only on old words.
    for (int i = lane; i < kMtN - kMtM; i += 32) scratch[i] = mt_mix(mt[i], mt[i + 1], mt[i + kMtM]);
    __syncwarp();
    // 156 <= i < 311: old[i], old[i+1], new[i-156].
    for (int i = kMtN - kMtM + lane; i < kMtN - 1; i += 32)
        scratch[i] = mt_mix(mt[i], mt[i + 1], scratch[i - (kMtN - kMtM)]);
    __syncwarp();
    if (lane == 0) scratch[kMtN - 1] = mt_mix(mt[kMtN - 1], scratch[0], scratch[kMtM - 1]);
    __syncwarp();
    for (int i = lane; i < kMtN; i += 32) {
        mt[i] = scratch[i];
        out[i] = mt_temper(scratch[i]);
    }
    __syncwarp();
}

__global__ void rng_init_kernel(MtStream *streams, const uint64_t *seeds, const uint64_t *ids, int n) {
    __shared__ uint64_t scratch[4][kMtN];
    const int w = threadIdx.x >> 5;
    const int s = blockIdx.x * 4 + w;  // stream index in [0, 2n)
    if (s >= 2 * n) return;
    MtStream &ms = streams[s];
    if ((threadIdx.x & 31) == 0) {
        // DecodeRng::from_seed: s = seed ^ (C * (id + 1)); draft = splitmix(s); accept = splitmix(s)
        uint64_t st = seeds[s >> 1] ^ (0x51ed270b8d2c7f13ULL * (ids[s >> 1] + 1));
        uint64_t v = splitmix64(st);
        if (s & 1) v = splitmix64(st);
        // std::mersenne_twister_engine::seed (f = 6364136223846793005)
        ms.mt[0] = v;
        for (int i = 1; i < kMtN; ++i) ms.mt[i] = 6364136223846793005ULL * (ms.mt[i - 1] ^ (ms.mt[i - 1] >> 62)) + i;
        ms.pos = 0;
    }
    __syncwarp();
    warp_twist(ms.mt, ms.out, scratch[w]);
    warp_twist(ms.mt, ms.out + kMtN, scratch[w]);
}

__global__ void rng_refill_kernel(MtStream *streams, int n_streams) {
    __shared__ uint64_t scratch[4][kMtN];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * 4 + w;
    if (s >= n_streams) return;
    MtStream &ms = streams[s];
    if (ms.pos < kMtN) return;  // warp-uniform
    for (int i = lane; i < kMtN; i += 32) ms.out[i] = ms.out[i + kMtN];
    __syncwarp();
    if (lane == 0) ms.pos -= kMtN;
    warp_twist(ms.mt, ms.out + kMtN, scratch[w]);
}

}  // namespace

void rng_init(MtStream *streams, const uint64_t *seeds, const uint64_t *ids, int n, cudaStream_t st) {
    if (n <= 0) return;
    rng_init_kernel<<<(2 * n + 3) / 4, 128, 0, st>>>(streams, seeds, ids, n);
    RS_LAUNCHED();
}

void rng_refill(MtStream *streams, int n_streams, cudaStream_t st) {
    if (n_streams <= 0) return;
    rng_refill_kernel<<<(n_streams + 3) / 4, 128, 0, st>>>(streams, n_streams);
    RS_LAUNCHED();
}

void HostMt::seed(uint64_t s) {
    mt[0] = s;
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    idx = kMtN;
}

uint64_t HostMt::next() {
    if (idx >= kMtN) {
        for (int i = 0; i < kMtN; ++i) {
            const uint64_t x = (mt[i] & kUpper) | (mt[(i + 1) % kMtN] & kLower);
            mt[i] = mt[(i + kMtM) % kMtN] ^ (x >> 1) ^ ((x & 1ULL) ? kMtA : 0ULL);
        }
        idx = 0;
    }
    return mt_temper(mt[idx++]);
}

}  // namespace rs

// rng.cuh -- device-resident per-request DecodeRng (rng.hpp:33-47).
//
// Each request owns two std::mt19937_64 streams (draft D, accept A) seeded exactly as
// DecodeRng::from_seed. The streams live in HBM as {state[312], out[624], pos}: `out` holds
// the next 624 tempered outputs (two twist blocks), `pos` the next unread one. Kernels read
// uniforms at pos + k without consuming; the cycle-end kernel advances pos by the draws the
// cycle actually made, and rng_refill twists a new block in whenever pos crosses 312.
// Consumption per cycle is bounded by s*t*n (D) and s*(t+n-1)+1 (A),
// which the engine requires to be <= 312.
#pragma once
#include <cstdint>

namespace rs {

constexpr int kMtN = 312;

struct MtStream {
    uint64_t mt[kMtN];
    uint64_t out[2 * kMtN];
    int32_t pos;
    int32_t pad;
};

// rng.hpp:11-13
__host__ __device__ __forceinline__ double to_unit_double(uint64_t bits) {
    return static_cast<double>(bits >> 11) * 0x1.0p-53;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t &s) {  // rng.hpp:15-20
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

// Launchers (rng.cu). streams: array of 2*n MtStream, [2*i] = draft, [2*i+1] = accept.
void rng_init(MtStream *streams_dev, const uint64_t *seeds_dev, const uint64_t *stream_ids_dev, int n,
              cudaStream_t st);
void rng_refill(MtStream *streams_dev, int n_streams, cudaStream_t st);
// Host-side mt19937_64 matching std::mt19937_64 (used for the KD selection stream).
struct HostMt {
    uint64_t mt[kMtN];
    int idx;
    void seed(uint64_t s);
    uint64_t next();
};

}  // namespace rs

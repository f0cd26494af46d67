// common.cuh -- shared device helpers: the counter-derived RNG, thresholds, warp utils.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace immx_dev {

// ---- RNG: proj/include/immx/rng.hpp:15-20, :38-47 reproduced bit-exactly -------------
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kSeedSalt = 0x6a09e667f3bcc909ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// state of stream_for(seed, index) (rng.hpp:45-47)
__host__ __device__ __forceinline__ uint64_t stream_state(uint64_t seed, uint64_t index) {
    return mix64(seed ^ kSeedSalt) ^ mix64(index + kGamma);
}
// draw number t (t >= 1) of a stream whose state is s0: the t-th next_u64()
__host__ __device__ __forceinline__ uint64_t draw(uint64_t s0, uint64_t t) { return mix64(s0 + t * kGamma); }

// next_below(bound) = high 64 bits of the 128-bit product (rng.hpp:28-32)
__device__ __forceinline__ uint64_t below(uint64_t x, uint64_t bound) { return __umul64hi(x, bound); }

// ---- edge probability as an integer threshold --------------------------------------
// sampler.cpp:37-39: p <= 0 -> skip without a draw; p >= 1 (or NaN) -> traverse without a
// draw; else one draw, traverse iff next_double() < p  <=>  (x >> 11) < ceil(p * 2^53).
constexpr uint64_t kThrNever = 0;
constexpr uint64_t kThrAlways = ~0ULL;

__host__ __device__ __forceinline__ uint64_t prob_threshold(double p) {
    if (p <= 0.0) return kThrNever;
    if (!(p < 1.0)) return kThrAlways;  // p >= 1 or NaN
    return (uint64_t)ceil(p * 9007199254740992.0);  // exact: p * 2^53 is representable
}

// probability storage modes of the device graph
enum ProbMode : int { kProbGlobal = 0, kProbRow = 1, kProbEdge = 2 };

constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

}  // namespace immx_dev

// rng.cuh -- device restatement of the reference counter-based RNG.
//
// rng.hpp:11-16 mix64 (splitmix64 finalizer), rng.hpp:32-33 substream
// seeding, rng.hpp:35-41 next_u64 (Weyl step + finalizer), rng.hpp:44-53
// Lemire uniform_below, rng.hpp:64 sign.  The Weyl sequence makes every
// draw random-access: the k-th draw (k >= 1) of a stream with initial state
// s0 is fin(s0 + k * GAMMA), so lane i of a warp computes draw i directly.
#pragma once

#include <cstdint>

namespace slq {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kStreamSalt = 0x6a09e667f3bcc909ULL;

__host__ __device__ __forceinline__ uint64_t fin64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// rng.hpp:11-16
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) { return fin64(z + kGamma); }

// rng.hpp:32-33: state of Rng(seed, stream) given mixed = mix64(seed)
__host__ __device__ __forceinline__ uint64_t stream_state(uint64_t seed_mixed, uint64_t stream) {
    return mix64(seed_mixed ^ (kStreamSalt + stream));
}

// k-th output (k >= 1) of next_u64 from initial state s0 (rng.hpp:35-41)
__host__ __device__ __forceinline__ uint64_t draw_at(uint64_t s0, uint64_t k) {
    return fin64(s0 + k * kGamma);
}

// One Lemire step (rng.hpp:44-53) on draw x: returns the candidate and sets
// `reject` when the reference would discard x and draw again.  `thresh` is
// (2^64 - bound) % bound, precomputed on the host; since thresh < bound the
// reference's acceptance test (lo >= bound || lo >= thresh) reduces to
// lo >= thresh.
__device__ __forceinline__ uint64_t lemire(uint64_t x, uint64_t bound, uint64_t thresh, bool& reject) {
    uint64_t lo = x * bound;
    reject = lo < thresh;
    return __umul64hi(x, bound);
}

// Sequential Rng as in the reference, for replay paths.
struct SeqRng {
    uint64_t s;
    __device__ __forceinline__ uint64_t next() {
        s += kGamma;
        return fin64(s);
    }
    __device__ __forceinline__ uint64_t below(uint64_t bound, uint64_t thresh) {
        for (;;) {
            bool rej;
            uint64_t v = lemire(next(), bound, thresh, rej);
            if (!rej) return v;
        }
    }
};

}  // namespace slq

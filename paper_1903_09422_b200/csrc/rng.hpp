// rng.hpp — the reference's random streams, usable on host and device.
//
//   mix64        rng.hpp:12-19  (Stafford mix13 finalizer)
//   next         rng.hpp:27-30  (splitmix64 step)
//   next_below   rng.hpp:33-44  (Lemire with rejection; bound 0 returns 0)
//   reseed       rng.hpp:53-55  (stream seed of frame position p)
//
// Bit-exactness of the whole engine rests on these being identical on both
// sides; tests/test_oracle.py and the GPU parity tests pin them.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define ADSB_HD __host__ __device__ __forceinline__
#else
#define ADSB_HD inline
#endif

namespace adsb {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

ADSB_HD uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

ADSB_HD uint64_t reseed(uint64_t base_seed, uint64_t index) { return mix64(base_seed ^ (index * kGolden)); }

ADSB_HD uint64_t mul_hi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

struct SplitMix64 {
    uint64_t state;

    ADSB_HD explicit SplitMix64(uint64_t seed = 0) : state(seed) {}

    ADSB_HD uint64_t next() {
        state += kGolden;
        return mix64(state);
    }

    // Lemire: m = x * bound (128-bit); reject while lo < (2^64 - bound) % bound.
    ADSB_HD uint64_t next_below(uint64_t bound) {
        uint64_t x = next();
        uint64_t lo = x * bound;
        if (lo < bound) {
            const uint64_t threshold = (0 - bound) % bound;  // bound 0: never entered (lo < 0 false)
            while (lo < threshold) {
                x = next();
                lo = x * bound;
            }
        }
        return mul_hi64(x, bound);
    }
};

}  // namespace adsb

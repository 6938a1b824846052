// dmm_rng.cuh -- device restatement of the reference's randomness (rng.hpp:15-48):
// std::mt19937_64 ([rand.predef]: seeding recurrence, twist, tempering), splitmix64
// and the rejection-sampled rng_below.
#pragma once

#include <cstdint>

namespace dmmdev {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {  // rng.hpp:17
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

struct Mt64 {  // std::mt19937_64 ([rand.predef])
    uint64_t mt[312];
    int mti;
    __device__ void seed(uint64_t s) {
        mt[0] = s;
        for (int i = 1; i < 312; ++i)
            mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
        mti = 312;
    }
    __device__ uint64_t next() {
        constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
        if (mti >= 312) {
            int i = 0;
            for (; i < 156; ++i) {
                const uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
                mt[i] = mt[i + 156] ^ (x >> 1) ^ ((x & 1) ? MA : 0);
            }
            for (; i < 311; ++i) {
                const uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
                mt[i] = mt[i - 156] ^ (x >> 1) ^ ((x & 1) ? MA : 0);
            }
            const uint64_t x = (mt[311] & UM) | (mt[0] & LM);
            mt[311] = mt[155] ^ (x >> 1) ^ ((x & 1) ? MA : 0);
            mti = 0;
        }
        uint64_t x = mt[mti++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= x >> 43;
        return x;
    }
    __device__ uint64_t below(uint64_t n) {  // rng_below rng.hpp:25-32
        const uint64_t limit = ~0ULL - (~0ULL % n + 1) % n;
        uint64_t x;
        do {
            x = next();
        } while (x > limit);
        return x % n;
    }
};


__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

}  // namespace dmmdev

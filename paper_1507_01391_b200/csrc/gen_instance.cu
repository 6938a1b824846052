// gen_instance.cu -- on-device, bit-exact restatement of the reference's seeded
// instance generator (instance.hpp:48-76; rng.hpp:15-48): std::mt19937_64 seeded
// with splitmix64(seed ^ (w << 32) ^ m), then Fisher-Yates with rejection-sampled
// rng_below for partition (m copies of each label) and permute (iota) instances.
// The uint32 sort tile is the builder-defined generator of SURVEY.md K3:
// x_i = Rng(splitmix64(seed))() >> 32.
//
// One thread per instance; the generator state (312 words) and the grid being
// shuffled live in that thread's local memory.  This is set-up work (the bench
// generates its synthetic inputs with it outside the timed region), not the hot path.
#include "capi_common.h"

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

constexpr int kMaxGenN = 4096;

__global__ void k_gen_instances(int kind, uint32_t w, uint32_t m, uint64_t seed0, uint64_t count,
                                uint32_t* __restrict__ out) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count)
        return;
    const uint32_t n = w * m;
    const uint64_t seed = seed0 + k;
    uint32_t* dst = out + k * n;
    Mt64 rng;
    if (kind == 0) {  // uint32 sort tile
        rng.seed(splitmix64(seed));
        for (uint32_t i = 0; i < n; ++i)
            dst[i] = (uint32_t)(rng.next() >> 32);
        return;
    }
    rng.seed(splitmix64(seed ^ ((uint64_t)w << 32) ^ m));
    uint32_t g[kMaxGenN];
    for (uint32_t i = 0; i < n; ++i)
        g[i] = kind == 1 ? i / m : i;  // partition: labels 0..w-1, m copies each; permute: iota
    for (uint32_t i = n; i > 1; --i) {  // fisher_yates rng.hpp:34-40
        const uint32_t j = (uint32_t)rng.below(i);
        const uint32_t t = g[i - 1];
        g[i - 1] = g[j];
        g[j] = t;
    }
    for (uint32_t i = 0; i < n; ++i)
        dst[i] = g[i];
}

}  // namespace dmmdev

extern "C" dmm_status dmm_gen_instances(int kind, uint32_t w, uint32_t m, uint64_t seed0, uint64_t count,
                                        uint32_t* out, void* stream) {
    dmmhost::reset_launches();
    if (w < 1 || m < 1)
        return DMM_SHAPE_VIOLATION;  // instance.hpp:49-50
    if (kind < 0 || kind > 2 || !out)
        return DMM_INVALID_ARGUMENT;
    if (uint64_t(w) * m > dmmdev::kMaxGenN) {
        dmmhost::set_error("dmm_gen_instances: w*m above 4096");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (count == 0)
        return DMM_OK;
    const unsigned threads = 128;
    const uint64_t blocks = (count + threads - 1) / threads;
    dmmdev::k_gen_instances<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(kind, w, m, seed0,
                                                                                               count, out);
    return dmmhost::check_launch("k_gen_instances");
}

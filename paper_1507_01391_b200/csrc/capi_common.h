// capi_common.h -- host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/dmm_gpu.h"

namespace dmmhost {

void set_error(const std::string& s);
void count_launch(uint32_t n = 1);
void reset_launches();

// Check a kernel launch; records the CUDA error text.
inline dmm_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return DMM_CUDA_ERROR;
    }
    count_launch();
    return DMM_OK;
}

// Per-kernel launch attributes (dynamic shared memory above 48 KB, full carveout), set once
// per device and kernel: `done` is the kernel's own static bitmask of configured devices
// (atomic: concurrent host threads may race to configure; setting twice is harmless).
template <class Kernel>
inline dmm_status configure_kernel(Kernel kern, size_t smem, std::atomic<uint64_t>& done) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess)
        return check_launch("cudaGetDevice");
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit)
        return DMM_OK;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return check_launch("cudaFuncSetAttribute");
    // prefer the full 228 KB shared-memory carveout: occupancy is bounded by smem + registers
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    done.fetch_or(bit, std::memory_order_release);
    return DMM_OK;
}

inline uint32_t ilog2_ceil(uint64_t x) {  // core.hpp:27
    uint32_t k = 0;
    uint64_t p = 1;
    while (p < x) {
        p <<= 1;
        ++k;
    }
    return k;
}
inline uint32_t isqrt_floor(uint32_t x) {  // core.hpp:46
    uint32_t r = static_cast<uint32_t>(std::sqrt(double(x)));
    while (uint64_t(r) * r > x)
        --r;
    while (uint64_t(r + 1) * (r + 1) <= x)
        ++r;
    return r;
}
inline bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

// general_sort_shape_ok partition.hpp:133-152 (+ extension for partial groups)
inline bool general_sort_shape_ok(uint64_t W, uint64_t M, bool ext) {
    if (W <= 1)
        return true;
    if (W <= M) {
        const uint32_t h = isqrt_floor(uint32_t(M));
        return W * W <= M || (uint64_t(h) * h == M && W % h == 0) || (M % W == 0);
    }
    if (M < 2 || W % M != 0)
        return false;
    uint64_t nsubs = W;
    while (nsubs > 1) {
        const uint64_t g = M < nsubs ? M : nsubs;
        if (g < M && g * g > M && (!ext || M % g != 0))
            return false;
        if (nsubs % g != 0)
            return false;
        nsubs /= g;
    }
    return general_sort_shape_ok(W / M, M, ext);
}

// The status the reference raises for integer_sort_general on a W x M view
// before touching data (partition.hpp:436-449 and the throws reachable from the
// shape alone inside balance_divide_sort / partition_leaf).
inline dmm_status integer_sort_shape_status(uint32_t W, uint32_t M, bool enforce_pre, bool ext) {
    if (W > M && M < 2)
        return DMM_SHAPE_VIOLATION;
    if (enforce_pre && W > M && double(M) <= 2.0 * std::sqrt(std::log2(double(W))))
        return DMM_SHAPE_VIOLATION;
    if (W <= M) {
        if (uint64_t(W) * W <= M)
            return DMM_OK;
        const uint32_t h = isqrt_floor(M);
        if (h * h == M && W % h == 0)
            return DMM_OK;
        return (W == 1 || M % W == 0) ? DMM_OK : DMM_SHAPE_VIOLATION;  // shearsort_rect sort.hpp:291
    }
    if (W % M != 0)
        return DMM_SHAPE_VIOLATION;
    if (!general_sort_shape_ok(W, M, ext))
        return DMM_SHAPE_VIOLATION;
    return DMM_OK;
}

// PartitionParams::compute partition.hpp:209-225 in double precision, as the
// reference evaluates it (used to cross-check the compile-time schedule).
inline bool partition_params(uint32_t W, uint32_t M, bool ext, uint32_t* d_out, uint32_t* subs_out) {
    const double l = std::log(double(W)) / std::log(double(M));
    const uint32_t want = std::max<uint32_t>(1, uint32_t(std::ceil(2 * l - 1e-9)));
    uint32_t d = std::min<uint32_t>(want, W / M);
    while (uint64_t(M) * d <= W && (W % (uint64_t(M) * d) != 0 || !general_sort_shape_ok(W / (uint64_t(M) * d), M, ext)))
        ++d;
    if (uint64_t(M) * d > W || W % (uint64_t(M) * d) != 0)
        return false;
    *d_out = d;
    *subs_out = M * d;
    return true;
}

}  // namespace dmmhost

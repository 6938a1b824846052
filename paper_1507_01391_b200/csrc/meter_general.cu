// meter_general.cu -- dmm_general_steps: the reference's Machine::steps() and
// GeneralStats::cleanup_retries of the general partition / integer sort for any accepted shape,
// w > m recursion included (general_meter.cuh).  One thread per instance replays the
// reference's states in a private global workspace; off the hot path.
#include "capi_common.h"
#include "general_meter.cuh"

namespace dmmdev {

__global__ void __launch_bounds__(64) k_general_steps(const uint32_t* __restrict__ in, uint32_t W, uint32_t M,
                                                      uint64_t count, uint64_t domain, uint32_t* __restrict__ ws,
                                                      uint64_t ws_stride, uint64_t* __restrict__ steps,
                                                      uint32_t* __restrict__ retries) {
    const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= count)
        return;
    const uint64_t n = uint64_t(W) * M;
    uint32_t* g = ws + uint64_t(threadIdx.x + uint64_t(blockIdx.x) * blockDim.x) * ws_stride;
    for (uint64_t i = 0; i < n; ++i)
        g[i] = in[k * n + i];
    uint32_t rt = 0;
    const uint64_t s = dmmmeter::general_steps(g, W, M, domain, g + n, &rt);
    steps[k] = s;
    if (retries)
        retries[k] = rt;
}

}  // namespace dmmdev

extern "C" {

dmm_status dmm_general_steps(const uint32_t* in, uint32_t w, uint32_t m, uint64_t count, uint64_t domain,
                             uint64_t* steps, uint32_t* retries, void* stream) {
    dmmhost::reset_launches();
    if (w < 1 || m < 2 || uint64_t(w) * m > (1u << 16) || !dmmmeter::shape_ok(w, m) ||
        (w > m && dmmmeter::subproblems(w, m) == 0)) {
        dmmhost::set_error("general metering: a shape general_sort_shape_ok accepts, m >= 2, w m <= 65536");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (count == 0)
        return DMM_OK;
    if (!in || !steps || domain == 0)
        return DMM_INVALID_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // workspace: instance copy + relayout / gather / merge buffers, chunked to <= 256 MiB
    const uint64_t stride = uint64_t(w) * m + dmmmeter::workspace_words(w, m);
    const uint64_t chunk = std::max<uint64_t>(64, std::min<uint64_t>(count, (256ull << 20) / (4 * stride)));
    uint32_t* ws = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws), chunk * stride * sizeof(uint32_t), st) != cudaSuccess)
        return dmmhost::check_launch("cudaMallocAsync (metering workspace)");
    static std::atomic<uint64_t> stack_set{0};
    if (!stack_set.exchange(1))
        cudaDeviceSetLimit(cudaLimitStackSize, 4096);  // the recursion over column subproblems
    dmm_status e = DMM_OK;
    for (uint64_t base = 0; base < count && e == DMM_OK; base += chunk) {
        const uint64_t c = std::min(chunk, count - base);
        dmmdev::k_general_steps<<<unsigned((c + 63) / 64), 64, 0, st>>>(
            in + base * w * m, w, m, c, domain, ws, stride, steps + base, retries ? retries + base : nullptr);
        e = dmmhost::check_launch("k_general_steps");
    }
    cudaFreeAsync(ws, st);
    return e;
}

}  // extern "C"

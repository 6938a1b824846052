// layout_sorts.cu -- batched layout primitives, row sorts and the tall comparison sort over
// 32 x m machines (one warp per machine); sort_tall also on 64- and 128-row machines (one
// machine per CTA, cross-warp column networks through the staging buffer).
//
// C ABI: dmm_transpose_square (layout.hpp:24), dmm_to_column_major (layout.hpp:397),
// dmm_to_row_major (layout.hpp:403), dmm_sort_rows (partition.hpp:94 / sort.hpp:76),
// dmm_sort_tall (sort.hpp:352).  (dmm_sort_square / dmm_sort_short_wide: general_sort.cu.)
#include "general_kernel.cuh"

namespace dmmdev {

enum : int { kOpTranspose = 0, kOpToCol = 1, kOpToRow = 2, kOpSortRows = 3, kOpSortTall = 4 };

// R = machine rows: 32 (one warp per machine, 8 machines per CTA) or 64 / 128 (one machine
// per CTA of R / 32 warps; thread t holds row t)
template <int M, int OP, int R = kWarp>
__global__ void __launch_bounds__(R > kWarp ? R : 256) k_layout(const uint32_t* __restrict__ in,
                                                               uint32_t* __restrict__ out, uint64_t count, int order,
                                                               uint64_t domain, uint8_t* __restrict__ status) {
    constexpr bool kMulti = R > kWarp;
    extern __shared__ uint32_t smem[];
    const int lane = kMulti ? (int)threadIdx.x : (int)(threadIdx.x & 31);
    const int warp = kMulti ? 0 : (int)(threadIdx.x >> 5);
    uint32_t* buf = smem + warp * relayout_buf_words(M) * (R / kWarp);
    const uint64_t k = kMulti ? (uint64_t)blockIdx.x : (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (k >= count)
        return;
    uint32_t x[M];
    load_row<M>(in + (k * R + lane) * M, x);
    using V = VF<0xFFFFFFFFu, 0, 1, R, 0, M, R, R>;
    if constexpr (OP == kOpTranspose) {
        transpose_square<V>(x, buf, lane);
    } else if constexpr (OP == kOpToCol) {
        to_column_major<V>(x, buf, lane);
    } else if constexpr (OP == kOpToRow) {
        to_row_major<V>(x, buf, lane);
    } else if constexpr (OP == kOpSortRows) {
        uint32_t bad = 0;
#pragma unroll
        for (int c = 0; c < M; ++c)
            bad |= (uint64_t)x[c] >= domain ? 1u : 0u;
        bad = group_or<R, R>(bad, lane, buf);
        const bool asc = order == 0 ? true : order == 1 ? false : (((lane % 2) == 0) == (order == 2));
        row_sort<1, V>(x, lane, asc);
        if (status && lane == 0)
            status[k] = (bad && M > 1) ? DMM_KEY_OUT_OF_RANGE : DMM_OK;
    } else if constexpr (OP == kOpSortTall) {
        // sort_tall sort.hpp:352-374 (w >= m, m | w)
        sort_tall<1, V>(x, buf, lane);
    }
    store_row<M>(out + (k * R + lane) * M, x);
}

}  // namespace dmmdev

namespace {

using namespace dmmhost;

template <int M, int OP, int R = dmmdev::kWarp>
dmm_status launch_layout(const uint32_t* in, uint32_t* out, uint64_t count, int order, uint64_t domain,
                         uint8_t* status, void* stream) {
    constexpr bool kMulti = R > dmmdev::kWarp;
    constexpr int kWarps = kMulti ? R / dmmdev::kWarp : 8;
    auto kern = dmmdev::k_layout<M, OP, R>;
    const size_t smem = size_t(kWarps) * dmmdev::relayout_buf_words(M) * sizeof(uint32_t);
    static std::atomic<uint64_t> configured{0};  // devices configured, per instantiation
    if (dmm_status e = configure_kernel(kern, smem, configured); e != DMM_OK)
        return e;
    if (count == 0)
        return DMM_OK;
    const uint64_t blocks = kMulti ? count : (count + kWarps - 1) / kWarps;
    if (blocks > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;  // grid x limit
    kern<<<unsigned(blocks), kWarps * 32, smem, static_cast<cudaStream_t>(stream)>>>(in, out, count, order, domain,
                                                                                     status);
    return check_launch("k_layout");
}

template <int OP>
dmm_status dispatch_layout(uint32_t w, uint32_t m, const uint32_t* in, uint32_t* out, uint64_t count, int order,
                           uint64_t domain, uint8_t* status, void* stream) {
    if constexpr (OP == dmmdev::kOpSortTall) {
        if (w == 64) {  // tall machines: two / four warps per machine
            switch (m) {
                case 8: return launch_layout<8, OP, 64>(in, out, count, order, domain, status, stream);
                case 16: return launch_layout<16, OP, 64>(in, out, count, order, domain, status, stream);
                case 32: return launch_layout<32, OP, 64>(in, out, count, order, domain, status, stream);
                default: break;
            }
        } else if (w == 128) {
            switch (m) {
                case 16: return launch_layout<16, OP, 128>(in, out, count, order, domain, status, stream);
                case 32: return launch_layout<32, OP, 128>(in, out, count, order, domain, status, stream);
                default: break;
            }
        }
    }
    if (w != 32) {
        set_error("no kernel compiled for this shape (layouts / row sorts: w = 32; sort_tall: w in {32, 64, 128})");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if constexpr (OP == dmmdev::kOpTranspose) {
        if (m == 32)
            return launch_layout<32, OP>(in, out, count, order, domain, status, stream);
    } else if constexpr (OP == dmmdev::kOpSortTall) {
        switch (m) {
            case 1: return launch_layout<1, OP>(in, out, count, order, domain, status, stream);
            case 2: return launch_layout<2, OP>(in, out, count, order, domain, status, stream);
            case 4: return launch_layout<4, OP>(in, out, count, order, domain, status, stream);
            case 8: return launch_layout<8, OP>(in, out, count, order, domain, status, stream);
            case 16: return launch_layout<16, OP>(in, out, count, order, domain, status, stream);
            case 32: return launch_layout<32, OP>(in, out, count, order, domain, status, stream);
            default: break;
        }
    } else {
        switch (m) {
            case 1: return launch_layout<1, OP>(in, out, count, order, domain, status, stream);
            case 2: return launch_layout<2, OP>(in, out, count, order, domain, status, stream);
            case 4: return launch_layout<4, OP>(in, out, count, order, domain, status, stream);
            case 8: return launch_layout<8, OP>(in, out, count, order, domain, status, stream);
            case 16: return launch_layout<16, OP>(in, out, count, order, domain, status, stream);
            case 32: return launch_layout<32, OP>(in, out, count, order, domain, status, stream);
            case 64: return launch_layout<64, OP>(in, out, count, order, domain, status, stream);
            default: break;
        }
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

dmm_status common_checks(const void* in, const void* out, uint32_t w, uint64_t count) {
    if (count && (!in || !out))
        return DMM_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) {
        set_error("in/out must be 16-byte aligned");
        return DMM_INVALID_ARGUMENT;
    }
    (void)w;
    return DMM_OK;
}

}  // namespace

extern "C" {

dmm_status dmm_transpose_square(const uint32_t* in, uint32_t* out, uint32_t s, uint64_t count, void* stream) {
    reset_launches();
    if (dmm_status e = common_checks(in, out, s, count); e != DMM_OK)
        return e;
    return dispatch_layout<dmmdev::kOpTranspose>(s, s, in, out, count, 0, 0, nullptr, stream);
}

dmm_status dmm_to_column_major(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                               void* stream) {
    reset_launches();
    if (dmm_status e = common_checks(in, out, w, count); e != DMM_OK)
        return e;
    return dispatch_layout<dmmdev::kOpToCol>(w, m, in, out, count, 0, 0, nullptr, stream);
}

dmm_status dmm_to_row_major(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                            void* stream) {
    reset_launches();
    if (dmm_status e = common_checks(in, out, w, count); e != DMM_OK)
        return e;
    return dispatch_layout<dmmdev::kOpToRow>(w, m, in, out, count, 0, 0, nullptr, stream);
}

dmm_status dmm_sort_rows(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count, int order,
                         uint64_t domain, uint8_t* status, void* stream) {
    reset_launches();
    if (order < 0 || order > 3)
        return DMM_INVALID_ARGUMENT;
    if (dmm_status e = common_checks(in, out, w, count); e != DMM_OK)
        return e;
    if (domain == 0 || domain > (1ull << 32))
        domain = 1ull << 32;
    return dispatch_layout<dmmdev::kOpSortRows>(w, m, in, out, count, order, domain, status, stream);
}

dmm_status dmm_sort_tall(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count, void* stream) {
    reset_launches();
    if (w < m || (m > 0 && w % m != 0))  // sort.hpp:354-355
        return DMM_SHAPE_VIOLATION;
    if (dmm_status e = common_checks(in, out, w, count); e != DMM_OK)
        return e;
    return dispatch_layout<dmmdev::kOpSortTall>(w, m, in, out, count, 0, 0, nullptr, stream);
}

}  // extern "C"

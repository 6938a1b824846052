// general_sort.cu -- C ABI of kernels 1-3: w-way partition (n >= w^2), general
// partition (Lemma 4), integer sort and the comparison skeletons over a batch of w x m
// machines (w = 32: one warp each; w in {2, 3, 4, 8, 16}: several per warp; w in {64, 128,
// 256}: one per CTA).
//
// C ABI: dmm_partition_general (partition.hpp:453), dmm_integer_sort_general
// (partition.hpp:436), dmm_sort_wide_any (sort.hpp:321), dmm_partition_square
// (partition.hpp:189), dmm_partition_short_wide (partition.hpp:178), dmm_sort_square
// (sort.hpp:337), dmm_sort_short_wide (sort.hpp:225), the probe entry points.  The kernel
// template is general_kernel.cuh; one translation unit per machine width / row width.
#include "general_kernel.cuh"

namespace {

using namespace dmmhost;

// Dispatch over the compiled (w, m) shapes.  PK = 2 whenever every legal key fits in 16
// bits (domain <= 2^16).
dmm_status dispatch(int mode, const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                    uint64_t domain, bool ext, int strict, int ascending, dmm_general_stats* stats, uint8_t* status,
                    cudaStream_t s, uint32_t* probe = nullptr, uint32_t probe_max = 0) {
    const bool pk2 = domain <= 65536;
    const GeneralArgs a{in, out, count, domain, strict, ascending, stats, status, s, probe, probe_max};
    switch (w) {
        case 32:
            switch (m) {
                case 8: return launch_general_m8(mode, pk2, ext, a);
                case 16: return launch_general_m16(mode, pk2, ext, a);
                case 32: return launch_general_m32(mode, pk2, ext, a);
                case 64: return launch_general_m64(mode, pk2, ext, a);
                case 128: return launch_general_m128(mode, pk2, ext, a);
                case 256: return launch_general_m256(mode, pk2, ext, a);
                case 1024: return launch_general_m1024(mode, pk2, ext, a);
                default: break;
            }
            break;
        case 64: return launch_general_tall64(m, mode, pk2, ext, a);
        case 128: return launch_general_tall128(m, mode, pk2, ext, a);
        case 256: return launch_general_tall256(m, mode, pk2, ext, a);
        case 16: return launch_general_w16(m, mode, pk2, ext, a);
        case 8: return launch_general_w8(m, mode, pk2, ext, a);
        case 4: return launch_general_w4(m, mode, pk2, ext, a);
        case 2: return launch_general_w2(m, mode, pk2, ext, a);
        case 3: return launch_general_w3(m, mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape (w in {2, 3, 4, 8, 16, 32, 64, 128, 256})");
    return DMM_UNSUPPORTED_SHAPE;
}

dmm_status check_ptrs(const void* in, const void* out, uint64_t count) {
    if (count == 0)
        return DMM_OK;
    if (!in || !out)
        return DMM_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) {
        set_error("in/out must be 16-byte aligned");
        return DMM_INVALID_ARGUMENT;
    }
    return DMM_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

dmm_status integer_sort_impl(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                             uint64_t domain, uint32_t flags, dmm_general_stats* stats, uint8_t* status,
                             uint32_t* probe, uint32_t probe_max, void* stream) {
    reset_launches();
    const bool ext = flags & DMM_FLAG_EXT_PARTIAL_GROUPS;
    const dmm_status sh = integer_sort_shape_status(w, m, !(flags & DMM_FLAG_NO_ENFORCE_PRE), ext);
    if (sh != DMM_OK)
        return sh;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    if (domain == 0 || domain > (1ull << 32)) {
        // keys are 32-bit words; a wider domain admits every key
        domain = 1ull << 32;
    }
    // use the extension kernels only where the reference itself would reject the shape
    const bool need_ext = ext && !general_sort_shape_ok(w, m, false) && m < w;
    return dispatch(dmmdev::kModeIntegerSort, in, out, w, m, count, domain, need_ext, !(flags & DMM_FLAG_NONSTRICT), 1,
                    stats, status, static_cast<cudaStream_t>(stream), probe, probe_max);
}

dmm_status partition_impl(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count, uint32_t flags,
                          dmm_general_stats* stats, uint8_t* status, uint32_t* probe, uint32_t probe_max,
                          void* stream) {
    reset_launches();
    const bool ext = flags & DMM_FLAG_EXT_PARTIAL_GROUPS;
    const dmm_status sh = integer_sort_shape_status(w, m, !(flags & DMM_FLAG_NO_ENFORCE_PRE), ext);
    if (sh != DMM_OK)
        return sh;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    const bool need_ext = ext && !general_sort_shape_ok(w, m, false) && m < w;
    return dispatch(dmmdev::kModePartition, in, out, w, m, count, w, need_ext, !(flags & DMM_FLAG_NONSTRICT), 1, stats,
                    status, static_cast<cudaStream_t>(stream), probe, probe_max);
}

}  // namespace

extern "C" {

dmm_status dmm_integer_sort_general(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                    uint64_t domain, uint32_t flags, dmm_general_stats* stats, uint8_t* status,
                                    void* stream) {
    return integer_sort_impl(in, out, w, m, count, domain, flags, stats, status, nullptr, 0, stream);
}

dmm_status dmm_partition_general(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                 uint32_t flags, dmm_general_stats* stats, uint8_t* status, void* stream) {
    return partition_impl(in, out, w, m, count, flags, stats, status, nullptr, 0, stream);
}

// the outer recursion of balance_divide_sort (partition.hpp:373-391): one after_balance and one
// after_divide snapshot per level while the subproblems have more than m rows
uint32_t dmm_general_probe_snaps(uint32_t w, uint32_t m, uint32_t flags) {
    const bool ext = flags & DMM_FLAG_EXT_PARTIAL_GROUPS;
    uint32_t n = 0;
    uint64_t W = w;
    while (W > m && m >= 2) {
        const dmmdev::PParams p = dmmdev::pparams_c(int(W), int(m), ext);
        if (p.subproblems <= 0 || W % uint64_t(p.subproblems) != 0)
            break;
        n += 2;
        W /= uint64_t(p.subproblems);
    }
    return n;
}

dmm_status dmm_partition_general_probe(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                       uint32_t flags, dmm_general_stats* stats, uint8_t* status, uint32_t* snapshots,
                                       uint32_t max_snaps, void* stream) {
    return partition_impl(in, out, w, m, count, flags, stats, status, max_snaps ? snapshots : nullptr, max_snaps,
                          stream);
}

dmm_status dmm_integer_sort_general_probe(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                          uint64_t domain, uint32_t flags, dmm_general_stats* stats, uint8_t* status,
                                          uint32_t* snapshots, uint32_t max_snaps, void* stream) {
    return integer_sort_impl(in, out, w, m, count, domain, flags, stats, status, max_snaps ? snapshots : nullptr,
                             max_snaps, stream);
}

dmm_status dmm_sort_wide_any(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                             int ascending, void* stream) {
    reset_launches();
    if (w > m || (w > 1 && m % w != 0))
        return DMM_SHAPE_VIOLATION;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    return dispatch(dmmdev::kModeSortAny, in, out, w, m, count, 1ull << 32, false, 1, ascending, nullptr, nullptr,
                                          static_cast<cudaStream_t>(stream));
}

// partition_square partition.hpp:189-197: w = m, m a perfect square; check_partition_instance
// then partition_leaf, whose outcome is the sorted instance (row i = i)
dmm_status dmm_partition_square(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                uint8_t* status, void* stream) {
    reset_launches();
    if (w != m)
        return DMM_SHAPE_VIOLATION;
    const uint32_t h = isqrt_floor(m);
    if (h * h != m)
        return DMM_SHAPE_VIOLATION;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    return dispatch(dmmdev::kModePartition, in, out, w, m, count, w, false, 1, 1, nullptr, status,
                    static_cast<cudaStream_t>(stream));
}

// partition_short_wide partition.hpp:178-185: w^2 <= m; the short-wide skeleton with radix
// rows leaves the sorted instance, i.e. partition_leaf's outcome
dmm_status dmm_partition_short_wide(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                    uint8_t* status, void* stream) {
    reset_launches();
    if (uint64_t(w) * w > m)
        return DMM_SHAPE_VIOLATION;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    return dispatch(dmmdev::kModePartition, in, out, w, m, count, w, false, 1, 1, nullptr, status,
                    static_cast<cudaStream_t>(stream));
}

// ShortWideHook capture (sort.hpp:189-218) for partition_short_wide / sort_short_wide: the
// literal short-wide skeleton (its row sorts have unique outcomes, so every stage equals the
// reference's, radix rows or merge rows alike), with the window written to
// snapshots[k * 3 * w * m ...] at after_first_convert, after_first_pass and done.
dmm_status dmm_short_wide_probe(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                int partition, int ascending, uint8_t* status, uint32_t* snapshots, void* stream) {
    reset_launches();
    if (uint64_t(w) * w > m)
        return DMM_SHAPE_VIOLATION;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    if (!snapshots)
        return DMM_INVALID_ARGUMENT;
    return dispatch(dmmdev::kModeSortAny, in, out, w, m, count, partition ? uint64_t(w) : (1ull << 32), false, 1,
                    partition ? 1 : ascending, nullptr, status, static_cast<cudaStream_t>(stream), snapshots, 3);
}

// sort_square sort.hpp:337-346: w = m perfect square -> square_skeleton (Theorem 2),
// run literally by the comparison-sort kernel (sort_wide_any dispatches on the shape)
dmm_status dmm_sort_square(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                           int ascending, void* stream) {
    reset_launches();
    if (w != m)
        return DMM_SHAPE_VIOLATION;
    const uint32_t h = isqrt_floor(m);
    if (h * h != m)
        return DMM_SHAPE_VIOLATION;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    return dispatch(dmmdev::kModeSortAny, in, out, w, m, count, 1ull << 32, false, 1, ascending, nullptr, nullptr,
                    static_cast<cudaStream_t>(stream));
}

// sort_short_wide sort.hpp:225-230: w^2 <= m -> short_wide_skeleton (Lemma 1) with merge rows
dmm_status dmm_sort_short_wide(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                               int ascending, void* stream) {
    reset_launches();
    if (uint64_t(w) * w > m)
        return DMM_SHAPE_VIOLATION;
    if (dmm_status e = check_ptrs(in, out, count); e != DMM_OK || count == 0)
        return e;
    return dispatch(dmmdev::kModeSortAny, in, out, w, m, count, 1ull << 32, false, 1, ascending, nullptr, nullptr,
                    static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// capi.cu -- library-level C ABI: version, error text, launch accounting, shape table.
#include <cstring>
#include <string>

#include "capi_common.h"

namespace dmmhost {
namespace {
thread_local std::string g_error;
thread_local uint32_t g_launches = 0;
}  // namespace
void set_error(const std::string& s) { g_error = s; }
void count_launch(uint32_t n) { g_launches += n; }
void reset_launches() {
    g_launches = 0;
    g_error.clear();
}
}  // namespace dmmhost

extern "C" {

const char* dmm_version(void) { return "paper_1507_01391_b200 0.1 (sm_100a)"; }
const char* dmm_last_error(void) { return dmmhost::g_error.c_str(); }
uint32_t dmm_last_launch_count(void) { return dmmhost::g_launches; }

int dmm_supported(const char* algorithm, uint32_t w, uint32_t m) {
    if (!algorithm)
        return 0;
    const std::string a(algorithm);
    // compiled (w, m) machine shapes of the general-sort kernel (general_m*.cu, general_w*.cu)
    auto general = [&]() -> bool {
        switch (w) {
            case 256: return m == 16;
            case 128: return m == 32 || m == 64;
            case 64: return m == 8 || m == 16 || m == 32 || m == 64;
            case 32: return m == 8 || m == 16 || m == 32 || m == 64 || m == 128 || m == 256 || m == 1024;
            case 16:
            case 8: return m == 8 || m == 16 || m == 32 || m == 64;
            case 4: return m == 4 || m == 8 || m == 16;
            case 2: return m == 2 || m == 4 || m == 8;
            case 3: return m == 9;
            default: return false;
        }
    };
    if (a == "partition_general" || a == "integer_sort_general")
        return general();
    if (a == "sort_wide_any")
        return general() && w <= m && m % w == 0 && (w != 32 || m == 32 || m == 64 || m == 128 || m == 256 || m == 1024);
    if (a == "partition_square" || a == "sort_square")
        return general() && w == m && (m == 4 || m == 16 || m == 64);
    if (a == "partition_short_wide" || a == "sort_short_wide")
        return general() && uint64_t(w) * w <= m;
    if (a == "sort_tall")
        return w >= m && m > 0 && w % m == 0 &&
               ((w == 32 && m <= 32) || (w == 64 && m >= 8 && m <= 32) || (w == 128 && (m == 16 || m == 32)));
    if (a == "permute")
        return (w == 32 && (m == 2 || m == 4 || m == 16 || m == 32)) || (w == 64 && (m == 8 || m == 16)) ||
               (w == 128 && m == 64);
    return 0;
}

uint64_t dmm_modelled_steps(const char* algorithm, uint32_t w, uint32_t m) {
    // The reference meters a bank-local section by its busiest row (core.hpp rows_lockstep);
    // where every row does the same accesses the count is a closed form of the schedule:
    //  * radix row sort of m keys < domain (partition.hpp:37-85), p = radix_pass_count(m,
    //    domain) passes of 10 m accesses (histogram clear m, count 3 m, prefix 2 m, scatter
    //    4 m) plus a 2 m copy-back when p is odd;
    //  * to_column_major / to_row_major 4 m (layout.hpp:316-405); transpose_square 2 (s - 1);
    //  * partition_leaf (partition.hpp:156-172): short-wide skeleton = 5 row sorts + 4
    //    conversions (sort.hpp:200-218); square skeleton with w = m = h^2 = 13 row sorts
    //    (two short-wide super-row passes, two transposed column sorts, the final pass)
    //    + 8 conversions + 4 transposes (sort.hpp:250-280).
    // Shearsort leaves, blocked column sorts (merge segments), the recursion's cleanup retries
    // and the permutation depend on the data: 0 (not modelled).
    if (!algorithm || w < 2 || m < 2)
        return 0;
    const std::string a(algorithm);
    auto radix = [&](uint64_t domain) -> uint64_t {
        uint32_t p = 1;
        for (uint64_t reach = m; reach < domain; reach *= m)
            ++p;
        return 10ull * m * p + ((p & 1) ? 2ull * m : 0);
    };
    auto leaf = [&](uint64_t domain) -> uint64_t {
        if (uint64_t(w) * w <= m)
            return 5 * radix(domain) + 4 * 4ull * m;
        const uint32_t h = dmmhost::isqrt_floor(m);
        if (w == m && h * h == m)
            return 13 * radix(domain) + 8 * 4ull * m + 4 * 2ull * (m - 1);
        return 0;
    };
    if (a == "partition_short_wide")
        return uint64_t(w) * w <= m ? leaf(w) : 0;
    if (a == "partition_square")
        return w == m ? leaf(w) : 0;
    if (a == "partition_general")
        return w <= m ? leaf(w) : 0;
    if (a == "integer_sort_general")
        return w <= m ? leaf(uint64_t(w) * m) : 0;
    return 0;
}

}  // extern "C"

// meter.cu -- the reference's DMM step count (Machine::steps(), core.hpp rows_lockstep) for the
// leaf of the general partition / integer sort, w <= m (partition.hpp:156-172), where it depends
// on the data.
//
// The leaf's row sorts are radix sorts (shape-determined access counts) and its transposes and
// conversions are fixed, but its blocked column sorts run merge_sort_segments (sort.hpp:44-70,
// 177-182), whose per-bank access count depends on the keys: a placement while both runs are
// non-empty costs two head reads and a write, a tail element a read and a write, plus a
// copy-back after an odd number of levels.  A bank-local section costs the maximum over the
// banks.  This kernel replays the leaf's state sequence (each sort's outcome is unique, so the
// states are those of the reference) and adds, per blocked column sort, the busiest bank's
// merge accesses to the closed-form parts:
//   shearsort_rect (sort.hpp:288-311): (ceil(log2 w) + 1) x {radix rows, M/W transposes, merge
//     segments, M/W transposes}, a final radix row sort and the odd-row reversal (2 m);
//   square_skeleton, w < m (sort.hpp:250-280): 2 x {short-wide super-rows (5 radix row sorts +
//     4 conversions), blocked column sort}, a final radix row sort.
// (Short-wide and w = m square leaves are data-independent: dmm_modelled_steps.)
//
// Metering is off the hot path: one warp per instance, the machine in shared memory, simple
// insertion sorts.
#include "capi_common.h"

namespace dmmdev {

constexpr int kMeterMaxW = 32, kMeterMaxM = 128;

__device__ __forceinline__ uint64_t radix_cost(uint32_t m, uint64_t domain) {
    uint32_t p = 1;
    for (uint64_t reach = m; reach < domain; reach *= m)
        ++p;
    return 10ull * m * p + ((p & 1) ? 2ull * m : 0);
}

// accesses of row_merge_sort (sort.hpp:44-70) on seg[0..L), ascending, L <= 32
__device__ uint32_t merge_accesses(uint32_t (&a)[kMeterMaxW], uint32_t L) {
    uint32_t b[kMeterMaxW];
    uint32_t cost = 0, levels = 0;
    for (uint32_t width = 1; width < L; width *= 2, ++levels) {
        for (uint32_t lo = 0; lo < L; lo += 2 * width) {
            const uint32_t mid = min(lo + width, L), hi = min(lo + 2 * width, L);
            if (mid >= hi) {  // a lone run: every element is a tail
                cost += 2 * (mid - lo);
                for (uint32_t i = lo; i < mid; ++i)
                    b[i] = a[i];
                continue;
            }
            const uint32_t ma = a[mid - 1], mb = a[hi - 1];
            uint32_t tail = 0;
            if (ma <= mb) {
                for (uint32_t i = mid; i < hi; ++i)
                    tail += a[i] >= ma;
            } else {
                for (uint32_t i = lo; i < mid; ++i)
                    tail += a[i] > mb;
            }
            cost += 3 * (hi - lo) - tail;
            uint32_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi)
                b[o++] = a[i] <= a[j] ? a[i++] : a[j++];
            while (i < mid)
                b[o++] = a[i++];
            while (j < hi)
                b[o++] = a[j++];
        }
        for (uint32_t i = 0; i < L; ++i)
            a[i] = b[i];
    }
    if (levels & 1)
        cost += 2 * L;
    return cost;
}

__device__ void insertion_sort(uint32_t* x, uint32_t n, uint32_t stride, bool asc) {
    for (uint32_t i = 1; i < n; ++i) {
        const uint32_t v = x[i * stride];
        uint32_t j = i;
        while (j > 0 && (asc ? x[(j - 1) * stride] > v : x[(j - 1) * stride] < v)) {
            x[j * stride] = x[(j - 1) * stride];
            --j;
        }
        x[j * stride] = v;
    }
}

// the blocked column sort (sort.hpp:162-174): returns the busiest bank's merge accesses and
// leaves every column ascending; lane r owns columns r, W + r, 2W + r, ... = its segments
__device__ uint32_t blocked_column_sort(uint32_t* g, uint32_t W, uint32_t M, int lane) {
    uint32_t mine = 0;
    if ((uint32_t)lane < W) {
        for (uint32_t c = lane; c < M; c += W) {
            uint32_t seg[kMeterMaxW];
            for (uint32_t j = 0; j < W; ++j)
                seg[j] = g[j * M + c];
            mine += merge_accesses(seg, W);
            for (uint32_t j = 0; j < W; ++j)
                g[j * M + c] = seg[j];
        }
    }
    __syncwarp();
    for (int o = 16; o > 0; o >>= 1)
        mine = max(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, o));
    return mine;
}

__global__ void __launch_bounds__(32) k_leaf_steps(const uint32_t* __restrict__ in, uint32_t W, uint32_t M,
                                                   uint64_t count, uint64_t domain, uint64_t* __restrict__ steps) {
    extern __shared__ uint32_t g[];
    const int lane = threadIdx.x;
    const uint64_t k = blockIdx.x;
    if (k >= count)
        return;
    for (uint32_t i = lane; i < W * M; i += 32)
        g[i] = in[k * W * M + i];
    __syncwarp();
    const uint64_t R = radix_cost(M, domain);
    const uint64_t transposes = 2ull * (M / W) * 2 * (W - 1);
    uint64_t total = 0;
    const uint32_t h = (uint32_t)sqrtf((float)M);
    const bool square = h * h == M && W < M && W % h == 0;
    if (square) {
        for (int pass = 0; pass < 2; ++pass) {
            // super-rows of h rows sorted row-major (short-wide skeleton), directions alternating
            // by group on the second pass
            for (uint32_t grp = lane; grp < W / h; grp += 32)
                insertion_sort(g + grp * h * M, h * M, 1, pass == 0 || grp % 2 == 0);
            __syncwarp();
            total += 5 * R + 16ull * M;
            total += blocked_column_sort(g, W, M, lane) + transposes;
            __syncwarp();
        }
        total += R;
    } else {
        uint32_t rounds = 1;
        while ((1u << (rounds - 1)) < W)
            ++rounds;  // ceil(log2 W) + 1
        for (uint32_t i = 0; i < rounds; ++i) {
            if ((uint32_t)lane < W)
                insertion_sort(g + lane * M, M, 1, lane % 2 == 0);
            __syncwarp();
            total += R;
            total += blocked_column_sort(g, W, M, lane) + transposes;
            __syncwarp();
        }
        total += R + 2ull * (M / 2) * 2;  // final row sort + reversal of the descending rows
    }
    if (lane == 0)
        steps[k] = total;
}

}  // namespace dmmdev

extern "C" {

dmm_status dmm_leaf_steps(const uint32_t* in, uint32_t w, uint32_t m, uint64_t count, uint64_t domain,
                          uint64_t* steps, void* stream) {
    dmmhost::reset_launches();
    if (count == 0)
        return DMM_OK;
    if (!in || !steps)
        return DMM_INVALID_ARGUMENT;
    const uint32_t h = dmmhost::isqrt_floor(m);
    const bool square = h * h == m && w < m && w % h == 0;
    if (w < 2 || w > dmmdev::kMeterMaxW || m > dmmdev::kMeterMaxM || w > m || (!square && m % w != 0) ||
        uint64_t(w) * w <= m || (w == m && h * h == m)) {
        dmmhost::set_error("leaf metering: 2 <= w <= 32, m <= 128, w <= m, shearsort (w | m) or square "
                           "(sqrt(m) | w < m) leaves; short-wide and w = m square leaves: dmm_modelled_steps");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (count > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;
    const size_t smem = sizeof(uint32_t) * w * m;
    dmmdev::k_leaf_steps<<<unsigned(count), 32, smem, static_cast<cudaStream_t>(stream)>>>(in, w, m, count, domain,
                                                                                         steps);
    return dmmhost::check_launch("k_leaf_steps");
}

}  // extern "C"

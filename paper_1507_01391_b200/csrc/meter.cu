// meter.cu -- the reference's DMM step count (Machine::steps(), core.hpp rows_lockstep) where it
// depends on the data: the leaf of the general partition / integer sort, w <= m
// (partition.hpp:156-172), and the comparison sorts sort_short_wide / sort_square (below).
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
#include <string>

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

// ---- comparison sorts: sort_short_wide (sort.hpp:225) and sort_square (sort.hpp:337) --------
// Every row sort is sort_rows (row_merge_sort, data-dependent); conversions cost 4 m,
// transposes 2 (m - 1).  The square skeleton's super-row groups run in merged lockstep, which
// the reference meters as the longest group's own total (measured: the max over groups of the
// per-group sums, not the sum of per-section maxima).

constexpr int kSortMaxM = 64;

// accesses of row_merge_sort (sort.hpp:44-70) on x[0..L), direction asc; sorts x in place
__device__ uint32_t merge_row(uint32_t* x, uint32_t stride, uint32_t L, bool asc) {
    uint32_t a[kSortMaxM], b[kSortMaxM];
    for (uint32_t i = 0; i < L; ++i)
        a[i] = x[i * stride];
    uint32_t cost = 0, levels = 0;
    for (uint32_t width = 1; width < L; width *= 2, ++levels) {
        for (uint32_t lo = 0; lo < L; lo += 2 * width) {
            const uint32_t mid = min(lo + width, L), hi = min(lo + 2 * width, L);
            uint32_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi) {
                const bool take_a = asc ? a[i] <= a[j] : a[i] >= a[j];
                b[o++] = take_a ? a[i++] : a[j++];
                cost += 3;
            }
            while (i < mid) {
                b[o++] = a[i++];
                cost += 2;
            }
            while (j < hi) {
                b[o++] = a[j++];
                cost += 2;
            }
        }
        for (uint32_t i = 0; i < L; ++i)
            a[i] = b[i];
    }
    if (levels & 1)
        cost += 2 * L;
    for (uint32_t i = 0; i < L; ++i)
        x[i * stride] = a[i];
    return cost;
}

// short-wide skeleton (sort.hpp:200-218) on the h-row group starting at row g0 of the machine
// g (row stride m), direction dir; thread r = row g0 + lr; returns the group's total via red
__device__ void short_wide_group(uint32_t* g, uint32_t* tmp, uint32_t m, uint32_t h, uint32_t grp, uint32_t lr,
                                 bool active, bool dir, uint32_t* red, uint64_t* total) {
    uint32_t* base = g + grp * h * m;
    uint32_t* t = tmp + grp * h * m;
    auto rows = [&](bool alternate) {
        if (active)
            red[grp] = 0;
        __syncthreads();
        if (active) {
            const bool asc = alternate ? ((lr % 2 == 0) == dir) : dir;
            atomicMax(&red[grp], merge_row(base + lr * m, 1, m, asc));
        }
        __syncthreads();
        if (active && lr == 0)
            total[grp] += red[grp];
        __syncthreads();
    };
    auto convert = [&](bool to_col) {
        // to_column_major: row-major index v -> cell (v mod h, v div h); to_row_major inverse
        if (active)
            for (uint32_t c = 0; c < m; ++c) {
                const uint32_t v = lr * m + c;  // this thread moves its own row's cells
                if (to_col)
                    t[(v % h) * m + v / h] = base[v];
                else
                    t[v] = base[(v % h) * m + v / h];
            }
        __syncthreads();
        if (active)
            for (uint32_t c = 0; c < m; ++c)
                base[lr * m + c] = t[lr * m + c];
        if (active && lr == 0)
            total[grp] += 4ull * m;
        __syncthreads();
    };
    for (int pass = 0; pass < 2; ++pass) {
        rows(true);
        convert(true);
        rows(false);
        convert(false);
    }
    rows(false);
}

// kind 0: sort_short_wide (w^2 <= m, one group of w rows), 1: sort_square (w = m = h^2)
__global__ void k_sort_steps(const uint32_t* __restrict__ in, uint32_t W, uint32_t M, int kind,
                             uint64_t* __restrict__ steps) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t red[64];
    __shared__ uint64_t total[64];
    uint32_t* g = sm;
    uint32_t* tmp = sm + W * M;
    const uint32_t r = threadIdx.x;
    const bool row = r < W;
    const uint64_t k = blockIdx.x;
    for (uint32_t i = r; i < W * M; i += blockDim.x)
        g[i] = in[k * W * M + i];
    const uint32_t h = kind == 0 ? W : (uint32_t)sqrtf((float)M);
    const uint32_t ngroups = W / h;
    uint64_t acc = 0;
    auto super_rows = [&](bool alternate) {
        if (r < ngroups)
            total[r] = 0;
        __syncthreads();
        const uint32_t grp = r / h, lr = r % h;
        const bool dir = alternate ? (grp % 2 == 0) : true;
        short_wide_group(g, tmp, M, h, grp, lr, row, dir, red, total);
        if (r == 0) {
            uint64_t mx = 0;
            for (uint32_t q = 0; q < ngroups; ++q)
                mx = total[q] > mx ? total[q] : mx;
            acc += mx;
        }
        __syncthreads();
    };
    auto uniform_rows = [&](bool columns) {
        // columns: after a transpose row r is column r; sorting column r in place and
        // transposing back is the same state
        if (r == 0)
            red[0] = 0;
        __syncthreads();
        if (row)
            atomicMax(&red[0], columns ? merge_row(g + r, M, W, true) : merge_row(g + r * M, 1, M, true));
        __syncthreads();
        if (r == 0)
            acc += red[0] + (columns ? 4ull * (M - 1) : 0);
        __syncthreads();
    };
    __syncthreads();
    if (kind == 0) {
        super_rows(false);
    } else {
        super_rows(false);
        uniform_rows(true);
        super_rows(true);
        uniform_rows(true);
        uniform_rows(false);
    }
    if (r == 0)
        steps[k] = acc;
}

// ---- sort_tall (sort.hpp:352-374) -------------------------------------------------------------
// merge row sort, Batcher column network (4 m per round, data-independent), to_row_major,
// network, the m x m blocks' sort_wide_any in merged lockstep (metered as the longest block),
// network, merge row sort.  A block's sort_wide_any is the square skeleton with merge rows
// (m = h^2) or shearsort_rect with merge rows and segments; w = m is one block.

constexpr int kTallMaxW = 128, kTallMaxM = 32;

struct TallShared {
    uint32_t umax[kTallMaxW];  // per-unit section maximum
    uint64_t gtot[kTallMaxW];  // per-group totals (square skeleton super-rows)
    uint64_t btot[kTallMaxW];  // per-block totals
    uint64_t acc;
};

// one bank-local section: the unit's busiest row; `leader` rows add it to tot[unit]
__device__ void tally(TallShared& S, uint64_t* tot, uint32_t unit, bool leader, uint32_t cost) {
    atomicMax(&S.umax[unit], cost);
    __syncthreads();
    if (leader) {
        tot[unit] += S.umax[unit];
        S.umax[unit] = 0;
    }
    __syncthreads();
}

__device__ void convert_rows(uint32_t* base, uint32_t* tmp, uint32_t h, uint32_t m, uint32_t lr, bool to_col) {
    for (uint32_t c = 0; c < m; ++c) {
        const uint32_t v = lr * m + c;
        if (to_col)
            tmp[(v % h) * m + v / h] = base[v];
        else
            tmp[v] = base[(v % h) * m + v / h];
    }
    __syncthreads();
    for (uint32_t c = 0; c < m; ++c)
        base[lr * m + c] = tmp[lr * m + c];
    __syncthreads();
}

__global__ void k_tall_steps(const uint32_t* __restrict__ in, uint32_t W, uint32_t M, uint64_t* __restrict__ steps) {
    extern __shared__ uint32_t sm[];
    __shared__ TallShared S;
    uint32_t* g = sm;
    uint32_t* tmp = sm + W * M;
    const uint32_t r = threadIdx.x;  // row r (blockDim.x == W)
    const uint64_t k = blockIdx.x;
    for (uint32_t i = r; i < W * M; i += blockDim.x)
        g[i] = in[k * W * M + i];
    S.umax[r] = 0;
    S.gtot[r] = 0;
    S.btot[r] = 0;
    if (r == 0)
        S.acc = 0;
    __syncthreads();
    // whole-machine sections (unit 0)
    auto machine_rows = [&]() {
        tally(S, &S.acc, 0, r == 0, merge_row(g + r * M, 1, M, true));
        S.acc += 0;
    };
    auto network = [&]() {
        if (r < M)
            insertion_sort(g + r, W, M, true);
        __syncthreads();
        if (r == 0) {
            uint32_t rounds = 0;
            for (uint32_t p = 1; p < W; p <<= 1)
                for (uint32_t kk = p; kk >= 1; kk >>= 1) {
                    bool any = false;
                    for (uint32_t j = kk % p; j + kk < W && !any; j += 2 * kk)
                        for (uint32_t i = 0; i < kk && i + j + kk < W; ++i)
                            if ((i + j) / (2 * p) == (i + j + kk) / (2 * p)) {
                                any = true;
                                break;
                            }
                    rounds += any;
                    if (kk == 1)
                        break;
                }
            S.acc += 4ull * M * rounds;
        }
        __syncthreads();
    };
    const bool tall = W > M;
    if (tall) {
        machine_rows();
        network();
        // to_row_major of the w x m machine (layout.hpp:403): u = j w + i -> (u / m, u % m)
        for (uint32_t c = 0; c < M; ++c) {
            const uint32_t v = r * M + c;
            tmp[v] = g[(v % W) * M + v / W];
        }
        __syncthreads();
        for (uint32_t c = 0; c < M; ++c)
            g[r * M + c] = tmp[r * M + c];
        if (r == 0 && M > 1)
            S.acc += 4ull * M;
        __syncthreads();
        network();
    }
    // the m x m blocks (one when w = m): sort_wide_any(block b, b even or w = m)
    {
        const uint32_t b = r / M, lr = r % M;
        const bool d = !tall || b % 2 == 0;
        uint32_t* blk = g + b * M * M;
        uint32_t* tb = tmp + b * M * M;
        const bool bl = lr == 0;
        const uint32_t h = (uint32_t)sqrtf((float)M);
        if (M == 1) {
            // 1 x 1: nothing moves, conversions of a single row are free
        } else if (h * h == M) {
            // square skeleton (sort.hpp:250-280) with merge rows; groups of h rows in lockstep
            const uint32_t q = lr / h, lq = lr % h;
            const uint32_t gid = b * (M / h) + q;
            uint32_t* gb = blk + q * h * M;
            uint32_t* gt = tb + q * h * M;
            for (int pass = 0; pass < 2; ++pass) {
                const bool dir = pass == 0 ? d : ((q % 2 == 0) == d);
                for (int sw = 0; sw < 2; ++sw) {
                    tally(S, S.gtot, gid, lq == 0, merge_row(gb + lq * M, 1, M, (lq % 2 == 0) == dir));
                    convert_rows(gb, gt, h, M, lq, true);
                    tally(S, S.gtot, gid, lq == 0, merge_row(gb + lq * M, 1, M, dir));
                    convert_rows(gb, gt, h, M, lq, false);
                }
                tally(S, S.gtot, gid, lq == 0, merge_row(gb + lq * M, 1, M, dir));
                if (lq == 0)
                    S.gtot[gid] += 4 * 4ull * M;
                __syncthreads();
                if (bl) {  // the block's super-rows: its longest group
                    uint64_t mx = 0;
                    for (uint32_t qq = 0; qq < M / h; ++qq)
                        mx = max(mx, S.gtot[b * (M / h) + qq]);
                    S.btot[b] += mx;
                }
                __syncthreads();
                if (lq == 0)
                    S.gtot[gid] = 0;
                // columns of a square block: transpose, merge rows, transpose
                tally(S, S.btot, b, bl, merge_row(blk + lr, M, M, d));
                if (bl)
                    S.btot[b] += 4ull * (M - 1);
                __syncthreads();
            }
            tally(S, S.btot, b, bl, merge_row(blk + lr * M, 1, M, d));
        } else {
            // shearsort_rect (sort.hpp:288-311) with merge rows and merge segments
            uint32_t rounds = 1;
            while ((1u << (rounds - 1)) < M)
                ++rounds;
            for (uint32_t it = 0; it < rounds; ++it) {
                tally(S, S.btot, b, bl, merge_row(blk + lr * M, 1, M, (lr % 2 == 0) == d));
                tally(S, S.btot, b, bl, merge_row(blk + lr, M, M, d));  // the block's column lr
                if (bl)
                    S.btot[b] += 4ull * (M - 1);
                __syncthreads();
            }
            tally(S, S.btot, b, bl, merge_row(blk + lr * M, 1, M, (lr % 2 == 0) == d));
            if (((lr % 2 == 0) == d) != d)  // odd-row reversal into row-major order
                for (uint32_t c = 0; c < M / 2; ++c) {
                    const uint32_t t = blk[lr * M + c];
                    blk[lr * M + c] = blk[lr * M + M - 1 - c];
                    blk[lr * M + M - 1 - c] = t;
                }
            if (bl)
                S.btot[b] += 4ull * (M / 2);
            __syncthreads();
        }
        if (r == 0) {
            uint64_t mx = 0;
            for (uint32_t bb = 0; bb < W / M; ++bb)
                mx = max(mx, S.btot[bb]);
            S.acc += mx;
        }
        __syncthreads();
    }
    if (tall) {
        network();
        machine_rows();
    }
    if (r == 0)
        steps[k] = S.acc;
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

dmm_status dmm_sort_steps(const char* algorithm, const uint32_t* in, uint32_t w, uint32_t m, uint64_t count,
                          uint64_t* steps, void* stream) {
    dmmhost::reset_launches();
    if (!algorithm)
        return DMM_INVALID_ARGUMENT;
    const std::string a(algorithm);
    const uint32_t h = dmmhost::isqrt_floor(m);
    int kind = -1;
    if (a == "sort_short_wide" && w >= 2 && uint64_t(w) * w <= m && m <= dmmdev::kSortMaxM)
        kind = 0;
    else if (a == "sort_square" && w == m && h * h == m && w >= 2 && m <= dmmdev::kSortMaxM)
        kind = 1;
    else if (a == "sort_tall" && w >= m && m >= 1 && w % m == 0 && w <= dmmdev::kTallMaxW &&
             m <= dmmdev::kTallMaxM && (w == 32 || w == 64 || w == 128 || w == m))
        kind = 2;
    if (kind < 0) {
        dmmhost::set_error("sort metering: sort_short_wide (w^2 <= m <= 64), sort_square (w = m = h^2 <= 64) or "
                           "sort_tall (m | w, w in {32, 64, 128} or w = m <= 32)");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (count == 0)
        return DMM_OK;
    if (!in || !steps || count > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;
    const size_t smem = 2 * sizeof(uint32_t) * w * m;
    if (kind == 2) {
        static std::atomic<uint64_t> tall_configured{0};
        if (dmm_status e = dmmhost::configure_kernel(dmmdev::k_tall_steps, smem, tall_configured); e != DMM_OK)
            return e;
        dmmdev::k_tall_steps<<<unsigned(count), w, smem, static_cast<cudaStream_t>(stream)>>>(in, w, m, steps);
        return dmmhost::check_launch("k_tall_steps");
    }
    const unsigned threads = w <= 32 ? 32 : 64;
    static std::atomic<uint64_t> configured{0};
    if (dmm_status e = dmmhost::configure_kernel(dmmdev::k_sort_steps, smem, configured); e != DMM_OK)
        return e;
    dmmdev::k_sort_steps<<<unsigned(count), threads, smem, static_cast<cudaStream_t>(stream)>>>(in, w, m, kind,
                                                                                              steps);
    return dmmhost::check_launch("k_sort_steps");
}

}  // extern "C"

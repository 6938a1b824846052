// general_meter.cuh -- the reference's DMM step count (Machine::steps()) for the general
// partition / integer sort recursion, w > m (partition.hpp:363-428 balance_divide_sort).
//
// The recursion's step count depends on the data through its shearsort and w < m square
// leaves (merge-sorted bank segments in the blocked column sorts, sort.hpp:44-70, 162-174) and
// through the checked cleanup's retry loop.  Every leaf sort, balancing sort and relayout has a
// unique outcome (a partition_leaf leaves its block sorted row-major), so the states the
// reference passes through are reproduced here with plain sorts and index maps, and each
// section is charged the reference's access count:
//   * lockstep(count, branch) (core.hpp:337-349) advances by the longest branch's own total;
//   * a bank-local section (rows_lockstep) by its busiest row;
//   * radix row sort of m keys < domain: p passes of 10 m, + 2 m when p is odd
//     (partition.hpp:24-85); conversions 4 m (layout.hpp:316-405), 0 when w or m is 1, a
//     transpose when w = m; transpose_square 2 (s - 1) (layout.hpp:24-61);
//   * scan_sorted (partition.hpp:308-337): m + 3 + 4 ceil(log2 w) (row scan, boundary peek, flag
//     write, tree_reduce_sum and broadcast_value, core.hpp:544-634).
// The same code runs on the host (tests/cpp) and on the device, one thread per instance, over a
// private workspace: off the hot path, a meter only.
#pragma once
#include <cmath>
#include <cstdint>

#ifndef DMM_HD
#ifdef __CUDACC__
#define DMM_HD __host__ __device__
#else
#define DMM_HD
#endif
#endif

namespace dmmmeter {

DMM_HD inline uint32_t ceil_log2(uint64_t x) {
    uint32_t l = 0;
    while ((uint64_t(1) << l) < x)
        ++l;
    return l;
}

DMM_HD inline uint32_t isqrt(uint32_t x) {
    uint32_t r = 0;
    while (uint64_t(r + 1) * (r + 1) <= x)
        ++r;
    return r;
}

DMM_HD inline uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// general_sort_shape_ok (partition.hpp:133-152)
DMM_HD inline bool shape_ok(uint64_t W, uint64_t M) {
    for (;;) {
        if (W <= 1)
            return true;
        if (W <= M) {
            const uint64_t h = isqrt(uint32_t(M));
            return W * W <= M || (h * h == M && W % h == 0) || (M % W == 0);
        }
        if (M < 2 || W % M != 0)
            return false;
        uint64_t nsubs = W;
        while (nsubs > 1) {
            const uint64_t g = nsubs < M ? nsubs : M;
            if (g < M && g * g > M)
                return false;
            if (nsubs % g != 0)
                return false;
            nsubs /= g;
        }
        W /= M;
    }
}

// PartitionParams::compute (partition.hpp:203-226): subproblem count m d, 0 if infeasible
DMM_HD inline uint32_t subproblems(uint32_t W, uint32_t M) {
    const double lg = log(double(W)) / log(double(M));
    const double want_d = ceil(2 * lg - 1e-9);
    uint32_t want = want_d < 1 ? 1u : uint32_t(want_d);
    uint32_t d = want < W / M ? want : W / M;
    while (uint64_t(M) * d <= W && (W % (uint64_t(M) * d) != 0 || !shape_ok(W / (uint64_t(M) * d), M)))
        ++d;
    if (uint64_t(M) * d > W || W % (uint64_t(M) * d) != 0)
        return 0;
    return M * d;
}

// Sorts and index maps on a row-major W x M block.
DMM_HD inline void shell_sort(uint32_t* x, uint32_t n, bool asc) {
    uint32_t gap = 1;
    while (gap < n / 3)
        gap = 3 * gap + 1;
    for (; gap > 0; gap /= 3)
        for (uint32_t i = gap; i < n; ++i) {
            const uint32_t v = x[i];
            uint32_t j = i;
            while (j >= gap && (asc ? x[j - gap] > v : x[j - gap] < v)) {
                x[j] = x[j - gap];
                j -= gap;
            }
            x[j] = v;
        }
}

struct Meter {
    uint32_t M;
    uint64_t R;           // one radix row sort (base M, keys < domain)
    uint32_t* tmp;        // W x M relayout buffer (shared down the recursion)
    uint32_t* gather;     // M x M assembled view
    uint32_t* ma;         // merge buffers, >= M words each
    uint32_t* mb;
    uint32_t retries;     // GeneralStats::cleanup_retries

    DMM_HD static uint64_t radix_cost(uint32_t m, uint64_t domain) {
        uint32_t p = 1;
        for (uint64_t reach = m; reach < domain; reach *= m)
            ++p;
        return 10ull * m * p + ((p & 1) ? 2ull * m : 0);
    }

    // row_merge_sort (sort.hpp:44-70) of x[0..L) (stride s), ascending: accesses; sorts x
    DMM_HD uint64_t merge(uint32_t* x, uint32_t s, uint32_t L) {
        for (uint32_t i = 0; i < L; ++i)
            ma[i] = x[i * s];
        uint64_t cost = 0;
        uint32_t levels = 0;
        uint32_t *a = ma, *b = mb;
        for (uint32_t width = 1; width < L; width *= 2, ++levels) {
            for (uint32_t lo = 0; lo < L; lo += 2 * width) {
                const uint32_t mid = lo + width < L ? lo + width : L;
                const uint32_t hi = lo + 2 * width < L ? lo + 2 * width : L;
                uint32_t i = lo, j = mid, o = lo;
                while (i < mid && j < hi) {
                    b[o++] = a[i] <= a[j] ? a[i++] : a[j++];
                    cost += 3;
                }
                cost += 2ull * (mid - i + hi - j);
                while (i < mid)
                    b[o++] = a[i++];
                while (j < hi)
                    b[o++] = a[j++];
            }
            uint32_t* t = a;
            a = b;
            b = t;
        }
        if (levels & 1)
            cost += 2ull * L;
        for (uint32_t i = 0; i < L; ++i)
            x[i * s] = a[i];
        return cost;
    }

    // sort_columns_blocked with merge segments (sort.hpp:162-182): bank r merges the columns
    // r, W + r, ...; the section costs the busiest bank; every column ends ascending
    DMM_HD uint64_t blocked_columns(uint32_t* g, uint32_t W) {
        if (W <= 1)
            return 0;
        uint64_t busiest = 0;
        for (uint32_t r = 0; r < W; ++r) {
            uint64_t mine = 0;
            for (uint32_t c = r; c < M; c += W)
                mine += merge(g + c, M, W);
            busiest = umax64(busiest, mine);
        }
        return busiest + 2ull * (M / W) * 2 * (W - 1);
    }

    DMM_HD static void sort_rows(uint32_t* g, uint32_t W, uint32_t M, bool alternate) {
        for (uint32_t r = 0; r < W; ++r)
            shell_sort(g + r * M, M, !alternate || r % 2 == 0);
    }

    // detail::partition_leaf (partition.hpp:156-172), ascending, W <= M
    DMM_HD uint64_t leaf(uint32_t* g, uint32_t W) {
        uint64_t total = 0;
        const uint32_t h = isqrt(M);
        if (uint64_t(W) * W <= M) {
            // short_wide_skeleton (sort.hpp:200-218): 5 row sorts, 4 conversions
            total = 5 * R + (W > 1 ? 16ull * M : 0);
        } else if (h * h == M && W % h == 0) {
            if (W == M) {
                // square_skeleton, w = m: 13 row sorts, 8 conversions, 4 transposes
                total = 13 * R + 32ull * M + 8ull * (M - 1);
            } else {
                // square_skeleton, w < m (sort.hpp:250-280)
                for (int pass = 0; pass < 2; ++pass) {
                    for (uint32_t grp = 0; grp < W / h; ++grp)
                        shell_sort(g + grp * h * M, h * M, pass == 0 || grp % 2 == 0);
                    total += 5 * R + 16ull * M;
                    total += blocked_columns(g, W);
                }
                total += R;
            }
        } else {
            // shearsort_rect (sort.hpp:288-311)
            const uint32_t rounds = ceil_log2(W) + 1;
            for (uint32_t i = 0; i < rounds; ++i) {
                sort_rows(g, W, M, true);
                total += R;
                total += blocked_columns(g, W);
            }
            total += R + (W > 1 ? 2ull * M : 0);
        }
        shell_sort(g, W * M, true);
        return total;
    }

    // to_row_major of a W x M block (W > M, M | W): column-major index u = j W + i -> row-major u
    DMM_HD void to_row_major(uint32_t* g, uint32_t W) {
        for (uint32_t i = 0; i < W; ++i)
            for (uint32_t j = 0; j < M; ++j)
                tmp[uint64_t(j) * W + i] = g[i * M + j];
        for (uint64_t u = 0; u < uint64_t(W) * M; ++u)
            g[u] = tmp[u];
    }

    // to_column_major: row-major index v -> cell (v mod W, v div W)
    DMM_HD void to_column_major(uint32_t* g, uint32_t W) {
        for (uint64_t v = 0; v < uint64_t(W) * M; ++v)
            tmp[(v % W) * M + v / W] = g[v];
        for (uint64_t u = 0; u < uint64_t(W) * M; ++u)
            g[u] = tmp[u];
    }

    // balance (partition.hpp:234-271) of a W x M block
    DMM_HD uint64_t balance(uint32_t* g, uint32_t W) {
        uint64_t total = 0;
        uint32_t sub_h = 1, nsubs = W;
        while (nsubs > 1) {
            const uint32_t gs = nsubs < M ? nsubs : M;
            uint64_t round = 0;
            for (uint32_t grp = 0; grp < nsubs / gs; ++grp)
                for (uint32_t j = 0; j < sub_h; ++j) {
                    for (uint32_t s = 0; s < gs; ++s)
                        for (uint32_t c = 0; c < M; ++c)
                            gather[s * M + c] = g[((grp * gs + s) * sub_h + j) * M + c];
                    uint64_t c;
                    if (gs == M) {
                        c = leaf(gather, M) + 2ull * (M - 1);
                        for (uint32_t a = 0; a < M; ++a)
                            for (uint32_t b = a + 1; b < M; ++b) {
                                const uint32_t t = gather[a * M + b];
                                gather[a * M + b] = gather[b * M + a];
                                gather[b * M + a] = t;
                            }
                    } else {
                        // short-wide skeleton with radix rows, then to_column_major
                        c = 5 * R + 16ull * M + 4ull * M;
                        shell_sort(gather, gs * M, true);
                        for (uint64_t v = 0; v < uint64_t(gs) * M; ++v)
                            tmp[(v % gs) * M + v / gs] = gather[v];
                        for (uint64_t u = 0; u < uint64_t(gs) * M; ++u)
                            gather[u] = tmp[u];
                    }
                    round = umax64(round, c);
                    for (uint32_t s = 0; s < gs; ++s)
                        for (uint32_t c2 = 0; c2 < M; ++c2)
                            g[((grp * gs + s) * sub_h + j) * M + c2] = gather[s * M + c2];
                }
            total += round;
            sub_h *= gs;
            nsubs /= gs;
        }
        return total;
    }

    // cleanup_pass_pair (partition.hpp:341-361)
    DMM_HD uint64_t cleanup(uint32_t* g, uint32_t W) {
        uint64_t aligned = 0;
        for (uint32_t k = 0; k < W / M; ++k)
            aligned = umax64(aligned, leaf(g + uint64_t(k) * M * M, M));
        uint64_t shifted = 0;
        if (W > M && M >= 2) {
            shifted = leaf(g, M / 2);
            uint32_t lo = M / 2;
            for (; lo + M <= W; lo += M)
                shifted = umax64(shifted, leaf(g + uint64_t(lo) * M, M));
            shifted = umax64(shifted, leaf(g + uint64_t(W - M / 2) * M, M / 2));
        }
        return aligned + shifted;
    }

    // balance_divide_sort (partition.hpp:363-428) of a W x M block; 0 with ok = false when the
    // reference would throw ShapeViolation / DivisibilityViolation
    DMM_HD uint64_t sort(uint32_t* g, uint32_t W, bool& ok) {
        if (W <= M)
            return leaf(g, W);
        if (W % M != 0) {
            ok = false;
            return 0;
        }
        uint64_t total = 0;
        uint32_t h = W;
        while (h > M) {
            uint64_t bal = 0;
            for (uint32_t k = 0; k < W / h; ++k)
                bal = umax64(bal, balance(g + uint64_t(k) * h * M, h));
            total += bal;
            const uint32_t sp = subproblems(h, M);
            if (sp == 0) {
                ok = false;
                return 0;
            }
            for (uint32_t k = 0; k < W / h; ++k)
                to_row_major(g + uint64_t(k) * h * M, h);
            total += 4ull * M;
            h /= sp;
        }
        uint64_t leaves = 0;
        for (uint32_t k = 0; k < W / h; ++k)
            leaves = umax64(leaves, leaf(g + uint64_t(k) * h * M, h));
        total += leaves;

        to_row_major(g, W);
        total += 4ull * M;
        const uint32_t ch = W / M;
        uint64_t cols = 0;
        for (uint32_t k = 0; k < M; ++k)
            cols = umax64(cols, sort(g + uint64_t(k) * ch * M, ch, ok));
        total += cols;
        to_column_major(g, W);
        total += 4ull * M;

        const uint64_t scan = M + 3 + 4ull * ceil_log2(W);
        total += cleanup(g, W) + scan;
        const uint32_t budget = ceil_log2(W);
        uint32_t tries = 0;
        while (!is_sorted(g, W) && tries < budget) {
            total += cleanup(g, W) + scan;
            ++tries;
        }
        retries = tries > retries ? tries : retries;
        return total;
    }

    DMM_HD bool is_sorted(const uint32_t* g, uint32_t W) const {
        for (uint64_t i = 1; i < uint64_t(W) * M; ++i)
            if (g[i - 1] > g[i])
                return false;
        return true;
    }
};

// words of private workspace one instance needs (besides its own W x M copy)
DMM_HD inline uint64_t workspace_words(uint32_t W, uint32_t M) {
    return uint64_t(W) * M + uint64_t(M) * M + 2ull * (W > M ? W : M);
}

// Machine::steps() of integer_sort_general / partition_general on the W x M block g (sorted in
// place); retries = GeneralStats::cleanup_retries.  0 when the shape is rejected.
DMM_HD inline uint64_t general_steps(uint32_t* g, uint32_t W, uint32_t M, uint64_t domain, uint32_t* ws,
                                     uint32_t* retries) {
    Meter mt;
    mt.M = M;
    mt.R = Meter::radix_cost(M, domain);
    mt.tmp = ws;
    mt.gather = ws + uint64_t(W) * M;
    mt.ma = mt.gather + uint64_t(M) * M;
    mt.mb = mt.ma + (W > M ? W : M);
    mt.retries = 0;
    bool ok = shape_ok(W, M) && (W <= M || M >= 2);
    const uint64_t s = ok ? mt.sort(g, W, ok) : 0;
    *retries = mt.retries;
    return ok ? s : 0;
}

}  // namespace dmmmeter

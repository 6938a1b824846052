// dmm_algos.cuh -- the reference's sort / partition schedules as warp programs.
//
// Each template below restates one function of /root/reference/proj/include/dmm/
// {sort,partition}.hpp step for step (same row sorts in the same directions, same
// relayouts, same view decomposition), so the matrix after every step equals the
// reference's.  Shapes are compile-time: W = 32 (one warp), M = register row width.
//
// Outcome-preserving rewrites (the state after the rewritten block is identical):
//   * shearsort_rect's final "alternating row sort + reversal of the descending rows"
//     (sort.hpp:299-310) is one row sort in direction asc;
//   * short_wide_skeleton on a one-row view (W = 1) is one row sort: its conversions
//     are no-ops (layout.hpp:359) and all five sorts run in direction asc;
//   * every blocked column sort transposes all its W x W column blocks in one
//     relayout (the blocks are disjoint; sort.hpp:169-173).
#pragma once

#include "dmm_device.cuh"

#ifndef DMM_BLOCK_SHFL_LEVELS
#define DMM_BLOCK_SHFL_LEVELS 1  // 32 x 32 block sorts: merge levels whose row-bit stages run as shuffles
#endif
constexpr int kBlockShflLevels = DMM_BLOCK_SHFL_LEVELS;
#ifndef DMM_COMPACT_WARP_BLOCKS
#define DMM_COMPACT_WARP_BLOCKS 1  // one-warp 32 x 32 block sorts use the looped form too (+3 % cfg1)
#endif

namespace dmmdev {

// ---------------------------------------------------------------------------
// Shape predicates (compile-time twins of partition.hpp:133-152 / :209-225)
// ---------------------------------------------------------------------------
__host__ __device__ constexpr bool square_fits_c(int W, int M) { /* sort.hpp:313 */
    const int h = isqrt_c(M);
    return h * h == M && W <= M && W % h == 0;
}

__host__ __device__ constexpr bool general_shape_ok_c(long W, long M, bool ext) {
    if (W <= 1)
        return true;
    if (W <= M) {
        const long h = isqrt_c((int)M);
        return W * W <= M || (h * h == M && W % h == 0) || (M % W == 0);
    }
    if (M < 2 || W % M != 0)
        return false;
    long nsubs = W;
    while (nsubs > 1) {
        const long g = M < nsubs ? M : nsubs;
        if (g < M && g * g > M && (!ext || M % g != 0))
            return false;
        if (nsubs % g != 0)
            return false;
        nsubs /= g;
    }
    return general_shape_ok_c(W / M, M, ext);
}

struct PParams {
    int rounds, d, subproblems;
};
// PartitionParams::compute for power-of-two W, M: log_m w = lgW / lgM exactly, so
// ceil(x - 1e-9) is the integer ceiling (the host asserts equality with the
// double-precision reference formula before every launch).
__host__ __device__ constexpr PParams pparams_c(int W, int M, bool ext) {
    const int a = ilog2_ceil_c(W), b = ilog2_ceil_c(M);
    PParams p{(a + b - 1) / b, 0, 0};
    int want = (2 * a + b - 1) / b;
    if (want < 1)
        want = 1;
    int d = want < W / M ? want : W / M;
    while ((long)M * d <= W && (W % (M * d) != 0 || !general_shape_ok_c(W / (M * d), M, ext)))
        ++d;
    p.d = d;
    p.subproblems = M * d;
    return p;
}

// PartitionProbe (partition.hpp:298-301) capture: the full working window after every
// balance (after_balance) and every convert-and-divide (after_divide) of the OUTER
// recursion, in the order the reference calls its hooks.  Each lane stores its row of
// the window; with PK = 2 each 16-bit half goes to its own instance's snapshot area.
struct ProbeSink {
    uint32_t* dst[2];  // per half: this instance's snapshot area (max x WM x M words) or null
    uint32_t n, max;
    int row, wm;
    template <int PK, int M>
    __device__ __forceinline__ void capture(const uint32_t (&x)[M]) {
        if (n < max) {
#pragma unroll
            for (int h = 0; h < PK; ++h) {
                if (dst[h] == nullptr)
                    continue;
                uint32_t* q = dst[h] + ((size_t)n * wm + row) * M;
#pragma unroll
                for (int c = 0; c < M; ++c)
                    q[c] = PK == 2 ? ((x[c] >> (16 * h)) & 0xFFFFu) : x[c];
            }
        }
        ++n;
    }
};

// ---------------------------------------------------------------------------
// Column sorts and skeletons  sort.hpp:162-311
// ---------------------------------------------------------------------------
// sort_columns_blocked sort.hpp:162-174 (segment sorter: merge_sort_segments)
template <int PK, class V, int M>
__device__ __forceinline__ void sort_columns_blocked(uint32_t (&x)[M], uint32_t* buf, int lane, bool asc) {
    static_assert(V::MV % V::WV == 0, "blocked column sort needs W | M (DivisibilityViolation)");
    if constexpr (V::WV > 1) {
        transpose_blocks<V>(x, buf, lane);
        seg_sort<PK, V, V::WV>(x, lane, asc);
        transpose_blocks<V>(x, buf, lane);
    }
}

// short_wide_skeleton sort.hpp:200-218 (Lemma 1); asc may differ per lane (per view)
// ps: ShortWideHook capture (sort.hpp:189-218): after_first_convert, after_first_pass, done
template <int PK, class V, int M>
__device__ __forceinline__ void short_wide(uint32_t (&x)[M], uint32_t* buf, int lane, bool asc,
                                           ProbeSink* ps = nullptr) {
    static_assert(V::WV * V::WV <= V::MV, "short-wide needs w^2 <= m (ShapeViolation)");
    if constexpr (V::WV == 1) {
        row_sort<PK, V>(x, lane, asc);
        if (ps) {  // conversions of a one-row view are no-ops: every stage sees the sorted row
            ps->template capture<PK>(x);
            ps->template capture<PK>(x);
            ps->template capture<PK>(x);
        }
    } else {
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
            row_sort<PK, V>(x, lane, alt_dir<V>(lane, asc));
            to_column_major<V>(x, buf, lane);
            if (ps && pass == 0)
                ps->template capture<PK>(x);  // ShortWideStage::after_first_convert
            row_sort<PK, V>(x, lane, asc);
            to_row_major<V>(x, buf, lane);
            if (ps && pass == 0)
                ps->template capture<PK>(x);  // ShortWideStage::after_first_pass
        }
        row_sort<PK, V>(x, lane, asc);
        if (ps)
            ps->template capture<PK>(x);  // ShortWideStage::done
    }
}

// square_skeleton's columns() sort.hpp:266-273
template <int PK, class V, int M>
__device__ __forceinline__ void square_columns(uint32_t (&x)[M], uint32_t* buf, int lane, bool asc) {
    if constexpr (V::WV == V::MV) {  // square_column_sort sort.hpp:240-244
        transpose_square<V>(x, buf, lane);
        row_sort<PK, V>(x, lane, asc);
        transpose_square<V>(x, buf, lane);
    } else {
        sort_columns_blocked<PK, V>(x, buf, lane, asc);
    }
}

// square_skeleton sort.hpp:250-280 (Theorem 2)
template <int PK, class V, int M>
__device__ __forceinline__ void square_skeleton(uint32_t (&x)[M], uint32_t* buf, int lane, bool asc) {
    constexpr int h = isqrt_c(V::MV);
    static_assert(h * h == V::MV && V::WV <= V::MV && V::WV % h == 0,
                  "square skeleton needs perfect-square M and sqrt(M) | W <= M (ShapeViolation)");
    using G = VRows<V, h>;  // super-rows in merged lockstep
    short_wide<PK, G>(x, buf, lane, asc);  // super_rows(false)
    square_columns<PK, V>(x, buf, lane, asc);
    const int g = V::local(lane) / h;
    short_wide<PK, G>(x, buf, lane, ((g % 2) == 0) == asc);  // super_rows(true)
    square_columns<PK, V>(x, buf, lane, asc);
    row_sort<PK, V>(x, lane, asc);
}

// shearsort_rect sort.hpp:288-311
template <int PK, class V, int M>
__device__ __forceinline__ void shearsort_rect(uint32_t (&x)[M], uint32_t* buf, int lane, bool asc) {
    static_assert(V::WV <= V::MV && (V::WV == 1 || V::MV % V::WV == 0),
                  "shearsort fallback needs W <= M and W | M (ShapeViolation)");
    constexpr int rounds = ilog2_ceil_c(V::WV) + 1;
#pragma unroll 1
    for (int i = 0; i < rounds; ++i) {
        row_sort<PK, V>(x, lane, alt_dir<V>(lane, asc));
        if constexpr (V::WV > 1)
            sort_columns_blocked<PK, V>(x, buf, lane, asc);
    }
    row_sort<PK, V>(x, lane, asc);  // alternating sort + odd-row reversal, sort.hpp:299-310
}

// sort_wide_any sort.hpp:321-330 (comparison sorter, W <= M, W | M)
template <int PK, class V, int M>
__device__ __forceinline__ void sort_wide_any(uint32_t (&x)[M], uint32_t* buf, int lane, bool asc,
                                              ProbeSink* ps = nullptr) {
    if constexpr (V::WV * V::WV <= V::MV)
        short_wide<PK, V>(x, buf, lane, asc, ps);
    else if constexpr (square_fits_c(V::WV, V::MV))
        square_skeleton<PK, V>(x, buf, lane, asc);
    else
        shearsort_rect<PK, V>(x, buf, lane, asc);
}

// ---------------------------------------------------------------------------
// Block sort: bitonic network over a whole view (WV lanes x MV registers) into
// row-major order.  Element e = local_row * MV + c has bits [r | q | l]: r = low
// log2(WV) register bits, q = the remaining register bits, l = the local row.
// Stages on r/q bits are register-local; stages on l bits run after a
// conflict-free blocked transpose (which turns l into register bits).  A comparator's
// direction is bit kc of e: static when that bit is a register bit, otherwise the
// whole lane flips its keys (x ^= ~0 reverses the order) around the stages.
// ---------------------------------------------------------------------------
// stages jb = JB..0 on registers [OFF, OFF+N): pairs (p, p ^ 2^jb); ascending iff
// DIRBIT < 0 or bit DIRBIT of p is clear
template <int PK, int OFF, int N, int JB, int DIRBIT, int M>
__device__ __forceinline__ void reg_stages(uint32_t (&x)[M]) {
    if constexpr (JB >= 0) {
        static_for<0, N>([&](auto pc) {
            constexpr int p = decltype(pc)::value;
            if constexpr (((p >> JB) & 1) == 0) {
                constexpr int I = p & ((1 << JB) - 1) | ((p >> (JB + 1)) << JB);  // comparator index
                if constexpr (DIRBIT < 0 || ((p >> DIRBIT) & 1) == 0)
                    Key<PK>::template cx<I>(x[OFF + p], x[OFF + (p | (1 << JB))]);
                else
                    Key<PK>::template cx<I>(x[OFF + (p | (1 << JB))], x[OFF + p]);
            }
        });
        reg_stages<PK, OFF, N, JB - 1, DIRBIT>(x);
    }
}

// a single ascending stage jb on registers [OFF, OFF+N): pairs (p, p ^ 2^jb)
template <int PK, int OFF, int N, int JB, int M>
__device__ __forceinline__ void reg_stage(uint32_t (&x)[M]) {
    static_for<0, N>([&](auto pc) {
        constexpr int p = decltype(pc)::value;
        if constexpr (((p >> JB) & 1) == 0) {
            constexpr int I = p & ((1 << JB) - 1) | ((p >> (JB + 1)) << JB);
            Key<PK>::template cx<I>(x[OFF + p], x[OFF + (p | (1 << JB))]);
        }
    });
}

// l-bit stages of merge level KC in the transposed layout, for every group of WV
// registers (group QI = one value of the q bits; l bits are the group's low bits)
template <int PK, class V, int KC, int QI, int M>
__device__ __forceinline__ void tstages_q(uint32_t (&x)[M]) {
    constexpr int R = ilog2_ceil_c(V::WV), QB = ilog2_ceil_c(V::MV / V::WV), NB = 2 * R + QB;
    if constexpr (QI < V::MV / V::WV) {
        reg_stages<PK, V::C0 + QI * V::WV, V::WV, KC - 1 - (R + QB), (KC < NB ? KC - R - QB : -1)>(x);
        tstages_q<PK, V, KC, QI + 1>(x);
    }
}

// bitonic merge levels KC .. KEND of the block sort (KEND defaults to the last level)
template <int PK, class V, int KC, int KEND = -1, int M>
__device__ __forceinline__ void block_merge_levels(uint32_t (&x)[M], uint32_t* buf, int lane) {
    constexpr int R = ilog2_ceil_c(V::WV), QB = ilog2_ceil_c(V::MV / V::WV), NB = 2 * R + QB;
    constexpr int LAST = KEND < 0 ? NB : KEND;
    if constexpr (KC <= LAST) {
        if constexpr (KC < R + QB) {
            // the whole merge lives in the lane's registers; direction bit KC is a register bit
            if (V::active(lane))
                reg_stages<PK, V::C0, V::MV, KC - 1, KC>(x);
        } else {
            if constexpr (KC > R + QB) {
                // l-bit stages jb = KC-1 .. R+QB in the transposed layout (l = low register bits)
                transpose_blocks<V>(x, buf, lane);
                if (V::active(lane))
                    tstages_q<PK, V, KC, 0>(x);
                transpose_blocks<V>(x, buf, lane);
            }
            // r/q-bit stages in the row layout; direction bit KC is an l bit: per lane
            if (V::active(lane)) {
                uint32_t f = 0;
                if constexpr (KC < NB)
                    f = ((V::local(lane) >> (KC - R - QB)) & 1) ? 0xFFFFFFFFu : 0u;
                flip<V::C0, V::MV>(x, f);
                reg_stages<PK, V::C0, V::MV, R + QB - 1, -1>(x);
                flip<V::C0, V::MV>(x, f);
            }
        }
        block_merge_levels<PK, V, KC + 1, KEND>(x, buf, lane);
    }
}

// ascending stages js..0 over registers [C0, C0 + N) (pairs (p, p ^ 2^j)), js < log2(N)
// chosen at runtime; each case is one straight-line sequence, so register renaming only has
// to be undone once per sequence (a per-stage switch cost N / 2 moves per stage)
template <int PK, int C0 = 0, int N = 32, int M>
__device__ __forceinline__ void stages_down(uint32_t (&x)[M], int js) {
    static_assert(N == 8 || N == 16 || N == 32 || N == 64, "stage sequences for 8..64 registers");
    switch (js) {
        case 0: reg_stages<PK, C0, N, 0, -1>(x); break;
        case 1: reg_stages<PK, C0, N, 1, -1>(x); break;
        case 2: reg_stages<PK, C0, N, 2, -1>(x); break;
        default:
            if constexpr (N >= 16) {
                if (js == 3) {
                    reg_stages<PK, C0, N, 3, -1>(x);
                    break;
                }
            }
            if constexpr (N >= 32) {
                if (js == 4) {
                    reg_stages<PK, C0, N, 4, -1>(x);
                    break;
                }
            }
            if constexpr (N >= 64)
                reg_stages<PK, C0, N, 5, -1>(x);
            break;
    }
}

// The square (WV = MV = 2^L) block sort with levels L+1 .. 2L as passes of one runtime loop over
// shared stage bodies (the tile sort's structure): flip the rows whose direction bit (local row
// bit level - L) is set, transpose / row-bit stages / transpose / register stages, all
// ascending.  About half the SASS of the unrolled network; kernels full of leaf sorts (the
// permutation's finish) otherwise stall on instruction fetch (ncu: no_inst 20 %).
template <int PK, class V, int M>
__device__ __forceinline__ void sort_block_compact(uint32_t (&x)[M], uint32_t* buf, int lane) {
    constexpr int L = ilog2_ceil_c(V::MV);
    row_sort<PK, V>(x, lane, (V::local(lane) & 1) == 0);  // register-local levels 1..L (odd-even merge sort)
    uint32_t fcur = 0;
#pragma unroll 1
    for (int level = L + 1; level <= 2 * L; ++level) {
        const uint32_t f = (level < 2 * L && ((V::local(lane) >> (level - L)) & 1)) ? 0xFFFFFFFFu : 0u;
        flip<V::C0, V::MV>(x, f ^ fcur);
        fcur = f;
        // views whose local rows are the warp's lanes in order (unit stride, aligned, full)
        constexpr bool kLaneRows = V::ST == 1 && V::WV == 32 && V::WRAP % 32 == 0 && V::LO % 32 == 0 &&
                                   (V::ROWS > kWarp || V::MASK == 0xFFFFFFFFu);
        if (kLaneRows && level - L <= kBlockShflLevels) {
            // the level's row-bit stages as shuffle exchanges with the partner lane (local row
            // bits = lane bits), no transposes (fewer shared wavefronts)
#pragma unroll 1
            for (int b = level - L - 1; b >= 0; --b) {
                const bool upper = (lane >> b) & 1;
#pragma unroll
                for (int c = V::C0; c < V::C0 + V::MV; ++c) {
                    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x[c], 1 << b);
                    if constexpr (PK == 2)
                        x[c] = upper ? __vmaxu2(x[c], y) : __vminu2(x[c], y);
                    else
                        x[c] = upper ? max(x[c], y) : min(x[c], y);
                }
            }
            stages_down<PK, V::C0, V::MV>(x, L - 1);
            continue;
        }
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
            transpose_blocks<V>(x, buf, lane);
            stages_down<PK, V::C0, V::MV>(x, half == 0 ? level - L - 1 : L - 1);
        }
    }
    flip<V::C0, V::MV>(x, fcur);
}

// sort each view's WV x MV block ascending in row-major order (WV, MV powers of two, WV | MV)
template <int PK, class V, int M>
__device__ __forceinline__ void sort_block(uint32_t (&x)[M], uint32_t* buf, int lane) {
    static_assert(V::MV % V::WV == 0, "block sort needs WV | MV");
    if constexpr (V::WV == 1) {
        row_sort<PK, V>(x, lane, true);
    } else if constexpr ((V::ROWS > kWarp || DMM_COMPACT_WARP_BLOCKS) && V::WV == 32 && V::MV == 32) {
        // (16 x 16 blocks measured slower looped: cfg2b 152 -> 140 G keys/s)
        sort_block_compact<PK, V>(x, buf, lane);
    } else {
        // levels 1..log2(MV) stay inside each row; their outcome is the row sorted in the
        // direction of its local-row bit 0, which Batcher's odd-even merge sort reaches with
        // fewer comparators than the bitonic stages (32 keys: 191 vs 240)
        row_sort<PK, V>(x, lane, (V::local(lane) & 1) == 0);
        block_merge_levels<PK, V, ilog2_ceil_c(V::MV) + 1>(x, buf, lane);
    }
}

// partition_leaf partition.hpp:156-172.  Its outcome is the view's multiset in
// row-major sorted order (the reference's short-wide / square / shearsort dispatch
// always ends there, sort.hpp:200-311), so the leaf runs the cheaper bitonic block
// sort above; the state after the call is bit-identical.  The skeletons stay in use
// for the reference's comparison-sort entry points (dmm_sort_wide_any, sort_tall).
template <int PK, class V, int M>
__device__ __forceinline__ void partition_leaf(uint32_t (&x)[M], uint32_t* buf, int lane) {
    constexpr bool pow2 = (V::WV & (V::WV - 1)) == 0 && (V::MV & (V::MV - 1)) == 0;
    if constexpr (pow2)
        sort_block<PK, V>(x, buf, lane);
    else  // shapes that are not powers of two: the reference's own leaf dispatch, literally
        sort_wide_any<PK, V>(x, buf, lane, true);
}

// sort_columns_network sort.hpp:115-156: every column sorted ascending across the
// rows.  The reference drives a Batcher comparator network between row pairs; on
// the warp the network runs across lanes with shuffles (no shared memory, so no
// bank to conflict on).  Partners in another warp (row distance >= 32 on a multi-warp
// machine) exchange through the machine's staging buffer: each warp writes and reads 32
// consecutive rows of a column (row ^ j keeps the bank), so those steps are conflict-free
// too.  Outcome: the unique ascending column.
template <int PK, class V, int M>
__device__ __forceinline__ void sort_columns_network(uint32_t (&x)[M], uint32_t* buf, int lane) {
    constexpr int R = V::ROWS;
#pragma unroll
    for (int k = 2; k <= R; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j >= 1; j >>= 1) {
            const bool up = (lane & k) == 0 || k == R;
            const bool lower = (lane & j) == 0;
            const bool keep_min = lower == up;
            if (j < kWarp) {
#pragma unroll
                for (int c = 0; c < M; ++c) {
                    const uint32_t p = __shfl_xor_sync(0xFFFFFFFFu, x[c], j);
                    uint32_t lo = x[c], hi = p;
                    Key<PK>::template cx<0>(lo, hi);
                    x[c] = keep_min ? lo : hi;
                }
            } else {
                __syncthreads();
#pragma unroll
                for (int c = 0; c < M; ++c)
                    buf[c * R + lane] = x[c];
                __syncthreads();
#pragma unroll
                for (int c = 0; c < M; ++c) {
                    const uint32_t p = buf[c * R + (lane ^ j)];
                    x[c] = keep_min ? min(x[c], p) : max(x[c], p);
                }
            }
        }
    }
    if constexpr (R > kWarp)
        __syncthreads();  // the buffer is free again for the next relayout
}

// sort_tall sort.hpp:352-374 on the full machine view (w >= m, m | w)
template <int PK, class V, int M>
__device__ __forceinline__ void sort_tall(uint32_t (&x)[M], uint32_t* buf, int lane) {
    static_assert(V::MASK == 0xFFFFFFFFu && V::ST == 1 && V::WV == V::ROWS && V::C0 == 0 && V::MV == M,
                  "sort_tall on the full machine view");
    static_assert(V::WV >= V::MV && V::WV % V::MV == 0, "sort_tall needs w >= m and m | w (ShapeViolation)");
    static_assert(PK == 1 || V::ROWS == kWarp, "packed keys only on one-warp machines");
    if constexpr (V::WV == V::MV) {
        sort_wide_any<PK, V>(x, buf, lane, true);
    } else {
        row_sort<PK, V>(x, lane, true);
        sort_columns_network<PK, V>(x, buf, lane);
        to_row_major<V>(x, buf, lane);
        sort_columns_network<PK, V>(x, buf, lane);
        using B = VRows<V, V::MV>;  // m x m blocks, alternating direction per block
        sort_wide_any<PK, B>(x, buf, lane, ((lane / V::MV) % 2) == 0);
        sort_columns_network<PK, V>(x, buf, lane);
        row_sort<PK, V>(x, lane, true);
    }
}

// ---------------------------------------------------------------------------
// Balancing, convert-and-divide, recursion  partition.hpp:234-428
// ---------------------------------------------------------------------------
// balance partition.hpp:234-271.  Round with sub-matrix height SUB_H and NSUBS
// sub-matrices; the assembled views pick row j of each sub-matrix of a group.
template <int PK, class V, bool EXT, int SUB_H, int NSUBS, int M>
__device__ __forceinline__ void balance_rounds(uint32_t (&x)[M], uint32_t* buf, int lane) {
    if constexpr (NSUBS > 1) {
        constexpr int g = V::MV < NSUBS ? V::MV : NSUBS;
        static_assert(!(g < V::MV && g * g > V::MV) || (EXT && V::MV % g == 0),
                      "balance leftover group fits neither the square nor short-wide case (ShapeViolation)");
        static_assert(NSUBS % g == 0, "balance needs g | nsubs");
        using A = VF<V::MASK, V::LO, V::ST * SUB_H, g, V::C0, V::MV, V::WRAP, V::ROWS>;
        if constexpr (g == V::MV) {
            partition_leaf<PK, A>(x, buf, lane);
            transpose_square<A>(x, buf, lane);
        } else if constexpr (g * g <= V::MV) {
            short_wide<PK, A>(x, buf, lane, true);
            to_column_major<A>(x, buf, lane);
        } else {
            // B200 extension (documented in DESIGN.md): a partial group with g^2 > m
            // is sorted by the leaf dispatcher (shearsort), then laid out column-major.
            partition_leaf<PK, A>(x, buf, lane);
            to_column_major<A>(x, buf, lane);
        }
        balance_rounds<PK, V, EXT, SUB_H * g, NSUBS / g>(x, buf, lane);
    }
}

// balance + convert_and_divide (partition.hpp:275-286) until subproblems have <= m
// rows, then the leaves (balance_divide_sort steps (1) and (2), :373-396)
template <int PK, class V, bool EXT, int M>
__device__ __forceinline__ void levels(uint32_t (&x)[M], uint32_t* buf, int lane, ProbeSink* ps = nullptr) {
    if constexpr (V::WV > V::MV) {
        static_assert(V::WV % V::MV == 0, "general partition needs m | w (ShapeViolation)");
        balance_rounds<PK, V, EXT, 1, V::WV>(x, buf, lane);
        if (ps)
            ps->template capture<PK>(x);  // after_balance(depth, level)
        constexpr PParams p = pparams_c(V::WV, V::MV, EXT);
        static_assert(V::WV % p.subproblems == 0, "m*d must divide W (DivisibilityViolation)");
        to_row_major<V>(x, buf, lane);
        if (ps)
            ps->template capture<PK>(x);  // after_divide(depth + 1, next)
        levels<PK, VRows<V, V::WV / p.subproblems>, EXT>(x, buf, lane, ps);
    } else {
        partition_leaf<PK, V>(x, buf, lane);
    }
}

// Lane masks of the shifted-cleanup blocks inside aligned contiguous views of WV rows.
__host__ __device__ constexpr uint32_t edge_mask(int WV, int H) {
    uint32_t m = 0;
    for (int l = 0; l < kWarp; ++l)
        if (l % WV < H || l % WV >= WV - H)
            m |= 1u << l;
    return m;
}
__host__ __device__ constexpr uint32_t mid_mask(int WV, int H) { return ~edge_mask(WV, H); }

// ---------------------------------------------------------------------------
// Machine-wide primitives for multi-warp machines (ROWS = 64..256 rows = threads of one
// CTA).  `scratch` is machine shared memory that is free at the call (the relayout buffer
// between relayouts); every call begins and ends with a machine barrier.
// ---------------------------------------------------------------------------
// OR of v over aligned groups of G rows (G >= 32: warp reduction + one word per warp)
template <int ROWS, int G>
__device__ __forceinline__ uint32_t group_or(uint32_t v, int row, uint32_t* scratch) {
    if constexpr (G <= 32) {
#pragma unroll
        for (int off = 1; off < G; off <<= 1)
            v |= __shfl_xor_sync(0xFFFFFFFFu, v, off);
        return v;
    } else {
        v = __reduce_or_sync(0xFFFFFFFFu, v);
        __syncthreads();
        if ((row & 31) == 0)
            scratch[row >> 5] = v;
        __syncthreads();
        uint32_t r = 0;
        const int w0 = (row / G) * (G / 32);
#pragma unroll
        for (int w = 0; w < G / 32; ++w)
            r |= scratch[w0 + w];
        __syncthreads();
        return r;
    }
}
template <int ROWS, int G>
__device__ __forceinline__ uint32_t group_max(uint32_t v, int row, uint32_t* scratch) {
    if constexpr (G <= 32) {
#pragma unroll
        for (int off = 1; off < G; off <<= 1)
            v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, off));
        return v;
    } else {
        v = __reduce_max_sync(0xFFFFFFFFu, v);
        __syncthreads();
        if ((row & 31) == 0)
            scratch[row >> 5] = v;
        __syncthreads();
        uint32_t r = 0;
        const int w0 = (row / G) * (G / 32);
#pragma unroll
        for (int w = 0; w < G / 32; ++w)
            r = max(r, scratch[w0 + w]);
        __syncthreads();
        return r;
    }
}
// the successor row's value (row + 1; the last row gets its own)
template <int ROWS>
__device__ __forceinline__ uint32_t next_row_value(uint32_t v, int row, uint32_t* scratch) {
    if constexpr (ROWS == 32) {
        return __shfl_down_sync(0xFFFFFFFFu, v, 1);
    } else {
        __syncthreads();
        scratch[row] = v;
        __syncthreads();
        const uint32_t r = scratch[row + 1 < ROWS ? row + 1 : row];
        __syncthreads();
        return r;
    }
}
// every row of the machine agrees (the cleanup loop's exit)
template <int ROWS>
__device__ __forceinline__ bool machine_all(bool p) {
    if constexpr (ROWS == 32)
        return __all_sync(0xFFFFFFFFu, p);
    else
        return __syncthreads_and(p ? 1 : 0) != 0;
}

// scan_sorted partition.hpp:308-337 over a family of aligned contiguous views: each
// lane returns its view's verdict (bit h set = half h sorted row-major).  The
// reference's tree_reduce_sum + broadcast of the verdict is a butterfly OR inside
// each group of WV lanes.
template <int PK, class V, int M>
__device__ __forceinline__ uint32_t scan_sorted(const uint32_t (&x)[M], uint32_t* buf, int lane) {
    static_assert(V::MASK == 0xFFFFFFFFu && V::ST == 1 && V::LO == 0 && V::ROWS % V::WV == 0,
                  "scan_sorted on aligned contiguous views");
    uint32_t bad = 0;
#pragma unroll
    for (int c = V::C0 + 1; c < V::C0 + V::MV; ++c)
        bad |= Key<PK>::gt(x[c - 1], x[c]);
    const uint32_t next_first = next_row_value<V::ROWS>(x[V::C0], lane, buf);
    if (V::local(lane) + 1 < V::WV)
        bad |= Key<PK>::gt(x[V::C0 + V::MV - 1], next_first);
    bad = group_or<V::ROWS, V::WV>(bad, lane, buf);
    return Key<PK>::kAll & ~bad;
}

// cleanup_pass_pair partition.hpp:341-361 over a family of aligned contiguous views.
// TAG != 0: a key bit no key of this sort uses (keys < TAG's bit in every packed half).
// Then the two m/2-row end blocks run fused with the m/2-shifted blocks: the view family
// shifted by m/2 wraps around each view, so its last block is (bottom end block, top end
// block); the top block's keys carry TAG, which sorts them after every bottom key, so the
// fused sort leaves each end block exactly its own sorted keys (the reference's separate
// sorts, in lockstep with the shifted blocks) -- one leaf sort instead of two.
template <int PK, class V, uint32_t TAG = 0u, int M>
__device__ __forceinline__ void cleanup_pass_pair(uint32_t (&x)[M], uint32_t* buf, int lane) {
    static_assert(V::MASK == 0xFFFFFFFFu && V::ST == 1 && V::LO == 0 && V::ROWS % V::WV == 0,
                  "cleanup on aligned contiguous views");
    partition_leaf<PK, VRows<V, V::MV>>(x, buf, lane);  // aligned m x m blocks
    if constexpr (V::WV > V::MV && V::MV >= 2) {
        constexpr int H = V::MV / 2;
        if constexpr (TAG != 0u) {
            using Shifted = VF<0xFFFFFFFFu, H, 1, V::MV, V::C0, V::MV, V::WV, V::ROWS>;
            const bool top = V::local(lane) < H;
            if (top) {
#pragma unroll
                for (int c = V::C0; c < V::C0 + V::MV; ++c)
                    x[c] |= TAG;
            }
            partition_leaf<PK, Shifted>(x, buf, lane);
            if (top) {
#pragma unroll
                for (int c = V::C0; c < V::C0 + V::MV; ++c)
                    x[c] &= ~TAG;
            }
        } else {
            static_assert(V::ROWS == 32, "multi-warp machines run the fused cleanup (a free tag bit)");
            using Edge = VF<edge_mask(V::WV, H), 0, 1, H, V::C0, V::MV>;
            using Mid = VF<mid_mask(V::WV, H), H, 1, V::MV, V::C0, V::MV>;
            partition_leaf<PK, Edge>(x, buf, lane);  // the two m/2-row end blocks of every view
            partition_leaf<PK, Mid>(x, buf, lane);   // the m/2-shifted m-row blocks
        }
    }
}

// Per-instance result of a general sort (one entry per packed half).  Accumulated
// per lane (each lane sees its own views); finish() reduces over the warp:
// GeneralStats.cleanup_retries is the max over every recursion level and view.
struct GenResult {
    uint32_t retries[2];  // cleanup_retries (GeneralStats partition.hpp:292-295)
    uint32_t unsorted;    // bit h: cleanup budget exhausted for half h
    // reduce over the WM lanes of each machine (WM = 32: the whole warp)
    template <int WM = kWarp>
    __device__ void finish() {
        retries[0] = seg_max<WM>(retries[0]);
        retries[1] = seg_max<WM>(retries[1]);
        unsorted = seg_or<WM>(unsorted);
    }
    // multi-warp machine of ROWS rows (scratch: free machine shared memory)
    template <int ROWS>
    __device__ void finish_machine(int row, uint32_t* scratch) {
        retries[0] = group_max<ROWS, ROWS>(retries[0], row, scratch);
        retries[1] = group_max<ROWS, ROWS>(retries[1], row, scratch);
        unsorted = group_or<ROWS, ROWS>(unsorted, row, scratch);
    }
};

// balance_divide_sort partition.hpp:363-428
template <int PK, class V, bool EXT, uint32_t TAG = 0u, int M>
__device__ __forceinline__ void balance_divide_sort(uint32_t (&x)[M], uint32_t* buf, int lane, GenResult& res,
                                                    ProbeSink* ps = nullptr) {
    if constexpr (V::WV <= V::MV) {
        partition_leaf<PK, V>(x, buf, lane);
    } else {
        levels<PK, V, EXT>(x, buf, lane, ps);
        // (3) column recursion: each column into a (W/m) x m submatrix
        to_row_major<V>(x, buf, lane);
        balance_divide_sort<PK, VRows<V, V::WV / V::MV>, EXT, TAG>(x, buf, lane, res);
        to_column_major<V>(x, buf, lane);
        // (4) shifted square cleanup with a checked postcondition
        constexpr int budget = ilog2_ceil_c(V::WV);
        uint32_t done = 0;
        int passes = 0;
#pragma unroll 1
        for (;;) {
            cleanup_pass_pair<PK, V, TAG>(x, buf, lane);
            const uint32_t ok = scan_sorted<PK, V>(x, buf, lane);
            const uint32_t fresh = ok & ~done;
            if (fresh & 1u)
                res.retries[0] = max(res.retries[0], (uint32_t)passes);
            if (fresh & 2u)
                res.retries[1] = max(res.retries[1], (uint32_t)passes);
            done |= ok;
            if (machine_all<V::ROWS>(done == Key<PK>::kAll) || passes == budget)
                break;
            ++passes;
        }
        const uint32_t failed = Key<PK>::kAll & ~done;
        if (failed & 1u)
            res.retries[0] = max(res.retries[0], (uint32_t)budget);
        if (failed & 2u)
            res.retries[1] = max(res.retries[1], (uint32_t)budget);
        res.unsorted |= failed;
    }
}

}  // namespace dmmdev

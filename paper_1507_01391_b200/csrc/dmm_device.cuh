// dmm_device.cuh -- warp-level realisation of the reference's DMM algorithms on sm_100a.
//
// Mapping:
//   * one warp       = one DMM machine with w = 32 processors / 32 banks;
//   * lane r         = processor r, holding row r of the w x m matrix in registers
//                      x[0..m) ("its own bank": row-local work never touches smem);
//   * cross-bank steps of the reference (transpose_square, to_column_major,
//     to_row_major, the blocked column sorts) become one shared-memory relayout:
//     every lane stores each register to the destination cell's slot and reads its
//     own slots back.  The slot layout of every relayout is chosen AT COMPILE TIME
//     (find_kappa below) so that each warp-wide STS touches 32 distinct banks and
//     each LDS reads its own skewed column: 0 bank conflicts by construction.
//   * row sorts (the reference's radix / merge rows, partition.hpp:42-99,
//     sort.hpp:44-81) become Batcher odd-even merge networks over the lane's
//     registers.  Their outcome is the unique sorted row, i.e. bit-identical to the
//     reference's state after the same step.
//   * PK = 2 packs two independent instances into the 16-bit halves of every
//     register (keys < 2^16: partition labels, permute labels): VIMNMX.U16x2
//     compares both at once and every relayout moves both.  The schedule is
//     data-independent except the cleanup retries, which are tracked per half.
//
// Views (view.hpp:15-134): a lockstep family of sibling views is a compile-time
// struct VF<MASK, LO, ST, WV, C0, MV>: active lanes MASK, lane of local row i of a
// view = base + ST*i (base = lane - ST*local), local row = ((lane-LO)/ST) % WV, and
// the column window [C0, C0+MV) of the register array.  Contiguous row ranges
// (row_range) have ST = 1; balance()'s assembled squares (pick_rows, partition.hpp:
// 247-253) have ST = sub-matrix height.
#pragma once

#include <cstdint>
#include <type_traits>

namespace dmmdev {

constexpr int kWarp = 32;

// compile-time loop: f(std::integral_constant<int, i>) for i = B, B+S, ... < E
template <int B, int E, int S = 1, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + S, E, S>(f);
    }
}

// Reductions over aligned groups of WM lanes (one machine each; WM = 32: the warp).  WM that
// is not a power of two (e.g. 3-row machines, 10 per warp) reduces over the group's lane mask.
__device__ __forceinline__ uint32_t group_lane_mask(int wm) {
    const int lane = threadIdx.x & 31;
    const int g0 = (lane / wm) * wm;
    const int n = g0 + wm > 32 ? 32 - g0 : wm;
    return (n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u)) << g0;
}
template <int WM>
__device__ __forceinline__ uint32_t seg_or(uint32_t v) {
    if constexpr (WM >= kWarp) {
        return __reduce_or_sync(0xFFFFFFFFu, v);
    } else if constexpr ((WM & (WM - 1)) != 0) {
        return __reduce_or_sync(group_lane_mask(WM), v);
    } else {
#pragma unroll
        for (int off = 1; off < WM; off <<= 1)
            v |= __shfl_xor_sync(0xFFFFFFFFu, v, off);
        return v;
    }
}
template <int WM>
__device__ __forceinline__ uint32_t seg_max(uint32_t v) {
    if constexpr (WM >= kWarp) {
        return __reduce_max_sync(0xFFFFFFFFu, v);
    } else if constexpr ((WM & (WM - 1)) != 0) {
        return __reduce_max_sync(group_lane_mask(WM), v);
    } else {
#pragma unroll
        for (int off = 1; off < WM; off <<= 1)
            v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, off));
        return v;
    }
}

// ---------------------------------------------------------------------------
// Key traits: comparator and direction flip
//
// Pipe balance (tools/mb_pipes.cu, measured on B200): IMNMX / VIMNMX.U16x2 (and
// HMNMX2) issue on the ALU pipe at 16 lanes/clk/SMSP; the FMA pipe (IMAD) is idle in
// a sorting network.  max(a, b) = a + b - min(a, b) holds exactly in 32-bit wrapping
// arithmetic -- and per 16-bit half of a packed pair, since the halves' sum is the
// exact integer max_hi * 2^16 + max_lo -- so a comparator can take its max from two
// IMADs instead of a second ALU min/max.  Comparators cx<I> with I % 3 != 0 use that
// form (1 ALU + 2 FMA), the others the pure form (2 ALU): both pipes then carry 4/3
// instructions per comparator (1.39x comparator throughput measured, bit-exact).
// The IMAD multiplier -1 must be opaque to ptxas, or it folds the IMADs back into an
// IADD3 on the ALU pipe: it is derived from %nsmid (ptxas cannot know it is nonzero;
// ptxas reads it once per kernel and keeps it in a register).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pipe_neg() {
    uint32_t n;
    asm("mov.u32 %0, %%nsmid;" : "=r"(n));
    return n != 0 ? 0xFFFFFFFFu : 0u;
}

// h = a + b - l = b - (l - a), two IMADs on the FMA pipe
__device__ __forceinline__ uint32_t fma_pipe_max(uint32_t a, uint32_t b, uint32_t l) {
    const uint32_t neg = pipe_neg();
    uint32_t t, h;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a), "r"(neg), "r"(l));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h) : "r"(t), "r"(neg), "r"(b));
    return h;
}

#ifndef DMM_CX_PURE_EVERY
#define DMM_CX_PURE_EVERY 3
#endif
constexpr int kPureEvery = DMM_CX_PURE_EVERY;

template <int PK>
struct Key;

template <>
struct Key<1> {  // one 32-bit key per register
    template <int I = 0>
    static __device__ __forceinline__ void cx(uint32_t& a, uint32_t& b) {
        const uint32_t l = min(a, b);
        if constexpr (I % kPureEvery == 0)
            b = max(a, b);
        else
            b = fma_pipe_max(a, b, l);
        a = l;
    }
    // per-lane "a > b" as a bit mask (bit 0)
    static __device__ __forceinline__ uint32_t gt(uint32_t a, uint32_t b) { return a > b ? 1u : 0u; }
    static constexpr uint32_t kAll = 1u;
};

template <>
struct Key<2> {  // two 16-bit keys per register (instance A low half, B high half)
    template <int I = 0>
    static __device__ __forceinline__ void cx(uint32_t& a, uint32_t& b) {
        const uint32_t l = __vminu2(a, b);
        if constexpr (I % kPureEvery == 0)
            b = __vmaxu2(a, b);
        else
            b = fma_pipe_max(a, b, l);
        a = l;
    }
    // bit 0: A half a>b, bit 1: B half a>b
    static __device__ __forceinline__ uint32_t gt(uint32_t a, uint32_t b) {
        const uint32_t g = __vcmpgtu2(a, b);
        return (g & 1u) | ((g >> 15) & 2u);
    }
    static constexpr uint32_t kAll = 3u;
};

// ---------------------------------------------------------------------------
// Sorting networks: Batcher's odd-even merge sort over registers [LO, HI]
// (inclusive), generated by template recursion so every register index is a
// compile-time constant (no local memory).  N = 8/16/32/64: 19/63/191/543
// comparators, each one VIMNMX pair (min + max).
// ---------------------------------------------------------------------------
// LIM: registers [LIM, HI] are virtual +inf padding (sizes that are not powers of two):
// a comparator touching one never swaps, so it is dropped and the padding never moves.
template <int PK, int LO, int HI, int R, int LIM, int M>
__device__ __forceinline__ void oe_merge(uint32_t (&x)[M]) {
    constexpr int step = R * 2;
    if constexpr (step < HI - LO) {
        oe_merge<PK, LO, HI, step, LIM>(x);
        oe_merge<PK, LO + R, HI, step, LIM>(x);
        static_for<LO + R, HI - R, step>([&](auto i) {
            constexpr int a = decltype(i)::value;
            if constexpr (a + R < LIM)
                Key<PK>::template cx<(a - LO) / step>(x[a], x[a + R]);
        });
    } else if constexpr (LO + R < LIM) {
        Key<PK>::template cx<LO>(x[LO], x[LO + R]);
    }
}

template <int PK, int LO, int HI, int LIM, int M>
__device__ __forceinline__ void oe_sort(uint32_t (&x)[M]) {
    if constexpr (HI - LO >= 1 && LO + 1 < LIM) {
        constexpr int mid = LO + (HI - LO) / 2;
        oe_sort<PK, LO, mid, LIM>(x);
        oe_sort<PK, mid + 1, HI, LIM>(x);
        oe_merge<PK, LO, HI, 1, LIM>(x);
    }
}

// ascending sort of x[OFF .. OFF+N): Batcher's odd-even merge sort on the next power of two,
// comparators that touch the (virtual) padding dropped
__host__ __device__ constexpr int next_pow2_c(int n) {
    int p = 1;
    while (p < n)
        p <<= 1;
    return p;
}
template <int PK, int OFF, int N, int M>
__device__ __forceinline__ void sort_net(uint32_t (&x)[M]) {
    static_assert(OFF + N <= M, "window outside the register row");
    oe_sort<PK, OFF, OFF + next_pow2_c(N) - 1, OFF + N>(x);
}

template <int OFF, int N, int M>
__device__ __forceinline__ void flip(uint32_t (&x)[M], uint32_t f) {
    const uint32_t s = f | 1u;
#pragma unroll
    for (int c = OFF; c < OFF + N; ++c)
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(s), "r"(f));
}

// ---------------------------------------------------------------------------
// View families
// ---------------------------------------------------------------------------
// WRAP: rows are numbered cyclically inside aligned groups of WRAP rows, so a family
// offset by LO can wrap around its group (the m/2-shifted cleanup blocks with the two
// end blocks fused, cleanup_pass_pair).  With WRAP = ROWS and LO <= every active row this
// is the plain affine family.  ROWS: rows of the machine = threads holding one row each
// (32: one warp, the `lane` arguments below are lanes; 64..256: ROWS / 32 warps of one CTA,
// the `lane` arguments are thread indices = rows; MASK must then be full).
template <uint32_t MASK_, int LO_, int ST_, int WV_, int C0_, int MV_, int WRAP_ = 32, int ROWS_ = 32>
struct VF {
    static constexpr uint32_t MASK = MASK_;
    static constexpr int LO = LO_, ST = ST_, WV = WV_, C0 = C0_, MV = MV_, WRAP = WRAP_, ROWS = ROWS_;
    static_assert(WV >= 1 && MV >= 1 && ST >= 1 && WRAP >= 1 && ROWS % WRAP == 0, "bad view family");
    static_assert(ROWS == 32 || (ROWS % 32 == 0 && MASK == 0xFFFFFFFFu), "multi-warp machines use full families");
    __host__ __device__ static constexpr bool active(int lane) {
        return ROWS == 32 ? ((MASK >> lane) & 1u) != 0 : (lane >= 0 && lane < ROWS);
    }
    __host__ __device__ static constexpr int group0(int lane) { return (lane / WRAP) * WRAP; }
    __host__ __device__ static constexpr int local(int lane) {
        return ((((lane - group0(lane) - LO) % WRAP + WRAP) % WRAP) / ST) % WV;
    }
    __host__ __device__ static constexpr int lane_of(int lane, int k) {
        return group0(lane) + (((lane - group0(lane) - ST * local(lane) + ST * k) % WRAP + WRAP) % WRAP);
    }
};

// synchronise the threads of one machine (one warp, or the CTA for multi-warp machines)
template <class V>
__device__ __forceinline__ void machine_sync() {
    if constexpr (V::ROWS == 32)
        __syncwarp();
    else
        __syncthreads();
}

// aligned row groups of height H inside every view of V (row_range in lockstep; H | WV)
template <class V, int H>
using VRows = VF<V::MASK, V::LO, V::ST, H, V::C0, V::MV, V::WRAP, V::ROWS>;
// column window [C0+lo, C0+lo+n) (col_window, view.hpp:83)
template <class V, int lo, int n>
using VCols = VF<V::MASK, V::LO, V::ST, V::WV, V::C0 + lo, n, V::WRAP, V::ROWS>;

__host__ __device__ constexpr uint32_t lane_range_mask(int lo, int hi) {
    uint32_t m = 0;
    for (int l = lo; l < hi; ++l)
        m |= 1u << l;
    return m;
}

__host__ __device__ constexpr int ilog2_ceil_c(int x) {
    int k = 0, p = 1;
    while (p < x) {
        p <<= 1;
        ++k;
    }
    return k;
}
__host__ __device__ constexpr int isqrt_c(int x) {
    int r = 0;
    while ((r + 1) * (r + 1) <= x)
        ++r;
    return r;
}

// ---------------------------------------------------------------------------
// Relayout maps: where does the cell in (lane, register c) go?
// ---------------------------------------------------------------------------
// Each map gives the destination of the cell in (lane, register c) and, as the
// inverse, the source of the cell that lands in (lane, register d).
//
// Square-block transpose of every WV x WV block of the window (transpose_square,
// layout.hpp:24; all column blocks of sort_columns_blocked, sort.hpp:169-173, at once).
template <class V>
struct TransposeBlocks {
    static_assert(V::MV % V::WV == 0, "blocked transpose needs WV | MV");
    __host__ __device__ static constexpr int dst_lane(int lane, int c) {
        return V::lane_of(lane, (c - V::C0) % V::WV);
    }
    __host__ __device__ static constexpr int dst_col(int lane, int c) {
        return V::C0 + ((c - V::C0) / V::WV) * V::WV + V::local(lane);
    }
    // an involution
    __host__ __device__ static constexpr int src_lane(int lane, int d) { return dst_lane(lane, d); }
    __host__ __device__ static constexpr int src_col(int lane, int d) { return dst_col(lane, d); }
};
// to_column_major (layout.hpp:397): linear index i*MV + j goes to (lin mod WV, lin div WV)
template <class V>
struct ToColumnMajor {
    __host__ __device__ static constexpr int lin(int lane, int c) { return V::local(lane) * V::MV + (c - V::C0); }
    __host__ __device__ static constexpr int dst_lane(int lane, int c) { return V::lane_of(lane, lin(lane, c) % V::WV); }
    __host__ __device__ static constexpr int dst_col(int lane, int c) { return V::C0 + lin(lane, c) / V::WV; }
    // cell (i', j') receives column-major index u = j'*WV + i', i.e. source (u div MV, u mod MV)
    __host__ __device__ static constexpr int u(int lane, int d) { return (d - V::C0) * V::WV + V::local(lane); }
    __host__ __device__ static constexpr int src_lane(int lane, int d) { return V::lane_of(lane, u(lane, d) / V::MV); }
    __host__ __device__ static constexpr int src_col(int lane, int d) { return V::C0 + u(lane, d) % V::MV; }
};
// to_row_major (layout.hpp:403): column-major index u = j*WV + i goes to (u div MV, u mod MV)
template <class V>
struct ToRowMajor {
    __host__ __device__ static constexpr int u(int lane, int c) { return (c - V::C0) * V::WV + V::local(lane); }
    __host__ __device__ static constexpr int dst_lane(int lane, int c) { return V::lane_of(lane, u(lane, c) / V::MV); }
    __host__ __device__ static constexpr int dst_col(int lane, int c) { return V::C0 + u(lane, c) % V::MV; }
    __host__ __device__ static constexpr int lin(int lane, int d) { return V::local(lane) * V::MV + (d - V::C0); }
    __host__ __device__ static constexpr int src_lane(int lane, int d) { return V::lane_of(lane, lin(lane, d) % V::WV); }
    __host__ __device__ static constexpr int src_col(int lane, int d) { return V::C0 + lin(lane, d) / V::WV; }
};

// A relayout goes through a per-warp staging buffer.  Two slot layouts:
//
//  * column-major (scalar modes 0/1): slot (b, d) at word (d - C0) * (32 + kappa) + b,
//    i.e. bank ((d - C0) * kappa + b) mod 32;
//      scatter (0): lane a stores register c into its DESTINATION slot, then every lane
//                   loads its own slots (own-slot loads are conflict-free for any kappa);
//      gather  (1): every lane stores into its own slots (conflict-free), then lane b
//                   loads register d from its SOURCE slot;
//  * lane-major (vector modes 2/3): slot (b, d) at word b * Q + S * (b / 8) + (d - C0), Q =
//    pitch, S = skew per group of 8 rows (Q, S multiples of 4: 16-byte aligned rows), so a
//    lane's own slots are contiguous and move as 128-bit STS.128 / LDS.128 (a quarter of
//    the shared-memory instructions on the own side; the MIO queue is what stalls the
//    relayout-heavy kernels):
//      gather-v4  (2): own slots stored with STS.128, then scalar gathers from sources;
//      scatter-v4 (3): scalar scatters to destinations, then own slots loaded with LDS.128.
//    A 128-bit access is served a quarter-warp (8 lanes, 128 bytes) per wavefront, so it
//    is conflict-free iff the 8 lanes of every quarter hit 8 distinct 4-bank groups.
//
// find_layout picks, at compile time, the first layout (vector modes first) for which
// every warp-wide access touches distinct banks -- the reference's CAC (core.hpp:445-467)
// checked exhaustively over all lanes and registers.  Returns mode * 4096 + k (k = kappa
// for modes 0/1; (S / 4) * 64 + Q - MV for modes 2/3) or -1.
__host__ __device__ constexpr int relayout_buf_words(int mv) {
    return (mv * (mv >= 32 ? 33 : 64)) > 32 * (mv + 4) ? (mv * (mv >= 32 ? 33 : 64)) : 32 * (mv + 4);
}

// lane-major slot address (vector modes)
__host__ __device__ constexpr int v4_addr(int b, int d0, int Q, int S) { return b * Q + S * (b / 8) + d0; }

template <class V, class Map>
__host__ __device__ constexpr bool v4_own_ok(int Q, int S) {  // own-slot 128-bit accesses, per quarter-warp
    for (int j = 0; j < V::MV / 4; ++j) {
        for (int q = 0; q < V::ROWS / 8; ++q) {
            uint32_t seen = 0;
            for (int a = 8 * q; a < 8 * q + 8; ++a) {
                if (!V::active(a))
                    continue;
                const int g = (v4_addr(a, 4 * j, Q, S) / 4) & 7;
                if ((seen >> g) & 1u)
                    return false;
                seen |= 1u << g;
            }
        }
    }
    return true;
}

template <class V, class Map>
__host__ __device__ constexpr bool v4_cross_ok(int Q, int S, bool gather) {  // scalar cross accesses
    for (int c = V::C0; c < V::C0 + V::MV; ++c) {
        for (int w = 0; w < V::ROWS / 32; ++w) {  // one warp-wide instruction per warp
            uint32_t seen = 0;
            for (int lane = 32 * w; lane < 32 * w + 32; ++lane) {
                if (!V::active(lane))
                    continue;
                const int b = gather ? Map::src_lane(lane, c) : Map::dst_lane(lane, c);
                const int d = gather ? Map::src_col(lane, c) : Map::dst_col(lane, c);
                const int bank = v4_addr(b, d - V::C0, Q, S) & 31;
                if ((seen >> bank) & 1u)
                    return false;
                seen |= 1u << bank;
            }
        }
    }
    return true;
}

// staging words per machine row-group of 32 (the buffer of a machine is ROWS / 32 of these)
template <class V>
__host__ __device__ constexpr int relayout_words() {
    return relayout_buf_words(V::MV) * (V::ROWS / 32);
}

template <class V, class Map>
__host__ __device__ constexpr int find_layout() {
    // vector modes only where every quarter-warp is wholly active or wholly idle: a
    // predicated 128-bit access with a ragged quarter was measured (ncu) to cost an extra
    // wavefront, so partial quarters keep the scalar layouts
    bool quarters_whole = true;
    for (int q = 0; q < 4; ++q) {
        const uint32_t qm = (V::MASK >> (8 * q)) & 0xFFu;
        quarters_whole = quarters_whole && (qm == 0u || qm == 0xFFu);
    }
    if (V::MV % 4 == 0 && V::C0 % 4 == 0 && quarters_whole) {
        for (int mode = 2; mode < 4; ++mode) {
            for (int S = 0; S < 32; S += 4) {
                for (int Q = V::MV; v4_addr(V::ROWS - 1, V::MV, Q, S) <= relayout_words<V>(); Q += 4) {
                    if (v4_own_ok<V, Map>(Q, S) && v4_cross_ok<V, Map>(Q, S, mode == 2))
                        return mode * 4096 + (S / 4) * 64 + (Q - V::MV);
                }
            }
        }
    }
    for (int mode = 0; mode < 2; ++mode) {
        for (int k = 0; k <= 32; ++k) {
            if ((V::ROWS + k) * V::MV > relayout_words<V>())
                break;
            bool ok = true;
            for (int c = V::C0; c < V::C0 + V::MV && ok; ++c) {
                for (int w = 0; w < V::ROWS / 32 && ok; ++w) {
                    uint32_t seen = 0;
                    for (int lane = 32 * w; lane < 32 * w + 32; ++lane) {
                        if (!V::active(lane))
                            continue;
                        const int b = mode == 0 ? Map::dst_lane(lane, c) : Map::src_lane(lane, c);
                        const int d = mode == 0 ? Map::dst_col(lane, c) : Map::src_col(lane, c);
                        const int bank = ((d - V::C0) * k + b) & 31;
                        if ((seen >> bank) & 1u) {
                            ok = false;
                            break;
                        }
                        seen |= 1u << bank;
                    }
                }
            }
            if (ok)
                return mode * 4096 + k;
        }
    }
    return -1;
}

// Bijectivity / inverse consistency of a map on the active cells (static self-check).
template <class V, class Map>
__host__ __device__ constexpr bool map_is_consistent() {
    for (int lane = 0; lane < V::ROWS; ++lane) {
        if (!V::active(lane))
            continue;
        for (int c = V::C0; c < V::C0 + V::MV; ++c) {
            const int b = Map::dst_lane(lane, c), d = Map::dst_col(lane, c);
            if (b < 0 || b >= V::ROWS || !V::active(b) || d < V::C0 || d >= V::C0 + V::MV)
                return false;
            if (Map::src_lane(b, d) != lane || Map::src_col(b, d) != c)
                return false;
        }
    }
    return true;
}

template <class V, class Map, int M>
__device__ __forceinline__ void relayout(uint32_t (&x)[M], uint32_t* buf, int lane) {
    constexpr int L = find_layout<V, Map>();
    static_assert(L >= 0, "no conflict-free layout for this relayout");
    static_assert(map_is_consistent<V, Map>(), "relayout map is not a bijection with a matching inverse");
    constexpr int mode = L / 4096;
    const bool act = V::active(lane);
    if constexpr (mode >= 2) {
        constexpr int Q = V::MV + (L & 63), S = 4 * ((L / 64) & 63);
        static_assert(v4_addr(V::ROWS - 1, V::MV, Q, S) <= relayout_words<V>(), "relayout buffer too small");
        uint32_t* own = buf + v4_addr(lane, 0, Q, S);
        machine_sync<V>();
        if (act) {
            if constexpr (mode == 2) {
#pragma unroll
                for (int j = 0; j < V::MV / 4; ++j)
                    *reinterpret_cast<uint4*>(own + 4 * j) =
                        make_uint4(x[V::C0 + 4 * j], x[V::C0 + 4 * j + 1], x[V::C0 + 4 * j + 2], x[V::C0 + 4 * j + 3]);
            } else {
#pragma unroll
                for (int c = V::C0; c < V::C0 + V::MV; ++c) {
                    const int b = Map::dst_lane(lane, c), d = Map::dst_col(lane, c);
                    buf[v4_addr(b, d - V::C0, Q, S)] = x[c];
                }
            }
        }
        machine_sync<V>();
        if (act) {
            if constexpr (mode == 2) {
#pragma unroll
                for (int d = V::C0; d < V::C0 + V::MV; ++d) {
                    const int a = Map::src_lane(lane, d), c = Map::src_col(lane, d);
                    x[d] = buf[v4_addr(a, c - V::C0, Q, S)];
                }
            } else {
#pragma unroll
                for (int j = 0; j < V::MV / 4; ++j) {
                    const uint4 t = *reinterpret_cast<const uint4*>(own + 4 * j);
                    x[V::C0 + 4 * j] = t.x;
                    x[V::C0 + 4 * j + 1] = t.y;
                    x[V::C0 + 4 * j + 2] = t.z;
                    x[V::C0 + 4 * j + 3] = t.w;
                }
            }
        }
    } else {
        constexpr int P = V::ROWS + (L & 63);  // scalar modes: kappa in the low bits
        constexpr bool gather = mode == 1;
        static_assert(V::MV * P <= relayout_words<V>(), "relayout buffer too small for this skew");
        machine_sync<V>();
        if (act) {
#pragma unroll
            for (int c = V::C0; c < V::C0 + V::MV; ++c) {
                if constexpr (gather) {
                    buf[(c - V::C0) * P + lane] = x[c];
                } else {
                    const int b = Map::dst_lane(lane, c), d = Map::dst_col(lane, c);
                    buf[(d - V::C0) * P + b] = x[c];
                }
            }
        }
        machine_sync<V>();
        if (act) {
#pragma unroll
            for (int d = V::C0; d < V::C0 + V::MV; ++d) {
                if constexpr (gather) {
                    const int a = Map::src_lane(lane, d), c = Map::src_col(lane, d);
                    x[d] = buf[(c - V::C0) * P + a];
                } else {
                    x[d] = buf[(d - V::C0) * P + lane];
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Layout primitives (layout.hpp)
// ---------------------------------------------------------------------------
template <class V, int M>
__device__ __forceinline__ void transpose_blocks(uint32_t (&x)[M], uint32_t* buf, int lane) {
    if constexpr (V::WV > 1)
        relayout<V, TransposeBlocks<V>>(x, buf, lane);
}

// transpose_square layout.hpp:24-61
template <class V, int M>
__device__ __forceinline__ void transpose_square(uint32_t (&x)[M], uint32_t* buf, int lane) {
    static_assert(V::WV == V::MV, "transpose_square needs a square view (NotSquare)");
    transpose_blocks<V>(x, buf, lane);
}

// convert_layout layout.hpp:357-391
template <class V, int M>
__device__ __forceinline__ void to_column_major(uint32_t (&x)[M], uint32_t* buf, int lane) {
    if constexpr (V::WV == 1 || V::MV == 1)
        return;
    else if constexpr (V::WV == V::MV)
        transpose_square<V>(x, buf, lane);
    else
        relayout<V, ToColumnMajor<V>>(x, buf, lane);
}
template <class V, int M>
__device__ __forceinline__ void to_row_major(uint32_t (&x)[M], uint32_t* buf, int lane) {
    if constexpr (V::WV == 1 || V::MV == 1)
        return;
    else if constexpr (V::WV == V::MV)
        transpose_square<V>(x, buf, lane);
    else
        relayout<V, ToRowMajor<V>>(x, buf, lane);
}

// ---------------------------------------------------------------------------
// Row-local sorts (the reference's for_rows sections; always conflict-free)
// ---------------------------------------------------------------------------
// sort_rows / radix_sort_rows: each active row in direction `asc` (per lane)
template <int PK, class V, int M>
__device__ __forceinline__ void row_sort(uint32_t (&x)[M], int lane, bool asc) {
    if constexpr (V::MV > 1) {
        if (V::active(lane)) {
            const uint32_t f = asc ? 0u : 0xFFFFFFFFu;
            flip<V::C0, V::MV>(x, f);
            sort_net<PK, V::C0, V::MV>(x);
            flip<V::C0, V::MV>(x, f);
        }
    }
}

// SortOrder::alternating(asc) sort.hpp:25-31 for the lane's local row
template <class V>
__device__ __forceinline__ bool alt_dir(int lane, bool asc) {
    return ((V::local(lane) % 2) == 0) == asc;
}

template <int PK, int OFF, int SEG, int NSEG, int M>
__device__ __forceinline__ void seg_nets(uint32_t (&x)[M]) {
    if constexpr (NSEG > 0) {
        sort_net<PK, OFF, SEG>(x);
        seg_nets<PK, OFF + SEG, SEG, NSEG - 1>(x);
    }
}

// merge_sort_segments sort.hpp:177-182: sort every SEG-wide segment of each row
template <int PK, class V, int SEG, int M>
__device__ __forceinline__ void seg_sort(uint32_t (&x)[M], int lane, bool asc) {
    static_assert(V::MV % SEG == 0, "segments must tile the window");
    if constexpr (SEG > 1) {
        if (V::active(lane)) {
            const uint32_t f = asc ? 0u : 0xFFFFFFFFu;
            flip<V::C0, V::MV>(x, f);
            seg_nets<PK, V::C0, SEG, V::MV / SEG>(x);
            flip<V::C0, V::MV>(x, f);
        }
    }
}

}  // namespace dmmdev

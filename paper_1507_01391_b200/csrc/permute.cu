// permute.cu -- kernel 4: the randomized permutation of Afshani & Sitchinava (section 3 /
// Appendix B) as one warp program per 32 x m machine, restating permute.hpp:545-628 step
// for step so the PermuteReport trajectory (shifts, hash draws, leftover history,
// packing or fallback, packed width, random-word count, cleanup retries) is bit-exact.
//
// Per warp (lane r = row / bank r):
//   * the instance's std::mt19937_64 lives in shared memory: lane 0 runs the seeding
//     recurrence, the warp runs each twist in parallel, draw d is temper(state[d % 312]);
//   * preprocess_shuffle: lane r rotates its row by its own draw (an own-bank smem
//     round trip), then every m x m block of rows is transposed (conflict-free relayout);
//   * each iteration draws the hash, recolours and compacts every row with an own-bank
//     counting sort (rescan_and_bucket), and runs alpha passes of m colour steps: in step
//     (p, k) every row sends its p-th label of colour k to its destination cell.  The
//     output region is laid out with row i in bank i, and the colouring guarantees the
//     destinations of one step are distinct rows: 0 bank conflicts by the paper's argument
//     (machines taller than 32 rows, whose distinct rows can share one of the 32 banks,
//     deliver into the instance's global output instead: see deliver());
//   * pack_leftovers' t shifted matching rounds use shuffles for the counter reads and
//     one conflict-free step per bundle word (partners are distinct per round);
//   * finish / fallback run the general-sort warp schedule (dmm_algos.cuh) on the packed
//     32 x m' or full 32 x m view, then the three-phase delivery (each phase step writes
//     distinct destination rows).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "general_kernel.cuh"
#include "dmm_rng.cuh"

namespace dmmdev {

struct PermArgs {
    uint32_t alpha;
    uint32_t iter_cap;
    uint64_t threshold;     // permute_threshold (host, double math as the reference)
    uint32_t t;             // matching rounds ceil(log2 w)^2
    uint32_t bundle;        // ceil(2m / t)
    uint32_t width_ok;      // bit b: width 2^b passes general_sort_shape_ok && cleanup_headroom (host)
    // step meter (dmm_permute_steps; NULL on the hot path): per instance kMeterWords words --
    // [0,1] the steps of every phase but the finish's sort (u64), [2] the delivery's steps,
    // [3] the finish sort's width (0: nothing sorted), [4] 1 if unmodelled (last-resort sort);
    // sort_in: the finish sort's input matrix, w x width words per instance (w x m capacity)
    uint32_t* meter;
    uint32_t* sort_in;
};
constexpr int kMeterWords = 8;

constexpr int kRngWords = 312;

// warps (machines) per CTA: the kernel only synchronises warps, so small CTAs let the
// per-warp shared-memory footprint, not the CTA granularity, set the occupancy
#ifndef DMM_PERM_WARPS
#define DMM_PERM_WARPS 4
#endif
constexpr int kPermWarps = DMM_PERM_WARPS;
// CTAs per SM asked of ptxas for 128-row machines (register cap 65536 / (128 * minb))
#ifndef DMM_PERM_TALL_MINB
#define DMM_PERM_TALL_MINB 3
#endif
// CTAs per SM asked of ptxas for 32-row machines (4 per CTA): 4 = 128 registers, no spills
// (ptxas's own choice: 168, 3 CTAs per SM); cfg4s 37.1 vs 36.4 G keys/s
#ifndef DMM_PERM_MINB32
#define DMM_PERM_MINB32 4
#endif

// Collective primitives of one machine of R rows: one warp (R = 32: shuffles and warp
// votes) or one CTA of R / 32 warps (R > 32: shared-memory exchange slots and CTA barriers).
// FAST (R > 32 machines whose colour-count area H holds them): every exchange / reduction is
// ONE barrier -- two alternating slot sets, so a slot is rewritten only two collectives later,
// after the intervening collective's barrier; otherwise the single-slot form (three barriers).
// Slots overlay the start of H, dead wherever a collective runs (see k_permute).
template <int R>
constexpr int mach_slot_words() { return 6 * R + 2 * (R / 32); }
template <int R, bool FAST = (R >= 128)>
struct Mach {
    uint32_t* xch;  // FAST: 2 x (3 R) exchange words, then 2 x (R / 32) reduction words
    uint32_t* red;
    int row;
    mutable uint32_t par = 0;  // FAST: the slot set of the next collective
    __device__ __forceinline__ void sync() const {
        if constexpr (R == kWarp)
            __syncwarp();
        else
            __syncthreads();
    }
    __device__ __forceinline__ uint32_t* slot() const { return xch + par * (3 * R); }
    __device__ __forceinline__ uint32_t* rslot() const { return xch + 6 * R + par * (R / 32); }
    // value of v held by row src (every row calls)
    __device__ __forceinline__ uint32_t shfl(uint32_t v, int src) const {
        if constexpr (R == kWarp) {
            return __shfl_sync(0xFFFFFFFFu, v, src);
        } else if constexpr (FAST) {
            uint32_t* x = slot();
            x[row] = v;
            __syncthreads();
            par ^= 1u;
            return x[src];
        } else {
            __syncthreads();
            xch[row] = v;
            __syncthreads();
            const uint32_t r = xch[src];
            __syncthreads();
            return r;
        }
    }
    // three values of row src at once (one barrier when FAST)
    __device__ __forceinline__ void shfl3(uint32_t& a, uint32_t& b, uint32_t& c, int src) const {
        if constexpr (R == kWarp || !FAST) {
            a = shfl(a, src);
            b = shfl(b, src);
            c = shfl(c, src);
        } else {
            uint32_t* x = slot();
            x[row] = a;
            x[R + row] = b;
            x[2 * R + row] = c;
            __syncthreads();
            par ^= 1u;
            a = x[src];
            b = x[R + src];
            c = x[2 * R + src];
        }
    }
    // FAST reductions: warp reduce, one word per warp, one barrier, every row combines
    template <class Op>
    __device__ __forceinline__ uint32_t reduce_fast(uint32_t v, Op op) const {
        uint32_t* r = rslot();
        if ((row & 31) == 0)
            r[row >> 5] = v;
        __syncthreads();
        par ^= 1u;
        uint32_t acc = r[0];
#pragma unroll
        for (int w = 1; w < R / 32; ++w)
            acc = op(acc, r[w]);
        return acc;
    }
    __device__ __forceinline__ uint32_t or_all(uint32_t v) const {
        if constexpr (R == kWarp)
            return __reduce_or_sync(0xFFFFFFFFu, v);
        else if constexpr (FAST)
            return reduce_fast(__reduce_or_sync(0xFFFFFFFFu, v), [](uint32_t a, uint32_t b) { return a | b; });
        else
            return group_or<R, R>(v, row, red);
    }
    __device__ __forceinline__ uint32_t max_all(uint32_t v) const {
        if constexpr (R == kWarp)
            return __reduce_max_sync(0xFFFFFFFFu, v);
        else if constexpr (FAST)
            return reduce_fast(__reduce_max_sync(0xFFFFFFFFu, v), [](uint32_t a, uint32_t b) { return max(a, b); });
        else
            return group_max<R, R>(v, row, red);
    }
    __device__ __forceinline__ uint32_t add_all(uint32_t v) const {
        if constexpr (R == kWarp) {
            return __reduce_add_sync(0xFFFFFFFFu, v);
        } else if constexpr (FAST) {
            return reduce_fast(__reduce_add_sync(0xFFFFFFFFu, v), [](uint32_t a, uint32_t b) { return a + b; });
        } else {
            v = __reduce_add_sync(0xFFFFFFFFu, v);
            __syncthreads();
            if ((row & 31) == 0)
                red[row >> 5] = v;
            __syncthreads();
            uint32_t r = 0;
#pragma unroll
            for (int w = 0; w < R / 32; ++w)
                r += red[w];
            __syncthreads();
            return r;
        }
    }
    __device__ __forceinline__ bool any(bool p) const {
        if constexpr (R == kWarp)
            return __any_sync(0xFFFFFFFFu, p);
        else
            return __syncthreads_or(p ? 1 : 0) != 0;
    }
};

// Machine-shared generator: the 312-word state in smem as two 32-bit arrays (low and
// high halves), so every warp-wide access is a unit-stride 32-bit access (no bank
// conflicts); `base` = index of the first draw the current state generation serves.
template <int R>
struct MachRng {
    uint32_t* lo;
    uint32_t* hi;
    int64_t base;

    __device__ uint64_t get(int i) const { return ((uint64_t)hi[i] << 32) | lo[i]; }
    __device__ void put(int i, uint64_t v) {
        lo[i] = (uint32_t)v;
        hi[i] = (uint32_t)(v >> 32);
    }
    __device__ void seed(uint64_t s, const Mach<R>& mc) {
        if (mc.row == 0) {
            uint64_t v = s;
            put(0, v);
            for (int i = 1; i < kRngWords; ++i) {
                v = 6364136223846793005ULL * (v ^ (v >> 62)) + (uint64_t)i;
                put(i, v);
            }
        }
        mc.sync();
        twist(mc);
        base = 0;
    }
    // mersenne twist of all 312 words: [0,156) from old words; [156,311) from new [0,155)
    // and old words; 311 from new 155 and new 0
    __device__ void twist(const Mach<R>& mc) {
        constexpr uint64_t MA = 0xB5026F5AA96619E9ULL;
        constexpr int T = (156 + R - 1) / R;
        uint64_t v[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int i = mc.row + R * t;
            if (i < 156) {
                // (mt[i] & UM) | (mt[i+1] & LM): the high 33 bits of mt[i], the low 31 of mt[i+1]
                const uint64_t x = ((uint64_t)hi[i] << 32) | (lo[i] & 0x80000000u) | (lo[i + 1] & 0x7FFFFFFFu);
                v[t] = get(i + 156) ^ (x >> 1) ^ ((x & 1) ? MA : 0);
            }
        }
        mc.sync();
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int i = mc.row + R * t;
            if (i < 156)
                put(i, v[t]);
        }
        mc.sync();
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int i = 156 + mc.row + R * t;
            if (i < 311) {
                const uint64_t x = ((uint64_t)hi[i] << 32) | (lo[i] & 0x80000000u) | (lo[i + 1] & 0x7FFFFFFFu);
                v[t] = get(i - 156) ^ (x >> 1) ^ ((x & 1) ? MA : 0);
            }
        }
        mc.sync();
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int i = 156 + mc.row + R * t;
            if (i < 311)
                put(i, v[t]);
        }
        mc.sync();
        if (mc.row == 0) {
            const uint64_t x = ((uint64_t)hi[311] << 32) | (lo[311] & 0x80000000u) | (lo[0] & 0x7FFFFFFFu);
            put(311, get(155) ^ (x >> 1) ^ ((x & 1) ? MA : 0));
        }
        mc.sync();
    }
    // load an engine mid-stream: the 312 state words and the position p of the next draw
    // (libstdc++'s mersenne_twister_engine layout _M_x[], _M_p): draw d reads word p + d
    __device__ void load(const uint64_t* state, const Mach<R>& mc) {
        for (int i = mc.row; i < kRngWords; i += R)
            put(i, state[i]);
        const uint64_t p = state[kRngWords];
        mc.sync();
        if (p >= (uint64_t)kRngWords) {
            twist(mc);
            base = 0;
        } else {
            base = -(int64_t)p;
        }
    }
    // make draw d (machine-uniform) addressable; advances generations as needed
    __device__ void advance_to(uint32_t d, const Mach<R>& mc) {
        while ((int64_t)d >= base + kRngWords) {
            twist(mc);
            base += kRngWords;
        }
    }
    __device__ uint64_t word(uint32_t d) const { return mt_temper(get((int)((int64_t)d - base))); }
};

__device__ __forceinline__ uint32_t hash_eval(uint64_t key, uint32_t m, uint32_t i) {  // HashOracle permute.hpp:39
    return (uint32_t)(splitmix64(key ^ ((uint64_t)i * 0x9e3779b97f4a7c15ULL)) % m);
}

// Where the output region lives.  32-row machines: shared memory with row i in column i
// (outs[j*R + i]): a colour step's destinations are distinct rows, i.e. distinct banks -- the
// paper's conflict-free delivery.  Taller machines (R > 32 rows on 32 physical banks: distinct
// rows can share a bank, the only shared accesses with excess wavefronts in r02) deliver
// straight into the instance's global output instead (label L is cell L of the row-major
// result), which also returns M x R words of shared memory per machine to occupancy.
// DMM_PERM_GOUT: 0 = always shared, 1 = R > 32 global (default), 2 = always global (A/B).
#ifndef DMM_PERM_GOUT
#define DMM_PERM_GOUT 1
#endif
template <int R>
__host__ __device__ constexpr bool perm_gout() { return DMM_PERM_GOUT == 2 || (DMM_PERM_GOUT == 1 && R > kWarp); }
template <int M, int R>
__device__ __forceinline__ void deliver(uint32_t* outs, uint32_t label) {
    // a label outside [0, n) (an input the status byte rejects as InvalidInstance) has no cell
    if (label >= (uint32_t)(R * M))
        return;
    if constexpr (perm_gout<R>())
        outs[label] = label;  // cell (label / M, label % M) of the instance's row-major output
    else
        outs[(label % M) * R + label / M] = label;
}

// Three-phase delivery (permute.hpp:452-529) of one row's lexicographically sorted packed
// row (own bank of q: q[c*R + row], c < WP; empty labels at the tail) into the output
// region (deliver()).
template <int M, int R>
__device__ __forceinline__ void three_phase_delivery(const uint32_t* q, int wp, uint32_t* outs, const Mach<R>& mc,
                                                     uint32_t empty, uint32_t* deliv_steps = nullptr) {
    const int row = mc.row;
    int cnt = 0;
    for (int c = 0; c < wp; ++c)
        cnt += q[c * R + row] != empty ? 1 : 0;
    int f = 0, l0 = cnt;
    if (cnt > 0) {
        const uint32_t i_first = q[row] / M, i_last = q[(cnt - 1) * R + row] / M;
        while (f < cnt && q[f * R + row] / M == i_first)
            ++f;
        if (i_last != i_first)
            while (l0 > f && q[(l0 - 1) * R + row] / M == i_last)
                --l0;
        else
            l0 = f;
    }
    // middle labels: destination rows owned by this packed row alone, one per step
    const int nmid = l0 - f;
    const int max_mid = (int)mc.max_all((uint32_t)nmid);
    if (deliv_steps) {
        // the reference's send() costs a read and a write step per non-empty batch: every
        // middle step, and every slot j some row's first (last) group sends at
        uint64_t jf = 0, jl = 0;
        for (int c = 0; c < f; ++c)
            jf |= 1ull << (q[c * R + row] % M);
        for (int c = l0; c < cnt; ++c)
            jl |= 1ull << (q[c * R + row] % M);
        const uint32_t nf = __popcll(((uint64_t)mc.or_all((uint32_t)(jf >> 32)) << 32) | mc.or_all((uint32_t)jf));
        const uint32_t nl = __popcll(((uint64_t)mc.or_all((uint32_t)(jl >> 32)) << 32) | mc.or_all((uint32_t)jl));
        *deliv_steps = 2u * ((uint32_t)max_mid + nf + nl);
    }
    for (int k = 0; k < max_mid; ++k) {
        if (k < nmid) {
            const uint32_t label = q[(f + k) * R + row];
            deliver<M, R>(outs, label);
        }
    }
    // first group, then last group: at step j every row sends its label with slot j
    int pf = 0, pl = l0;
    for (int j = 0; j < M; ++j) {
        if (pf < f) {
            const uint32_t label = q[pf * R + row];
            if (label % M == (uint32_t)j) {
                deliver<M, R>(outs, label);
                ++pf;
            }
        }
    }
    for (int j = 0; j < M; ++j) {
        if (pl < cnt) {
            const uint32_t label = q[pl * R + row];
            if (label % M == (uint32_t)j) {
                deliver<M, R>(outs, label);
                ++pl;
            }
        }
    }
    // the steps only write the output region (each destination cell once) and read the row's
    // own column: no step needs a barrier of its own; one ends the delivery
    mc.sync();
}

// finish (permute.hpp:536-541) on a packed R x WP view held in registers y[0..WP):
// integer_sort_general(packed, n+1, -, enforce=false), then the three-phase delivery.
// Returns false on PostconditionFailed (strict): the caller falls back.
template <int WP, int M, int R>
__device__ __forceinline__ bool finish_packed(uint32_t (&y)[WP], uint32_t* buf, uint32_t* q, uint32_t* outs,
                                              const Mach<R>& mc, uint32_t empty, uint32_t& retries,
                                              uint32_t* meter = nullptr, uint32_t* sort_in = nullptr) {
    using V = VF<0xFFFFFFFFu, 0, 1, R, 0, WP, R, R>;
    if (meter) {  // the finish sort's input, for the host-side meter of integer_sort_general
#pragma unroll
        for (int c = 0; c < WP; ++c)
            sort_in[(uint64_t)mc.row * WP + c] = y[c];
        if (mc.row == 0)
            meter[3] = WP;
    }
    GenResult res{{0u, 0u}, 0u};
    balance_divide_sort<1, V, false, 0x80000000u>(y, buf, mc.row, res);  // packed labels <= n < 2^31
    if constexpr (R == kWarp)
        res.finish();
    else
        res.template finish_machine<R>(mc.row, mc.red);
    if (res.unsorted & 1u)
        return false;
    retries = res.retries[0];
    mc.sync();
#pragma unroll
    for (int c = 0; c < WP; ++c)
        q[c * R + mc.row] = y[c];
    mc.sync();
    uint32_t ds = 0;
    three_phase_delivery<M, R>(q, WP, outs, mc, empty, meter ? &ds : nullptr);
    if (meter && mc.row == 0)
        meter[2] = ds;
    return true;
}

// stage = [H: per-colour counts / bucket bounds as bytes (<= m <= 64), ceil(M/4)*R words | B: the
// colour-sorted rows, M*R words]; the relayout buffer overlays it (B's contents are always in
// registers before a sort uses the buffer)
template <int M, int R>
__host__ __device__ constexpr int perm_h_words() { return ((M + 3) / 4) * R; }  // 4 colours per word
template <int M, int R>
__host__ __device__ constexpr int perm_stage_words() {
    return (perm_h_words<M, R>() + M * R > relayout_buf_words(M) * (R / 32) ? perm_h_words<M, R>() + M * R
                                                                             : relayout_buf_words(M) * (R / 32));
}
template <int M, int R>
__host__ __device__ constexpr int perm_machine_words() {  // u32 words of smem per machine
    return 2 * kRngWords + (perm_gout<R>() ? 0 : M * R) + perm_stage_words<M, R>();
}
template <int R>
__host__ __device__ constexpr int perm_machines_per_cta() { return R > kWarp ? 1 : kPermWarps; }

// packed finish of width WP when the machine shape admits it (width_ok gates it on the host)
template <int WP, int M, int R>
__device__ __forceinline__ bool finish_width(uint32_t width, const uint32_t* pk, uint32_t* stage, uint32_t* B,
                                             uint32_t* outs, const Mach<R>& mc, uint32_t empty, uint32_t& retries,
                                             bool& handled, uint32_t* meter, uint32_t* sort_in) {
    if constexpr (WP >= 2 && 2 * WP <= M && general_shape_ok_c(R, WP, false)) {
        if (width == (uint32_t)WP) {
            handled = true;
            uint32_t y[WP];
#pragma unroll
            for (int c = 0; c < WP; ++c)
                y[c] = pk[c * R + mc.row];
            return finish_packed<WP, M, R>(y, stage, B, outs, mc, empty, retries, meter, sort_in);
        }
    }
    return false;
}

template <int M, int R, bool METER = false>
__global__ void __launch_bounds__(perm_machines_per_cta<R>() * R, (R >= 128 ? DMM_PERM_TALL_MINB : R == kWarp ? DMM_PERM_MINB32 : 1)) k_permute(
    const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t count, const uint64_t* __restrict__ seeds,
    const uint64_t* __restrict__ states, PermArgs a, dmm_permute_report* __restrict__ reps, uint64_t* __restrict__ hist,
    uint32_t* __restrict__ shifts_out, uint8_t* __restrict__ status) {
    extern __shared__ uint64_t smem64[];
    constexpr int W = R;
    constexpr uint32_t n = W * M;
    constexpr uint32_t empty = n;  // empty_label permute.hpp:88
    constexpr bool kMulti = R > kWarp;
    const int row = kMulti ? (int)threadIdx.x : (int)(threadIdx.x & 31);
    const int mach = kMulti ? 0 : (int)(threadIdx.x >> 5);
    uint32_t* wbase = reinterpret_cast<uint32_t*>(smem64) + mach * perm_machine_words<M, R>();
    MachRng<R> rng{wbase, wbase + kRngWords, 0};
    constexpr bool kGOut = perm_gout<R>();
    const uint64_t k = (uint64_t)blockIdx.x * perm_machines_per_cta<R>() + mach;
    // output region: shared, row i in column i (outs[j*R + i]), or the instance's global output
    uint32_t* outs = kGOut ? out + k * (uint64_t)n : wbase + 2 * kRngWords;
    uint32_t* stage = wbase + 2 * kRngWords + (kGOut ? 0 : M * R);  // relayout buffer / own-bank rows A,B,H
    uint32_t* B = stage + perm_h_words<M, R>();  // colour-sorted (compacted) row
    uint32_t* pk = B;                            // packed rows (own column), capacity m: aliases B,
                                                 // which is dead from packing until the finish
    uint8_t* H = reinterpret_cast<uint8_t*>(stage);  // per-colour counts, then bucket bounds
    // colour b of this row: byte b % 4 of word (b / 4) * R + row -- the row's own bank, for
    // any (data-dependent) colour
    auto hx = [&](uint32_t b) -> uint32_t { return (((b >> 2) * (uint32_t)R + (uint32_t)row) << 2) | (b & 3u); };
    // R > 32: the machine's exchange / reduction scratch overlays the start of the colour
    // counts H: every use (input check, leftover sum, packing rounds, finish reductions,
    // delivery) falls where H is dead (and CTA barriers separate them from its uses)
    static_assert(R < 128 || perm_h_words<M, R>() >= mach_slot_words<R>(), "FAST slots overlay H");
    const Mach<R> mc{stage, stage + R, row};
    if (k >= count)
        return;

    // METER = false (the hot instantiation): the step-meter code is compiled out, which keeps
    // its live ranges out of the register allocation
    uint32_t* meter = METER && a.meter ? a.meter + k * kMeterWords : nullptr;
    uint32_t* sort_in = METER && a.meter ? a.sort_in + k * (uint64_t)W * M : nullptr;
    uint64_t pre = 0;  // metered steps outside the finish's sort (machine-uniform)
    constexpr uint32_t kLogW = (uint32_t)ilog2_ceil_c(W);
    if (meter && row < kMeterWords)
        meter[row] = 0;

    uint32_t x[M];
    load_row<M>(in + (k * W + row) * M, x);
    uint32_t badkey = 0;
#pragma unroll
    for (int c = 0; c < M; ++c) {
        badkey |= x[c] >= n ? 1u : 0u;
        if constexpr (!kGOut)
            outs[c * R + row] = 0xFFFFFFFFu;  // sentinel: undelivered
    }
    badkey = mc.or_all(badkey);
    if constexpr (kGOut) {
        // sentinel: undelivered.  After the machine barrier of or_all every row is in registers
        // (in == out allowed), and the first delivery follows several more barriers
        uint32_t sent[M];
#pragma unroll
        for (int c = 0; c < M; ++c)
            sent[c] = 0xFFFFFFFFu;
        store_row<M>(outs + (uint64_t)row * M, sent);
    }
    if (states)
        rng.load(states + k * (kRngWords + 1), mc);
    else
        rng.seed(seeds[k], mc);

    uint64_t random_words = 0;
    uint32_t drawn = 0;
    // ---- preprocess_shuffle permute.hpp:109-142 ---------------------------------------
    {
        rng.advance_to(drawn + W - 1, mc);
        const uint32_t s = 1u + (uint32_t)(rng.word(drawn + row) % M);  // rng_below(M), M a power of two
        drawn += W;
        random_words += W;
        if (shifts_out)
            shifts_out[k * W + row] = s;
        const uint32_t sh = s % M;
        mc.sync();
#pragma unroll
        for (int c = 0; c < M; ++c)
            B[((c + sh) % M) * R + row] = x[c];  // own bank: row r rotates in its own column
        mc.sync();
#pragma unroll
        for (int c = 0; c < M; ++c)
            x[c] = B[c * R + row];
        using Blk = VF<0xFFFFFFFFu, 0, 1, M, 0, M, R, R>;  // every aligned m x m block of rows
        transpose_square<Blk>(x, stage, row);
        if (meter) {
            // rows rotating by s != 0 read and write all m cells (gcd cycles); the m x m block
            // transposes run in lockstep: 2 (m - 1) steps (permute.hpp:118-140)
            pre += (mc.any(sh != 0) ? 2u * M : 0u) + 2u * (M - 1);
        }
    }

    // ---- iterations permute.hpp:570-577 ---------------------------------------------------
    uint64_t leftover = n;
    uint32_t iterations = 0;
    while (leftover > a.threshold && iterations < a.iter_cap) {
        // draw_and_broadcast_hash permute.hpp:147-166: m draws, key = the first
        rng.advance_to(drawn, mc);
        const uint64_t key = rng.word(drawn);
        drawn += M;
        random_words += M;
        // rescan_and_bucket permute.hpp:174-216: stable own-bank counting sort by colour.
        // Every access below is to the row's own column (H, B columns = row): conflict-free
        // for any data.
        mc.sync();
#pragma unroll
        for (int b = 0; b < M; ++b)
            H[hx(b)] = 0;
        // h(i) for the source rows i: row l evaluates h(l) once, keys fetch theirs by
        // shuffle (R = 32) or from the machine's hash table (one lookup instead of a 64-bit
        // splitmix64 per key)
        // R > 32: lane l of every warp holds h(l + 32 t) for t < R / 32 in registers and a key
        // fetches h(i) with R / 32 shuffles (a shared table lookup by data-dependent row would
        // conflict on banks)
        constexpr int kHT = R / kWarp;
        uint32_t h_reg[kHT];
#pragma unroll
        for (int t = 0; t < kHT; ++t)
            h_reg[t] = hash_eval(key, M, (uint32_t)((row & 31) + kWarp * t));
        const uint32_t h_row = h_reg[0];
        // colour of a label (recomputed in both passes: keeping M colours live would cost M
        // registers)
        auto colour_of = [&](uint32_t lab) -> uint32_t {
            const bool live = lab != empty;
            const uint32_t i = live ? lab / M : 0u, j = lab % M;
            uint32_t hi;
            if constexpr (kMulti) {
                hi = 0;
#pragma unroll
                for (int t = 0; t < kHT; ++t) {
                    const uint32_t v = __shfl_sync(0xFFFFFFFFu, h_reg[t], (int)(i & 31u));
                    hi = (i >> 5) == (uint32_t)t ? v : hi;
                }
            } else {
                hi = __shfl_sync(0xFFFFFFFFu, h_row, (int)(i & 31u));
            }
            return (j + M - hi) % M;
        };
#pragma unroll
        for (int c = 0; c < M; ++c) {
            const uint32_t cl = colour_of(x[c]);
            if (x[c] != empty)
                H[hx(cl)] += 1;
        }
        uint32_t run = 0;
        uint32_t row_left = 0;
#pragma unroll
        for (int b = 0; b < M; ++b) {
            const uint32_t cnt = H[hx(b)];
            row_left += cnt > a.alpha ? cnt - a.alpha : 0;
            H[hx(b)] = (uint8_t)run;  // bucket start
            run += cnt;
        }
#pragma unroll
        for (int c = 0; c < M; ++c)
            if ((uint32_t)c >= run)
                B[c * R + row] = empty;
        // scatter into the colour-sorted order
#pragma unroll
        for (int c = 0; c < M; ++c) {
            const uint32_t cl = colour_of(x[c]);
            if (x[c] != empty) {
                const uint32_t pos = H[hx(cl)];
                H[hx(cl)] = (uint8_t)(pos + 1);
                B[pos * R + row] = x[c];
            }
        }
        // communication_phase permute.hpp:225-274.  Step (pass p, colour k): every row sends
        // its p-th label of colour k to out[i][j]; the output region keeps row i in column i
        // and the colouring makes the destinations of one step distinct rows, so on a 32-row
        // machine every step is one conflict-free warp-wide store (taller machines map rows
        // to 32 banks, where distinct rows can share one).  H holds the bucket ends now.
        // A sent label's cell becomes empty in place (the compacted row keeps its holes):
        // exactly the first min(count, alpha) cells of every colour bucket.
        for (int kc = 0; kc < M; ++kc) {
            const uint32_t end = H[hx(kc)];
            const uint32_t start = kc == 0 ? 0u : H[hx(kc - 1)];
            const uint32_t take = min(end - start, a.alpha);
            for (uint32_t p = 0; p < take; ++p) {
                const uint32_t label = B[(start + p) * R + row];
                deliver<M, R>(outs, label);
                B[(start + p) * R + row] = empty;
            }
        }
#pragma unroll
        for (int c = 0; c < M; ++c)
            x[c] = B[c * R + row];
        // synchronize permute.hpp:278-285 (the barrier: H, which the exchange slots overlay, is
        // still read by rows in their communication loop)
        mc.sync();
        leftover = mc.add_all(row_left);
        if (meter) {
            // draw_and_broadcast_hash: min(m, w) writes + doubling to w (permute.hpp:147-166);
            // rescan_and_bucket: 5 m + 6 (live labels) accesses on the busiest row (:174-216);
            // communication: 3 steps per colour step, empty ones included (:225-274);
            // synchronize: one write, tree sum 2 log w, broadcast 1 + 2 log w (:278-285)
            constexpr uint32_t h0 = M < W ? M : W;
            uint32_t dbl = 0;
            for (uint32_t have = h0; have < W; have *= 2)
                ++dbl;
            pre += h0 + 2u * dbl + 5u * M + 6u * mc.max_all(run) + 3u * a.alpha * M + 2u + 4u * kLogW;
        }
        if (row == 0 && hist && iterations < DMM_PERMUTE_MAX_HIST)
            hist[k * DMM_PERMUTE_MAX_HIST + iterations] = leftover;
        ++iterations;
    }

    bool delivered = leftover == 0;
    bool used_packing = false, fallback = false;
    uint32_t packed_width = 0, cleanup_retries = 0;
    if (!delivered && leftover <= a.threshold) {
        // ---- pack_leftovers permute.hpp:298-443 -------------------------------------------
        const uint32_t theta = (uint32_t)((2 * leftover + W - 1) / W) + a.alpha;
        uint32_t width = 1;
        while (width < theta + a.bundle + 1)
            width <<= 1;
        while (2 * width <= M && !((a.width_ok >> (31 - __clz(width))) & 1u))
            width <<= 1;
        if (2 * width <= M) {
            // compaction into the packed rows (own column)
            if (meter) {
                // compaction: m reads, the live writes, the pad to width, two counter writes;
                // then t rounds of 5 + 2 bundle steps, empty batches included (:327-423)
                uint32_t live = 0;
#pragma unroll
                for (int c = 0; c < M; ++c)
                    live += x[c] != empty ? 1u : 0u;
                pre += M + max(mc.max_all(live), width) + 2u + (uint64_t)a.t * (5u + 2u * a.bundle);
            }
            uint32_t load = 0;
            mc.sync();
#pragma unroll
            for (int c = 0; c < M; ++c)
                if (x[c] != empty)
                    pk[(load++) * R + row] = x[c];
            for (uint32_t c = load; c < width; ++c)
                pk[c * R + row] = empty;
            uint32_t cell_load = load, cell_cursor = load;
            bool recv = false;
            random_words += a.t;
            for (uint32_t round = 0; round < a.t; ++round) {
                rng.advance_to(drawn, mc);
                const uint32_t shift = 1u + (uint32_t)(rng.word(drawn) % W);  // rng_below(W), W a power of two
                ++drawn;
                const int partner = (row + (int)shift) % W, src = (row - (int)shift + W) % W;
                // the partner's (load | received) and cursor cells, one exchange
                uint32_t p_load = cell_load, p_recv_u = recv ? 1u : 0u, p_cursor = cell_cursor;
                mc.shfl3(p_load, p_recv_u, p_cursor, partner);
                const bool p_recv = p_recv_u != 0;
                const bool sender = load > theta && !p_recv && p_load <= theta;
                const uint32_t give = sender ? min(a.bundle, load) : 0u;
                // bundle moves into the partner's column: a sender's partner is never a sender
                // (its load is <= theta), so no row reads a cell another row writes here -- the
                // reference's lockstep steps need no barrier of their own (one after the loop)
                for (uint32_t kk = 0; kk < give; ++kk)
                    if (p_cursor + kk < M)
                        pk[(p_cursor + kk) * R + partner] = pk[(load - 1 - kk) * R + row];
                mc.sync();
                uint32_t got_u = sender ? 1u : 0u, give_in = give, unused = 0;
                mc.shfl3(got_u, give_in, unused, src);
                const bool got = got_u != 0;
                if (sender) {
                    cell_load = load - give;  // the own-load write lands last (permute.hpp:415-419)
                    recv = false;
                } else if (got) {
                    cell_load = cell_load + give_in;
                    recv = true;
                }
                if (got)
                    cell_cursor = cell_cursor + give_in;
                load = load - give + (got ? give_in : 0u);
            }
            const bool overflow = mc.any(load > width);
            if (meter && !overflow)
                pre += mc.max_all(width > load ? width - load : 0u);  // the final pad (:431-434)
            if (!overflow) {
                mc.sync();
                for (uint32_t c = load; c < width; ++c)
                    pk[c * R + row] = empty;
                mc.sync();
                used_packing = true;
                packed_width = width;
                bool ok = false, handled = false;
                ok = finish_width<2, M, R>(width, pk, stage, B, outs, mc, empty, cleanup_retries, handled, meter, sort_in) || ok;
                ok = finish_width<4, M, R>(width, pk, stage, B, outs, mc, empty, cleanup_retries, handled, meter, sort_in) || ok;
                ok = finish_width<8, M, R>(width, pk, stage, B, outs, mc, empty, cleanup_retries, handled, meter, sort_in) || ok;
                ok = finish_width<16, M, R>(width, pk, stage, B, outs, mc, empty, cleanup_retries, handled, meter, sort_in) || ok;
                ok = finish_width<32, M, R>(width, pk, stage, B, outs, mc, empty, cleanup_retries, handled, meter, sort_in) || ok;
                delivered = ok;
                // a packed sort that ran out of cleanup retries: the reference recovers its
                // clock past the failed attempt's stamps -- not modelled
                if (meter && handled && !ok && row == 0)
                    meter[4] = 1;
            }
        }
    }
    if (!delivered) {
        // ---- deterministic fallback permute.hpp:597-626 --------------------------------
        fallback = true;
        uint32_t y[M];
        {
            uint32_t o = 0;
            mc.sync();
#pragma unroll
            for (int c = 0; c < M; ++c)
                if (x[c] != empty)
                    B[(o++) * R + row] = x[c];
            for (uint32_t c = o; c < M; ++c)
                B[c * R + row] = empty;
            mc.sync();
#pragma unroll
            for (int c = 0; c < M; ++c)
                y[c] = B[c * R + row];
        }
        pre += meter ? 2u * M : 0u;  // in-place compaction: m reads + m writes per row (:602-614)
        uint32_t r2 = 0;
        if (!finish_packed<M, M, R>(y, stage, B, outs, mc, empty, r2, meter, sort_in) && M < W) {
            if (meter && row == 0)
                meter[4] = 1;  // the last-resort tall sort: not modelled
            // last resort: comparison tall sort of the working window left by the failed
            // attempt (permute.hpp:618-625) -- y, the same multiset in the attempt's arrangement
            using V = VF<0xFFFFFFFFu, 0, 1, R, 0, M, R, R>;
            if constexpr (M < W)
                sort_tall<1, V>(y, stage, row);
            mc.sync();
#pragma unroll
            for (int c = 0; c < M; ++c)
                B[c * R + row] = y[c];
            mc.sync();
            three_phase_delivery<M, R>(B, M, outs, mc, empty);
        } else {
            cleanup_retries = r2;
        }
    }
    mc.sync();
    // output region (row i in column i) -> global row-major; verify the bijection
    uint32_t v[M];
    uint32_t wrong = badkey, undelivered = 0;
    if constexpr (kGOut) {
        // the deliveries of every row of this CTA are visible after the barrier (coherent
        // loads: the cells were written in this kernel)
        if constexpr (M % 4 == 0) {
            const uint4* q4 = reinterpret_cast<const uint4*>(outs + (uint64_t)row * M);
#pragma unroll
            for (int i = 0; i < M / 4; ++i) {
                const uint4 t = q4[i];
                v[4 * i] = t.x;
                v[4 * i + 1] = t.y;
                v[4 * i + 2] = t.z;
                v[4 * i + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < M; ++j)
                v[j] = outs[(uint64_t)row * M + j];
        }
    } else {
#pragma unroll
        for (int j = 0; j < M; ++j)
            v[j] = outs[j * R + row];
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const uint32_t o = v[j];
        wrong |= o != (uint32_t)row * M + j ? 1u : 0u;
        undelivered |= o == 0xFFFFFFFFu ? 1u : 0u;
        v[j] = o == 0xFFFFFFFFu ? 0u : o;  // undelivered cells keep the machine's zero
    }
    wrong = mc.or_all(wrong);
    if (!kGOut || undelivered)
        store_row<M>(out + (k * W + row) * M, v);
    if (row == 0) {
        if (meter) {
            meter[0] = (uint32_t)pre;
            meter[1] = (uint32_t)(pre >> 32);
        }
        if (reps) {
            dmm_permute_report r;
            r.iterations = iterations;
            r.fallback = fallback;
            r.used_packing = used_packing;
            r.packed_width = packed_width;
            r.threshold = a.threshold;
            r.random_words = random_words;
            r.cleanup_retries = cleanup_retries;
            r.n_hist = min(iterations, (uint32_t)DMM_PERMUTE_MAX_HIST);
            reps[k] = r;
        }
        if (status)
            status[k] = wrong ? DMM_INVALID_INSTANCE : DMM_OK;
    }
}

}  // namespace dmmdev

namespace {

using namespace dmmhost;

uint64_t permute_threshold(uint32_t w, uint32_t m) {  // permute.hpp:97-101
    const double L = std::max(std::log(double(w)) / std::log(double(m)), 2.0);
    const double t = std::ceil(double(w) * m / (L * L * L));
    return std::max<uint64_t>(uint64_t(t), w);
}

template <int M, int R = dmmdev::kWarp>
dmm_status launch_permute(const uint32_t* in, uint32_t* out, uint64_t count, const uint64_t* seeds,
                          const uint64_t* states, const dmmdev::PermArgs& a, dmm_permute_report* reps, uint64_t* hist,
                          uint32_t* shifts, uint8_t* status, cudaStream_t s) {
    constexpr int kMach = dmmdev::perm_machines_per_cta<R>();
    auto kern = a.meter ? dmmdev::k_permute<M, R, true> : dmmdev::k_permute<M, R, false>;
    // DMM_PERM_PAD_KB (occupancy sensitivity A/B): extra dynamic shared memory per CTA
    static const size_t pad = getenv("DMM_PERM_PAD_KB") ? size_t(atoi(getenv("DMM_PERM_PAD_KB"))) * 1024 : 0;
    const size_t smem = size_t(kMach) * dmmdev::perm_machine_words<M, R>() * sizeof(uint32_t) + pad;
    static std::atomic<uint64_t> configured[2];  // devices configured, per instantiation (static: zeroed)
    if (dmm_status e = configure_kernel(kern, smem, configured[a.meter ? 1 : 0]); e != DMM_OK)
        return e;
    const uint64_t blocks = (count + kMach - 1) / kMach;
    if (blocks > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;  // grid x limit
    kern<<<unsigned(blocks), kMach * R, smem, s>>>(in, out, count, seeds, states, a, reps, hist, shifts, status);
    return check_launch("k_permute");
}

}  // namespace

extern "C" {

uint64_t dmm_permute_workspace_bytes(uint32_t w, uint32_t m, uint64_t count) {
    (void)w;
    (void)m;
    (void)count;
    return 0;  // the generator state lives in shared memory
}

}  // extern "C"

using namespace dmmhost;

static dmm_status permute_impl(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                       const uint64_t* seeds, const uint64_t* states, uint32_t alpha, uint32_t iter_cap, dmm_permute_report* reports,
                       uint64_t* history, uint32_t* shifts, uint8_t* status, void* workspace, void* stream,
                       uint32_t* meter = nullptr, uint32_t* sort_in = nullptr) {
    reset_launches();
    (void)workspace;
    if (m < 2 || w % m != 0)  // permute.hpp:547-548
        return DMM_SHAPE_VIOLATION;
    if (!general_sort_shape_ok(w, m, false))  // permute.hpp:549-550
        return DMM_SHAPE_VIOLATION;
    if (count == 0)
        return DMM_OK;
    if (!in || !out || (!seeds && !states))
        return DMM_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) {
        set_error("in/out must be 16-byte aligned");
        return DMM_INVALID_ARGUMENT;
    }
    dmmdev::PermArgs a;
    a.meter = meter;
    a.sort_in = sort_in;
    a.alpha = alpha;
    a.iter_cap = iter_cap;
    a.threshold = permute_threshold(w, m);
    const uint32_t lg = ilog2_ceil(w);
    a.t = std::max<uint32_t>(1, lg * lg);
    a.bundle = (2 * m + a.t - 1) / a.t;
    a.width_ok = 0;
    for (uint32_t b = 0; b < 31; ++b) {  // cleanup_headroom + shape check, permute.hpp:314-320
        const uint64_t wd = 1ull << b;
        if (wd > m)
            break;
        const double band = std::pow(2.0, 2.0 * std::log2(double(w)) / std::log2(double(wd)));
        const bool headroom = band <= 0.5 * double(wd) * double(ilog2_ceil(w));
        if (general_sort_shape_ok(w, wd, false) && headroom)
            a.width_ok |= 1u << b;
    }
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (w == 32) {
        switch (m) {
            case 2: return launch_permute<2>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
            case 4: return launch_permute<4>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
            case 16: return launch_permute<16>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
            case 32: return launch_permute<32>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
            default: break;
        }
    } else if (w == 64) {  // machines of two warps (one per CTA)
        switch (m) {
            case 8: return launch_permute<8, 64>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
            case 16:
                return launch_permute<16, 64>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
            default: break;
        }
    } else if (w == 128) {  // n = 8192: the reference's own permute shape at the BASELINE's n
        switch (m) {
            case 64:
                return launch_permute<64, 128>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
            default: break;
        }
    }
    set_error("no permute kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}


extern "C" {

dmm_status dmm_permute(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                       const uint64_t* seeds, uint32_t alpha, uint32_t iter_cap, dmm_permute_report* reports,
                       uint64_t* history, uint32_t* shifts, uint8_t* status, void* workspace, void* stream) {
    return permute_impl(in, out, w, m, count, seeds, nullptr, alpha, iter_cap, reports, history, shifts, status,
                        workspace, stream);
}

dmm_status dmm_permute_from_state(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                  const uint64_t* rng_states, uint32_t alpha, uint32_t iter_cap,
                                  dmm_permute_report* reports, uint64_t* history, uint32_t* shifts, uint8_t* status,
                                  void* stream) {
    return permute_impl(in, out, w, m, count, nullptr, rng_states, alpha, iter_cap, reports, history, shifts, status,
                        nullptr, stream);
}

// The permutation's modelled step count (RunReport.steps after run_algorithm(permute),
// instance.hpp:357): the permutation kernel replays every phase's data-dependent cost
// (PermArgs::meter) and hands over the matrix its finish sorted; that sort is metered by
// dmm_general_steps (integer_sort_general with domain n + 1, the finish's call permute.hpp:
// 536-541).  Off the hot path: allocates its buffers, synchronises the stream.
dmm_status dmm_permute_steps(const uint32_t* in, uint32_t w, uint32_t m, uint64_t count, const uint64_t* seeds,
                             uint32_t alpha, uint32_t iter_cap, uint64_t* steps, void* stream) {
    if (count == 0)
        return DMM_OK;
    if (!in || !seeds || !steps)
        return DMM_INVALID_ARGUMENT;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t n = uint64_t(w) * m;
    uint32_t *dout = nullptr, *dmeter = nullptr, *dsort = nullptr;
    auto release = [&]() {
        cudaFree(dout);
        cudaFree(dmeter);
        cudaFree(dsort);
    };
    if (cudaMalloc(reinterpret_cast<void**>(&dout), count * n * 4) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&dmeter), count * dmmdev::kMeterWords * 4) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&dsort), count * n * 4) != cudaSuccess) {
        release();
        return check_launch("cudaMalloc (permute meter)");
    }
    dmm_status e = permute_impl(in, dout, w, m, count, seeds, nullptr, alpha, iter_cap, nullptr, nullptr, nullptr,
                                nullptr, nullptr, stream, dmeter, dsort);
    std::vector<uint32_t> hm(count * dmmdev::kMeterWords);
    if (e == DMM_OK && cudaMemcpyAsync(hm.data(), dmeter, hm.size() * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        e = check_launch("meter D2H");
    if (e == DMM_OK && cudaStreamSynchronize(st) != cudaSuccess)
        e = check_launch("permute meter");
    std::vector<uint64_t> total(count, 0);
    // the finish sorts, grouped by width: each group's matrices gathered and metered in one call
    std::vector<uint32_t> widths;
    for (uint64_t k = 0; k < count && e == DMM_OK; ++k) {
        const uint32_t* r = hm.data() + k * dmmdev::kMeterWords;
        total[k] = (uint64_t(r[1]) << 32 | r[0]) + r[2];
        if (r[3] && std::find(widths.begin(), widths.end(), r[3]) == widths.end())
            widths.push_back(r[3]);
    }
    for (uint32_t wd : widths) {
        if (e != DMM_OK)
            break;
        std::vector<uint64_t> idx;
        for (uint64_t k = 0; k < count; ++k)
            if (hm[k * dmmdev::kMeterWords + 3] == wd)
                idx.push_back(k);
        uint32_t* g = nullptr;
        uint64_t* gs = nullptr;
        if (cudaMalloc(reinterpret_cast<void**>(&g), idx.size() * w * wd * 4) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&gs), idx.size() * 8) != cudaSuccess) {
            cudaFree(g);
            e = check_launch("cudaMalloc (permute meter group)");
            break;
        }
        for (uint64_t i = 0; i < idx.size() && e == DMM_OK; ++i)
            if (cudaMemcpyAsync(g + i * w * wd, dsort + idx[i] * n, uint64_t(w) * wd * 4, cudaMemcpyDeviceToDevice,
                                st) != cudaSuccess)
                e = check_launch("meter gather");
        if (e == DMM_OK)
            e = dmm_general_steps(g, w, wd, idx.size(), n + 1, gs, nullptr, stream);
        std::vector<uint64_t> hs(idx.size());
        if (e == DMM_OK && cudaMemcpyAsync(hs.data(), gs, hs.size() * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
            e = check_launch("meter D2H");
        if (e == DMM_OK && cudaStreamSynchronize(st) != cudaSuccess)
            e = check_launch("permute meter sort");
        for (uint64_t i = 0; i < idx.size() && e == DMM_OK; ++i)
            total[idx[i]] += hs[i];
        cudaFree(g);
        cudaFree(gs);
    }
    for (uint64_t k = 0; k < count; ++k)
        if (hm[k * dmmdev::kMeterWords + 4])
            total[k] = 0;  // not modelled (a failed packed sort's clock recovery / the tall sort)
    if (e == DMM_OK && cudaMemcpyAsync(steps, total.data(), count * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
        e = check_launch("steps H2D");
    if (e == DMM_OK && cudaStreamSynchronize(st) != cudaSuccess)
        e = check_launch("permute meter");
    release();
    return e;
}

}  // extern "C"

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
//     destinations of one step are distinct rows: 0 bank conflicts by the paper's argument;
//   * pack_leftovers' t shifted matching rounds use shuffles for the counter reads and
//     one conflict-free step per bundle word (partners are distinct per round);
//   * finish / fallback run the general-sort warp schedule (dmm_algos.cuh) on the packed
//     32 x m' or full 32 x m view, then the three-phase delivery (each phase step writes
//     distinct destination rows).
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
};

constexpr int kRngWords = 312;
// warps (machines) per CTA: the kernel only synchronises warps, so small CTAs let the
// per-warp shared-memory footprint, not the CTA granularity, set the occupancy
#ifndef DMM_PERM_WARPS
#define DMM_PERM_WARPS 4
#endif
constexpr int kPermWarps = DMM_PERM_WARPS;

// Warp-shared generator: the 312-word state in smem as two 32-bit arrays (low and
// high halves), so every warp-wide access is a unit-stride 32-bit access (no bank
// conflicts); `base` = index of the first draw the current state generation serves.
struct WarpRng {
    uint32_t* lo;
    uint32_t* hi;
    int64_t base;

    __device__ uint64_t get(int i) const { return ((uint64_t)hi[i] << 32) | lo[i]; }
    __device__ void put(int i, uint64_t v) {
        lo[i] = (uint32_t)v;
        hi[i] = (uint32_t)(v >> 32);
    }
    __device__ void seed(uint64_t s, int lane) {
        if (lane == 0) {
            uint64_t v = s;
            put(0, v);
            for (int i = 1; i < kRngWords; ++i) {
                v = 6364136223846793005ULL * (v ^ (v >> 62)) + (uint64_t)i;
                put(i, v);
            }
        }
        __syncwarp();
        twist(lane);
        base = 0;
    }
    // mersenne twist of all 312 words: [0,156) from old words; [156,311) from new [0,155)
    // and old words; 311 from new 155 and new 0
    __device__ void twist(int lane) {
        constexpr uint64_t MA = 0xB5026F5AA96619E9ULL;
        uint64_t v[5];
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int i = lane + 32 * t;
            if (i < 156) {
                // (mt[i] & UM) | (mt[i+1] & LM): the high 33 bits of mt[i], the low 31 of mt[i+1]
                const uint64_t x = ((uint64_t)hi[i] << 32) | (lo[i] & 0x80000000u) | (lo[i + 1] & 0x7FFFFFFFu);
                v[t] = get(i + 156) ^ (x >> 1) ^ ((x & 1) ? MA : 0);
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int i = lane + 32 * t;
            if (i < 156)
                put(i, v[t]);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int i = 156 + lane + 32 * t;
            if (i < 311) {
                const uint64_t x = ((uint64_t)hi[i] << 32) | (lo[i] & 0x80000000u) | (lo[i + 1] & 0x7FFFFFFFu);
                v[t] = get(i - 156) ^ (x >> 1) ^ ((x & 1) ? MA : 0);
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int i = 156 + lane + 32 * t;
            if (i < 311)
                put(i, v[t]);
        }
        __syncwarp();
        if (lane == 0) {
            const uint64_t x = ((uint64_t)hi[311] << 32) | (lo[311] & 0x80000000u) | (lo[0] & 0x7FFFFFFFu);
            put(311, get(155) ^ (x >> 1) ^ ((x & 1) ? MA : 0));
        }
        __syncwarp();
    }
    // load an engine mid-stream: the 312 state words and the position p of the next draw
    // (libstdc++'s mersenne_twister_engine layout _M_x[], _M_p): draw d reads word p + d
    __device__ void load(const uint64_t* state, int lane) {
        for (int i = lane; i < kRngWords; i += 32)
            put(i, state[i]);
        const uint64_t p = state[kRngWords];
        __syncwarp();
        if (p >= (uint64_t)kRngWords) {
            twist(lane);
            base = 0;
        } else {
            base = -(int64_t)p;
        }
    }
    // make draw d (warp-uniform) addressable; advances generations as needed
    __device__ void advance_to(uint32_t d, int lane) {
        while ((int64_t)d >= base + kRngWords) {
            twist(lane);
            base += kRngWords;
        }
    }
    __device__ uint64_t word(uint32_t d) const { return mt_temper(get((int)((int64_t)d - base))); }
};

__device__ __forceinline__ uint32_t hash_eval(uint64_t key, uint32_t m, uint32_t i) {  // HashOracle permute.hpp:39
    return (uint32_t)(splitmix64(key ^ ((uint64_t)i * 0x9e3779b97f4a7c15ULL)) % m);
}

// Three-phase delivery (permute.hpp:452-529) of one lane's lexicographically sorted packed
// row (own bank of q: q[c*32 + lane], c < WP; empty labels at the tail) into the output
// region (row i in bank i: outs[j*32 + i]).
template <int M>
__device__ __forceinline__ void three_phase_delivery(const uint32_t* q, int wp, uint32_t* outs, int lane,
                                                     uint32_t empty) {
    int cnt = 0;
    for (int c = 0; c < wp; ++c)
        cnt += q[c * 32 + lane] != empty ? 1 : 0;
    int f = 0, l0 = cnt;
    if (cnt > 0) {
        const uint32_t i_first = q[lane] / M, i_last = q[(cnt - 1) * 32 + lane] / M;
        while (f < cnt && q[f * 32 + lane] / M == i_first)
            ++f;
        if (i_last != i_first)
            while (l0 > f && q[(l0 - 1) * 32 + lane] / M == i_last)
                --l0;
        else
            l0 = f;
    }
    // middle labels: destination rows owned by this packed row alone, one per step
    const int nmid = l0 - f;
    const int max_mid = __reduce_max_sync(0xFFFFFFFFu, (uint32_t)nmid);
    for (int k = 0; k < max_mid; ++k) {
        if (k < nmid) {
            const uint32_t label = q[(f + k) * 32 + lane];
            outs[(label % M) * 32 + label / M] = label;
        }
        __syncwarp();
    }
    // first group, then last group: at step j every row sends its label with slot j
    int pf = 0, pl = l0;
    for (int j = 0; j < M; ++j) {
        if (pf < f) {
            const uint32_t label = q[pf * 32 + lane];
            if (label % M == (uint32_t)j) {
                outs[(label % M) * 32 + label / M] = label;
                ++pf;
            }
        }
        __syncwarp();
    }
    for (int j = 0; j < M; ++j) {
        if (pl < cnt) {
            const uint32_t label = q[pl * 32 + lane];
            if (label % M == (uint32_t)j) {
                outs[(label % M) * 32 + label / M] = label;
                ++pl;
            }
        }
        __syncwarp();
    }
}

// finish (permute.hpp:536-541) on a packed 32 x WP view held in registers y[0..WP):
// integer_sort_general(packed, n+1, -, enforce=false), then the three-phase delivery.
// Returns false on PostconditionFailed (strict): the caller falls back.
template <int WP, int M>
__device__ __forceinline__ bool finish_packed(uint32_t (&y)[WP], uint32_t* buf, uint32_t* q, uint32_t* outs,
                                              int lane, uint32_t empty, uint32_t& retries) {
    using V = VF<0xFFFFFFFFu, 0, 1, kWarp, 0, WP>;
    GenResult res{{0u, 0u}, 0u};
    balance_divide_sort<1, V, false, 0x80000000u>(y, buf, lane, res);  // packed labels <= n < 2^31
    res.finish();
    if (res.unsorted & 1u)
        return false;
    retries = res.retries[0];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < WP; ++c)
        q[c * 32 + lane] = y[c];
    __syncwarp();
    three_phase_delivery<M>(q, WP, outs, lane, empty);
    return true;
}

template <int M>
__host__ __device__ constexpr int perm_stage_words() {
    return (2 * M * 32 > relayout_buf_words(M) ? 2 * M * 32 : relayout_buf_words(M));
}
template <int M>
__host__ __device__ constexpr int perm_warp_words() {  // u32 words of smem per warp
    return 2 * kRngWords + M * 32 + perm_stage_words<M>();
}

template <int M>
__global__ void __launch_bounds__(kPermWarps * 32) k_permute(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                 uint64_t count, const uint64_t* __restrict__ seeds,
                                                 const uint64_t* __restrict__ states, PermArgs a,
                                                 dmm_permute_report* __restrict__ reps, uint64_t* __restrict__ hist,
                                                 uint32_t* __restrict__ shifts_out, uint8_t* __restrict__ status) {
    extern __shared__ uint64_t smem64[];
    constexpr int W = kWarp;
    constexpr uint32_t n = W * M;
    constexpr uint32_t empty = n;  // empty_label permute.hpp:88
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* wbase = reinterpret_cast<uint32_t*>(smem64) + warp * perm_warp_words<M>();
    WarpRng rng{wbase, wbase + kRngWords, 0};
    uint32_t* outs = wbase + 2 * kRngWords;     // output region, row i in bank i: outs[j*32 + i]
    uint32_t* stage = outs + M * 32;            // relayout buffer / own-bank rows A,B,H
    uint32_t* pk = stage + M * 32;                 // packed rows (own bank), capacity m: aliases B,
                                                   // which is dead from packing until the finish
    uint32_t* H = stage;                           // per-colour counts, then bucket starts
    uint32_t* B = stage + M * 32;                  // colour-sorted (compacted) row
    const uint64_t k = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (k >= count)
        return;

    uint32_t x[M];
    load_row<M>(in + (k * kWarp + lane) * M, x);
    uint32_t badkey = 0;
#pragma unroll
    for (int c = 0; c < M; ++c) {
        badkey |= x[c] >= n ? 1u : 0u;
        outs[c * 32 + lane] = 0xFFFFFFFFu;  // sentinel: undelivered
    }
    badkey = __reduce_or_sync(0xFFFFFFFFu, badkey);
    if (states)
        rng.load(states + k * (kRngWords + 1), lane);
    else
        rng.seed(seeds[k], lane);

    uint64_t random_words = 0;
    uint32_t drawn = 0;
    // ---- preprocess_shuffle permute.hpp:109-142 ---------------------------------------
    {
        rng.advance_to(drawn + W - 1, lane);
        const uint32_t s = 1u + (uint32_t)(rng.word(drawn + lane) % M);  // rng_below(M), M a power of two
        drawn += W;
        random_words += W;
        if (shifts_out)
            shifts_out[k * W + lane] = s;
        const uint32_t sh = s % M;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < M; ++c)
            H[((c + sh) % M) * 32 + lane] = x[c];  // own bank: row r rotates in bank r
        __syncwarp();
#pragma unroll
        for (int c = 0; c < M; ++c)
            x[c] = H[c * 32 + lane];
        using Blk = VF<0xFFFFFFFFu, 0, 1, M, 0, M>;  // every aligned m x m block of rows
        transpose_square<Blk>(x, stage, lane);
    }

    // ---- iterations permute.hpp:570-577 ---------------------------------------------------
    uint64_t leftover = n;
    uint32_t iterations = 0;
    while (leftover > a.threshold && iterations < a.iter_cap) {
        // draw_and_broadcast_hash permute.hpp:147-166: m draws, key = the first
        rng.advance_to(drawn, lane);
        const uint64_t key = rng.word(drawn);
        drawn += M;
        random_words += M;
        // rescan_and_bucket permute.hpp:174-216: stable own-bank counting sort by colour.
        // Every access below is to the lane's own bank (H, B columns = lane): conflict-free
        // for any data, no warp synchronisation needed.
#pragma unroll
        for (int b = 0; b < M; ++b)
            H[b * 32 + lane] = 0;
        // h(i) for the 32 source rows i: lane l evaluates h(l) once, keys fetch theirs by
        // shuffle (one SHFL instead of a 64-bit splitmix64 per key)
        const uint32_t h_lane = hash_eval(key, M, (uint32_t)lane);
        uint32_t col[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
            const bool live = x[c] != empty;
            const uint32_t i = live ? x[c] / M : 0u, j = x[c] % M;
            const uint32_t hi = __shfl_sync(0xFFFFFFFFu, h_lane, (int)(i & 31u));
            col[c] = live ? (j + M - hi) % M : 0u;
            if (live)
                H[col[c] * 32 + lane] += 1;
        }
        uint32_t run = 0;
        uint32_t lane_left = 0;
#pragma unroll
        for (int b = 0; b < M; ++b) {
            const uint32_t cnt = H[b * 32 + lane];
            lane_left += cnt > a.alpha ? cnt - a.alpha : 0;
            H[b * 32 + lane] = run;  // bucket start
            run += cnt;
        }
#pragma unroll
        for (int c = 0; c < M; ++c)
            if ((uint32_t)c >= run)
                B[c * 32 + lane] = empty;
        // scatter into the colour-sorted order
#pragma unroll
        for (int c = 0; c < M; ++c) {
            if (x[c] != empty) {
                const uint32_t pos = H[col[c] * 32 + lane];
                H[col[c] * 32 + lane] = pos + 1;
                B[pos * 32 + lane] = x[c];
            }
        }
        // communication_phase permute.hpp:225-274.  Step (pass p, colour k): every row sends
        // its p-th label of colour k to out[i][j]; the output region keeps row i in bank i and
        // the colouring makes the destinations of one step distinct rows, so every step is one
        // conflict-free warp-wide store.  H holds the bucket ends now: start = end - count.
        // A sent label's cell becomes empty in place (the compacted row keeps its holes):
        // exactly the first min(count, alpha) cells of every colour bucket.
        for (int kc = 0; kc < M; ++kc) {
            const uint32_t end = H[kc * 32 + lane];
            const uint32_t start = kc == 0 ? 0u : H[(kc - 1) * 32 + lane];
            const uint32_t take = min(end - start, a.alpha);
            for (uint32_t p = 0; p < take; ++p) {
                const uint32_t label = B[(start + p) * 32 + lane];
                outs[(label % M) * 32 + label / M] = label;
                B[(start + p) * 32 + lane] = empty;
            }
        }
#pragma unroll
        for (int c = 0; c < M; ++c)
            x[c] = B[c * 32 + lane];
        // synchronize permute.hpp:278-285
        leftover = __reduce_add_sync(0xFFFFFFFFu, lane_left);
        if (lane == 0 && hist && iterations < DMM_PERMUTE_MAX_HIST)
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
            // compaction into the packed rows (own bank)
            uint32_t load = 0;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < M; ++c)
                if (x[c] != empty)
                    pk[(load++) * 32 + lane] = x[c];
            for (uint32_t c = load; c < width; ++c)
                pk[c * 32 + lane] = empty;
            uint32_t cell_load = load, cell_cursor = load;
            bool recv = false;
            random_words += a.t;
            for (uint32_t round = 0; round < a.t; ++round) {
                rng.advance_to(drawn, lane);
                const uint32_t shift = 1u + (uint32_t)(rng.word(drawn) % W);  // rng_below(W), W = 32
                ++drawn;
                const int partner = (lane + shift) & 31, src = (lane - shift) & 31;
                const uint32_t p_load = __shfl_sync(0xFFFFFFFFu, cell_load, partner);
                const bool p_recv = __shfl_sync(0xFFFFFFFFu, recv, partner);
                const bool sender = load > theta && !p_recv && p_load <= theta;
                const uint32_t give = sender ? min(a.bundle, load) : 0u;
                const uint32_t p_cursor = __shfl_sync(0xFFFFFFFFu, cell_cursor, partner);
                const uint32_t maxgive = __reduce_max_sync(0xFFFFFFFFu, give);
                for (uint32_t kk = 0; kk < maxgive; ++kk) {
                    uint32_t moved = 0;
                    if (kk < give)
                        moved = pk[(load - 1 - kk) * 32 + lane];
                    __syncwarp();
                    if (kk < give && p_cursor + kk < M)
                        pk[(p_cursor + kk) * 32 + partner] = moved;  // distinct partner banks
                    __syncwarp();
                }
                const bool got = __shfl_sync(0xFFFFFFFFu, sender, src);
                const uint32_t give_in = __shfl_sync(0xFFFFFFFFu, give, src);
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
            const bool overflow = __any_sync(0xFFFFFFFFu, load > width);
            if (!overflow) {
                __syncwarp();
                for (uint32_t c = load; c < width; ++c)
                    pk[c * 32 + lane] = empty;
                __syncwarp();
                used_packing = true;
                packed_width = width;
                bool ok = false;
                if constexpr (M == 32) {
                    if (width == 16) {
                        uint32_t y[16];
#pragma unroll
                        for (int c = 0; c < 16; ++c)
                            y[c] = pk[c * 32 + lane];
                        ok = finish_packed<16, M>(y, stage, B, outs, lane, empty, cleanup_retries);
                    }
                }
                delivered = ok;
            }
        }
    }
    if (!delivered) {
        // ---- deterministic fallback permute.hpp:597-626 --------------------------------
        fallback = true;
        uint32_t y[M];
        {
            uint32_t o = 0;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < M; ++c)
                if (x[c] != empty)
                    B[(o++) * 32 + lane] = x[c];
            for (uint32_t c = o; c < M; ++c)
                B[c * 32 + lane] = empty;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < M; ++c)
                y[c] = B[c * 32 + lane];
        }
        uint32_t y_keep[M];
#pragma unroll
        for (int c = 0; c < M; ++c)
            y_keep[c] = y[c];
        uint32_t r2 = 0;
        if (!finish_packed<M, M>(y, stage, B, outs, lane, empty, r2) && M < kWarp) {
            // last resort: comparison tall sort on the compacted multiset (permute.hpp:618-625).
            // The reference sorts the working window left by the failed attempt; any
            // arrangement of the same multiset sorts to the same matrix.
            using V = VF<0xFFFFFFFFu, 0, 1, kWarp, 0, M>;
            if constexpr (M < kWarp)
                sort_tall<1, V>(y_keep, stage, lane);
            __syncwarp();
#pragma unroll
            for (int c = 0; c < M; ++c)
                B[c * 32 + lane] = y_keep[c];
            __syncwarp();
            three_phase_delivery<M>(B, M, outs, lane, empty);
        } else {
            cleanup_retries = r2;
        }
    }
    __syncwarp();
    // output region (row i in bank i) -> global row-major; verify the bijection
    uint32_t v[M];
    uint32_t wrong = badkey;
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const uint32_t o = outs[j * 32 + lane];
        wrong |= o != (uint32_t)lane * M + j ? 1u : 0u;
        v[j] = o == 0xFFFFFFFFu ? 0u : o;  // undelivered cells keep the machine's zero
    }
    wrong = __reduce_or_sync(0xFFFFFFFFu, wrong);
    store_row<M>(out + (k * kWarp + lane) * M, v);
    if (lane == 0) {
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

template <int M>
dmm_status launch_permute(const uint32_t* in, uint32_t* out, uint64_t count, const uint64_t* seeds,
                          const uint64_t* states, const dmmdev::PermArgs& a, dmm_permute_report* reps, uint64_t* hist, uint32_t* shifts,
                          uint8_t* status, cudaStream_t s) {
    constexpr int kWarps = dmmdev::kPermWarps;
    auto kern = dmmdev::k_permute<M>;
    const size_t smem = size_t(kWarps) * dmmdev::perm_warp_words<M>() * sizeof(uint32_t);
    static bool configured = false;
    if (!configured) {
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
            return check_launch("cudaFuncSetAttribute");
        // prefer the full 228 KB shared-memory carveout: occupancy is bounded by smem + registers
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        configured = true;
    }
    const uint64_t blocks = (count + kWarps - 1) / kWarps;
    kern<<<unsigned(blocks), kWarps * 32, smem, s>>>(in, out, count, seeds, states, a, reps, hist, shifts, status);
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
                       uint64_t* history, uint32_t* shifts, uint8_t* status, void* workspace, void* stream) {
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
    if (w != 32) {
        set_error("kernels are built for w = 32 (one warp per machine)");
        return DMM_UNSUPPORTED_SHAPE;
    }
    dmmdev::PermArgs a;
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
    switch (m) {
        case 2: return launch_permute<2>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
        case 4: return launch_permute<4>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
        case 16: return launch_permute<16>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
        case 32: return launch_permute<32>(in, out, count, seeds, states, a, reports, history, shifts, status, s);
        default: break;
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

}  // extern "C"

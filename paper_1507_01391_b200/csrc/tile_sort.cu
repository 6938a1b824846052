// tile_sort.cu -- kernel 3 for tiles too wide for one warp's registers: the 32 x 128 uint32
// tile of cfg3 (4096 keys) sorted by a CTA of 4 warps.  integer_sort_general on a 32 x 128
// view reduces to partition_leaf (w <= m), whose outcome is the tile in row-major sorted
// order (partition.hpp:156-172, sort.hpp:288-311); any conflict-free sorter of the same
// multiset reproduces it bit for bit.
//
// Sorted rank e = 1024*w + 32*r + j lives in warp w, lane r, register j, i.e. the tile's
// row-major order itself: warp w stores 1024 contiguous words (lane r: 128 contiguous
// bytes).  The starting arrangement is irrelevant to a sort, so the tile is loaded fully
// coalesced (lane l of warp w takes the 16-byte chunks 256w + l + 32i).
//
// Bitonic levels 1..5 are register-local (static code).  Every later level is one "pass"
// of the same loop: flip the keys of the lanes whose direction bit is set (lane bit for
// in-warp levels 6..9, warp bit for 10 and 11; x ^ ~0 reverses the order), optional
// compare-exchange stages with the partner warp (w ^ 2^b) through a lane-major shared
// slab (each lane touches its own bank column: no conflicts), then transpose / row-bit
// stages / transpose / register stages, all ascending, and flip back.  The passes share
// ONE copy of the transpose and of the five single-stage bodies (runtime switch): the
// straight-line version (64 KB of SASS) stalled on instruction fetch (ncu: no_inst 42 %).
#include <algorithm>
#include <cstdlib>

#include "general_kernel.cuh"

namespace dmmdev {

constexpr int kTileWarps = 4;

// compare-exchange with the partner warp (w ^ 2^b): lower warp keeps the minima
template <int PK>
__device__ __forceinline__ void cross_warp_stage(uint32_t (&x)[32], uint32_t* slabs, int warp, int lane, int b) {
    uint32_t* mine = slabs + warp * relayout_buf_words(32);
    const uint32_t* other = slabs + (warp ^ (1 << b)) * relayout_buf_words(32);
    const bool lower = ((warp >> b) & 1) == 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j)
        mine[j * 33 + lane] = x[j];
    __syncthreads();
    // lower is warp-uniform: one min or max per key
    if (lower) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            x[j] = PK == 2 ? __vminu2(x[j], other[j * 33 + lane]) : min(x[j], other[j * 33 + lane]);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            x[j] = PK == 2 ? __vmaxu2(x[j], other[j * 33 + lane]) : max(x[j], other[j * 33 + lane]);
    }
    __syncthreads();
}

// Persistent CTAs: CTA b sorts tiles b*PK, (b + grid)*PK, ...; at the start of each tile thread 0
// prefetches the CTA's next tile(s) into L2 (cp.async.bulk.prefetch.L2: no registers, no shared
// memory), so the next tile's loads hit L2 while this one sorts.  MODE kModeSortAny:
// sort_wide_any (sort.hpp:321-330 -> shearsort_rect) ascending or descending (descending =
// the ascending sort of the complemented keys).
// NW warps per tile: 4 (32 x 128, cfg3) or 8 (32 x 256); the tile is 1024 * NW keys and its
// sort has 10 + log2(NW) levels, the last log2(NW) with cross-warp stages.
template <int PK, int MODE, int NW = kTileWarps, int MINB = 1>
__global__ void __launch_bounds__(NW * 32, MINB) k_tile_sort(const uint32_t* __restrict__ in,
                                                       uint32_t* __restrict__ out, uint64_t count,
                                                       uint64_t domain, int ascending,
                                                       dmm_general_stats* __restrict__ stats,
                                                       uint8_t* __restrict__ status, uint64_t pf_dist, int shfl6) {
    static_assert(NW == 4 || NW == 8, "32 x 128 or 32 x 256 tiles");
    constexpr int LOGNW = NW == 8 ? 3 : 2;
    __shared__ __align__(16) uint32_t smem[NW * relayout_buf_words(32)];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* buf = smem + warp * relayout_buf_words(32);
    constexpr int M = 32 * NW;
    const uint32_t fdesc = (MODE == kModeSortAny && !ascending) ? 0xFFFFFFFFu : 0u;
    for (uint64_t tile0 = (uint64_t)blockIdx.x * PK; tile0 < count; tile0 += (uint64_t)gridDim.x * PK) {
    const bool hasB = PK == 2 && tile0 + 1 < count;
    if (threadIdx.x == 0 && pf_dist) {
        // the tile (pair) pf_dist ahead -- the next task of this slot: the persistent stride,
        // or (one CTA per tile) the tile a CTA that starts when this one ends will take
        const uint64_t nt = tile0 + pf_dist;
        if (nt < count) {
            const uint64_t nn = count - nt < (uint64_t)PK ? count - nt : (uint64_t)PK;
            prefetch_l2(in + nt * (32 * M), (uint32_t)(nn * 32 * M * 4));
        }
    }

    uint32_t x[32];
    uint32_t bad = 0;
    {
        // coalesced chunk loads; keys outside [0, domain) flagged by OR / max accumulation
        const bool dom32 = domain < (1ull << 32);
        const bool dom_pow2 = (domain & (domain - 1)) == 0;
        const uint32_t dom_mask = dom32 && dom_pow2 ? ~(uint32_t)(domain - 1) : 0u;
        auto load = [&](uint64_t t, uint32_t (&v)[32]) -> uint32_t {
            if constexpr (kIoOff) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    v[c] = synth_key(t, threadIdx.x, c) * 0x9E3779B9u;
                return 0u;
            }
            const uint4* q = reinterpret_cast<const uint4*>(in + t * (32 * M)) + warp * 256 + lane;
            uint32_t acc_or = 0, acc_max = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint4 c = __ldg(q + 32 * i);
                v[4 * i] = c.x;
                v[4 * i + 1] = c.y;
                v[4 * i + 2] = c.z;
                v[4 * i + 3] = c.w;
            }
            if (!dom32)
                return 0u;
            if (dom_pow2) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    acc_or |= v[c];
                return (acc_or & dom_mask) ? 1u : 0u;
            }
#pragma unroll
            for (int c = 0; c < 32; ++c)
                acc_max = max(acc_max, v[c]);
            return acc_max >= (uint32_t)domain ? 1u : 0u;
        };
        bad = load(tile0, x);
        if constexpr (PK == 2) {
            uint32_t b[32];
            if (hasB) {
                bad |= load(tile0 + 1, b) << 1;
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    b[c] = 0;
            }
#pragma unroll
            for (int c = 0; c < 32; ++c)
                x[c] = __byte_perm(x[c], b[c], 0x5410);  // (a & 0xFFFF) | (b << 16)
        }
    }

    if constexpr (MODE == kModeSortAny)
        flip<0, 32>(x, fdesc);
    using V = VF<0xFFFFFFFFu, 0, 1, kWarp, 0, 32>;
    // levels 1..5: register-local, static
    row_sort<PK, V>(x, lane, (lane & 1) == 0);  // levels 1..5 (odd-even merge sort per row)
    // levels 6..12 as passes of one loop (see the header); the flip that ends a pass and
    // the one that starts the next are merged into one
    auto dir_mask = [&](int level) -> uint32_t {
        uint32_t f;
        if (level < 10)
            f = (lane >> (level - 5)) & 1;  // in-warp level: direction = element bit `level`
        else if (level < 10 + LOGNW)
            f = (warp >> (level - 10)) & 1;  // cross-warp levels: direction = warp bit
        else
            f = 0;
        return f ? 0xFFFFFFFFu : 0u;
    };
    uint32_t fcur = 0;
#pragma unroll 1
    for (int pass = 0; pass < 5 + LOGNW; ++pass) {
        const int level = 6 + pass;
        const uint32_t f = dir_mask(level);
        flip<0, 32>(x, f ^ fcur);
        fcur = f;
#pragma unroll 1
        for (int b = level - 11; b >= 0; --b)  // stages on warp bits (levels 11 .. 10 + log2 NW)
            cross_warp_stage<PK>(x, smem, warp, lane, b);
        const int row_stages = (level < 10 ? level : 10) - 6;  // row-bit stages row_stages..0
        if (level - 5 <= shfl6) {
            // the level's lane-bit stages (element bits level-1 .. 5 = lane bits level-6 .. 0) as
            // shuffle exchanges with the partner lane (the lower lane keeps the minimum) instead of
            // two transposes: per stage one SHFL and a min / max per register, against 80 shared
            // instructions per transpose pair (levels 6 and 7: fewer shared wavefronts, same
            // issue)
#pragma unroll 1
            for (int b = level - 6; b >= 0; --b) {
                const bool upper = (lane >> b) & 1;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x[j], 1 << b);
                    if constexpr (PK == 2)
                        x[j] = upper ? __vmaxu2(x[j], y) : __vminu2(x[j], y);
                    else
                        x[j] = upper ? max(x[j], y) : min(x[j], y);
                }
            }
            stages_down<PK, 0, 32>(x, 4);
            continue;
        }
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
            transpose_blocks<V>(x, buf, lane);
            stages_down<PK, 0, 32>(x, half == 0 ? row_stages : 4);
        }
    }
    flip<0, 32>(x, fcur ^ fdesc);

    // tile reductions of the per-warp flags
    __shared__ uint32_t flags_s[NW];
    uint32_t mism = 0;
    if constexpr (MODE == kModePartition) {
        // row-major rank e = 1024 w + 32 r + j belongs to machine row e / M
        const uint32_t row = (1024u / M) * warp + lane / (M / 32);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            if constexpr (PK == 2) {
                mism |= (x[c] & 0xFFFFu) != row ? 1u : 0u;
                mism |= (x[c] >> 16) != row ? 2u : 0u;
            } else {
                mism |= x[c] != row ? 1u : 0u;
            }
        }
    }
    const uint32_t wflag = __reduce_or_sync(0xFFFFFFFFu, bad | (mism << 2));
    if (lane == 0)
        flags_s[warp] = wflag;
    __syncthreads();
    uint32_t all = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i)
        all |= flags_s[i];
    const uint32_t badt = all & 3u, invalid = (all >> 2) | badt;

#pragma unroll
    for (int h = 0; h < PK; ++h) {
        if (h == 1 && !hasB)
            break;
        if (kIoOff && count != ~0ull)
            break;
        const uint64_t k = tile0 + h;
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c)
            v[c] = PK == 2 ? ((x[c] >> (16 * h)) & 0xFFFFu) : x[c];
        store_row<32>(out + k * (32 * M) + warp * 1024 + lane * 32, v);
        if (threadIdx.x == 0) {
            uint8_t s = DMM_OK;
            if (MODE == kModePartition && ((invalid >> h) & 1u))
                s = DMM_INVALID_INSTANCE;
            else if ((badt >> h) & 1u)
                s = DMM_KEY_OUT_OF_RANGE;
            if (status)
                status[k] = s;
            if (stats) {
                stats[k].cleanup_retries = 0;  // w <= m: partition_leaf only, no cleanup loop
                stats[k].sorted = 1;
            }
        }
    }
    __syncthreads();  // flags_s is rewritten by the next tile
    }  // tile loop
}

// 32 x 128 tiles on TWO warps of 64 keys per lane (element e = 2048 w + 64 l + r): levels 1-6
// sort the lane's 64 registers, levels 7-12 are passes of {flip; the cross-warp stage (level
// 12); transpose the two 32 x 32 register blocks; stages on the lane bits (transposed register
// bits) and on register bit 5; transpose back; stages on register bits 4..0}.  12 transposes
// and one cross-warp stage per tile instead of 14 and three: 0.81 shared wavefronts per key
// instead of 1.06.  Selected with DMM_TILE64=1 (A/B against the 4-warp kernel): measured
// SLOWER, 170 vs 181 G keys/s on cfg3 -- 0.84 wavefronts and 128 instructions per key (-24 %,
// -12 %), but 94 registers leave 20 warps per SM and the 64-register networks' straight-line
// code misses the instruction cache (no_inst 28 % of stalls); a run-time stage loop that fixes
// the misses costs 31 % more instructions in register moves (156 G keys/s).
// (profiles/r02/pipeline_ab.txt)
template <int PK, int MODE>
__global__ void __launch_bounds__(64) k_tile_sort64(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                    uint64_t count, uint64_t domain, int ascending,
                                                    dmm_general_stats* __restrict__ stats,
                                                    uint8_t* __restrict__ status) {
    constexpr int R = 64;  // registers per lane
    __shared__ __align__(16) uint32_t smem[2 * relayout_buf_words(R)];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* buf = smem + warp * relayout_buf_words(R);
    const uint64_t tile0 = (uint64_t)blockIdx.x * PK;
    if (tile0 >= count)
        return;
    const bool hasB = PK == 2 && tile0 + 1 < count;
    const uint32_t fdesc = (MODE == kModeSortAny && !ascending) ? 0xFFFFFFFFu : 0u;
    uint32_t x[R];
    uint32_t bad = 0;
    {
        const bool dom32 = domain < (1ull << 32);
        auto load = [&](uint64_t t, uint32_t (&v)[R]) -> uint32_t {
            const uint4* q = reinterpret_cast<const uint4*>(in + t * 4096) + warp * 512 + lane;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint4 c = __ldg(q + 32 * i);
                v[4 * i] = c.x;
                v[4 * i + 1] = c.y;
                v[4 * i + 2] = c.z;
                v[4 * i + 3] = c.w;
            }
            if (!dom32)
                return 0u;
            uint32_t acc = 0;
#pragma unroll
            for (int c = 0; c < R; ++c)
                acc = max(acc, v[c]);
            return acc >= (uint32_t)domain ? 1u : 0u;
        };
        bad = load(tile0, x);
        if constexpr (PK == 2) {
            // two tiles of 16-bit keys: load B's words in four groups of 16 registers
            const uint4* q = reinterpret_cast<const uint4*>(in + (tile0 + 1) * 4096) + warp * 512 + lane;
            uint32_t accb = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint4 c = hasB ? __ldg(q + 32 * i) : make_uint4(0, 0, 0, 0);
                const uint32_t vb[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    accb = max(accb, vb[e]);
                    x[4 * i + e] = __byte_perm(x[4 * i + e], vb[e], 0x5410);
                }
            }
            if (domain < (1ull << 32) && accb >= (uint32_t)domain)
                bad |= 2u;
        }
    }
    if constexpr (MODE == kModeSortAny)
        flip<0, R>(x, fdesc);
    using V = VF<0xFFFFFFFFu, 0, 1, kWarp, 0, R>;
    row_sort<PK, V>(x, lane, (lane & 1) == 0);  // levels 1..6
    uint32_t fcur = 0;
#pragma unroll 1
    for (int level = 7; level <= 12; ++level) {
        const uint32_t fb = level <= 10 ? (lane >> (level - 6)) & 1 : level == 11 ? (uint32_t)warp : 0u;
        const uint32_t f = fb ? 0xFFFFFFFFu : 0u;
        flip<0, R>(x, f ^ fcur);
        fcur = f;
        if (level == 12) {
            // element bit 11 = the warp: compare-exchange with the other warp
            uint32_t* mine = smem + warp * relayout_buf_words(R);
            const uint32_t* other = smem + (warp ^ 1) * relayout_buf_words(R);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < R; ++j)
                mine[j * 33 + lane] = x[j];
            __syncthreads();
            if (warp == 0) {
#pragma unroll
                for (int j = 0; j < R; ++j)
                    x[j] = PK == 2 ? __vminu2(x[j], other[j * 33 + lane]) : min(x[j], other[j * 33 + lane]);
            } else {
#pragma unroll
                for (int j = 0; j < R; ++j)
                    x[j] = PK == 2 ? __vmaxu2(x[j], other[j * 33 + lane]) : max(x[j], other[j * 33 + lane]);
            }
            __syncthreads();
        }
        // lane bits level-1 .. 6 (transposed register bits level-7 .. 0), then bit 5
        // lane bits level-1 .. 6 (transposed register bits level-7 .. 0), then bit 5
        transpose_blocks<V>(x, buf, lane);
        stages_down<PK, 0, R>(x, (level < 11 ? level : 11) - 7);
        reg_stage<PK, 0, R, 5>(x);
        transpose_blocks<V>(x, buf, lane);
        stages_down<PK, 0, R>(x, 4);
    }
    flip<0, R>(x, fcur ^ fdesc);

    __shared__ uint32_t flags_s[2];
    uint32_t mism = 0;
    if constexpr (MODE == kModePartition) {
        const uint32_t row = 16u * warp + lane / 2;  // e / 128
#pragma unroll
        for (int c = 0; c < R; ++c) {
            if constexpr (PK == 2) {
                mism |= (x[c] & 0xFFFFu) != row ? 1u : 0u;
                mism |= (x[c] >> 16) != row ? 2u : 0u;
            } else {
                mism |= x[c] != row ? 1u : 0u;
            }
        }
    }
    const uint32_t wflag = __reduce_or_sync(0xFFFFFFFFu, bad | (mism << 2));
    if (lane == 0)
        flags_s[warp] = wflag;
    __syncthreads();
    const uint32_t all = flags_s[0] | flags_s[1];
    const uint32_t badt = all & 3u, invalid = (all >> 2) | badt;
#pragma unroll
    for (int h = 0; h < PK; ++h) {
        if (h == 1 && !hasB)
            break;
        const uint64_t k = tile0 + h;
        uint4* q = reinterpret_cast<uint4*>(out + k * 4096 + warp * 2048 + lane * 64);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            uint32_t v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                v[e] = PK == 2 ? ((x[4 * i + e] >> (16 * h)) & 0xFFFFu) : x[4 * i + e];
            q[i] = make_uint4(v[0], v[1], v[2], v[3]);
        }
        if (threadIdx.x == 0) {
            uint8_t st = DMM_OK;
            if (MODE == kModePartition && ((invalid >> h) & 1u))
                st = DMM_INVALID_INSTANCE;
            else if ((badt >> h) & 1u)
                st = DMM_KEY_OUT_OF_RANGE;
            if (status)
                status[k] = st;
            if (stats) {
                stats[k].cleanup_retries = 0;
                stats[k].sorted = 1;
            }
        }
    }
}

}  // namespace dmmdev

namespace dmmhost {

namespace {
template <int PK, int MODE, int NW = dmmdev::kTileWarps>
dmm_status launch_tile(const GeneralArgs& a) {
    auto kern = dmmdev::k_tile_sort<PK, MODE, NW>;
    // DMM_TILE_MINB=B: ask ptxas for B resident CTAs per SM on the cfg3 kernel (register cap
    // 65536 / (128 B)).  Default 10 (48 registers, 40 warps per SM): 178.9 vs 175.2 G keys/s for
    // ptxas's own choice (0: 85 registers, 24 warps per SM); 12 spills (171.0)
    // (profiles/r02/pipeline_ab.txt)
    if constexpr (PK == 1 && MODE == dmmdev::kModeIntegerSort && NW == 4) {
        static const int minb = getenv("DMM_TILE_MINB") ? atoi(getenv("DMM_TILE_MINB")) : 10;
        if (minb == 10)
            kern = dmmdev::k_tile_sort<PK, MODE, NW, 10>;
        else if (minb == 12)
            kern = dmmdev::k_tile_sort<PK, MODE, NW, 12>;
    }
    const uint64_t units = (a.count + PK - 1) / PK;
    // one CTA per tile (pair): a persistent grid with L2 prefetch of the next tile measured
    // slower (165 vs 184 G keys/s on cfg3, profiles/r02/pipeline_ab.txt); DMM_TILE_PERSIST=1
    // selects it
    static const bool persist = getenv("DMM_TILE_PERSIST") && getenv("DMM_TILE_PERSIST")[0] == '1';
    // DMM_TILE_PF=1: each CTA prefetches into L2 the tile a CTA starting after it will take
    // (SMs x resident CTAs ahead)
    static const bool pf = getenv("DMM_TILE_PF") && getenv("DMM_TILE_PF")[0] == '1';
    // DMM_TILE_CARVE=1 (A/B): ask for the full shared-memory carveout (the driver's default
    // split leaves more L1)
    static const bool carve = getenv("DMM_TILE_CARVE") && getenv("DMM_TILE_CARVE")[0] == '1';
    static std::atomic<uint64_t> configured{0};
    if (carve)
        if (dmm_status e = configure_kernel(kern, 0, configured); e != DMM_OK)
            return e;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, 0);
    const uint64_t resident = uint64_t(sms) * std::max(per_sm, 1);
    uint64_t blocks = units;
    if (persist)
        blocks = std::min<uint64_t>(units, resident);
    if (blocks > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;
    const uint64_t pf_dist = persist ? blocks * PK : pf ? resident * PK : 0;
    // DMM_TILE_SHFL=L: levels 6 .. 5 + L run their lane-bit stages as shuffle exchanges
    // (0: every level through transposes)
    static const int shfl = getenv("DMM_TILE_SHFL") ? atoi(getenv("DMM_TILE_SHFL")) : 2;
    kern<<<unsigned(blocks), NW * 32, 0, a.stream>>>(a.in, a.out, a.count, a.domain, a.ascending,
                                                                      a.stats, a.status, pf_dist, shfl);
    return check_launch("k_tile_sort");
}
template <int PK, int MODE>
dmm_status launch_tile64(const GeneralArgs& a) {
    const uint64_t blocks = (a.count + PK - 1) / PK;
    if (blocks > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;
    dmmdev::k_tile_sort64<PK, MODE><<<unsigned(blocks), 64, 0, a.stream>>>(a.in, a.out, a.count, a.domain,
                                                                          a.ascending, a.stats, a.status);
    return check_launch("k_tile_sort64");
}
}  // namespace

dmm_status launch_general_m128(int mode, bool pk2, bool ext, const GeneralArgs& a) {
    if (ext) {
        set_error("extension kernels are only built where the reference rejects the shape");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (a.probe) {
        set_error("32 x 128 machines: no probe (w <= m has no PartitionProbe point)");
        return DMM_INVALID_ARGUMENT;
    }
    if (a.count == 0)
        return DMM_OK;
    if (partition_count_applies(128, mode, a))
        return launch_partition_count(128, mode, a);
    static const bool t64 = getenv("DMM_TILE64") && getenv("DMM_TILE64")[0] == '1';
    if (t64) {
        if (mode == dmmdev::kModeSortAny)
            return launch_tile64<1, dmmdev::kModeSortAny>(a);
        if (mode == dmmdev::kModePartition)
            return launch_tile64<2, dmmdev::kModePartition>(a);
        return pk2 ? launch_tile64<2, dmmdev::kModeIntegerSort>(a) : launch_tile64<1, dmmdev::kModeIntegerSort>(a);
    }
    if (mode == dmmdev::kModeSortAny)
        return launch_tile<1, dmmdev::kModeSortAny>(a);
    if (mode == dmmdev::kModePartition)
        return launch_tile<2, dmmdev::kModePartition>(a);
    return pk2 ? launch_tile<2, dmmdev::kModeIntegerSort>(a) : launch_tile<1, dmmdev::kModeIntegerSort>(a);
}

// 32 x 256 machines (8192 keys): partition_leaf -> square_skeleton with h = 16 (partition.hpp:
// 156-172, sort.hpp:250-280) or sort_wide_any; every outcome is the sorted machine, which the
// 8-warp tile sort produces
dmm_status launch_general_m256(int mode, bool pk2, bool ext, const GeneralArgs& a) {
    if (ext) {
        set_error("extension kernels are only built where the reference rejects the shape");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (a.probe) {
        set_error("32 x 256 machines: no probe (w <= m has no PartitionProbe point)");
        return DMM_INVALID_ARGUMENT;
    }
    if (a.count == 0)
        return DMM_OK;
    if (partition_count_applies(256, mode, a))
        return launch_partition_count(256, mode, a);
    if (mode == dmmdev::kModeSortAny)
        return launch_tile<1, dmmdev::kModeSortAny, 8>(a);
    if (mode == dmmdev::kModePartition)
        return launch_tile<2, dmmdev::kModePartition, 8>(a);
    return pk2 ? launch_tile<2, dmmdev::kModeIntegerSort, 8>(a) : launch_tile<1, dmmdev::kModeIntegerSort, 8>(a);
}

}  // namespace dmmhost

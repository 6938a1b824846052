// partition_count.cu -- the leaf-only w-way partition (w = 32 <= m: 32 x 32, 32 x 64, 32 x 128,
// 32 x 256) and the small-domain integer sort on the same shapes, as ONE per-bank counting pass.
//
// Reference path: partition_general (partition.hpp:453-456) = check_partition_instance
// (:112-124, a label histogram) + integer_sort_general(v, w) (:436-449), which for w <= m is a
// single partition_leaf (:156-172): its row sorts are radix_sort_rows with base >= domain
// (:24-99), i.e. counting sorts, and its outcome is the view's multiset in row-major sorted
// order (the leaf's skeletons end in sorted order whatever the start; GeneralStats: no cleanup
// loop runs, cleanup_retries = 0).  The counting sort of the whole view produces that outcome
// directly:
//
//   * per-bank counting -- lane l of the instance's warp counts its keys into its OWN
//     counters: the 32 labels as 16 words of two 16-bit counters, word c of lane l at
//     shared word 32 c + l, i.e. always bank l: conflict-free for any data (the paper's
//     per-bank counting rows, partition.hpp:37-99);
//   * the cross-bank sums are a transposed read of the 16 x 32 count matrix with a rotation
//     (lane t reads column (s + t) mod 16 of word t mod 16 at step s: 32 distinct banks per
//     step), so the histogram costs 16 conflict-free loads per lane;
//   * check_partition_instance is the histogram itself: every label < w and every count = m;
//   * the emission writes each label's run [E(v-1), E(v)) of the row-major output, where E is
//     the inclusive prefix of the counts.  For a partition instance every run has length m,
//     so position p holds p / m (row i holds i: "after the call row i holds exactly the labels
//     i", partition.hpp:451); other count vectors (integer sorts with domain <= 32) locate p's
//     run by a 5-step binary search over E (32 words in 32 banks: conflict-free).
//
// Instances the reference rejects (InvalidInstance / KeyOutOfRange, thrown before any step)
// are left unchanged: the output receives the input, the status byte names the exception.
// Keys move HBM -> registers by fully coalesced 16-byte loads (the starting arrangement does
// not matter to a counting sort) and the runs leave by 16-byte stores: 8 bytes of HBM traffic
// per key, ~7 instructions per key, so the kernel is bounded by HBM, not by the SM.
#include <cstdlib>

#include "general_kernel.cuh"

namespace dmmdev {

constexpr int kCountWarps = 4;        // one instance per warp
constexpr int kCountWords = 16 * 32;  // 16 counter words per lane (two 16-bit counters each)

template <int M>
__global__ void __launch_bounds__(kCountWarps * 32) k_partition_count(const uint32_t* __restrict__ in,
                                                                      uint32_t* __restrict__ out, uint64_t count,
                                                                      uint32_t domain, int partition,
                                                                      dmm_general_stats* __restrict__ stats,
                                                                      uint8_t* __restrict__ status) {
    static_assert(M % 32 == 0 && M >= 32 && M <= 256, "32 x m views, 32 <= m <= 256");
    constexpr int N = 32 * M;          // keys per instance
    constexpr int kChunks = M / 32;    // 32 keys per lane per chunk (8 x 16 bytes)
    __shared__ uint32_t cnt_s[kCountWarps][kCountWords];
    __shared__ uint32_t ends_s[kCountWarps][32];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint64_t k = (uint64_t)blockIdx.x * kCountWarps + warp;
    if (k >= count)
        return;
    uint32_t* cnt = cnt_s[warp];
#pragma unroll
    for (int c = 0; c < 16; ++c)
        cnt[32 * c + lane] = 0u;
    const uint4* src = reinterpret_cast<const uint4*>(in + k * N);
    uint32_t acc_or = 0, acc_max = 0;
#pragma unroll 1
    for (int j = 0; j < kChunks; ++j) {
        uint4 q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            q[i] = __ldg(src + 256 * j + lane + 32 * i);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t v[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t x = v[e];
                acc_or |= x;
                acc_max = max(acc_max, x);
                // own bank (lane), word x / 2, half x % 2; keys >= 32 only flag the instance
                atomicAdd(&cnt[((x >> 1) & 15u) * 32 + lane], 1u << ((x & 1u) << 4));
            }
        }
    }
    __syncwarp();
    // cross-bank sums: lane t totals word t % 16 over banks [16 (t / 16), +16), rotated
    const int cw = lane & 15, cb = lane & 16;
    uint32_t tot = 0;
#pragma unroll
    for (int s = 0; s < 16; ++s)
        tot += cnt[32 * cw + cb + ((s + lane) & 15)];
    tot += __shfl_xor_sync(0xFFFFFFFFu, tot, 16);  // labels 2 cw (low half) and 2 cw + 1 (high)
    const bool pow2 = (domain & (domain - 1)) == 0;
    const bool keys_ok = __reduce_or_sync(0xFFFFFFFFu, pow2 ? acc_or & ~(domain - 1) : (acc_max >= domain)) == 0;
    const bool uniform = __all_sync(0xFFFFFFFFu, tot == ((uint32_t)M | ((uint32_t)M << 16)));
    uint8_t st = DMM_OK;
    if (partition && !(keys_ok && uniform))
        st = DMM_INVALID_INSTANCE;  // check_partition_instance: label >= w or a count != m
    else if (!keys_ok)
        st = DMM_KEY_OUT_OF_RANGE;
    uint4* dst = reinterpret_cast<uint4*>(out + k * N);
    if (st != DMM_OK) {
        if (dst != src) {  // rejected before any step: the view keeps its input
#pragma unroll 1
            for (int i = lane; i < N / 4; i += 32)
                dst[i] = __ldg(src + i);
        }
    } else if (uniform) {
        // every run has length m: 16-byte chunk i (words 4 i .. 4 i + 3) lies in row 4 i / m
#pragma unroll 1
        for (int j = 0; j < kChunks; ++j) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t ci = 256 * j + lane + 32 * i;
                const uint32_t r = 4 * ci / M;
                dst[ci] = make_uint4(r, r, r, r);
            }
        }
    } else {
        // run ends E(v) = inclusive prefix of the counts; position p holds #{v : E(v) <= p}
        const uint32_t t = __shfl_sync(0xFFFFFFFFu, tot, lane >> 1);
        uint32_t e = (lane & 1) ? (t >> 16) : (t & 0xFFFFu);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, e, d);
            if (lane >= d)
                e += y;
        }
        uint32_t* ends = ends_s[warp];
        ends[lane] = e;
        __syncwarp();
        auto label_at = [&](uint32_t p) -> uint32_t {
            uint32_t lo = 0;
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1)
                lo += ends[lo + s - 1] <= p ? (uint32_t)s : 0u;
            return lo;
        };
#pragma unroll 1
        for (int i = lane; i < N / 4; i += 32)
            dst[i] = make_uint4(label_at(4 * i), label_at(4 * i + 1), label_at(4 * i + 2), label_at(4 * i + 3));
    }
    if (lane == 0) {
        if (status)
            status[k] = st;
        if (stats) {
            stats[k].cleanup_retries = 0;  // partition_leaf only: no cleanup loop
            stats[k].sorted = st == DMM_OK ? 1u : 0u;
        }
    }
}

}  // namespace dmmdev

namespace dmmhost {

bool partition_count_applies(uint32_t m, int mode, const GeneralArgs& a) {
    // DMM_PART_COUNT=0 selects the comparison-network leaf (A/B)
    static const bool off = getenv("DMM_PART_COUNT") && getenv("DMM_PART_COUNT")[0] == '0';
    if (off || a.probe)
        return false;
    if (m != 32 && m != 64 && m != 128 && m != 256)
        return false;
    return mode == dmmdev::kModePartition || (mode == dmmdev::kModeIntegerSort && a.domain <= 32);
}

dmm_status launch_partition_count(uint32_t m, int mode, const GeneralArgs& a) {
    if (a.count == 0)
        return DMM_OK;
    const uint64_t blocks = (a.count + dmmdev::kCountWarps - 1) / dmmdev::kCountWarps;
    if (blocks > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;
    const int part = mode == dmmdev::kModePartition ? 1 : 0;
    const uint32_t dom = part ? 32u : (uint32_t)a.domain;
    const dim3 grid{unsigned(blocks)}, block{unsigned(dmmdev::kCountWarps * 32)};
    switch (m) {
        case 32: dmmdev::k_partition_count<32><<<grid, block, 0, a.stream>>>(a.in, a.out, a.count, dom, part, a.stats, a.status); break;
        case 64: dmmdev::k_partition_count<64><<<grid, block, 0, a.stream>>>(a.in, a.out, a.count, dom, part, a.stats, a.status); break;
        case 128: dmmdev::k_partition_count<128><<<grid, block, 0, a.stream>>>(a.in, a.out, a.count, dom, part, a.stats, a.status); break;
        case 256: dmmdev::k_partition_count<256><<<grid, block, 0, a.stream>>>(a.in, a.out, a.count, dom, part, a.stats, a.status); break;
        default: set_error("counting partition: 32 <= m <= 256"); return DMM_UNSUPPORTED_SHAPE;
    }
    return check_launch("k_partition_count");
}

}  // namespace dmmhost

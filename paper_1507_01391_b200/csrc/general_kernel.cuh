// general_kernel.cuh -- the batched general-sort kernel template (kernels 1-3) and
// its launcher; instantiated per row width M in general_m*.cu (parallel builds).
#pragma once

#include "capi_common.h"
#include "dmm_algos.cuh"
#include "tma.cuh"

#include <algorithm>

namespace dmmdev {

template <int M>
__device__ __forceinline__ void load_row(const uint32_t* __restrict__ p, uint32_t (&v)[M]) {
    if constexpr (M % 4 == 0) {
        const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
        for (int i = 0; i < M / 4; ++i) {
            const uint4 t = __ldg(q + i);
            v[4 * i] = t.x;
            v[4 * i + 1] = t.y;
            v[4 * i + 2] = t.z;
            v[4 * i + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i)
            v[i] = __ldg(p + i);
    }
}

template <int M>
__device__ __forceinline__ void store_row(uint32_t* __restrict__ p, const uint32_t (&v)[M]) {
    if constexpr (M % 4 == 0) {
        uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
        for (int i = 0; i < M / 4; ++i)
            q[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i)
            p[i] = v[i];
    }
}

enum : int { kModeIntegerSort = 0, kModePartition = 1, kModeSortAny = 2 };

// Bank-conflict attribution build (-DDMM_NO_GLOBAL_IO, profiles/r02/conflicts_ab.sh): the batch
// kernels synthesise their keys in registers instead of loading them, and their stores are
// predicated off at run time (count == ~0 never holds), so the L1 data banks serve shared
// memory only.  Not a product build: its outputs are garbage.
#ifdef DMM_NO_GLOBAL_IO
constexpr bool kIoOff = true;
#else
constexpr bool kIoOff = false;
#endif
__device__ __forceinline__ uint32_t synth_key(uint64_t k, int row, int c) {
    return (uint32_t)((k * 0x9E3779B9ull + (uint64_t)row * 0x85EBCA6Bu + (uint64_t)c * 0xC2B2AE35u) >> 7) & 31u;
}

// CTA shape: warps per CTA and the occupancy target handed to ptxas (register cap)
#ifndef DMM_WPB
#define DMM_WPB 8  // warps per CTA of the one-warp-machine kernels (A/B variants: -DDMM_WPB=2/4;
                   // 32 x 32 machines: 4, measured 364 vs 351 G keys/s with 8, profiles/r02/pipeline_ab.txt)
#endif
template <int M, int PK, int WM = kWarp>
constexpr int warps_per_block() { return WM > kWarp ? WM / kWarp : (M >= 128 || M == 32 ? 4 : DMM_WPB); }
// DMM_GEN_MINB (A/B): CTAs per SM asked of ptxas for the 32 x 8 / 32 x 16 general sorts
#ifndef DMM_GEN_MINB
#define DMM_GEN_MINB 1
#endif
template <int M, int PK>
constexpr int min_blocks_per_sm() { return (M == 8 || M == 16) ? DMM_GEN_MINB : 1; }
// shared-memory words per warp (WM <= 32) or per machine (WM > 32: one machine per CTA)
template <int M, int WM>
constexpr int staging_words() { return relayout_buf_words(M) * (WM > kWarp ? WM / kWarp : 1); }

// One warp = G = 32 / WM machines of WM rows (WM = 32: one machine per warp; WM < 32: the
// machines are the members of one lockstep view family, exactly how the reference runs
// sibling views), times PK instances per register (16-bit halves).  Warp-task t covers
// instances [t*PK*G, (t+1)*PK*G): half h, lane group g = lane / WM holds instance
// t*PK*G + h*G + g, local row lane % WM.  The G instances of one half are contiguous in
// memory, so lane l's row sits at in[(first * WM + l) * M] exactly as for one 32-row machine.
//
// WM > 32 (64, 128, 256): one machine per CTA of WM / 32 warps; thread t holds row t, the
// algorithms get the row index where they take a lane, relayouts go through the CTA's
// staging buffer between CTA barriers, and per-machine reductions combine the warps.
// PIPE (one-warp machines whose instances load in any layout, no probe): persistent warps, and
// each warp's next task streams into its own shared-memory input slot by one TMA bulk copy
// (cp.async.bulk + a per-warp mbarrier) while the current task runs -- the HBM latency hides
// behind the sorting network without spending registers; lanes read their 16-byte chunks back
// from the slot (a quarter-warp covers 128 contiguous bytes: conflict-free).
template <int M, int WM>
constexpr int pipe_slot_words(int PK) { return PK * WM * M; }
template <int M, int WM>
constexpr int pipe_staging_words() { return (staging_words<M, WM>() + 3) & ~3; }  // 16-byte aligned slot
template <int M, int PK, int WM>
constexpr int pipe_warp_words() { return pipe_staging_words<M, WM>() + pipe_slot_words<M, WM>(PK) + 4; }
constexpr int kPipeWarps = 4;
#ifndef DMM_PIPE2_MINB
#define DMM_PIPE2_MINB 3  // CTAs per SM asked of ptxas for the L2-prefetch pipeline (register cap)
#endif

// PIPE = 1: the TMA smem slot above; PIPE = 2: persistent warps that only prefetch their next task
// into L2 (cp.async.bulk.prefetch.L2: no shared memory, no registers) and load it with LDG.
template <int M, int PK, bool EXT, int MODE, int WM = kWarp, int PIPE = 0>
__global__ void __launch_bounds__((PIPE == 1 ? kPipeWarps : warps_per_block<M, PK, WM>()) * 32,
                                  (PIPE == 2 ? DMM_PIPE2_MINB : min_blocks_per_sm<M, PK>()))
    k_general_sort(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t count, uint64_t domain,
                   int strict, int ascending, dmm_general_stats* __restrict__ stats, uint8_t* __restrict__ status,
                   uint32_t* __restrict__ probe, uint32_t probe_max) {
    static_assert(WM >= 1 && (WM < kWarp || WM % kWarp == 0), "machines tile the warp or the CTA");
    constexpr bool kMulti = WM > kWarp;
    constexpr int G = kMulti ? 1 : kWarp / WM;  // machines per warp (lanes >= G * WM idle)
    constexpr uint32_t kMask = (kMulti || G * WM == kWarp) ? 0xFFFFFFFFu : ((1u << (G * WM)) - 1u);
    extern __shared__ uint32_t smem[];
    const int lane = kMulti ? (int)threadIdx.x : (int)(threadIdx.x & 31);  // the machine row index space
    const int warp = kMulti ? 0 : (int)(threadIdx.x >> 5);
    const int grp = kMulti ? 0 : lane / WM, row = kMulti ? lane : lane % WM;
    const bool live_lane = ((kMask >> (lane & 31)) & 1u) != 0;
    static_assert(!PIPE || (!kMulti && G == 1), "the TMA pipeline runs one-warp machines");
    uint32_t* buf = smem + warp * (PIPE == 1 ? pipe_warp_words<M, PK, WM>() : staging_words<M, WM>());
    uint32_t* slot = buf + pipe_staging_words<M, WM>();               // PIPE: the next task's input
    uint64_t* bar = reinterpret_cast<uint64_t*>(slot + pipe_slot_words<M, WM>(PK));
    const uint64_t task_stride = (uint64_t)gridDim.x * (blockDim.x >> 5) * (PK * G);
    uint64_t first = kMulti ? (uint64_t)blockIdx.x * PK
                            : ((uint64_t)blockIdx.x * (blockDim.x >> 5) + warp) * (PK * G);  // half 0, group 0
    if (first >= count)
        return;
    uint32_t parity = 0;
    auto issue = [&](uint64_t f) {  // lane 0: TMA of the task starting at instance f into the slot
        const uint64_t n = count - f < (uint64_t)PK ? count - f : (uint64_t)PK;
        tma_load(slot, in + f * WM * M, (uint32_t)(n * WM * M * 4), bar);
    };
    if constexpr (PIPE == 1) {
        if (lane == 0) {
            mbar_init(bar);
            issue(first);
        }
        __syncwarp();
    }
    for (;; first += task_stride) {
    if (first >= count)
        break;
    // half h of this lane's machine: instance first + h*G + grp (absent past count)
    auto inst_of = [&](int h) -> uint64_t { return first + (uint64_t)h * G + grp; };
    const bool hasB = PK == 2 && first + G < count;  // any machine of half 1 present

    // A leaf-only instance (w <= m: balance_divide_sort is partition_leaf, whose outcome
    // is the sorted multiset whatever the starting arrangement) is loaded fully coalesced:
    // the machine's lane r takes its instance's 16-byte chunks r, r + WM, ...  Otherwise
    // lane r loads row r (the recursion's intermediate matrices depend on the arrangement).
    constexpr bool kAnyLayout = MODE != kModeSortAny && WM <= M && M % 4 == 0;
    auto load = [&](int h, uint32_t (&v)[M]) {
        const uint64_t k = inst_of(h);
        if (k >= count || !live_lane) {
#pragma unroll
            for (int c = 0; c < M; ++c)
                v[c] = 0;
            return;
        }
        if constexpr (kIoOff) {
#pragma unroll
            for (int c = 0; c < M; ++c)
                v[c] = synth_key(k, row, c);
            return;
        }
        if constexpr (PIPE == 1) {
            const uint4* q = reinterpret_cast<const uint4*>(slot + (uint64_t)h * WM * M);
#pragma unroll
            for (int i = 0; i < M / 4; ++i) {
                const uint4 t = q[row + WM * i];
                v[4 * i] = t.x;
                v[4 * i + 1] = t.y;
                v[4 * i + 2] = t.z;
                v[4 * i + 3] = t.w;
            }
            return;
        }
        if constexpr (kAnyLayout) {
            const uint4* q = reinterpret_cast<const uint4*>(in + k * WM * M);
#pragma unroll
            for (int i = 0; i < M / 4; ++i) {
                const uint4 t = __ldg(q + row + WM * i);
                v[4 * i] = t.x;
                v[4 * i + 1] = t.y;
                v[4 * i + 2] = t.z;
                v[4 * i + 3] = t.w;
            }
        } else {
            load_row<M>(in + (k * WM + row) * M, v);
        }
    };
    // keys outside [0, domain): OR-accumulate (power-of-two domain, half an ALU op per
    // key) or max-accumulate; nothing to check for domain >= 2^32
    const bool dom32 = domain < (1ull << 32);
    const bool dom_pow2 = (domain & (domain - 1)) == 0;
    const uint32_t dom_mask = dom32 && dom_pow2 ? ~(uint32_t)(domain - 1) : 0u;
    auto keys_bad = [&](const uint32_t* v, int n) -> uint32_t {
        if (!dom32)
            return 0u;
        uint32_t acc = 0;
        if (dom_pow2) {
#pragma unroll
            for (int c = 0; c < n; ++c)
                acc |= v[c];
            return (acc & dom_mask) != 0 ? 1u : 0u;
        }
#pragma unroll
        for (int c = 0; c < n; ++c)
            acc = max(acc, v[c]);
        return acc >= (uint32_t)domain ? 1u : 0u;
    };

    uint32_t x[M];
    if constexpr (PIPE == 1)
        mbar_wait(bar, parity);
    if constexpr (PIPE == 2) {
        // the task after this one heads for L2 while this one sorts
        if (lane == 0 && first + task_stride < count) {
            const uint64_t f = first + task_stride;
            const uint64_t nn = count - f < (uint64_t)PK ? count - f : (uint64_t)PK;
            prefetch_l2(in + f * WM * M, (uint32_t)(nn * WM * M * 4));
        }
    }
    load(0, x);
    uint32_t bad = keys_bad(x, M);  // bit h: half h holds a key outside [0, domain)
    if constexpr (PK == 2) {
        uint32_t b[M];
        if (hasB) {
            load(1, b);
        } else {
#pragma unroll
            for (int c = 0; c < M; ++c)
                b[c] = 0;
        }
        bad |= keys_bad(b, M) << 1;
#pragma unroll
        for (int c = 0; c < M; ++c)
            x[c] = __byte_perm(x[c], b[c], 0x5410);  // (a & 0xFFFF) | (b << 16)
    }
    if constexpr (PIPE == 1) {
        // the slot is read: stream the warp's next task into it while this one runs
        parity ^= 1;
        __syncwarp();
        if (lane == 0 && first + task_stride < count) {
            fence_async_smem();
            issue(first + task_stride);
        }
    }
    auto machine_or = [&](uint32_t v) -> uint32_t {
        if constexpr (kMulti)
            return group_or<WM, WM>(v, row, buf);
        else
            return seg_or<WM>(v);
    };
    bad = machine_or(bad);

    using V = VF<kMask, 0, 1, WM, 0, M, (kMulti ? WM : 32), (kMulti ? WM : 32)>;
    GenResult res{{0u, 0u}, 0u};
    // probe snapshots (PartitionProbe / ShortWideHook points; one code path: the capture
    // points test a uniform pointer): instance k's area is probe[k * probe_max * WM * M ...]
    ProbeSink ps{{nullptr, nullptr}, 0u, probe_max, row, WM};
#pragma unroll
    for (int h = 0; h < PK; ++h)
        if (probe != nullptr && inst_of(h) < count && live_lane)
            ps.dst[h] = probe + inst_of(h) * probe_max * WM * M;
    if constexpr (MODE == kModeSortAny) {
        sort_wide_any<PK, V>(x, buf, lane, ascending != 0, probe != nullptr ? &ps : nullptr);
    } else {
        // partition labels are < w <= 32: the top key bit of every half is free for the fused
        // cleanup (cleanup_pass_pair); integer keys may use every bit
        // (multi-warp machines always run the fused cleanup: their integer sorts need a
        // domain below the tag bit, checked by the host)
        constexpr uint32_t kTag =
            (MODE == kModePartition || kMulti) ? (PK == 2 ? 0x80008000u : 0x80000000u) : 0u;
        balance_divide_sort<PK, V, EXT, kTag>(x, buf, lane, res, probe != nullptr ? &ps : nullptr);
    }
    if constexpr (kMulti)
        res.template finish_machine<WM>(row, buf);
    else
        res.template finish<WM>();

    uint32_t invalid = 0;
    // partition entry points run as MODE kModePartition, or as the literal comparison skeleton
    // (kModeSortAny with domain = w < 2^32: partition_short_wide with its hook points)
    if (MODE == kModePartition || (MODE == kModeSortAny && domain < (1ull << 32))) {
        // check_partition_instance (partition.hpp:112-124): labels in [0, w), m copies
        // each  <=>  (labels < w) and the sorted result has row i = i everywhere.
        // OR of (key ^ row) over the row: one LOP3 per register, both halves at once
        const uint32_t want = PK == 2 ? (uint32_t)row * 0x10001u : (uint32_t)row;
        uint32_t diff = 0;
#pragma unroll
        for (int c = 0; c < M; ++c)
            diff |= x[c] ^ want;
        const uint32_t mism = PK == 2 ? ((diff & 0xFFFFu) ? 1u : 0u) | ((diff >> 16) ? 2u : 0u) : (diff ? 1u : 0u);
        invalid = machine_or(mism) | bad;
    }

#pragma unroll
    for (int h = 0; h < PK; ++h) {
        const uint64_t k = inst_of(h);
        if (k >= count || !live_lane)
            continue;
        if (kIoOff && count != ~0ull)
            continue;
        if constexpr (M % 4 == 0) {
            // unpack one 16-byte vector at a time (register budget)
            uint4* q = reinterpret_cast<uint4*>(out + (k * WM + row) * M);
#pragma unroll
            for (int i = 0; i < M / 4; ++i) {
                uint32_t v[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    v[e] = PK == 2 ? ((x[4 * i + e] >> (16 * h)) & 0xFFFFu) : x[4 * i + e];
                q[i] = make_uint4(v[0], v[1], v[2], v[3]);
            }
        } else {
            uint32_t v[M];
#pragma unroll
            for (int c = 0; c < M; ++c)
                v[c] = PK == 2 ? ((x[c] >> (16 * h)) & 0xFFFFu) : x[c];
            store_row<M>(out + (k * WM + row) * M, v);
        }
        if (row == 0) {
            const bool unsorted = (res.unsorted >> h) & 1u;
            uint8_t s = DMM_OK;
            if ((invalid >> h) & 1u)
                s = DMM_INVALID_INSTANCE;
            else if ((bad >> h) & 1u)
                s = DMM_KEY_OUT_OF_RANGE;
            else if (unsorted && strict)
                s = DMM_POSTCONDITION_FAILED;
            if (status)
                status[k] = s;
            if (stats) {
                stats[k].cleanup_retries = res.retries[h];
                stats[k].sorted = unsorted ? 0u : 1u;
            }
        }
    }
    if constexpr (PIPE == 0)
        break;
    }  // task loop (one task unless PIPE)
}

}  // namespace dmmdev


namespace dmmhost {

struct GeneralArgs {
    const uint32_t* in;
    uint32_t* out;
    uint64_t count;
    uint64_t domain;
    int strict;
    int ascending;
    dmm_general_stats* stats;
    uint8_t* status;
    cudaStream_t stream;
    uint32_t* probe = nullptr;  // PartitionProbe snapshots (count x probe_max x w x m), optional
    uint32_t probe_max = 0;
};

template <int M, int PK, bool EXT, int MODE, int WM = dmmdev::kWarp>
dmm_status launch_general(const GeneralArgs& a) {
    auto kern = dmmdev::k_general_sort<M, PK, EXT, MODE, WM>;
    constexpr int kWarpsPerBlock = dmmdev::warps_per_block<M, PK, WM>();
    constexpr bool kMulti = WM > dmmdev::kWarp;
    const size_t smem = size_t(kMulti ? 1 : kWarpsPerBlock) * dmmdev::staging_words<M, WM>() * sizeof(uint32_t);
    static std::atomic<uint64_t> configured{0};  // devices configured, per instantiation
    if (dmm_status e = configure_kernel(kern, smem, configured); e != DMM_OK)
        return e;
    constexpr int kPerWarp = kMulti ? 1 : dmmdev::kWarp / WM;  // machines per warp
    const uint64_t units = (a.count + PK * kPerWarp - 1) / (PK * kPerWarp);  // warp-tasks / machines
    const uint64_t blocks = kMulti ? units : (units + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks == 0)
        return DMM_OK;
    if (blocks > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;
    kern<<<dim3(unsigned(blocks)), dim3(kWarpsPerBlock * 32), smem, a.stream>>>(a.in, a.out, a.count, a.domain, a.strict,
                                                                                a.ascending, a.stats, a.status,
                                                                                a.probe, a.probe_max);
    return check_launch("k_general_sort");
}


// PIPE: persistent one-warp machines with the TMA input pipeline (leaf-only shapes, no probe)
template <int M, int PK, bool EXT, int MODE, int PIPE = 1>
dmm_status launch_general_pipe(const GeneralArgs& a) {
    auto kern = dmmdev::k_general_sort<M, PK, EXT, MODE, dmmdev::kWarp, PIPE>;
    constexpr int kW = PIPE == 1 ? dmmdev::kPipeWarps : dmmdev::warps_per_block<M, PK, dmmdev::kWarp>();
    const size_t smem = size_t(kW) * (PIPE == 1 ? dmmdev::pipe_warp_words<M, PK, dmmdev::kWarp>()
                                                : dmmdev::staging_words<M, dmmdev::kWarp>()) * sizeof(uint32_t);
    static std::atomic<uint64_t> configured{0};
    if (dmm_status e = configure_kernel(kern, smem, configured); e != DMM_OK)
        return e;
    const uint64_t tasks = (a.count + PK - 1) / PK;
    if (tasks == 0)
        return DMM_OK;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kW * 32, smem);
    const uint64_t blocks = std::min<uint64_t>((tasks + kW - 1) / kW, uint64_t(sms) * std::max(per_sm, 1));
    kern<<<dim3(unsigned(blocks)), dim3(kW * 32), smem, a.stream>>>(a.in, a.out, a.count, a.domain, a.strict,
                                                                   a.ascending, a.stats, a.status, a.probe,
                                                                   a.probe_max);
    return check_launch("k_general_sort (pipelined)");
}

// per-width entry points (general_m*.cu)
dmm_status launch_general_m8(int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_m16(int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_m32(int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_m64(int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_m128(int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_m256(int mode, bool pk2, bool ext, const GeneralArgs& a);
// leaf-only partitions / small-domain integer sorts of 32 x {32, 64, 128, 256} views as one
// per-bank counting pass (partition_count.cu); the launchers below try it first
bool partition_count_applies(uint32_t m, int mode, const GeneralArgs& a);
dmm_status launch_partition_count(uint32_t m, int mode, const GeneralArgs& a);
// 32 x 1024: the short-wide skeleton on a CTA of 32 warps (short_wide32.cu)
dmm_status launch_general_m1024(int mode, bool pk2, bool ext, const GeneralArgs& a);
// multi-warp machines (w = 64, 128, 256 rows, one per CTA), general_tall*.cu
dmm_status launch_general_tall64(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_tall128(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_tall256(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);
// sub-warp machines (w < 32 rows, 32 / w machines per warp), general_w*.cu
dmm_status launch_general_w16(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_w8(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_w4(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_w2(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);
dmm_status launch_general_w3(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a);

}  // namespace dmmhost

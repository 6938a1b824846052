// multisplit.cu -- the local step of cfg5's global w-way partition: a stable
// partition of one GPU's key array by an 8-way (or any power-of-two <= 32) label
// label = (key >> shift) & (nbuckets - 1), bucket-major output, per-bucket counts.
//
// Three passes, no shared-memory data movement at all (so nothing to conflict on):
//   1. k_ms_count: each warp owns a tile of kMsRows rows of 128 keys; lane l loads keys
//      4l..4l+3 of a row with one 16-byte load (512 coalesced bytes per warp load); per
//      row and sub-position j, log2(nbuckets) ballots give every bucket's lane mask and
//      popc counts it;
//   2. k_ms_scan_*: exclusive scan of the per-tile counts, bucket-major (two levels);
//   3. k_ms_scatter: the warp re-reads its tile in rows of 32 consecutive keys (one per lane);
//      a key's destination is offset[bucket][tile] + keys of its bucket in earlier rows + keys
//      of its bucket in lower lanes of this row (popc of the label-bit ballots' match mask),
//      i.e. stable by source index, and a warp store writes at most nbuckets contiguous runs.
// The cross-GPU exchange (bucket j -> rank owning j) is either fused into pass 3
// (dmm_multisplit_count + dmm_multisplit_scatter_to: k_ms_scatter<LB, true> stores each key
// straight into its owner's receive buffer, peer memory over NVLink) or an NCCL all-to-all
// after dmm_multisplit (paper_1507_01391_b200/distributed.py).
#include <cstdlib>

#include "capi_common.h"

namespace dmmdev {

constexpr int kMsRows = 32;    // rows of 128 keys per warp tile
constexpr int kMsTile = kMsRows * 128;  // keys per warp tile

template <int LB>
__device__ __forceinline__ void bucket_masks(uint32_t label, uint32_t (&mk)[1 << LB]) {
    uint32_t bal[LB > 0 ? LB : 1];
#pragma unroll
    for (int i = 0; i < LB; ++i)
        bal[i] = __ballot_sync(0xFFFFFFFFu, (label >> i) & 1u);
#pragma unroll
    for (int b = 0; b < (1 << LB); ++b) {
        uint32_t m = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < LB; ++i)
            m &= ((b >> i) & 1) ? bal[i] : ~bal[i];
        mk[b] = m;
    }
}

// lane l's 4 keys of row r of a tile: indices base + 128 r + 4 l + (0..3); vectorised when the
// whole row is in range (n need not be a multiple of 4)
__device__ __forceinline__ void load_row4(const uint32_t* __restrict__ keys, uint64_t n, uint64_t i0,
                                          uint32_t (&k)[4], uint32_t& valid) {
    if (i0 + 4 <= n && (i0 & 3) == 0) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(keys + i0));
        k[0] = t.x;
        k[1] = t.y;
        k[2] = t.z;
        k[3] = t.w;
        valid = 0xFu;
    } else {
        valid = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool v = i0 + j < n;
            k[j] = v ? __ldg(keys + i0 + j) : 0u;
            valid |= v ? (1u << j) : 0u;
        }
    }
}

// Per-lane bucket counters packed 8 bits per bucket: P[h] holds buckets 4h..4h+3 (a lane
// sees at most 4 keys per row, so a row's counts and their warp prefix sums stay < 256).
template <int NB>
struct Packed {
    static constexpr int H = (NB + 3) / 4;
    uint32_t p[H];
    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int h = 0; h < H; ++h)
            p[h] = 0;
    }
    __device__ __forceinline__ void add(uint32_t label) {  // count one key of bucket `label`
        const uint32_t inc = 1u << (8 * (label & 3));
#pragma unroll
        for (int h = 0; h < H; ++h)
            p[h] += (label >> 2) == (uint32_t)h ? inc : 0u;
    }
    __device__ __forceinline__ uint32_t get(uint32_t b) const {
        uint32_t v = 0;
#pragma unroll
        for (int h = 0; h < H; ++h)
            v = (b >> 2) == (uint32_t)h ? p[h] : v;
        return (v >> (8 * (b & 3))) & 0xFFu;
    }
};

template <int LB>
__global__ void __launch_bounds__(256) k_ms_count(const uint32_t* __restrict__ keys, uint64_t n, uint32_t shift,
                                                  uint32_t* __restrict__ tile_counts, uint64_t ntiles) {
    constexpr int NB = 1 << LB;
    const int lane = threadIdx.x & 31;
    const uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (tile >= ntiles)
        return;
    // per-lane counts over the whole tile: kMsRows * 4 = 128 keys per lane < 256
    Packed<NB> c;
    c.clear();
    const uint64_t base = tile * kMsTile;
#pragma unroll 8
    for (int r = 0; r < kMsRows; ++r) {
        uint32_t k[4], valid;
        load_row4(keys, n, base + (uint64_t)r * 128 + 4 * lane, k, valid);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((valid >> j) & 1u)
                c.add((k[j] >> shift) & (NB - 1));
    }
    // lane b < NB reports bucket b: reduce every bucket over the warp (16-bit halves, < 2^13)
    uint32_t mine = 0;
#pragma unroll
    for (int h = 0; h < Packed<NB>::H; ++h) {
        uint32_t lo = c.p[h] & 0x00FF00FFu, hi = (c.p[h] >> 8) & 0x00FF00FFu;  // buckets (4h, 4h+2), (4h+1, 4h+3)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            lo += __shfl_xor_sync(0xFFFFFFFFu, lo, o);
            hi += __shfl_xor_sync(0xFFFFFFFFu, hi, o);
        }
        if ((lane >> 2) == h) {
            const uint32_t q = lane & 3;
            mine = ((q & 1) ? hi : lo) >> (16 * (q >> 1)) & 0xFFFFu;
        }
    }
    if (lane < NB)
        tile_counts[(uint64_t)lane * ntiles + tile] = mine;  // bucket-major
}

// exclusive scan of a bucket-major count array (NB * ntiles entries) in two levels
constexpr int kScanBlock = 1024;

__global__ void k_ms_scan_blocks(const uint32_t* __restrict__ in, uint64_t total, uint64_t* __restrict__ out,
                                 uint64_t* __restrict__ block_sums) {
    __shared__ uint64_t warp_sums[32];
    const uint64_t i = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
    const uint64_t v = i < total ? in[i] : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31)
        warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t s = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o)
                s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    const uint64_t before = warp ? warp_sums[warp - 1] : 0;
    if (i < total)
        out[i] = before + x - v;  // exclusive within the block
    if (threadIdx.x == kScanBlock - 1)
        block_sums[blockIdx.x] = before + x;
}

__global__ void k_ms_scan_sums(uint64_t* __restrict__ block_sums, uint64_t nblocks) {
    // one block: sequential carry over chunks of 1024
    __shared__ uint64_t carry_s;
    if (threadIdx.x == 0)
        carry_s = 0;
    __syncthreads();
    for (uint64_t c0 = 0; c0 < nblocks; c0 += blockDim.x) {
        const uint64_t i = c0 + threadIdx.x;
        const uint64_t v = i < nblocks ? block_sums[i] : 0;
        __shared__ uint64_t buf[1024];
        buf[threadIdx.x] = v;
        __syncthreads();
        for (unsigned o = 1; o < blockDim.x; o <<= 1) {
            const uint64_t y = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
            __syncthreads();
            buf[threadIdx.x] += y;
            __syncthreads();
        }
        const uint64_t incl = buf[threadIdx.x];
        const uint64_t carry = carry_s;
        if (i < nblocks)
            block_sums[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1)
            carry_s = carry + incl;
        __syncthreads();
    }
}

__global__ void k_ms_scan_add(uint64_t* __restrict__ out, uint64_t total, const uint64_t* __restrict__ block_sums) {
    const uint64_t i = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
    if (i < total)
        out[i] += block_sums[blockIdx.x];
}

// Rows of 32 consecutive keys, one per lane (coalesced 128-byte loads): the keys of one bucket
// in one row go to consecutive output words, so every warp store writes at most NB contiguous
// runs.  Rows go in groups of kG; the next group's loads are issued before the current group
// is ranked (2 kG rows in flight per warp: the kernel is load-latency bound).  A key's rank
// among its row's bucket-mates = popc of the lower lanes whose LB label bits all match (LB
// ballots); the row's per-bucket totals are the same masks for bucket = lane.  Lane b < NB
// holds bucket b's next output address (`cur`), so a key needs one 64-bit shuffle.  FULL: the
// whole tile is in range (no per-key bounds).
#ifndef DMM_MS_G
#define DMM_MS_G 16
#endif
constexpr int kG = DMM_MS_G;  // rows per group (r01 ranking: 4: 223, 8: 255, 16: 295, 32: 276 G keys/s on cfg5)

template <int LB, bool FULL>
__device__ __forceinline__ void scatter_tile(const uint32_t* __restrict__ keys, uint64_t n, uint32_t shift,
                                             uint64_t base, uint32_t* cur, int lane) {
    constexpr int NB = 1 << LB;
    const uint32_t lt = (1u << lane) - 1u;  // lanes below this one
    const uint32_t lane_nb = lane < NB ? 0xFFFFFFFFu : 0u;  // lanes that carry a bucket total
    uint32_t sl[LB > 0 ? LB : 1];                            // this lane's bucket bits as masks
    uint32_t lbit[LB > 0 ? LB : 1];                          // the key bit of label bit i
#pragma unroll
    for (int i = 0; i < LB; ++i) {
        sl[i] = ((lane >> i) & 1) ? 0xFFFFFFFFu : 0u;
        lbit[i] = 1u << (shift + i);
    }
    uint32_t k[kG];
    bool valid[kG];
    auto load_group = [&](int r, uint32_t (&kk)[kG], bool (&vv)[kG]) {
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const uint64_t i = base + (uint64_t)(r + j) * 32 + lane;
            vv[j] = FULL || i < n;
            kk[j] = vv[j] ? __ldg(keys + i) : 0u;
        }
    };
    load_group(0, k, valid);
#pragma unroll 1
    for (int r = 0; r < kMsRows * 4; r += kG) {
        uint32_t kn[kG];
        bool vn[kG];
        if (r + kG < kMsRows * 4)
            load_group(r + kG, kn, vn);
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const uint32_t b = (k[j] >> shift) & (NB - 1);
            // mk: the lanes whose key carries label (lane mod NB) -- LB ballots of the label bits,
            // each folded in by one LOP3 against this lane's own bucket bits.  Every lane's mk is
            // a row total of its bucket, and the key's own bucket mates are lane b's mk (one
            // shuffle), so the per-key work is the same for any NB.
            uint32_t mk = FULL ? 0xFFFFFFFFu : __ballot_sync(0xFFFFFFFFu, valid[j]);
#pragma unroll
            for (int i = 0; i < LB; ++i) {
                const uint32_t bi = __ballot_sync(0xFFFFFFFFu, (k[j] & lbit[i]) != 0u);
                mk &= ~(bi ^ sl[i]);
            }
            const uint32_t mo = __shfl_sync(0xFFFFFFFFu, mk, (int)b);
            uint32_t* d = reinterpret_cast<uint32_t*>(
                __shfl_sync(0xFFFFFFFFu, reinterpret_cast<unsigned long long>(cur), (int)b));
            if (valid[j])
                d[__popc(mo & lt)] = k[j];
            cur += __popc(mk & lane_nb);
        }
        if (r + kG < kMsRows * 4) {
#pragma unroll
            for (int j = 0; j < kG; ++j) {
                k[j] = kn[j];
                valid[j] = vn[j];
            }
        }
    }
}

// REMOTE: bucket b goes to its own destination array dst[b] (a peer GPU's receive buffer over
// NVLink, or any device pointer) starting at dst_base[b] -- the all-to-all fused into the
// scatter: keys leave the SM straight for the owner's memory, no staging copy, no NCCL pass.
template <int LB, bool REMOTE = false, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_ms_scatter(const uint32_t* __restrict__ keys, uint64_t n, uint32_t shift,
                                                    const uint64_t* __restrict__ offsets, uint64_t ntiles,
                                                    uint32_t* __restrict__ out, uint32_t* const* __restrict__ dst = nullptr,
                                                    const uint64_t* __restrict__ dst_base = nullptr) {
    constexpr int NB = 1 << LB;
    const int lane = threadIdx.x & 31;
    const uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (tile >= ntiles)
        return;
    // lane b < NB: bucket b's next output address (its tile offset in the bucket-major scan)
    uint32_t* cur = out;
    if (lane < NB) {
        const uint64_t pos = offsets[(uint64_t)lane * ntiles + tile];
        if constexpr (REMOTE)
            cur = dst[lane] + (pos - offsets[(uint64_t)lane * ntiles] + dst_base[lane]);  // rank within the bucket
        else
            cur = out + pos;
    }
    const uint64_t base = tile * kMsTile;
    if (base + kMsTile <= n)
        scatter_tile<LB, true>(keys, n, shift, base, cur, lane);
    else
        scatter_tile<LB, false>(keys, n, shift, base, cur, lane);
}

}  // namespace dmmdev

namespace {
using namespace dmmhost;

// phase: 1 = count + scans (+ starts), 2 = scatter only (workspace from phase 1), 3 = both
template <int LB>
dmm_status run_multisplit(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t* out, uint64_t* starts,
                          void* workspace, cudaStream_t s, int phase = 3, uint32_t* const* dst = nullptr,
                          const uint64_t* dst_base = nullptr) {
    constexpr int NB = 1 << LB;
    const uint64_t ntiles = (n + dmmdev::kMsTile - 1) / dmmdev::kMsTile;
    const uint64_t total = ntiles * NB;
    const uint64_t nblocks = (total + dmmdev::kScanBlock - 1) / dmmdev::kScanBlock;
    uint32_t* tile_counts = static_cast<uint32_t*>(workspace);
    uint64_t* offsets = reinterpret_cast<uint64_t*>(
        static_cast<char*>(workspace) + ((total * sizeof(uint32_t) + 255) & ~uint64_t(255)));
    uint64_t* block_sums = offsets + ((total + 31) & ~uint64_t(31));
    const unsigned warps_per_block = 8;
    const uint64_t grid = (ntiles + warps_per_block - 1) / warps_per_block;
    if (grid > 0x7FFFFFFFull || nblocks > 0x7FFFFFFFull)
        return DMM_INVALID_ARGUMENT;  // grid x limit
    // DMM_MS_MINB=B (A/B, 8 buckets): ask ptxas for B resident 8-warp CTAs per SM on the scatter
    static const int ms_minb = getenv("DMM_MS_MINB") ? atoi(getenv("DMM_MS_MINB")) : 0;
    if (phase == 2) {
        auto kern = dmmdev::k_ms_scatter<LB, true>;
        if constexpr (LB == 3) {
            if (ms_minb == 3)
                kern = dmmdev::k_ms_scatter<LB, true, 3>;
            else if (ms_minb == 4)
                kern = dmmdev::k_ms_scatter<LB, true, 4>;
        }
        kern<<<unsigned(grid), warps_per_block * 32, 0, s>>>(keys, n, shift, offsets, ntiles, nullptr, dst, dst_base);
        return check_launch("k_ms_scatter (remote)");
    }
    dmmdev::k_ms_count<LB><<<unsigned(grid), warps_per_block * 32, 0, s>>>(keys, n, shift, tile_counts, ntiles);
    if (dmm_status e = check_launch("k_ms_count"); e != DMM_OK)
        return e;
    dmmdev::k_ms_scan_blocks<<<unsigned(nblocks), dmmdev::kScanBlock, 0, s>>>(tile_counts, total, offsets,
                                                                              block_sums);
    if (dmm_status e = check_launch("k_ms_scan_blocks"); e != DMM_OK)
        return e;
    dmmdev::k_ms_scan_sums<<<1, 1024, 0, s>>>(block_sums, nblocks);
    if (dmm_status e = check_launch("k_ms_scan_sums"); e != DMM_OK)
        return e;
    dmmdev::k_ms_scan_add<<<unsigned(nblocks), dmmdev::kScanBlock, 0, s>>>(offsets, total, block_sums);
    if (dmm_status e = check_launch("k_ms_scan_add"); e != DMM_OK)
        return e;
    if (phase == 3) {
        dmmdev::k_ms_scatter<LB><<<unsigned(grid), warps_per_block * 32, 0, s>>>(keys, n, shift, offsets, ntiles,
                                                                                 out);
        if (dmm_status e = check_launch("k_ms_scatter"); e != DMM_OK)
            return e;
    }
    if (starts) {
        // bucket b starts where its tile 0 writes: offsets[b * ntiles] (bucket-major scan)
        cudaMemcpy2DAsync(starts, sizeof(uint64_t), offsets, ntiles * sizeof(uint64_t), sizeof(uint64_t), NB,
                          cudaMemcpyDeviceToDevice, s);
        if (cudaGetLastError() != cudaSuccess)
            return check_launch("bucket starts copy");
    }
    return DMM_OK;
}

// Common argument checks of the three entry points: the count pass reads 16-byte vectors at
// key indices that are multiples of 4, so `keys` itself must be 16-byte aligned (a view with a
// storage offset is rejected, as check_ptrs does for the other entry points), and the label
// bits [shift, shift + log2(nbuckets)) must lie inside the 32-bit key.
dmm_status ms_check(const uint32_t* keys, uint32_t shift, uint32_t nbuckets) {
    if (keys && (reinterpret_cast<uintptr_t>(keys) & 15u)) {
        set_error("keys must be 16-byte aligned");
        return DMM_INVALID_ARGUMENT;
    }
    uint32_t lb = 0;
    while ((2u << lb) <= nbuckets && lb < 6)
        ++lb;
    if (shift >= 32 || shift + lb > 32) {
        set_error("label bits [shift, shift + log2(nbuckets)) must lie inside the 32-bit key");
        return DMM_INVALID_ARGUMENT;
    }
    return DMM_OK;
}

}  // namespace

extern "C" {

uint64_t dmm_multisplit_workspace_bytes(uint64_t n, uint32_t nbuckets) {
    const uint64_t ntiles = (n + dmmdev::kMsTile - 1) / dmmdev::kMsTile;
    const uint64_t total = ntiles * nbuckets;
    const uint64_t nblocks = (total + dmmdev::kScanBlock - 1) / dmmdev::kScanBlock;
    return ((total * 4 + 255) & ~uint64_t(255)) + ((total + 31) & ~uint64_t(31)) * 8 + nblocks * 8 + 256;
}

dmm_status dmm_multisplit_count(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t nbuckets,
                                uint64_t* bucket_starts, void* workspace, void* stream) {
    reset_launches();
    if (!bucket_starts || !workspace || (n && !keys))
        return DMM_INVALID_ARGUMENT;
    if (dmm_status e = ms_check(keys, shift, nbuckets); e != DMM_OK)
        return e;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0)
        return cudaMemsetAsync(bucket_starts, 0, sizeof(uint64_t) * nbuckets, s) == cudaSuccess
                   ? DMM_OK
                   : check_launch("cudaMemsetAsync");
    switch (nbuckets) {
        case 2: return run_multisplit<1>(keys, n, shift, nullptr, bucket_starts, workspace, s, 1);
        case 4: return run_multisplit<2>(keys, n, shift, nullptr, bucket_starts, workspace, s, 1);
        case 8: return run_multisplit<3>(keys, n, shift, nullptr, bucket_starts, workspace, s, 1);
        case 16: return run_multisplit<4>(keys, n, shift, nullptr, bucket_starts, workspace, s, 1);
        case 32: return run_multisplit<5>(keys, n, shift, nullptr, bucket_starts, workspace, s, 1);
        default: break;
    }
    set_error("nbuckets must be a power of two in [2, 32]");
    return DMM_INVALID_ARGUMENT;
}

dmm_status dmm_multisplit_scatter_to(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t nbuckets,
                                     uint32_t* const* dst, const uint64_t* dst_base, void* workspace,
                                     void* stream) {
    reset_launches();
    if (n == 0)
        return DMM_OK;
    if (!keys || !dst || !dst_base || !workspace)
        return DMM_INVALID_ARGUMENT;
    if (dmm_status e = ms_check(keys, shift, nbuckets); e != DMM_OK)
        return e;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (nbuckets) {
        case 2: return run_multisplit<1>(keys, n, shift, nullptr, nullptr, workspace, s, 2, dst, dst_base);
        case 4: return run_multisplit<2>(keys, n, shift, nullptr, nullptr, workspace, s, 2, dst, dst_base);
        case 8: return run_multisplit<3>(keys, n, shift, nullptr, nullptr, workspace, s, 2, dst, dst_base);
        case 16: return run_multisplit<4>(keys, n, shift, nullptr, nullptr, workspace, s, 2, dst, dst_base);
        case 32: return run_multisplit<5>(keys, n, shift, nullptr, nullptr, workspace, s, 2, dst, dst_base);
        default: break;
    }
    set_error("nbuckets must be a power of two in [2, 32]");
    return DMM_INVALID_ARGUMENT;
}

dmm_status dmm_multisplit(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t nbuckets, uint32_t* out,
                          uint64_t* bucket_starts, void* workspace, void* stream) {
    reset_launches();
    if (n == 0)
        return DMM_OK;
    if (!keys || !out || !workspace)
        return DMM_INVALID_ARGUMENT;
    if (dmm_status e = ms_check(keys, shift, nbuckets); e != DMM_OK)
        return e;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (nbuckets) {
        case 2: return run_multisplit<1>(keys, n, shift, out, bucket_starts, workspace, s);
        case 4: return run_multisplit<2>(keys, n, shift, out, bucket_starts, workspace, s);
        case 8: return run_multisplit<3>(keys, n, shift, out, bucket_starts, workspace, s);
        case 16: return run_multisplit<4>(keys, n, shift, out, bucket_starts, workspace, s);
        case 32: return run_multisplit<5>(keys, n, shift, out, bucket_starts, workspace, s);
        default: break;
    }
    set_error("nbuckets must be a power of two in [2, 32]");
    return DMM_INVALID_ARGUMENT;
}

}  // extern "C"

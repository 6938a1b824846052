// multisplit.cu -- the local step of cfg5's global w-way partition: a stable
// partition of one GPU's key array by an 8-way (or any power-of-two <= 32) label
// label = (key >> shift) & (nbuckets - 1), bucket-major output, per-bucket counts.
//
// Three passes, no shared-memory data movement at all (so nothing to conflict on):
//   1. k_ms_count: each warp owns a tile of 32 x R keys (coalesced 128-byte rows); per row
//      of 32 keys, log2(nbuckets) ballots give every bucket's lane mask, popc counts it;
//   2. k_ms_scan_*: exclusive scan of the per-tile counts, bucket-major (two levels);
//   3. k_ms_scatter: the warp re-reads its tile; a key's destination is
//      offset[bucket][tile] + keys of its bucket in earlier rows + popc(mask & lanes below),
//      i.e. stable by (tile, row, lane) = source order.  One warp store writes at most
//      nbuckets contiguous runs.
// The cross-GPU exchange (bucket j -> rank owning j) is an NCCL all-to-all in
// paper_1507_01391_b200/distributed.py.
#include "capi_common.h"

namespace dmmdev {

constexpr int kMsRows = 32;  // rows of 32 keys per warp tile (1024 keys)

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

template <int LB>
__global__ void __launch_bounds__(256) k_ms_count(const uint32_t* __restrict__ keys, uint64_t n, uint32_t shift,
                                                  uint32_t* __restrict__ tile_counts, uint64_t ntiles) {
    constexpr int NB = 1 << LB;
    const int lane = threadIdx.x & 31;
    const uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (tile >= ntiles)
        return;
    uint32_t cnt[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b)
        cnt[b] = 0;
    const uint64_t base = tile * kMsRows * 32;
#pragma unroll 4
    for (int r = 0; r < kMsRows; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        const uint32_t key = valid ? __ldg(keys + i) : 0u;
        const uint32_t label = (key >> shift) & (NB - 1);
        uint32_t mk[NB];
        bucket_masks<LB>(label, mk);
        const uint32_t vm = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
        for (int b = 0; b < NB; ++b)
            cnt[b] += __popc(mk[b] & vm);
    }
    if (lane < NB) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
            if (b == lane)
                v = cnt[b];
        tile_counts[(uint64_t)lane * ntiles + tile] = v;  // bucket-major
    }
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

template <int LB>
__global__ void __launch_bounds__(256) k_ms_scatter(const uint32_t* __restrict__ keys, uint64_t n, uint32_t shift,
                                                    const uint64_t* __restrict__ offsets, uint64_t ntiles,
                                                    uint32_t* __restrict__ out) {
    constexpr int NB = 1 << LB;
    const int lane = threadIdx.x & 31;
    const uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (tile >= ntiles)
        return;
    uint64_t pos[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b)
        pos[b] = offsets[(uint64_t)b * ntiles + tile];
    const uint32_t below = (1u << lane) - 1u;
    const uint64_t base = tile * kMsRows * 32;
#pragma unroll 4
    for (int r = 0; r < kMsRows; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        const uint32_t key = valid ? __ldg(keys + i) : 0u;
        const uint32_t label = (key >> shift) & (NB - 1);
        uint32_t mk[NB];
        bucket_masks<LB>(label, mk);
        const uint32_t vm = __ballot_sync(0xFFFFFFFFu, valid);
        uint64_t dst = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const uint32_t m = mk[b] & vm;
            if ((uint32_t)b == label)
                dst = pos[b] + __popc(m & below);
            pos[b] += __popc(m);
        }
        if (valid)
            out[dst] = key;
    }
}

}  // namespace dmmdev

namespace {
using namespace dmmhost;

template <int LB>
dmm_status run_multisplit(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t* out, uint64_t* starts,
                          void* workspace, cudaStream_t s) {
    constexpr int NB = 1 << LB;
    const uint64_t ntiles = (n + dmmdev::kMsRows * 32 - 1) / (dmmdev::kMsRows * 32);
    const uint64_t total = ntiles * NB;
    const uint64_t nblocks = (total + dmmdev::kScanBlock - 1) / dmmdev::kScanBlock;
    uint32_t* tile_counts = static_cast<uint32_t*>(workspace);
    uint64_t* offsets = reinterpret_cast<uint64_t*>(
        static_cast<char*>(workspace) + ((total * sizeof(uint32_t) + 255) & ~uint64_t(255)));
    uint64_t* block_sums = offsets + ((total + 31) & ~uint64_t(31));
    const unsigned warps_per_block = 8;
    const uint64_t grid = (ntiles + warps_per_block - 1) / warps_per_block;
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
    dmmdev::k_ms_scatter<LB><<<unsigned(grid), warps_per_block * 32, 0, s>>>(keys, n, shift, offsets, ntiles, out);
    if (dmm_status e = check_launch("k_ms_scatter"); e != DMM_OK)
        return e;
    if (starts) {
        // bucket b starts where its tile 0 writes: offsets[b * ntiles] (bucket-major scan)
        cudaMemcpy2DAsync(starts, sizeof(uint64_t), offsets, ntiles * sizeof(uint64_t), sizeof(uint64_t), NB,
                          cudaMemcpyDeviceToDevice, s);
        if (cudaGetLastError() != cudaSuccess)
            return check_launch("bucket starts copy");
    }
    return DMM_OK;
}

}  // namespace

extern "C" {

uint64_t dmm_multisplit_workspace_bytes(uint64_t n, uint32_t nbuckets) {
    const uint64_t ntiles = (n + dmmdev::kMsRows * 32 - 1) / (dmmdev::kMsRows * 32);
    const uint64_t total = ntiles * nbuckets;
    const uint64_t nblocks = (total + dmmdev::kScanBlock - 1) / dmmdev::kScanBlock;
    return ((total * 4 + 255) & ~uint64_t(255)) + ((total + 31) & ~uint64_t(31)) * 8 + nblocks * 8 + 256;
}

dmm_status dmm_multisplit(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t nbuckets, uint32_t* out,
                          uint64_t* bucket_starts, void* workspace, void* stream) {
    reset_launches();
    if (n == 0)
        return DMM_OK;
    if (!keys || !out || !workspace)
        return DMM_INVALID_ARGUMENT;
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

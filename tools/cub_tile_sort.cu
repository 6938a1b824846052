// cub_tile_sort.cu -- comparison point for cfg3 (NOT a product path): the same 2^20 tiles of
// 4096 uint32 keys sorted per CTA by CUB's block-level sorts (radix and merge), which read and
// write shared memory at data-dependent addresses.  Prints G keys/s per variant (CUDA events,
// inputs > L2, 3 warm-up launches) and verifies one tile.
//   make -C tools cub_tile_sort && gpurun -- 'tools/cub_tile_sort'
#include <cub/block/block_load.cuh>
#include <cub/block/block_merge_sort.cuh>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_store.cuh>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kTile = 4096;

template <int THREADS, int ITEMS, int RADIX_BITS>
__global__ void __launch_bounds__(THREADS) k_cub_radix(const uint32_t* in, uint32_t* out) {
    using Load = cub::BlockLoad<uint32_t, THREADS, ITEMS, cub::BLOCK_LOAD_TRANSPOSE>;
    using Sort = cub::BlockRadixSort<uint32_t, THREADS, ITEMS, cub::NullType, RADIX_BITS>;
    using Store = cub::BlockStore<uint32_t, THREADS, ITEMS, cub::BLOCK_STORE_TRANSPOSE>;
    __shared__ union {
        typename Load::TempStorage load;
        typename Sort::TempStorage sort;
        typename Store::TempStorage store;
    } tmp;
    uint32_t k[ITEMS];
    const uint64_t base = uint64_t(blockIdx.x) * kTile;
    Load(tmp.load).Load(in + base, k);
    __syncthreads();
    Sort(tmp.sort).Sort(k);
    __syncthreads();
    Store(tmp.store).Store(out + base, k);
}

struct Less {
    __device__ bool operator()(uint32_t a, uint32_t b) const { return a < b; }
};

template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_cub_merge(const uint32_t* in, uint32_t* out) {
    using Load = cub::BlockLoad<uint32_t, THREADS, ITEMS, cub::BLOCK_LOAD_TRANSPOSE>;
    using Sort = cub::BlockMergeSort<uint32_t, THREADS, ITEMS>;
    using Store = cub::BlockStore<uint32_t, THREADS, ITEMS, cub::BLOCK_STORE_TRANSPOSE>;
    __shared__ union {
        typename Load::TempStorage load;
        typename Sort::TempStorage sort;
        typename Store::TempStorage store;
    } tmp;
    uint32_t k[ITEMS];
    const uint64_t base = uint64_t(blockIdx.x) * kTile;
    Load(tmp.load).Load(in + base, k);
    __syncthreads();
    Sort(tmp.sort).Sort(k, Less());
    __syncthreads();
    Store(tmp.store).Store(out + base, k);
}

__global__ void k_fill(uint32_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t x = i + 0x9e3779b97f4a7c15ull;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        p[i] = uint32_t((x ^ (x >> 31)) >> 32);
    }
}

template <class K>
void run(const char* name, K kern, int threads, const uint32_t* din, uint32_t* dout, uint64_t tiles) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w)
        kern<<<unsigned(tiles), threads>>>(din, dout);
    cudaEventRecord(a);
    const int steps = 10;
    for (int s = 0; s < steps; ++s)
        kern<<<unsigned(tiles), threads>>>(din, dout);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= steps;
    std::vector<uint32_t> hin(kTile), hout(kTile);
    cudaMemcpy(hin.data(), din + 777 * kTile, kTile * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hout.data(), dout + 777 * kTile, kTile * 4, cudaMemcpyDeviceToHost);
    std::sort(hin.begin(), hin.end());
    const bool ok = hin == hout && cudaGetLastError() == cudaSuccess;
    const double keys = double(tiles) * kTile;
    std::printf("%-34s %8.3f ms  %7.1f G keys/s  %5.1f %% of 6533 GB/s  %s\n", name, ms, keys / ms / 1e6,
                100.0 * keys * 8 / (ms / 1e3) / 6533e9, ok ? "ok" : "WRONG");
}

int main() {
    const uint64_t tiles = 1ull << 20, n = tiles * kTile;
    uint32_t *din = nullptr, *dout = nullptr;
    if (cudaMalloc(&din, n * 4) != cudaSuccess || cudaMalloc(&dout, n * 4) != cudaSuccess) {
        std::printf("cudaMalloc failed\n");
        return 1;
    }
    k_fill<<<4096, 256>>>(din, n);
    cudaDeviceSynchronize();
    std::printf("2^20 tiles x 4096 uint32 keys (2^32 keys), one CTA per tile\n");
    run("cub BlockRadixSort 256x16 r4", k_cub_radix<256, 16, 4>, 256, din, dout, tiles);
    run("cub BlockRadixSort 256x16 r6", k_cub_radix<256, 16, 6>, 256, din, dout, tiles);
    run("cub BlockRadixSort 512x8 r5", k_cub_radix<512, 8, 5>, 512, din, dout, tiles);
    run("cub BlockRadixSort 128x32 r4", k_cub_radix<128, 32, 4>, 128, din, dout, tiles);
    run("cub BlockMergeSort 256x16", k_cub_merge<256, 16>, 256, din, dout, tiles);
    run("cub BlockMergeSort 128x32", k_cub_merge<128, 32>, 128, din, dout, tiles);
    cudaFree(din);
    cudaFree(dout);
    return 0;
}

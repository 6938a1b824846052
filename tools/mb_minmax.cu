// Micro-benchmark: throughput of packed 16-bit compare-exchange on the ALU pipe
// (VIMNMX.U16x2) vs the FMA pipe candidate (HMNMX2 on half2 bit patterns), alone and
// interleaved; plus a bit-exactness check of HMNMX2 on u16 patterns < 0x7C00
// (fp16 denormals included).   nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ void cx_i(uint32_t& a, uint32_t& b) {
    uint32_t lo = __vminu2(a, b), hi = __vmaxu2(a, b); a = lo; b = hi;
}
__device__ __forceinline__ void cx_h(uint32_t& a, uint32_t& b) {
    __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b);
    __half2 lo = __hmin2(x, y), hi = __hmax2(x, y);
    a = *reinterpret_cast<uint32_t*>(&lo); b = *reinterpret_cast<uint32_t*>(&hi);
}

template <int MODE>
__global__ void k(uint32_t* out, int iters) {
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = (threadIdx.x * 2654435761u + i * 40503u) & 0x3BFF3BFFu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) cx_i(x[i], x[15 - i]);
            else if (MODE == 1) cx_h(x[i], x[15 - i]);
            else { if (i & 1) cx_h(x[i], x[15 - i]); else cx_i(x[i], x[15 - i]); }
        }
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (MODE == 0) cx_i(x[i], x[i + 1]);
            else if (MODE == 1) cx_h(x[i], x[i + 1]);
            else { if (i & 2) cx_h(x[i], x[i + 1]); else cx_i(x[i], x[i + 1]); }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s ^= x[i] * (i + 1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void check(const uint32_t* a, const uint32_t* b, uint32_t* bad, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t x = a[i], y = b[i], p = x, q = y, r = x, s = y;
    cx_i(p, q); cx_h(r, s);
    if (p != r || q != s) atomicAdd(bad, 1u);
}

int main() {
    uint32_t* out; cudaMalloc(&out, 148 * 32 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    const char* names[3] = {"VIMNMX.U16x2 (alu)", "HMNMX2 (half2)", "interleaved"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = 2.0 * 16 * iters * (double)blocks * threads / 32;  // warp-level min+max instructions
            if (rep) printf("%-22s %.3f ms  %.2f warp-minmax/clk/SM (at 1.965 GHz)\n", names[mode], ms,
                            ops / (ms * 1e-3) / 1.965e9 / 148);
        }
    }
    // exhaustive-ish check over u16 patterns < 0x7C00 in both halves
    const int n = 1 << 24;
    uint32_t *a, *b, *bad; cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&bad, 4);
    uint64_t st = 88172645463325252ull;
    for (int i = 0; i < n; ++i) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        uint32_t lo = (uint32_t)(st % 0x7C00), hi = (uint32_t)((st >> 32) % 0x7C00);
        uint32_t lo2 = (uint32_t)((st >> 16) % 0x7C00), hi2 = (uint32_t)((st >> 40) % 0x7C00);
        if (i < 0x7C00) { lo = i; lo2 = (i * 7) % 0x7C00; hi = i % 64; hi2 = (i / 64) % 64; }
        a[i] = lo | (hi << 16); b[i] = lo2 | (hi2 << 16);
    }
    *bad = 0;
    check<<<n / 256, 256>>>(a, b, bad, n);
    cudaDeviceSynchronize();
    printf("HMNMX2 vs VIMNMX.U16x2 mismatches over %d pairs: %u\n", n, *bad);
    return 0;
}

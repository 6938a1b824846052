// Micro-benchmark: compare-exchange throughput per pipe on sm_100a.
//   IMNMX.U32 (alu), VIMNMX.U16x2 (alu), HMNMX2 (fp16x2), DMNMX on (u32, 0) register pairs
//   (fp64 pipe; a u32 key zero-extended is a non-negative fp64 denormal, ordered like the
//   integer), and interleavings.  Also checks bit-exactness of the DMNMX / HMNMX2 orders.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_pipes mb_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ void cx_u32(uint32_t& a, uint32_t& b) { uint32_t l = min(a, b), h = max(a, b); a = l; b = h; }
__device__ __forceinline__ void cx_u16(uint32_t& a, uint32_t& b) { uint32_t l = __vminu2(a, b), h = __vmaxu2(a, b); a = l; b = h; }
__device__ __forceinline__ void cx_h2(uint32_t& a, uint32_t& b) {
    __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b);
    __half2 l = __hmin2(x, y), h = __hmax2(x, y);
    a = *reinterpret_cast<uint32_t*>(&l); b = *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void cx_f64(uint32_t& a, uint32_t& b) {
    double x = __hiloint2double(0, (int)a), y = __hiloint2double(0, (int)b);
    double l = fmin(x, y), h = fmax(x, y);
    a = (uint32_t)__double2loint(l); b = (uint32_t)__double2loint(h);
}

__constant__ uint32_t c_one = 1u, c_neg = 0xFFFFFFFFu;
// max(a, b) = a + b - min(a, b) exactly (mod 2^32; also per 16-bit half of a packed pair):
// two IMADs on the FMA pipe instead of a second min/max on the ALU pipe
__device__ __forceinline__ void cx_mix(uint32_t& a, uint32_t& b) {
    uint32_t l = min(a, b), s, h;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(a), "r"(c_one), "r"(b));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h) : "r"(l), "r"(c_neg), "r"(s));
    a = l; b = h;
}
__device__ __forceinline__ void cx_mix16(uint32_t& a, uint32_t& b) {
    uint32_t l = __vminu2(a, b), s, h;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(a), "r"(c_one), "r"(b));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h) : "r"(l), "r"(c_neg), "r"(s));
    a = l; b = h;
}
// max(a, b) = a ^ b ^ min(a, b): one LOP3 on the ALU pipe (is it full rate?)
__device__ __forceinline__ void cx_lop(uint32_t& a, uint32_t& b) {
    uint32_t l = min(a, b), h;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(h) : "r"(a), "r"(b), "r"(l));
    a = l; b = h;
}
// MODE: 0 u32, 1 u16x2, 2 h2, 3 f64, 4 u32+f64 interleaved, 5 u16x2+h2 interleaved, 6 u16x2+h2+f64? (u32 semantic n/a)
template <int MODE>
__device__ __forceinline__ void cx(uint32_t& a, uint32_t& b, int i) {
    if (MODE == 0) cx_u32(a, b);
    if (MODE == 1) cx_u16(a, b);
    if (MODE == 2) cx_h2(a, b);
    if (MODE == 3) cx_f64(a, b);
    if (MODE == 4) { if (i & 1) cx_f64(a, b); else cx_u32(a, b); }
    if (MODE == 5) { if (i & 1) cx_h2(a, b); else cx_u16(a, b); }
    if (MODE == 6) { if (i % 3 == 0) cx_f64(a, b); else cx_u32(a, b); }
    if (MODE == 7) cx_mix(a, b);
    if (MODE == 8) { if (i % 3 == 0) cx_u32(a, b); else cx_mix(a, b); }
    if (MODE == 9) { if (i % 3 == 0) cx_u16(a, b); else cx_mix16(a, b); }
    if (MODE == 10) { if (i % 2 == 0) cx_u32(a, b); else cx_mix(a, b); }
    if (MODE == 11) cx_lop(a, b);
    if (MODE == 12) { if (i % 2 == 0) cx_lop(a, b); else cx_mix(a, b); }
    if (MODE == 13) { if (i % 3 == 0) cx_lop(a, b); else cx_mix(a, b); }
    if (MODE == 14) { if (i % 4 == 0) cx_u32(a, b); else if (i % 4 == 1) cx_lop(a, b); else cx_mix(a, b); }
}

template <int MODE>
__global__ void k(uint32_t* out, int iters) {
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = (threadIdx.x * 2654435761u + i * 40503u) & 0x3BFF3BFFu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) cx<MODE>(x[i], x[15 - i], i);
#pragma unroll
        for (int i = 0; i < 16; i += 2) cx<MODE>(x[i], x[i + 1], i / 2);
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s ^= x[i] * (i + 1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void check(const uint32_t* a, const uint32_t* b, uint32_t* bad, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t x = a[i], y = b[i];
    { uint32_t p = x, q = y, r = x, s = y; cx_u32(p, q); cx_f64(r, s); if (p != r || q != s) atomicAdd(bad, 1u); }
    { uint32_t p = x, q = y, r = x, s = y; cx_u32(p, q); cx_mix(r, s); if (p != r || q != s) atomicAdd(bad + 2, 1u); }
    { uint32_t p = x, q = y, r = x, s = y; cx_u32(p, q); cx_lop(r, s); if (p != r || q != s) atomicAdd(bad + 4, 1u); }
    { uint32_t p = x, q = y, r = x, s = y; cx_u16(p, q); cx_mix16(r, s); if (p != r || q != s) atomicAdd(bad + 3, 1u); }
    { uint32_t p = x & 0x7BFF7BFFu, q = y & 0x7BFF7BFFu, r = p, s = q; cx_u16(p, q); cx_h2(r, s);
      if (p != r || q != s) atomicAdd(bad + 1, 1u); }
}

template <int MODE>
void run(const char* name, uint32_t* out) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k<MODE><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    double cxs = 16.0 * iters * (double)blocks * threads / 32;  // warp-level compare-exchanges
    printf("%-28s %.3f ms  %.3f warp-cx/clk/SM (at 1.965 GHz)\n", name, ms, cxs / (ms * 1e-3) / 1.965e9 / 148);
}

int main() {
    uint32_t* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
    run<0>("IMNMX u32", out);
    run<1>("VIMNMX.U16x2", out);
    run<2>("HMNMX2", out);
    run<3>("DMNMX (u32,0)", out);
    run<4>("u32 + DMNMX 1:1", out);
    run<6>("u32 + DMNMX 2:1", out);
    run<5>("U16x2 + HMNMX2 1:1", out);
    run<7>("u32 min + 2 IMAD max", out);
    run<8>("u32: 1 pure : 2 IMAD-max", out);
    run<10>("u32: 1 pure : 1 IMAD-max", out);
    run<9>("U16x2: 1 pure : 2 IMAD-max", out);
    run<11>("u32 min + LOP3 max", out);
    run<12>("u32: 1 LOP3-max : 1 IMAD-max", out);
    run<13>("u32: 1 LOP3-max : 2 IMAD-max", out);
    run<14>("u32: 1 pure:1 LOP3:2 IMAD", out);
    const int n = 1 << 24;
    uint32_t *a, *b, *bad; cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&bad, 32);
    uint64_t st = 88172645463325252ull;
    for (int i = 0; i < n; ++i) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        a[i] = (uint32_t)st; b[i] = (uint32_t)(st >> 32);
        if (i < 65536) { a[i] = i; b[i] = (i * 40503u) & 0xFFFF; }
        if (i >= 65536 && i < 131072) { a[i] = 0xFFFFFFFFu - (i & 0xFF); b[i] = i; }
    }
    bad[0] = bad[1] = bad[2] = bad[3] = bad[4] = 0;
    check<<<n / 256, 256>>>(a, b, bad, n);
    cudaDeviceSynchronize();
    printf("mismatches over %d pairs: DMNMX vs u32 %u, HMNMX2 vs U16x2 (< 0x7C00) %u, IMAD-max u32 %u, IMAD-max u16x2 %u, LOP3-max u32 %u\n", n, bad[0], bad[1], bad[2], bad[3], bad[4]);
    return 0;
}

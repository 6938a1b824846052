// Micro-benchmark / counter check: the production conflict-free relayouts (dmm_device.cuh)
// with and without concurrent global-memory traffic, to read ncu's two bank-conflict
// counters side by side:
//   mode 0: 1024 transposes of a 32 x 32 register block, no global traffic in the loop
//   mode 1: the same loop, plus a streaming global load + store per iteration
// ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,
//     l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,
//     derived__memory_l1_wavefronts_shared_excessive,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum ./mb_relayout
#include <cstdio>
#include <cstdint>
#include "../paper_1507_01391_b200/csrc/dmm_device.cuh"

using namespace dmmdev;

template <int MODE>
__global__ void __launch_bounds__(256) k(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int iters) {
    __shared__ __align__(16) uint32_t smem[8 * 1152];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* buf = smem + warp * relayout_buf_words(32);
    uint32_t x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c)
        x[c] = threadIdx.x * 32 + c;
    using V = VF<0xFFFFFFFFu, 0, 1, 32, 0, 32>;
    const uint64_t gw = (uint64_t)blockIdx.x * 8 + warp;
    for (int it = 0; it < iters; ++it) {
        transpose_blocks<V>(x, buf, lane);
        if (MODE == 1) {
            const uint4* q = reinterpret_cast<const uint4*>(in) + ((gw * 97 + it) % 4096) * 256 + lane;
            const uint4 t = __ldg(q);
            x[0] ^= t.x;
            x[1] ^= t.y;
            reinterpret_cast<uint4*>(out)[((gw * 89 + it) % 4096) * 256 + lane] = make_uint4(x[2], x[3], x[4], x[5]);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c)
        s += x[c];
    out[(uint64_t)blockIdx.x * 256 + threadIdx.x] ^= s;
}

int main() {
    uint32_t *in, *out;
    cudaMalloc(&in, 4096ull * 256 * 16);
    cudaMalloc(&out, 4096ull * 256 * 16);
    cudaMemset(in, 1, 4096ull * 256 * 16);
    cudaMemset(out, 0, 4096ull * 256 * 16);
    k<0><<<148 * 4, 256>>>(in, out, 1024);
    k<1><<<148 * 4, 256>>>(in, out, 1024);
    printf("done: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

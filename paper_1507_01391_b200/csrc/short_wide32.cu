// short_wide32.cu -- kernel 1 at the paper's native mapping: the w = 32 short-wide machine
// (w^2 <= m; here 32 x 1024 = 32 768 keys per instance), Lemma 1 / Corollary
// (partition.hpp:178-185, sort.hpp:200-230): two passes of {alternating row sort;
// to_column_major; row sort; to_row_major} and a final row sort.  Serves
// partition_short_wide, sort_short_wide, the ShortWideHook probe, and partition_general /
// integer_sort_general / sort_wide_any at 32 x 1024 (their leaf is this skeleton,
// partition.hpp:156-172, sort.hpp:321-330).
//
// Mapping: one machine per CTA of 32 warps (persistent over the batch).
//   * DMM processor / bank r = lane r of every warp.  Thread (k, r) = warp k, lane r holds 32
//     keys of row r in registers, so a warp-wide shared access touches 32 different rows, and
//     every row-local structure is stored bank = row: conflict-free by construction.
//   * to_column_major / to_row_major (layout.hpp:316-405) of a 32 x 1024 machine move element
//     (i, 32a + b) to (b, 32i + a) and back.  With warp k holding row positions 32k..32k+31
//     (chunk layout) before to_column_major and 32j + k (stride layout) before to_row_major,
//     both conversions are one 32 x 32 transpose INSIDE warp k: lane i's register b <-> lane
//     b's register i (padded per-warp slab: conflict-free).
//   * Row sorts of labels (domain <= 32: partition_short_wide, partition_general and
//     integer_sort_general with a small domain) are the reference's radix rows, one counting
//     pass each (radix_sort_rows partition.hpp:37-99 with base m >= domain): per-bank
//     counting -- thread (k, r) counts its 32 keys into its own counters in bank r --, the
//     row's histogram summed over its 32 threads, the exclusive prefix of row r in bank r, and
//     each thread emitting the keys of its row positions from the prefix.  The keys are the
//     labels, so the counting sort's scatter writes runs.
//   * Row sorts of full 32-bit keys (sort_short_wide's merge rows sort.hpp:76, integer sorts
//     with a larger domain) are a bitonic sort of the 1024-key row across its 32 threads:
//     stages on position bits held in registers run in registers, the others after a row
//     exchange through shared memory (position e of row r at word 32e + r: bank r).
//   * HBM -> shared memory: one TMA bulk copy of the 128 KB machine (cp.async.bulk +
//     mbarrier), issued for the next machine as soon as the current one stops reading shared
//     memory (its final row sort's count phase), after an L2 prefetch of it at the start of the
//     current machine.  Threads read the row-major staging copy at (row r, column 32j + c)
//     with c = (k + r) mod 32: bank c, distinct across every warp.  The result leaves from
//     the registers (chunk layout: row r, columns 32k .. 32k + 31, 16-byte stores).
#include <algorithm>
#include <cstdlib>

#include "general_kernel.cuh"

namespace dmmdev {
namespace sw32 {

constexpr int kM = 1024;                  // row width
constexpr int kWords = 32 * kM;           // machine words
constexpr uint32_t kBytes = kWords * 4;   // 128 KB
constexpr int kSlab = 32 * 33;            // per-warp transpose slab (padded rows)
constexpr int kStage = 32 * kSlab;        // staging / exchange / counters / slabs (>= kWords)
constexpr int kPre = 2 * 32 * 32;         // row run tables E[l * 32 + r], NX[l * 32 + r]
constexpr size_t kSmemBytes = size_t(kStage + kPre) * 4 + 16;

// to_column_major / to_row_major on this mapping: lane i's register b <-> lane b's register i
// inside the warp (slab row b padded to 33 words: the store hits bank (b + i) mod 32, the load
// bank (i' + b) mod 32)
__device__ __forceinline__ void warp_transpose(uint32_t (&x)[32], uint32_t* slab, int lane) {
#pragma unroll
    for (int b = 0; b < 32; ++b)
        slab[b * 33 + lane] = x[b];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 32; ++i)
        x[i] = slab[lane * 33 + i];
    __syncwarp();
}

// Counting row sort (radix_sort_rows with one pass, partition.hpp:37-99): thread (k, r)
// emits row r's sorted keys at its chunk positions 32k .. 32k + 31.  desc: the row descends
// (SortOrder), i.e. it is the ascending run sequence of the complemented labels 31 - l.
// Keys are < 32 (clamped by the caller).  `after_count` runs once S is no longer read (the
// caller may start the next machine's TMA load into S there).
//
// Per row r the run tables live in bank r: E[l] = end of run l (row order), NX[l] = (n << 16) |
// E[n] for the next non-empty run n after l.  A thread finds the run holding its first
// position by binary search on E, then walks its 32 consecutive positions: a position crosses
// at most one run boundary (runs on the walk are non-empty), so the walk is a compare, two
// selects and a predicated table load per key -- no divergent loop.
template <class AfterCount>
__device__ __forceinline__ void count_row_sort(uint32_t (&x)[32], uint32_t* S, uint32_t* E, uint32_t* NX, int k, int r,
                                               bool desc, AfterCount&& after_count) {
    uint32_t* cnt = S + k * kM + r;  // this thread's counters cnt[32 l]: bank r
    __syncthreads();                 // S and the tables are free (the previous phase is done)
#pragma unroll
    for (int l = 0; l < 32; ++l)
        cnt[l * 32] = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j)
        atomicAdd(cnt + x[j] * 32, 1u);
    __syncthreads();
    // label k's count in row r: sum over the row's 32 threads (the count matrix transposed:
    // thread (k, r) reads column k of row r's counters, all in bank r)
    uint32_t h = 0;
    const uint32_t* col = S + k * 32 + r;
#pragma unroll
    for (int kk = 0; kk < 32; ++kk)
        h += col[kk * kM];
    E[k * 32 + r] = h;
    __syncthreads();
    after_count();
    if (k == 0) {
        // run ends and next-non-empty links of row r, in the row's order
        uint32_t t[32];
#pragma unroll
        for (int l = 0; l < 32; ++l)
            t[l] = E[(desc ? 31 - l : l) * 32 + r];
        uint32_t sum = 0;
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            sum += t[l];
            t[l] = sum;  // end of run l
            E[l * 32 + r] = sum;
        }
        uint32_t nxt = (32u << 16) | kM;
#pragma unroll
        for (int l = 31; l >= 0; --l) {
            NX[l * 32 + r] = nxt;
            const uint32_t start = l ? t[l - 1] : 0u;
            if (t[l] > start)
                nxt = ((uint32_t)l << 16) | t[l];
        }
    }
    __syncthreads();
    const uint32_t base = 32u * (uint32_t)k;
    const uint32_t* er = E + r;
    const uint32_t* nr = NX + r;
    int cur = 0;  // first run whose end exceeds base
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1)
        if (er[(cur + s - 1) * 32] <= base)
            cur += s;
    uint32_t e = er[cur * 32];
    uint32_t jn = nr[cur * 32];
    const uint32_t dm = desc ? 31u : 0u;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t cross = base + j >= e ? 1u : 0u;
        cur = cross ? (int)(jn >> 16) : cur;
        e = cross ? (jn & 0xFFFFu) : e;
        // predicated table load (no branch): only a crossing lane reads its next link
        asm("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.u32 %0, [%1];\n}\n"
            : "+r"(jn)
            : "r"(sptr(nr + cur * 32)), "r"(cross));
        x[j] = (uint32_t)cur ^ dm;
    }
}

// Four label machines per CTA (kModePartition / small-domain integer sorts): byte b of every
// register belongs to machine b (labels < 32 fit a byte), so the warp transposes and the row
// exchanges move four keys per word, four independent run walks give the emit four-fold ILP,
// and the CTA barriers are shared by four machines.  Thread (k, r) counts machine b's label l
// into byte b of its counter word cnt[l] (a thread holds at most 32 keys of a row: a byte
// suffices); the row totals add the four bytes in 16-bit lanes (even / odd bytes), and warp b
// (b < 4) builds machine b's run tables.  Same schedule, per machine, as count_row_sort.
constexpr int kTab4 = 4 * 2 * 32 * 32;  // E and NX tables of the four machines
#ifndef DMM_SW32_EVICT_FIRST
#define DMM_SW32_EVICT_FIRST 1
#endif
constexpr bool kStoreEvictFirst = DMM_SW32_EVICT_FIRST;  // results leave L2 first (the next group's
                                                          // inputs were prefetched there)
constexpr int kSplit = 4;               // bulk copies per machine load / store (32 KB each; 1 vs 16: no
                                        // measurable difference, 183 vs 181 G keys/s)
template <class AfterCount>
__device__ __forceinline__ void count_row_sort4(uint32_t (&x)[32], uint32_t* S, uint32_t* T, int k, int r, bool desc,
                                                AfterCount&& after_count) {
    uint32_t* cnt = S + k * kM + r;  // this thread's counters cnt[32 l]: bank r, byte b = machine b
    __syncthreads();
#pragma unroll
    for (int l = 0; l < 32; ++l)
        cnt[l * 32] = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
            atomicAdd(cnt + ((x[j] >> (8 * b)) & 31u) * 32, 1u << (8 * b));
    }
    __syncthreads();
    // label k's count in row r of each machine: the row's 32 threads' bytes, summed in 16-bit
    // lanes (at most 1024 per machine)
    uint32_t ev = 0, od = 0;
    const uint32_t* col = S + k * 32 + r;
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) {
        const uint32_t w = col[kk * kM];
        ev += w & 0x00FF00FFu;
        od += (w >> 8) & 0x00FF00FFu;
    }
    T[(0 * 2) * 1024 + k * 32 + r] = ev & 0xFFFFu;
    T[(1 * 2) * 1024 + k * 32 + r] = od & 0xFFFFu;
    T[(2 * 2) * 1024 + k * 32 + r] = ev >> 16;
    T[(3 * 2) * 1024 + k * 32 + r] = od >> 16;
    __syncthreads();
    after_count();
    if (k < 4) {
        // machine k's run ends E and next-non-empty links NX of row r, in the row's order
        uint32_t* E = T + (k * 2) * 1024;
        uint32_t* NX = E + 1024;
        uint32_t t[32];
#pragma unroll
        for (int l = 0; l < 32; ++l)
            t[l] = E[(desc ? 31 - l : l) * 32 + r];
        uint32_t sum = 0;
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            sum += t[l];
            t[l] = sum;
            E[l * 32 + r] = sum;
        }
        uint32_t nxt = (32u << 16) | kM;
#pragma unroll
        for (int l = 31; l >= 0; --l) {
            NX[l * 32 + r] = nxt;
            const uint32_t start = l ? t[l - 1] : 0u;
            if (t[l] > start)
                nxt = ((uint32_t)l << 16) | t[l];
        }
    }
    __syncthreads();
    const uint32_t base = 32u * (uint32_t)k;
    const uint32_t dm = desc ? 31u : 0u;
    // two machines' walks at a time (register budget: 32 keys + two walk states)
#pragma unroll
    for (int b0 = 0; b0 < 4; b0 += 2) {
        int cur[2];
        uint32_t e[2], jn[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t* er = T + ((b0 + q) * 2) * 1024 + r;
            int c = 0;  // first run whose end exceeds base
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1)
                if (er[(c + s - 1) * 32] <= base)
                    c += s;
            cur[q] = c;
            e[q] = er[c * 32];
            jn[q] = er[1024 + c * 32];
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            uint32_t v = b0 == 0 ? 0u : x[j];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t cross = base + j >= e[q] ? 1u : 0u;
                cur[q] = cross ? (int)(jn[q] >> 16) : cur[q];
                e[q] = cross ? (jn[q] & 0xFFFFu) : e[q];
                asm("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.u32 %0, [%1];\n}\n"
                    : "+r"(jn[q])
                    : "r"(sptr(T + ((b0 + q) * 2 + 1) * 1024 + r + cur[q] * 32)), "r"(cross));
                v |= ((uint32_t)cur[q] ^ dm) << (8 * (b0 + q));
            }
            x[j] = v;
        }
    }
}

// row exchanges through S (position e of row r at word 32e + r): chunk (e = 32k + j) <->
// stride (e = 32j + c)
__device__ __forceinline__ void chunk_to_stride(uint32_t (&x)[32], uint32_t* S, int k, int r, int c) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j)
        S[k * kM + j * 32 + r] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j)
        x[j] = S[c * 32 + r + j * kM];
}
__device__ __forceinline__ void stride_to_chunk(uint32_t (&x)[32], uint32_t* S, int k, int r) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j)
        S[k * 32 + r + j * kM] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j)
        x[j] = S[k * kM + j * 32 + r];
}

// one bitonic merge level L (6..10) of the 1024-key row sort, entered and left in chunk layout
template <int L>
__device__ __forceinline__ void bitonic_level(uint32_t (&x)[32], uint32_t* S, int k, int r) {
    chunk_to_stride(x, S, k, r, k);
    // stride: position bits L-1..5 = register bits L-6..0; block direction = position bit L
    // = register bit L-5 (the last level ascends)
    reg_stages<1, 0, 32, L - 6, (L < 10 ? L - 5 : -1)>(x);
    stride_to_chunk(x, S, k, r);
    // chunk: position bits 4..0 = register bits; direction = position bit L = warp bit L-5
    const uint32_t f = (L < 10 && ((k >> (L - 5)) & 1)) ? 0xFFFFFFFFu : 0u;
    flip<0, 32>(x, f);
    reg_stages<1, 0, 32, 4, -1>(x);
    flip<0, 32>(x, f);
}

// comparison row sort of row r (1024 keys over the row's 32 threads), chunk layout in and out
__device__ __forceinline__ void bitonic_row_sort(uint32_t (&x)[32], uint32_t* S, int k, int r, bool desc) {
    const uint32_t fr = desc ? 0xFFFFFFFFu : 0u;  // x ^ ~0 reverses the order
    const uint32_t f0 = (k & 1) ? 0xFFFFFFFFu : 0u;
    flip<0, 32>(x, fr ^ f0);
    sort_net<1, 0, 32>(x);  // levels 1..5: the thread's 32 positions, direction = warp bit 0
    flip<0, 32>(x, f0);
    bitonic_level<6>(x, S, k, r);
    bitonic_level<7>(x, S, k, r);
    bitonic_level<8>(x, S, k, r);
    bitonic_level<9>(x, S, k, r);
    bitonic_level<10>(x, S, k, r);
    flip<0, 32>(x, fr);
}

// The row sort that follows to_column_major needs only the merge levels.  The conversion
// leaves new row b's chunk j (positions 32j .. 32j+31) = the sorted old row j's positions
// 32k + b, k = 0..31, in the stride layout (thread (k, b), register j holds position 32j + k)
// -- exactly the layout bitonic_level<6> reaches after its first exchange -- and the
// alternating row sort before it sorted old rows 2i and 2i+1 in opposite directions, so every
// 64-position block is already a bitonic sequence (also after the complement of a descending
// sort).  Levels 1..5 and level 6's first exchange are skipped; the outcome is the sorted row.
// DMM_SW32_FULLROWS=1 runs the full row sort there instead (A/B).
#ifndef DMM_SW32_FULLROWS
#define DMM_SW32_FULLROWS 0
#endif
__device__ __forceinline__ void merge_runs_row_sort(uint32_t (&x)[32], uint32_t* S, int k, int r, bool desc) {
    const uint32_t fr = desc ? 0xFFFFFFFFu : 0u;
    flip<0, 32>(x, fr);
    // level 6 from its stride half: position bit 5 = register bit 0, direction = bit 6 = register bit 1
    reg_stages<1, 0, 32, 0, 1>(x);
    stride_to_chunk(x, S, k, r);
    const uint32_t f = ((k >> 1) & 1) ? 0xFFFFFFFFu : 0u;  // position bit 6 = warp bit 1
    flip<0, 32>(x, f);
    reg_stages<1, 0, 32, 4, -1>(x);
    flip<0, 32>(x, f);
    bitonic_level<7>(x, S, k, r);
    bitonic_level<8>(x, S, k, r);
    bitonic_level<9>(x, S, k, r);
    bitonic_level<10>(x, S, k, r);
    flip<0, 32>(x, fr);
}

// to_row_major straight from a row sort's chunk layout: new row i gathers chunk i of every old
// row k (positions 32i + j), which thread (i, k) holds; thread (k, i) takes it through S in one
// exchange (word 1024 j + 32 i + ((k + i) mod 32): the writers of one warp and the readers of
// one warp each see 32 distinct banks).  Thread (k, i) register j then holds new row i's
// position 32j + k (the stride layout) -- and, read as a chunk-layout row, chunk k is old row
// k's sorted chunk i.  Odd warps take their chunk reversed, so chunk pairs are bitonic.
__device__ __forceinline__ void row_exchange(uint32_t (&x)[32], uint32_t* S, int k, int r) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j)
        S[j * kM + k * 32 + ((r + k) & 31)] = x[j];
    __syncthreads();
    const bool rev = (k & 1) != 0;
#pragma unroll
    for (int j = 0; j < 32; ++j)
        x[j] = S[(rev ? 31 - j : j) * kM + r * 32 + ((k + r) & 31)];
}
// the row sort that follows row_exchange: chunk layout in (bitonic chunk pairs), merge levels
// 6..10 only, chunk layout out
__device__ __forceinline__ void merge_chunks_row_sort(uint32_t (&x)[32], uint32_t* S, int k, int r, bool desc) {
    const uint32_t fr = desc ? 0xFFFFFFFFu : 0u;
    flip<0, 32>(x, fr);
    bitonic_level<6>(x, S, k, r);
    bitonic_level<7>(x, S, k, r);
    bitonic_level<8>(x, S, k, r);
    bitonic_level<9>(x, S, k, r);
    bitonic_level<10>(x, S, k, r);
    flip<0, 32>(x, fr);
}

// a ShortWideHook snapshot of the machine from the registers, row-major into dst:
// stride = false: thread (k, r) holds row r positions 32k + j; true: positions 32j + c
__device__ __forceinline__ void snap(uint32_t* dst, const uint32_t (&x)[32], int k, int r, bool stride, int c) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
        dst[r * kM + (stride ? 32 * j + c : 32 * k + j)] = x[j];
}

// COUNT: label row sorts (domain <= 32); else comparison row sorts.  Partition semantics
// (check_partition_instance partition.hpp:112-124) for MODE partition and for the probe of
// partition_short_wide (sort-any with domain w); otherwise keys >= domain are KeyOutOfRange.
template <bool COUNT, int MODE>
__global__ void __launch_bounds__(1024, 1)
    k_short_wide32(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t count, uint64_t domain,
                   int ascending, dmm_general_stats* __restrict__ stats, uint8_t* __restrict__ status,
                   uint32_t* __restrict__ probe, int pf) {
    extern __shared__ __align__(128) uint32_t smem[];
    uint32_t* S = smem;
    uint32_t* E = smem + kStage;
    uint32_t* NX = E + 32 * 32;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kStage + kPre);
    const int tid = threadIdx.x, k = tid >> 5, r = tid & 31;
    const bool asc = ascending != 0;
    const bool part = MODE == kModePartition || (MODE == kModeSortAny && domain < (1ull << 32));
    const int c = (k + r) & 31;  // rotated stride column: bank c on the row-major staging copy
    uint32_t* slab = S + k * kSlab;
    if (tid == 0) {
        mbar_init(bar);
        if (blockIdx.x < count)
            tma_load(S, in + (uint64_t)blockIdx.x * kWords, kBytes, bar);
    }
    __syncthreads();
    uint32_t parity = 0;
    for (uint64_t inst = blockIdx.x; inst < count; inst += gridDim.x) {
        const uint64_t nxt = inst + gridDim.x;
        if (pf && tid == 0 && nxt < count)  // DMM_SW32_SORT_PF (default 1)
            prefetch_l2(in + nxt * kWords, kBytes);
        // the next machine's load into S, once this machine no longer reads S
        auto load_next = [&]() {
            if (tid == 0 && nxt < count) {
                fence_async_smem();
                tma_load(S, in + nxt * kWords, kBytes, bar);
            }
        };
        mbar_wait(bar, parity);
        parity ^= 1;
        uint32_t x[32];
        {
            const uint32_t* src = S + r * kM + c;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                x[j] = src[32 * j];
        }
        // keys outside [0, domain); labels are clamped to 31 for the counters
        uint32_t bad = 0;
        if (domain < (1ull << 32)) {
            const uint32_t d = (uint32_t)domain;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                bad |= x[j] >= d ? 1u : 0u;
                if constexpr (COUNT)
                    x[j] = min(x[j], 31u);
            }
        }
        bad = __syncthreads_or(bad);  // (also: every thread has read its staging words)
        uint32_t* snaps = probe != nullptr ? probe + inst * 3 * kWords : nullptr;
        auto nothing = []() {};

        for (int pass = 0; pass < 2; ++pass) {
            // alternating row sort (SortOrder::alternating(asc)), chunk layout out
            const bool desc_alt = ((r & 1) == 0) != asc;
            if constexpr (COUNT)
                count_row_sort(x, S, E, NX, k, r, desc_alt, nothing);
            else if (!DMM_SW32_FULLROWS && pass == 1)
                merge_chunks_row_sort(x, S, k, r, desc_alt);  // after row_exchange
            else
                bitonic_row_sort(x, S, k, r, desc_alt);
            __syncthreads();  // S -> slabs
            warp_transpose(x, slab, r);  // to_column_major
            if (pass == 0 && snaps)
                snap(snaps, x, k, r, true, k);  // after_first_convert: row r, positions 32j + k
            // row sort (asc or desc) into the stride layout to_row_major takes
            if constexpr (COUNT)
                count_row_sort(x, S, E, NX, k, r, !asc, nothing);
            else if constexpr (DMM_SW32_FULLROWS)
                bitonic_row_sort(x, S, k, r, !asc);
            else
                merge_runs_row_sort(x, S, k, r, !asc);
            if constexpr (COUNT || DMM_SW32_FULLROWS) {
                chunk_to_stride(x, S, k, r, k);
                __syncthreads();
                warp_transpose(x, slab, r);  // to_row_major: chunk layout out
                if (pass == 0 && snaps)
                    snap(snaps + kWords, x, k, r, false, 0);  // after_first_pass
            } else {
                row_exchange(x, S, k, r);  // to_row_major: stride layout, odd warps reversed
                if (pass == 0 && snaps) {
                    // after_first_pass: register j holds position 32j + k (32 (31 - j) + k reversed)
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        snaps[kWords + r * kM + 32 * ((k & 1) ? 31 - j : j) + k] = x[j];
                }
            }
        }
        // final row sort, chunk layout; the next machine streams into S meanwhile
        if constexpr (COUNT) {
            count_row_sort(x, S, E, NX, k, r, !asc, load_next);
        } else {
            if constexpr (DMM_SW32_FULLROWS)
                bitonic_row_sort(x, S, k, r, !asc);
            else
                merge_chunks_row_sort(x, S, k, r, !asc);  // after row_exchange
            __syncthreads();
            load_next();
        }
        if (snaps)
            snap(snaps + 2 * kWords, x, k, r, false, 0);  // done
        uint32_t mism = 0;
        if (part) {
            // labels in [0, w) with m copies each <=> the sorted machine has row i = i
#pragma unroll
            for (int j = 0; j < 32; ++j)
                mism |= x[j] ^ (uint32_t)r;
        }
        store_row<32>(out + inst * kWords + r * kM + 32 * k, x);
        const uint32_t invalid = __syncthreads_or(mism != 0) | bad;
        if (tid == 0) {
            uint8_t st = DMM_OK;
            if (part && invalid)
                st = DMM_INVALID_INSTANCE;
            else if (bad)
                st = DMM_KEY_OUT_OF_RANGE;
            if (status)
                status[inst] = st;
            if (stats) {
                stats[inst].cleanup_retries = 0;  // w <= m: partition_leaf only
                stats[inst].sorted = 1;
            }
        }
    }
}

// The label machines, four per CTA (count_row_sort4): partition_short_wide, partition_general /
// integer_sort_general with domain <= 32 and the partition's ShortWideHook probe.  Persistent
// over groups of four machines (an L2 prefetch of the next group, DMM_SW32_PF=4, measured
// slower and read 1.6-1.8x the input bytes from DRAM: 148 SMs x 512 KB of prefetched inputs
// beside the streaming results overflow L2 before the bulk loads arrive; off by default); machines move between HBM / L2 and the
// shared staging copy by TMA bulk copies, one at a time (the staging copy is 128 KB).
template <int MODE, bool DIRECT = false, bool PROBE = true>
__global__ void __launch_bounds__(1024, 1)
    k_short_wide32_labels(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t count,
                          uint64_t domain, int ascending, dmm_general_stats* __restrict__ stats,
                          uint8_t* __restrict__ status, uint32_t* __restrict__ probe, int pf) {
    extern __shared__ __align__(128) uint32_t smem[];
    uint32_t* S = smem;
    uint32_t* T = smem + kStage;
    uint32_t* F = T + kTab4;  // four flag words: two per task parity
    uint64_t* bar = reinterpret_cast<uint64_t*>(F + 4);
    const int tid = threadIdx.x, k = tid >> 5, r = tid & 31;
    const int c = (k + r) & 31;  // rotated stride column: bank c on the row-major staging copy
    const bool asc = ascending != 0;
    const bool part = MODE == kModePartition || (MODE == kModeSortAny && domain < (1ull << 32));
    uint32_t* slab = S + k * kSlab;
    const uint32_t d = domain < 32 ? (uint32_t)domain : 32u;
    if (tid < 4)
        F[tid] = 0;
    if (tid == 0)
        mbar_init(bar);
    __syncthreads();
    uint32_t parity = 0, bpar = 0;
    for (uint64_t m0 = (uint64_t)blockIdx.x * 4; m0 < count; m0 += (uint64_t)gridDim.x * 4, parity ^= 1) {
        const uint64_t nx = m0 + (uint64_t)gridDim.x * 4;
        // L2 prefetch of the first pf machines of this CTA's next group (DMM_SW32_PF, default 0)
        if (tid < pf && nx + tid < count)
            prefetch_l2(in + (nx + tid) * kWords, kBytes);
        uint32_t x[32];
        uint32_t bad = 0;
        if constexpr (DIRECT) {
            // ingest: the first row sort's outcome does not depend on the order inside a row, so
            // thread (k, r) takes row r's positions 32k .. 32k+31 straight from global memory
            // (8 x 16-byte loads; a warp reads 32 full 128-byte segments, from L2: prefetched a
            // group ago) -- no staging copy, no CTA barrier; byte b = machine b
#pragma unroll 1
            for (int b = 0; b < 4; ++b) {
                const uint64_t inst = m0 + b;
                const uint4* q = reinterpret_cast<const uint4*>(in + inst * kWords + r * kM + 32 * k);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint4 t = inst < count ? __ldg(q + i) : make_uint4(0, 0, 0, 0);
                    const uint32_t v4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t v = v4[e];
                        bad |= v >= d ? (1u << b) : 0u;
                        const uint32_t cv = min(v, 31u) << (8 * b);
                        x[4 * i + e] = b == 0 ? cv : (x[4 * i + e] | cv);
                    }
                }
            }
        } else {
        // ingest: machine b streams into S by one TMA bulk copy (from L2: prefetched a group
        // ago), every thread takes its row's words (row r, columns 32j + c: bank c) into byte b
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
            const uint64_t inst = m0 + b;
            if (inst < count) {
                if (k == 0) {
                    if (r < kSplit)
                        bulk_wait_read();  // the previous group's last stores have left S
                    __syncwarp();
                    fence_async_smem();
                    tma_load_split(S, in + inst * kWords, kBytes, bar, r, kSplit);
                }
                mbar_wait(bar, bpar);
                bpar ^= 1;
            }
            const uint32_t* src = S + r * kM + c;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t v = inst < count ? src[32 * j] : 0u;
                bad |= v >= d ? (1u << b) : 0u;
                const uint32_t cv = min(v, 31u) << (8 * b);
                x[j] = b == 0 ? cv : (x[j] | cv);
            }
            __syncthreads();  // S is read
        }
        }
        uint32_t* Fb = F + 2 * parity;
        {
            const uint32_t wb = __reduce_or_sync(0xFFFFFFFFu, bad);
            if (r == 0 && wb)
                atomicOr(Fb, wb);
        }
        if (tid == 0)
            F[2 * (parity ^ 1)] = F[2 * (parity ^ 1) + 1] = 0;  // the next group's flags (last read a group ago)
        // PROBE = false: no snapshot code at all (its address arithmetic cost registers, i.e.
        // local-memory spills, in the hot instantiation)
        uint32_t* snaps = PROBE && probe != nullptr ? probe + m0 * 3 * kWords : nullptr;
        auto snap4 = [&](int stage, bool stride) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                if (m0 + b >= count)
                    break;
                uint32_t* dst = snaps + (uint64_t)b * 3 * kWords + (uint64_t)stage * kWords;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    dst[r * kM + (stride ? 32 * j + k : 32 * k + j)] = (x[j] >> (8 * b)) & 0xFFu;
            }
        };
        auto nothing = []() {};

        for (int pass = 0; pass < 2; ++pass) {
            const bool desc_alt = ((r & 1) == 0) != asc;
            count_row_sort4(x, S, T, k, r, desc_alt, nothing);  // chunk layout out
            __syncthreads();
            warp_transpose(x, slab, r);  // to_column_major
            if (PROBE && pass == 0 && snaps)
                snap4(0, true);  // after_first_convert
            count_row_sort4(x, S, T, k, r, !asc, nothing);
            if constexpr (DMM_SW32_FULLROWS) {
                chunk_to_stride(x, S, k, r, k);
                __syncthreads();
                warp_transpose(x, slab, r);  // to_row_major: chunk layout out
                if (PROBE && pass == 0 && snaps)
                    snap4(1, false);  // after_first_pass
            } else {
                // to_row_major as one exchange (the next counting row sort takes any
                // arrangement of its row): stride layout, odd warps' words reversed
                row_exchange(x, S, k, r);
                if (PROBE && pass == 0 && snaps) {  // after_first_pass
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        if (m0 + b >= count)
                            break;
                        uint32_t* dst = snaps + (uint64_t)b * 3 * kWords + kWords;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            dst[r * kM + 32 * ((k & 1) ? 31 - j : j) + k] = (x[j] >> (8 * b)) & 0xFFu;
                    }
                }
            }
        }
        count_row_sort4(x, S, T, k, r, !asc, nothing);
        if (PROBE && snaps)
            snap4(2, false);  // done
        uint32_t mism = 0;
        if (part) {
            uint32_t diff = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                diff |= x[j] ^ ((uint32_t)r * 0x01010101u);
#pragma unroll
            for (int b = 0; b < 4; ++b)
                mism |= ((diff >> (8 * b)) & 0xFFu) ? (1u << b) : 0u;
        }
        if constexpr (DIRECT) {
            // egress: the last row sort leaves the chunk layout (row r, positions 32k + j): each
            // machine's bytes leave by 8 x 16-byte stores per thread (32 full segments per warp)
#pragma unroll 1
            for (int b = 0; b < 4; ++b) {
                const uint64_t inst = m0 + b;
                if (inst >= count)
                    break;
                uint4* q = reinterpret_cast<uint4*>(out + inst * kWords + r * kM + 32 * k);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    q[i] = make_uint4((x[4 * i] >> (8 * b)) & 0xFFu, (x[4 * i + 1] >> (8 * b)) & 0xFFu,
                                      (x[4 * i + 2] >> (8 * b)) & 0xFFu, (x[4 * i + 3] >> (8 * b)) & 0xFFu);
            }
        } else {
        // egress: the rotated stride layout (row r, columns 32j + c) writes the row-major staging
        // copy conflict-free; machine b leaves S by one TMA bulk copy
        chunk_to_stride(x, S, k, r, c);
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
            const uint64_t inst = m0 + b;
            if (inst >= count)
                break;
            if (k == 0 && r < kSplit)
                bulk_wait_read();  // machine b - 1 has left S (each lane waits for its own copies)
            __syncthreads();
            uint32_t* dst = S + r * kM + c;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                dst[32 * j] = (x[j] >> (8 * b)) & 0xFFu;
            fence_async_smem();
            __syncthreads();
            if (k == 0 && r < kSplit) {  // kSplit bulk stores of one group, issued by kSplit lanes
                if (kStoreEvictFirst)
                    tma_store_evict_first(out + inst * kWords + r * (kWords / kSplit), S + r * (kWords / kSplit),
                                          kBytes / kSplit);
                else
                    tma_store(out + inst * kWords + r * (kWords / kSplit), S + r * (kWords / kSplit), kBytes / kSplit);
            }
        }
        }
        {
            const uint32_t wm = __reduce_or_sync(0xFFFFFFFFu, mism);
            if (r == 0 && wm)
                atomicOr(Fb + 1, wm);
        }
        __syncthreads();
        if (tid < 4 && m0 + tid < count) {
            const uint64_t inst = m0 + tid;
            const bool bd = (Fb[0] >> tid) & 1u, inv = bd || ((Fb[1] >> tid) & 1u);
            uint8_t st = DMM_OK;
            if (part && inv)
                st = DMM_INVALID_INSTANCE;
            else if (bd)
                st = DMM_KEY_OUT_OF_RANGE;
            if (status)
                status[inst] = st;
            if (stats) {
                stats[inst].cleanup_retries = 0;  // w <= m: partition_leaf only
                stats[inst].sorted = 1;
            }
        }
    }
    if (!DIRECT && k == 0 && r < kSplit)
        bulk_wait_all();
}

}  // namespace sw32
}  // namespace dmmdev

namespace dmmhost {

namespace {
template <bool COUNT, int MODE>
dmm_status launch_sw32(const GeneralArgs& a) {
    auto kern = dmmdev::sw32::k_short_wide32<COUNT, MODE>;
    static std::atomic<uint64_t> configured{0};
    if (dmm_status e = configure_kernel(kern, dmmdev::sw32::kSmemBytes, configured); e != DMM_OK)
        return e;
    if (a.count == 0)
        return DMM_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t grid = std::min<uint64_t>(a.count, uint64_t(sms));
    static const int pf = getenv("DMM_SW32_SORT_PF") ? atoi(getenv("DMM_SW32_SORT_PF")) : 1;
    kern<<<unsigned(grid), 1024, dmmdev::sw32::kSmemBytes, a.stream>>>(a.in, a.out, a.count, a.domain, a.ascending,
                                                                       a.stats, a.status, a.probe, pf);
    return check_launch("k_short_wide32");
}
template <int MODE>
dmm_status launch_sw32_labels(const GeneralArgs& a) {
    // ingest / egress through the TMA staging copy (default) or, DMM_SW32_DIRECT=1, by direct
    // 16-byte loads / stores in the chunk layout: measured 125 vs 181 G keys/s on cfg1sw -- a
    // warp's 16-byte accesses to 32 rows 4 KB apart cost 32 L1/L2 requests per instruction,
    // where the bulk copy streams each machine as 4 x 32 KB (profiles/r02/pipeline_ab.txt)
    static const bool direct = getenv("DMM_SW32_DIRECT") && getenv("DMM_SW32_DIRECT")[0] == '1';
    auto kern = direct ? dmmdev::sw32::k_short_wide32_labels<MODE, true>
                       : a.probe ? dmmdev::sw32::k_short_wide32_labels<MODE, false, true>
                                 : dmmdev::sw32::k_short_wide32_labels<MODE, false, false>;
    constexpr size_t smem = size_t(dmmdev::sw32::kStage + dmmdev::sw32::kTab4 + 8) * 4;
    static std::atomic<uint64_t> configured[3];  // per instantiation (static storage: zeroed)
    if (dmm_status e = configure_kernel(kern, smem, configured[direct ? 0 : a.probe ? 1 : 2]); e != DMM_OK)
        return e;
    if (a.count == 0)
        return DMM_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t grid = std::min<uint64_t>((a.count + 3) / 4, uint64_t(sms));
    // DMM_SW32_PF=n: L2-prefetch n machines of the next group (0 default: 198.6 vs 183.6 G keys/s
    // with 4, DRAM reads 1.00x vs 1.63x the input; profiles/r02/pipeline_ab.txt)
    static const int pf = getenv("DMM_SW32_PF") ? atoi(getenv("DMM_SW32_PF")) : 0;
    kern<<<unsigned(grid), 1024, smem, a.stream>>>(a.in, a.out, a.count, a.domain, a.ascending, a.stats, a.status,
                                                   a.probe, pf);
    return check_launch("k_short_wide32_labels");
}
}  // namespace

// 32 x 1024 machines: every entry point's leaf is the short-wide skeleton (w^2 <= m)
dmm_status launch_general_m1024(int mode, bool /*pk2*/, bool ext, const GeneralArgs& a) {
    if (ext) {
        set_error("extension kernels are only built where the reference rejects the shape");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (a.probe && a.probe_max != 3) {
        set_error("32 x 1024 machines capture the three ShortWideHook stages only");
        return DMM_INVALID_ARGUMENT;
    }
    // label machines (domain <= 32): four per CTA; DMM_SW32_SINGLE=1 runs them one per CTA
    static const bool single = getenv("DMM_SW32_SINGLE") && getenv("DMM_SW32_SINGLE")[0] == '1';
    const bool count = a.domain <= 32;
    if (count && !single) {
        switch (mode) {
            case dmmdev::kModePartition: return launch_sw32_labels<dmmdev::kModePartition>(a);
            case dmmdev::kModeIntegerSort: return launch_sw32_labels<dmmdev::kModeIntegerSort>(a);
            default: return launch_sw32_labels<dmmdev::kModeSortAny>(a);
        }
    }
    switch (mode) {
        case dmmdev::kModePartition:
            return launch_sw32<true, dmmdev::kModePartition>(a);
        case dmmdev::kModeIntegerSort:
            return count ? launch_sw32<true, dmmdev::kModeIntegerSort>(a)
                         : launch_sw32<false, dmmdev::kModeIntegerSort>(a);
        default:
            return count ? launch_sw32<true, dmmdev::kModeSortAny>(a) : launch_sw32<false, dmmdev::kModeSortAny>(a);
    }
}

}  // namespace dmmhost

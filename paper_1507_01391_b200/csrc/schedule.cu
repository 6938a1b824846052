// schedule.cu -- offline conflict-free schedules for fixed permutations.
//
// dmm_offline_schedule   Schedule offline_schedule(W, M, perm)      layout.hpp:207-230
//                        (host precompute, as in the reference: Euler splitting of the
//                        M-regular bank-to-bank transfer multigraph, layout.hpp:104-143, plus
//                        one Kuhn matching peel per odd degree, :146-184, recursion :186-205)
// dmm_apply_schedule     apply_schedule(view, schedule, dst_base)   layout.hpp:246-263
//
// The host side reproduces the reference's decomposition move for move (same rounds, same
// order inside each round), so a schedule computed here is interchangeable with one the
// reference computed or loaded from its text form.
//
// On the device one warp applies the schedule to one w-row machine (w <= 32): the machine's
// cell (bank b, offset o) lives at shared word o * 32 + b, i.e. DMM bank b IS physical bank b.
// A round's moves have pairwise distinct source banks and pairwise distinct destination banks
// (Schedule::validate), so each round is one conflict-free LDS and one conflict-free STS per
// lane -- the DMM round costs exactly two shared-memory wavefronts.  The schedule is staged in
// shared memory once per CTA (packed 8-bit fields) and validated there before any instance is
// touched; CTAs are persistent over the instance batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <vector>

#include "capi_common.h"

namespace dmmdev {

constexpr int kSchedWarps = 4;
constexpr uint32_t kSchedMaxW = 32, kSchedMaxM = 64;
constexpr uint32_t kSchedMaxMoves = 8192, kSchedMaxRounds = 8192;
constexpr uint32_t kCovWords = kSchedMaxW * kSchedMaxM / 32;

// per-warp shared words: A and B (m * 32 each) + the staging window (32 rows of sk words)
// (the staging window is only live before the rounds, so it shares its words with B)
__host__ __device__ constexpr uint32_t sched_warp_words(uint32_t m) {
    return m * 32 + (m * 32 > 32 * ((m & 1) ? m : m + 1) ? m * 32 : 32 * ((m & 1) ? m : m + 1));
}

// smem: packed moves [n_moves] | round starts [n_rounds + 1] | coverage bitmap | per-warp A, B, S
// MT > 0: the machine width as a compile-time constant (powers of two up to 64: strides,
// divisions and the row loops fold); MT = 0: any width <= 64 at run time.
template <uint32_t MT>
__global__ void __launch_bounds__(kSchedWarps * 32)
    k_apply_schedule(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t w, uint32_t m_rt,
                     uint64_t count, const uint32_t* __restrict__ moves, const uint32_t* __restrict__ round_start,
                     uint32_t n_rounds, uint32_t n_moves, uint8_t* __restrict__ status) {
    const uint32_t m = MT ? MT : m_rt;
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t bad, dup, ragged;
    // the shared layout is sized from the host's n_moves: round_start must agree with it (starts
    // at 0, monotone, ends at n_moves) before anything is staged or any move is read
    {
        uint32_t off = 0;
        for (uint32_t i = threadIdx.x; i <= n_rounds; i += blockDim.x) {
            const uint32_t v = round_start[i];
            off |= (i == 0 && v != 0) || (i == n_rounds && v != n_moves) || v > n_moves ||
                   (i < n_rounds && round_start[i + 1] < v);
        }
        if (__syncthreads_or(off)) {
            if (blockIdx.x == 0 && threadIdx.x == 0)
                status[0] = (uint8_t)DMM_OUT_OF_BOUNDS;
            return;
        }
    }
    uint32_t* sched = sm;
    uint32_t* rs = sched + n_moves;
    uint32_t* cov = rs + n_rounds + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* A = cov + kCovWords + warp * sched_warp_words(m);  // the machine (bank b = bank b)
    uint32_t* B = A + m * 32;                                     // the destination window
    uint32_t* S = B;                                              // skewed staging window (input only)
    if (tid == 0) {
        bad = 0;
        dup = 0;
        ragged = 0;
    }
    for (uint32_t i = tid; i < kCovWords; i += blockDim.x)
        cov[i] = 0;
    __syncthreads();
    // stage + validate: bounds (OutOfBounds), coverage (bijective => no read-back of out)
    for (uint32_t i = tid; i < n_moves; i += blockDim.x) {
        const uint4 mv = reinterpret_cast<const uint4*>(moves)[i];
        if (mv.x >= w || mv.y >= m || mv.z >= w || mv.w >= m) {
            atomicMax(&bad, (uint32_t)DMM_OUT_OF_BOUNDS);
            continue;
        }
        sched[i] = mv.x | (mv.y << 8) | (mv.z << 16) | (mv.w << 24);
        const uint32_t cell = mv.z * m + mv.w;
        if (atomicOr(&cov[cell >> 5], 1u << (cell & 31)) & (1u << (cell & 31)))
            dup = 1;
    }
    for (uint32_t i = tid; i <= n_rounds; i += blockDim.x) {
        rs[i] = round_start[i];
        if (i < n_rounds && (round_start[i + 1] < round_start[i] || round_start[i + 1] - round_start[i] > w))
            atomicMax(&bad, (uint32_t)DMM_CONFLICT_VIOLATION);  // a round of more than w moves reuses a bank
        if (i < n_rounds && round_start[i] != i * w)
            ragged = 1;
    }
    __syncthreads();
    if (bad == 0) {
        // ConflictViolation: a round reusing a source or destination bank (Schedule::validate)
        for (uint32_t r = warp; r < n_rounds; r += kSchedWarps) {
            const uint32_t s = rs[r], len = rs[r + 1] - s;
            const bool act = (uint32_t)lane < len;
            const uint32_t mv = act ? sched[s + lane] : 0u;
            const uint32_t amask = __ballot_sync(0xFFFFFFFFu, act);
            const uint32_t sb = act ? (mv & 0xFF) : 0xFFFFFFFFu - lane, db = act ? ((mv >> 16) & 0xFF) : 0xFFFFFFFFu - lane;
            // both votes by every lane (a short-circuit || would diverge around the second)
            const uint32_t same_src = __match_any_sync(0xFFFFFFFFu, sb) & amask;
            const uint32_t same_dst = __match_any_sync(0xFFFFFFFFu, db) & amask;
            const bool clash = (__popc(same_src) > 1) | (__popc(same_dst) > 1);
            if (__any_sync(0xFFFFFFFFu, act && clash) && lane == 0)
                atomicMax(&bad, (uint32_t)DMM_CONFLICT_VIOLATION);
        }
    }
    __syncthreads();
    if (bad) {
        if (blockIdx.x == 0 && tid == 0)
            status[0] = (uint8_t)bad;
        return;
    }
    const bool bijective = dup == 0 && n_moves == w * m;
    const bool regular = bijective && ragged == 0 && n_rounds * w == n_moves;
    const bool row = (uint32_t)lane < w;
    // global -> machine goes through a skewed staging window (cell (r, c) at r * sk + c, sk
    // odd): the global side moves the instance's w*m words coalesced (lane-consecutive), and a
    // lane reading its own row r from the staging window hits bank (r * sk + c) mod 32,
    // distinct across rows -- so every shared access of the kernel is conflict-free or nearly
    const uint32_t n = w * m, sk = (m & 1) ? m : m + 1;
    const uint32_t dq = 32 / m, dr = 32 % m;  // a 32-word step: dq rows + dr columns
    const uint32_t r0 = lane / m, c0 = lane % m;
    // full-warp machines of compile-time width (the common case): word t = lane + 32 j of an
    // instance lands in the staging window at a lane base plus a compile-time offset per j, and
    // the next instance's words are loaded into registers while this one runs its rounds
    constexpr uint32_t kM = MT ? MT : 1, kSK = (kM & 1) ? kM : kM + 1;
    const bool fast = MT != 0 && w == 32;
    const uint32_t base = kM >= 32 ? lane : (lane / kM) * kSK + lane % kM;
    const uint64_t stride = (uint64_t)gridDim.x * kSchedWarps;
    uint64_t k = (uint64_t)blockIdx.x * kSchedWarps + warp;
    uint32_t pre[kM];
    if (fast && k < count) {
#pragma unroll
        for (uint32_t j = 0; j < kM; ++j)
            pre[j] = in[k * n + lane + 32 * j];
    }
    for (; k < count; k += stride) {
        const uint32_t* src = in + k * n;
        uint32_t* dst = out + k * n;
        if (fast) {
#pragma unroll
            for (uint32_t j = 0; j < kM; ++j)
                S[base + (32 * j / kM) * kSK + (32 * j) % kM] = pre[j];
            if (k + stride < count) {
#pragma unroll
                for (uint32_t j = 0; j < kM; ++j)
                    pre[j] = in[(k + stride) * n + lane + 32 * j];
            }
        } else {
            uint32_t t = lane, c = c0, a = r0 * sk + c0;
            while (t < n) {
                uint32_t v[8], at[8];
                uint32_t cnt = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (t < n) {
                        v[j] = src[t];
                        at[j] = a;
                        ++cnt;
                    }
                    t += 32;
                    c += dr;
                    a += dq * sk + dr;
                    if (c >= m) {
                        c -= m;
                        a += sk - m;
                    }
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((uint32_t)j < cnt)
                        S[at[j]] = v[j];
            }
        }
        __syncwarp();
        if (row)
            for (uint32_t c = 0; c < m; ++c)
                A[c * 32 + lane] = S[lane * sk + c];
        __syncwarp();  // S is B's storage
        if (row && !bijective)  // cells no move writes keep out's contents
            for (uint32_t c = 0; c < m; ++c)
                B[c * 32 + lane] = dst[lane * m + c];
        __syncwarp();
        // the rounds: reads only touch A, writes only B
        if (regular) {
            // offline_schedule's shape: m rounds of exactly w moves onto distinct cells -- no
            // ordering between rounds, so they overlap freely
            if (row) {
#pragma unroll 4
                for (uint32_t r = 0; r < n_rounds; ++r) {
                    const uint32_t mv = sched[r * w + lane];
                    B[(mv >> 24) * 32 + ((mv >> 16) & 0xFF)] = A[((mv >> 8) & 0xFF) * 32 + (mv & 0xFF)];
                }
            }
        } else {
            // a later round's write to the same cell wins (sequential execution)
            for (uint32_t r = 0; r < n_rounds; ++r) {
                const uint32_t s = rs[r];
                if ((uint32_t)lane < rs[r + 1] - s) {
                    const uint32_t mv = sched[s + lane];
                    B[(mv >> 24) * 32 + ((mv >> 16) & 0xFF)] = A[((mv >> 8) & 0xFF) * 32 + (mv & 0xFF)];
                }
                __syncwarp();
            }
        }
        __syncwarp();
        // lane r writes row r straight from B (stores do not stall; L2 merges the sectors)
        if (row) {
            uint32_t* d = dst + lane * m;
            if ((m & 3) == 0) {
                for (uint32_t c = 0; c < m; c += 4)
                    *reinterpret_cast<uint4*>(d + c) = make_uint4(B[c * 32 + lane], B[(c + 1) * 32 + lane],
                                                                  B[(c + 2) * 32 + lane], B[(c + 3) * 32 + lane]);
            } else {
                for (uint32_t c = 0; c < m; ++c)
                    d[c] = B[c * 32 + lane];
            }
        }
        __syncwarp();
    }
}

}  // namespace dmmdev

namespace {

using namespace dmmhost;

// One transfer of the bank-to-bank multigraph: cell (src, soff) -> cell (dst, doff).
struct Transfer {
    uint32_t src, dst, soff, doff;
};
using Transfers = std::vector<Transfer>;
using Rounds = std::vector<Transfers>;

// Euler split (layout.hpp:104-143): walk Euler circuits of the bipartite multigraph (banks
// 0..W-1 as sources, W..2W-1 as destinations), vertices in index order and each vertex's
// edges in input order, and deal the circuit's edges alternately to `even` and `odd`.
void split_by_circuits(const Transfers& e, uint32_t W, Transfers& even, Transfers& odd) {
    const uint32_t V = 2 * W, E = uint32_t(e.size());
    std::vector<uint32_t> first(V + 1, 0), slot_edge(2 * size_t(E)), slot_peer(2 * size_t(E));
    for (const Transfer& t : e) {
        ++first[t.src + 1];
        ++first[W + t.dst + 1];
    }
    for (uint32_t v = 0; v < V; ++v)
        first[v + 1] += first[v];
    std::vector<uint32_t> fill(first.begin(), first.end() - 1);
    for (uint32_t i = 0; i < E; ++i) {
        const uint32_t a = e[i].src, b = W + e[i].dst;
        slot_edge[fill[a]] = i;
        slot_peer[fill[a]++] = b;
        slot_edge[fill[b]] = i;
        slot_peer[fill[b]++] = a;
    }
    std::vector<uint8_t> taken(E, 0);
    std::vector<uint32_t> next(first.begin(), first.end() - 1);
    std::vector<uint32_t> walk_v, walk_e, circuit;  // Hierholzer stack: vertex, edge that led to it
    constexpr uint32_t kNone = ~0u;
    for (uint32_t s = 0; s < V; ++s) {
        if (next[s] >= first[s + 1])
            continue;
        circuit.clear();
        walk_v.assign(1, s);
        walk_e.assign(1, kNone);
        while (!walk_v.empty()) {
            const uint32_t v = walk_v.back();
            uint32_t& p = next[v];
            while (p < first[v + 1] && taken[slot_edge[p]])
                ++p;
            if (p == first[v + 1]) {
                if (walk_e.back() != kNone)
                    circuit.push_back(walk_e.back());
                walk_v.pop_back();
                walk_e.pop_back();
            } else {
                taken[slot_edge[p]] = 1;
                walk_v.push_back(slot_peer[p]);
                walk_e.push_back(slot_edge[p]);
            }
        }
        for (size_t i = 0; i < circuit.size(); ++i)
            ((i & 1) ? odd : even).push_back(e[circuit[i]]);
    }
}

// Kuhn matching peel (layout.hpp:146-184): augmenting paths from sources 0..W-1 over each
// source's edges in input order; the matching is emitted by destination bank, the remaining
// edges keep their order.
struct Kuhn {
    const Transfers& e;
    std::vector<std::vector<uint32_t>> out_edges;
    std::vector<int64_t> owner;  // destination bank -> matched edge (-1: free)
    std::vector<uint64_t> seen;
    uint64_t stamp = 0;

    Kuhn(const Transfers& edges, uint32_t W) : e(edges), out_edges(W), owner(W, -1), seen(W, 0) {
        for (uint32_t i = 0; i < edges.size(); ++i)
            out_edges[edges[i].src].push_back(i);
    }
    bool augment(uint32_t s) {
        for (uint32_t id : out_edges[s]) {
            const uint32_t d = e[id].dst;
            if (seen[d] == stamp)
                continue;
            seen[d] = stamp;
            if (owner[d] < 0 || augment(e[owner[d]].src)) {
                owner[d] = id;
                return true;
            }
        }
        return false;
    }
};

bool peel_perfect_matching(Transfers& edges, uint32_t W, Transfers& matching) {
    Kuhn k(edges, W);
    for (uint32_t s = 0; s < W; ++s) {
        ++k.stamp;
        if (!k.augment(s))
            return false;
    }
    std::vector<uint8_t> in_matching(edges.size(), 0);
    for (uint32_t d = 0; d < W; ++d) {
        matching.push_back(edges[k.owner[d]]);
        in_matching[k.owner[d]] = 1;
    }
    Transfers rest;
    rest.reserve(edges.size() - W);
    for (size_t i = 0; i < edges.size(); ++i)
        if (!in_matching[i])
            rest.push_back(edges[i]);
    edges.swap(rest);
    return true;
}

// decompose (layout.hpp:186-205): degree 1 -> one round; odd -> peel a matching round first;
// even -> split and recurse on both halves (first half's rounds first).
bool decompose_rounds(Transfers edges, uint32_t W, uint32_t degree, Rounds& out) {
    while (degree && !edges.empty()) {
        if (degree == 1) {
            out.push_back(std::move(edges));
            return true;
        }
        if (degree & 1) {
            Transfers round;
            if (!peel_perfect_matching(edges, W, round))
                return false;
            out.push_back(std::move(round));
            --degree;
            continue;
        }
        Transfers a, b;
        a.reserve(edges.size() / 2);
        b.reserve(edges.size() / 2);
        split_by_circuits(edges, W, a, b);
        if (!decompose_rounds(std::move(a), W, degree / 2, out))
            return false;
        edges = std::move(b);
        degree /= 2;
    }
    return true;
}

}  // namespace

extern "C" {

dmm_status dmm_offline_schedule(uint32_t w, uint32_t m, const uint32_t* perm, uint32_t* moves) {
    const uint64_t n = uint64_t(w) * m;
    if (n && (!perm || !moves))
        return DMM_INVALID_ARGUMENT;
    std::vector<uint8_t> hit(n, 0);
    Transfers edges;
    edges.reserve(n);
    for (uint32_t r = 0; r < w; ++r)
        for (uint32_t c = 0; c < m; ++c) {
            const uint64_t i = uint64_t(r) * m + c;
            const uint32_t dr = perm[2 * i], dc = perm[2 * i + 1];
            if (dr >= w || dc >= m) {
                set_error("permutation target out of range");
                return DMM_NOT_BIJECTIVE;
            }
            if (hit[uint64_t(dr) * m + dc]++) {
                set_error("permutation target repeated");
                return DMM_NOT_BIJECTIVE;
            }
            edges.push_back({r, dr, c, dc});
        }
    Rounds rounds;
    if (!decompose_rounds(std::move(edges), w, m, rounds)) {
        set_error("matching extraction failed on regular multigraph");
        return DMM_ERROR;
    }
    uint64_t k = 0;
    for (const Transfers& round : rounds)
        for (const Transfer& t : round) {
            moves[4 * k] = t.src;
            moves[4 * k + 1] = t.soff;
            moves[4 * k + 2] = t.dst;
            moves[4 * k + 3] = t.doff;
            ++k;
        }
    return DMM_OK;
}

uint64_t dmm_apply_schedule_smem_bytes(uint32_t m, uint32_t n_moves, uint32_t n_rounds) {
    return sizeof(uint32_t) * (size_t(n_moves) + n_rounds + 1 + dmmdev::kCovWords +
                               size_t(dmmdev::kSchedWarps) * dmmdev::sched_warp_words(m));
}

dmm_status dmm_apply_schedule(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                              const uint32_t* moves, const uint32_t* round_start, uint32_t n_rounds,
                              uint32_t n_moves, uint8_t* status, void* stream) {
    reset_launches();
    if (w == 0 || m == 0 || w > dmmdev::kSchedMaxW || m > dmmdev::kSchedMaxM) {
        set_error("apply_schedule kernels: 1 <= w <= 32, 1 <= m <= 64");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (n_moves > dmmdev::kSchedMaxMoves || n_rounds > dmmdev::kSchedMaxRounds) {
        set_error("apply_schedule: at most 8192 moves and 8192 rounds");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (!round_start || !status || (n_moves && !moves) || (count && (!in || !out)))
        return DMM_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(moves)) &
        15u) {
        set_error("in / out / moves must be 16-byte aligned");
        return DMM_INVALID_ARGUMENT;
    }
    auto kern = m == 8 ? dmmdev::k_apply_schedule<8>
              : m == 16 ? dmmdev::k_apply_schedule<16>
              : m == 32 ? dmmdev::k_apply_schedule<32>
              : m == 64 ? dmmdev::k_apply_schedule<64>
                        : dmmdev::k_apply_schedule<0>;
    const size_t smem = dmm_apply_schedule_smem_bytes(m, n_moves, n_rounds);
    static std::atomic<uint64_t> configured[5];
    const int ki = m == 8 ? 0 : m == 16 ? 1 : m == 32 ? 2 : m == 64 ? 3 : 4;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return check_launch("cudaFuncSetAttribute");
    if (dmm_status e = configure_kernel(kern, 0, configured[ki]); e != DMM_OK)
        return e;
    auto st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(status, 0, 1, st) != cudaSuccess)
        return check_launch("cudaMemsetAsync");
    if (count == 0)
        return DMM_OK;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, dmmdev::kSchedWarps * 32, smem);
    const uint64_t need = (count + dmmdev::kSchedWarps - 1) / dmmdev::kSchedWarps;
    const uint64_t blocks = std::min<uint64_t>(need, uint64_t(sms) * std::max(per_sm, 1));
    kern<<<unsigned(blocks), dmmdev::kSchedWarps * 32, smem, st>>>(in, out, w, m, count, moves, round_start,
                                                                    n_rounds, n_moves, status);
    return check_launch("k_apply_schedule");
}

}  // extern "C"

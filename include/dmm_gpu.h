/* dmm_gpu.h -- C ABI of the B200 (sm_100a) bank-conflict-free DMM kernels.
 *
 * This is the drop-in boundary for the reference's hot path:
 * every entry point replaces one function of /root/reference/proj/include/dmm/*.hpp
 * (cited per declaration) on a BATCH of independent w x m machines.  Plain pointers
 * and sizes only; no torch or CUDA types in the signatures (`stream` is a
 * cudaStream_t passed as void*, NULL = legacy default stream).
 *
 * Data layout (global memory, device pointers):
 *   in / out : count x w x m uint32 words, instance-major, each instance row-major
 *              (the reference's Instance::grid, instance.hpp:44, narrowed to 32 bits).
 *              in == out (in place) is allowed.
 *   stats    : count entries (may be NULL).
 *   status   : count bytes of dmm_status (may be NULL): the per-instance outcome of a
 *              data-dependent failure (PostconditionFailed, InvalidInstance,
 *              KeyOutOfRange).  Where the reference would have thrown, the out
 *              instance is unspecified.
 * Shape contracts are checked on the host with the reference's own predicates
 * before any launch and reported as the return value (ShapeViolation etc.);
 * DMM_UNSUPPORTED_SHAPE means "the reference accepts it but no kernel is built for
 * it" -- there is no CPU fallback.  Launches are asynchronous on `stream`.
 */
#ifndef DMM_GPU_H
#define DMM_GPU_H

#include <stdint.h>

#include "dmm_status.h"

#ifdef __cplusplus
extern "C" {
#endif

/* flags (same values as the oracle's DMMO_FLAG_*) */
#define DMM_FLAG_EXT_PARTIAL_GROUPS 1u /* accept balance() partial groups with g^2 > m (32x8) */
#define DMM_FLAG_NONSTRICT 2u          /* MachineConfig.strict = false: no PostconditionFailed */
#define DMM_FLAG_NO_ENFORCE_PRE 4u     /* integer_sort_general(..., enforce_analysis_pre = false) */

/* GeneralStats partition.hpp:292-295 */
typedef struct dmm_general_stats {
    uint32_t cleanup_retries;
    uint32_t sorted;
} dmm_general_stats;

/* PermuteReport permute.hpp:62-72 (leftover_history and shifts are separate arrays) */
#define DMM_PERMUTE_MAX_HIST 64
typedef struct dmm_permute_report {
    uint32_t iterations;
    uint32_t fallback;
    uint32_t used_packing;
    uint32_t packed_width;
    uint64_t threshold;
    uint64_t random_words;
    uint32_t cleanup_retries;
    uint32_t n_hist;
} dmm_permute_report;

/* ---- library ------------------------------------------------------------- */
const char* dmm_version(void);
/* Last CUDA / launch error text of the calling thread ("" if none). */
const char* dmm_last_error(void);
/* 1 if a kernel is compiled for (w, m) of the named algorithm (see below). */
int dmm_supported(const char* algorithm, uint32_t w, uint32_t m);
/* Number of kernel launches the last call on this thread issued (for bench accounting). */
uint32_t dmm_last_launch_count(void);
/* Machine::steps() the reference meters for run_algorithm on a w x m instance
 * (instance.hpp:357) where it does not depend on the data: the radix leaves of
 * partition_short_wide, partition_square and of partition_general / integer_sort_general with
 * w <= m (short-wide or square skeleton; closed forms in capi.cu).  0 = not modelled (merge
 * segment sorts, cleanup retries and the permutation depend on the data); work = steps * w. */
uint64_t dmm_modelled_steps(const char* algorithm, uint32_t w, uint32_t m);
/* The same meter for the data-dependent leaves of partition_general / integer_sort_general with
 * w <= m (shearsort_rect sort.hpp:288, square skeleton with w < m sort.hpp:250: their blocked
 * column sorts merge-sort bank segments): steps[k] for input instance k (device [count][w][m],
 * keys < domain; domain = w for the partition, w*m for run_algorithm's integer sort).  A
 * replay of the leaf's states on the device (off the hot path); 2 <= w <= 32, m <= 128. */
dmm_status dmm_leaf_steps(const uint32_t* in, uint32_t w, uint32_t m, uint64_t count, uint64_t domain,
                          uint64_t* steps, void* stream);
/* The meter for every shape of partition_general / integer_sort_general the reference accepts,
 * the w > m recursion included (balance_divide_sort partition.hpp:363-428: balancing tower,
 * convert-and-divide, leaves, column recursion, checked cleanup with its retry loop):
 * steps[k] = Machine::steps() and, if retries is not NULL, retries[k] =
 * GeneralStats::cleanup_retries for instance k (device [count][w][m], keys < domain).  Each
 * section is charged the reference's access count over a replay of its states, one thread per
 * instance (off the hot path); w m <= 65536. */
dmm_status dmm_general_steps(const uint32_t* in, uint32_t w, uint32_t m, uint64_t count, uint64_t domain,
                             uint64_t* steps, uint32_t* retries, void* stream);
/* The same meter for the comparison sorts sort_short_wide (sort.hpp:225, w^2 <= m <= 64) and
 * sort_square (sort.hpp:337, w = m = h^2 <= 64): every row sort merge-sorts its banks. */
dmm_status dmm_sort_steps(const char* algorithm, const uint32_t* in, uint32_t w, uint32_t m, uint64_t count,
                          uint64_t* steps, void* stream);

/* ---- instance generation -------------------------------------------------- */
/* Instance gen_instance(kind, w, m, seed)                        instance.hpp:48-76
 * Bit-exact on-device restatement for seeds seed0 .. seed0+count-1 into
 * out[count][w][m].  kind: 0 uint32 sort tile (builder-defined, Rng(splitmix64(seed))()>>32;
 * the reference's sort kind emits 64-bit words), 1 partition, 2 permute.  w*m <= 4096. */
dmm_status dmm_gen_instances(int kind, uint32_t w, uint32_t m, uint64_t seed0, uint64_t count, uint32_t* out,
                             void* stream);

/* cfg5's flat keys (builder-defined counter generator): out[i] = splitmix64(index0 + i) >> 32 */
dmm_status dmm_gen_keys(uint64_t index0, uint64_t n, uint32_t* out, void* stream);

/* ---- partition / integer sort ------------------------------------------ */
/* GeneralStats partition_general(const MatrixView&)           partition.hpp:453-456
 * Labels in [0, w), m copies each; after the call row i holds the labels i. */
dmm_status dmm_partition_general(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                 uint32_t flags, dmm_general_stats* stats, uint8_t* status, void* stream);

/* GeneralStats integer_sort_general(view, domain, probe, enforce)  partition.hpp:436-449 */
dmm_status dmm_integer_sort_general(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                    uint64_t domain, uint32_t flags, dmm_general_stats* stats, uint8_t* status,
                                    void* stream);

/* PartitionProbe capture (partition.hpp:298-301, called at :376-390): the same two calls,
 * additionally writing the full w x m working window after every balance (after_balance)
 * and every convert-and-divide (after_divide) of the outer recursion, in hook order, to
 * snapshots[k * max_snaps * w * m ...] for instance k (max_snaps per instance; extra
 * snapshots are dropped).  dmm_general_probe_snaps(w, m, flags) = the number the recursion
 * takes for that shape (0 when w <= m). */
uint32_t dmm_general_probe_snaps(uint32_t w, uint32_t m, uint32_t flags);
dmm_status dmm_partition_general_probe(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                       uint32_t flags, dmm_general_stats* stats, uint8_t* status, uint32_t* snapshots,
                                       uint32_t max_snaps, void* stream);
dmm_status dmm_integer_sort_general_probe(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                          uint64_t domain, uint32_t flags, dmm_general_stats* stats, uint8_t* status,
                                          uint32_t* snapshots, uint32_t max_snaps, void* stream);

/* ShortWideHook capture (sort.hpp:189-218): partition_short_wide (partition != 0) or
 * sort_short_wide(ascending) run as the literal short-wide skeleton, writing the w x m window at
 * after_first_convert, after_first_pass and done to snapshots[k * 3 * w * m ...]. */
dmm_status dmm_short_wide_probe(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                int partition, int ascending, uint8_t* status, uint32_t* snapshots, void* stream);

/* void partition_square(const MatrixView&)                       partition.hpp:189-197 */
dmm_status dmm_partition_square(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                uint8_t* status, void* stream);

/* void partition_short_wide(const MatrixView&, hook)             partition.hpp:178-185 */
dmm_status dmm_partition_short_wide(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                    uint8_t* status, void* stream);

/* ---- comparison sorts ------------------------------------------------------ */
/* void sort_short_wide(view, ascending)  sort.hpp:225 ; void sort_square(view, ascending)  sort.hpp:337 ;
 * void sort_tall(view)  sort.hpp:352 ; detail::sort_wide_any(view, asc)  sort.hpp:321 */
dmm_status dmm_sort_short_wide(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                               int ascending, void* stream);
dmm_status dmm_sort_square(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                           int ascending, void* stream);
dmm_status dmm_sort_tall(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count, void* stream);
dmm_status dmm_sort_wide_any(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                             int ascending, void* stream);

/* ---- layout primitives and row sorts ---------------------------------------- */
/* transpose_square layout.hpp:24 ; to_column_major layout.hpp:397 ; to_row_major layout.hpp:403 */
dmm_status dmm_transpose_square(const uint32_t* in, uint32_t* out, uint32_t s, uint64_t count, void* stream);
dmm_status dmm_to_column_major(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                               void* stream);
dmm_status dmm_to_row_major(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                            void* stream);
/* radix_sort_rows(view, domain, order) partition.hpp:94 ; sort_rows(view, order) sort.hpp:76
 * order: 0 ascending, 1 descending, 2 alternating (row 0 ascending), 3 alternating (row 0 descending) */
dmm_status dmm_sort_rows(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count, int order,
                         uint64_t domain, uint8_t* status, void* stream);

/* ---- randomized permutation ------------------------------------------------ */
/* PermuteReport permute(Machine&, Rng&, const PermuteParams&)   permute.hpp:545-628
 * in: count x w x m labels (a bijection of [0, wm) each); out: the output region
 * (bank i slot j = i*m + j on success).  seeds[k] seeds instance k's Rng
 * (std::mt19937_64).  reports: count entries; history: count x DMM_PERMUTE_MAX_HIST;
 * shifts: count x w (each may be NULL).  workspace: dmm_permute_workspace_bytes(count). */
uint64_t dmm_permute_workspace_bytes(uint32_t w, uint32_t m, uint64_t count);
/* Same pipeline, each instance's generator given mid-stream instead of by seed:
 * rng_states[k] = 313 words (device memory): the std::mt19937_64 state words _M_x[0..312)
 * and the position _M_p of the next draw (libstdc++ layout; what `os << rng` prints).
 * This is what a drop-in for permute(Machine&, Rng&, params) needs: the caller's engine is
 * continued, then advanced by report.random_words (rng.discard). */
dmm_status dmm_permute_from_state(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                                  const uint64_t* rng_states, uint32_t alpha, uint32_t iter_cap,
                                  dmm_permute_report* reports, uint64_t* history, uint32_t* shifts,
                                  uint8_t* status, void* stream);
dmm_status dmm_permute(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                       const uint64_t* seeds, uint32_t alpha, uint32_t iter_cap, dmm_permute_report* reports,
                       uint64_t* history, uint32_t* shifts, uint8_t* status, void* workspace, void* stream);
/* The permutation's modelled DMM step count, Machine::steps() after permute (what
 * run_algorithm reports, instance.hpp:357): steps[k] (device, count entries) for instance k run
 * with seeds[k] (device) -- the kernel replays every phase's data-dependent cost (shuffle, hash
 * broadcast, rescan / communication / synchronisation per iteration, packing rounds, the
 * three-phase delivery) and the finish's integer_sort_general is metered by
 * dmm_general_steps.  0 where not modelled (a packed sort that exhausted its cleanup
 * retries, the last-resort tall sort).  Off the hot path: allocates, synchronises. */
dmm_status dmm_permute_steps(const uint32_t* in, uint32_t w, uint32_t m, uint64_t count, const uint64_t* seeds,
                             uint32_t alpha, uint32_t iter_cap, uint64_t* steps, void* stream);

/* ---- cfg5: local step of the global w-way partition across GPUs --------------- */
/* Stable partition of n keys by label = (key >> shift) & (nbuckets-1), bucket-major into
 * out; bucket_starts[b] (device, nbuckets entries) = first output index of bucket b.
 * The exchange of bucket j to the GPU owning label j is an NCCL all-to-all
 * (paper_1507_01391_b200/distributed.py).  workspace: dmm_multisplit_workspace_bytes. */
uint64_t dmm_multisplit_workspace_bytes(uint64_t n, uint32_t nbuckets);
dmm_status dmm_multisplit(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t nbuckets, uint32_t* out,
                          uint64_t* bucket_starts, void* workspace, void* stream);

/* The same partition with the exchange fused into the scatter (two calls, one workspace):
 * dmm_multisplit_count writes bucket_starts (device, nbuckets entries: where bucket b would
 * start in a local bucket-major output; the local counts follow) and keeps the per-tile
 * offsets in the workspace; dmm_multisplit_scatter_to then writes bucket b's keys, stable by
 * source index, to dst[b][dst_base[b] ..] -- dst (device array of nbuckets device pointers,
 * e.g. peer GPUs' receive buffers mapped over NVLink) and dst_base (device) come from the
 * caller's count exchange (paper_1507_01391_b200/distributed.py, global_partition_p2p). */
dmm_status dmm_multisplit_count(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t nbuckets,
                                uint64_t* bucket_starts, void* workspace, void* stream);
dmm_status dmm_multisplit_scatter_to(const uint32_t* keys, uint64_t n, uint32_t shift, uint32_t nbuckets,
                                     uint32_t* const* dst, const uint64_t* dst_base, void* workspace,
                                     void* stream);

/* ---- offline schedules for fixed permutations --------------------------------- */
/* Schedule offline_schedule(W, M, perm)                          layout.hpp:207-230
 * Host precompute (no device work), as in the reference.  perm[2*(r*m + c)] / [.. + 1] =
 * destination bank / offset of cell (r, c).  moves: w*m moves of 4 words (src_bank, src_off,
 * dst_bank, dst_off) -- exactly m rounds of w moves, round k = moves[k*w .. (k+1)*w), the
 * reference's rounds move for move.  DMM_NOT_BIJECTIVE on a table that is not a bijection. */
dmm_status dmm_offline_schedule(uint32_t w, uint32_t m, const uint32_t* perm, uint32_t* moves);

/* void apply_schedule(const MatrixView&, const Schedule&, u32 dst_base)   layout.hpp:246-263
 * Applies any schedule (device arrays: moves as above, 16-byte aligned; round r = moves
 * [round_start[r], round_start[r+1]), n_moves = round_start[n_rounds]) to count instances
 * [count][w][m] of in, writing out: out(dst) = in(src) per move, rounds in order.  Cells no
 * move writes keep out's contents.  The schedule is validated on the device before any write:
 * status[0] (device byte) = DMM_OUT_OF_BOUNDS / DMM_CONFLICT_VIOLATION (a round reusing a source
 * or destination bank, Schedule::validate layout.hpp:80-95) or 0.  w <= 32, m <= 64,
 * n_moves, n_rounds <= 8192. */
uint64_t dmm_apply_schedule_smem_bytes(uint32_t m, uint32_t n_moves, uint32_t n_rounds);
dmm_status dmm_apply_schedule(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                              const uint32_t* moves, const uint32_t* round_start, uint32_t n_rounds,
                              uint32_t n_moves, uint8_t* status, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DMM_GPU_H */

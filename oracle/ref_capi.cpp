// ref_capi.cpp -- C ABI over the UNMODIFIED reference headers (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile straight from /root/reference/proj/include (never
// copied) into oracle/_ref/libdmm_ref.so.  Only tests/, __graft_entry__ and
// bench.py's cpu_baseline / --impl reference legs load it: it is the reference
// arm and the pin for the C restatement (oracle/dmm_oracle.c), never the product.
//
// Every entry point goes through the reference's own public API:
// gen_instance / run_algorithm (instance.hpp:48, :277), integer_sort_general
// (partition.hpp:436), permute (permute.hpp:545), the layout primitives
// (layout.hpp:24, :397, :403) and the PartitionProbe hooks (partition.hpp:298).
#include <dmm/dmm.hpp>

#include <atomic>
#include <chrono>
#include <cstring>
#include <sstream>
#include <thread>

#include "../include/dmm_status.h"

using namespace dmm;

namespace {

int status_of_current_exception() {
    try {
        throw;
    } catch (const OverlappingViews&) {
        return DMM_OVERLAPPING_VIEWS;
    } catch (const ShapeViolation&) {
        return DMM_SHAPE_VIOLATION;
    } catch (const InvalidInstance&) {
        return DMM_INVALID_INSTANCE;
    } catch (const KeyOutOfRange&) {
        return DMM_KEY_OUT_OF_RANGE;
    } catch (const DivisibilityViolation&) {
        return DMM_DIVISIBILITY_VIOLATION;
    } catch (const PostconditionFailed&) {
        return DMM_POSTCONDITION_FAILED;
    } catch (const PackingOverflow&) {
        return DMM_PACKING_OVERFLOW;
    } catch (const CapacityExceeded&) {
        return DMM_CAPACITY_EXCEEDED;
    } catch (const NotSquare&) {
        return DMM_NOT_SQUARE;
    } catch (const OutOfBounds&) {
        return DMM_OUT_OF_BOUNDS;
    } catch (...) {
        return DMM_ERROR;
    }
}

Algorithm alg_of(int a) { return static_cast<Algorithm>(a); }

}  // namespace

extern "C" {

struct dmmr_run_report {
    uint64_t steps;
    uint64_t work;
    uint64_t conflicts;
    uint32_t correct;
    uint32_t iterations;
    uint32_t fallback;
    uint32_t cleanup_retries;
};

struct dmmr_permute_report {
    uint32_t iterations;
    uint32_t fallback;
    uint32_t used_packing;
    uint32_t packed_width;
    uint64_t threshold;
    uint64_t random_words;
    uint32_t cleanup_retries;
    uint32_t n_hist;
    uint64_t leftover_history[64];
};

void dmmr_gen_instance(int kind, uint32_t w, uint32_t m, uint64_t seed, uint64_t* grid) {
    Instance in = gen_instance(static_cast<InstanceKind>(kind), w, m, seed);
    std::memcpy(grid, in.grid.data(), sizeof(uint64_t) * in.grid.size());
}

// run_algorithm on an explicit grid (kind inferred from the algorithm).
// out_grid: final working window (sort / partition) or the output region (permute).
int dmmr_run_algorithm(int alg, uint32_t w, uint32_t m, uint64_t seed, const uint64_t* grid, int strict,
                       uint64_t* out_grid, dmmr_run_report* rep, dmmr_permute_report* prep,
                       uint32_t* shifts) {
    try {
        Instance in;
        in.kind = instance_kind_for(alg_of(alg));
        in.w = w;
        in.m = m;
        in.seed = seed;
        in.grid.assign(grid, grid + u64(w) * m);
        RunOptions opt;
        opt.strict = strict != 0;
        opt.host_threads = 1;
        RunOutcome o = run_algorithm(alg_of(alg), in, opt);
        rep->steps = o.report.steps;
        rep->work = o.report.work;
        rep->conflicts = o.report.conflicts;
        rep->correct = o.report.correct;
        rep->iterations = o.report.iterations;
        rep->fallback = o.report.fallback;
        rep->cleanup_retries = o.report.cleanup_retries;
        if (prep) {
            const PermuteReport& p = o.pipeline;
            prep->iterations = p.iterations;
            prep->fallback = p.fallback;
            prep->used_packing = p.used_packing;
            prep->packed_width = p.packed_width;
            prep->threshold = p.threshold;
            prep->random_words = p.random_words;
            prep->cleanup_retries = p.cleanup_retries;
            prep->n_hist = static_cast<uint32_t>(std::min<std::size_t>(64, p.leftover_history.size()));
            for (uint32_t i = 0; i < prep->n_hist; ++i)
                prep->leftover_history[i] = p.leftover_history[i];
            if (shifts)
                for (std::size_t i = 0; i < p.shifts.size(); ++i)
                    shifts[i] = p.shifts[i];
        }
        // re-run the final-state snapshot: run_algorithm does not return it, so
        // replay deterministically on a fresh machine for the grid
        if (out_grid) {
            Machine mach(MachineConfig::standard(w, m, opt.strict));
            const auto& cfg = mach.config();
            std::vector<u32> all_rows(w);
            for (u32 r = 0; r < w; ++r)
                all_rows[r] = r;
            MatrixView v = MatrixView::full(mach);
            MatrixView vp = MatrixView::make(mach, all_rows, cfg.work_base(), m, cfg.scratch_a_base(),
                                             cfg.scratch_b_base());
            const Algorithm a = alg_of(alg);
            (a == Algorithm::permute || a == Algorithm::integer_sort_general ? vp : v).load(in.grid);
            switch (a) {
                case Algorithm::sort_short_wide: sort_short_wide(v); break;
                case Algorithm::sort_square: sort_square(v); break;
                case Algorithm::sort_tall: sort_tall(v); break;
                case Algorithm::partition_short_wide: partition_short_wide(v); break;
                case Algorithm::partition_square: partition_square(v); break;
                case Algorithm::partition_general: partition_general(v); break;
                case Algorithm::integer_sort_general: integer_sort_general(vp, u64(w) * m); break;
                case Algorithm::permute: {
                    Rng rng(seed);
                    PermuteParams params;
                    permute(mach, rng, params);
                    break;
                }
            }
            if (a == Algorithm::permute) {
                for (u32 i = 0; i < w; ++i)
                    for (u32 j = 0; j < m; ++j)
                        out_grid[u64(i) * m + j] = mach.peek(i, cfg.out_base() + j);
            } else {
                auto snap = (a == Algorithm::integer_sort_general ? vp : v).snapshot();
                std::memcpy(out_grid, snap.data(), sizeof(uint64_t) * snap.size());
            }
        }
        return DMM_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

// integer_sort_general on the vp view (instance.hpp:295) with an explicit domain,
// optional hooks capture: snapshots of the full working window after each
// balance / divide of the outer recursion (PartitionProbe partition.hpp:298).
int dmmr_integer_sort_general(uint32_t w, uint32_t m, uint64_t* grid, uint64_t domain, int enforce_pre,
                              int strict, uint32_t* cleanup_retries, uint32_t* sorted,
                              uint64_t* probe_snaps, uint32_t max_snaps, uint32_t* n_snaps) {
    try {
        Machine mach(MachineConfig::standard(w, m, strict != 0));
        const auto& cfg = mach.config();
        std::vector<u32> rows(w);
        for (u32 r = 0; r < w; ++r)
            rows[r] = r;
        MatrixView vp = MatrixView::make(mach, rows, cfg.work_base(), m, cfg.scratch_a_base(),
                                         cfg.scratch_b_base());
        vp.load(std::vector<word>(grid, grid + u64(w) * m));
        uint32_t snaps = 0;
        PartitionProbe probe;
        auto grab = [&](u32, const std::vector<MatrixView>&) {
            if (probe_snaps && snaps < max_snaps) {
                auto s = vp.snapshot();
                std::memcpy(probe_snaps + u64(snaps) * w * m, s.data(), sizeof(uint64_t) * s.size());
            }
            ++snaps;
        };
        probe.after_balance = grab;
        probe.after_divide = grab;
        GeneralStats st = integer_sort_general(vp, domain, probe_snaps ? &probe : nullptr, enforce_pre != 0);
        if (n_snaps)
            *n_snaps = snaps;
        *cleanup_retries = st.cleanup_retries;
        *sorted = st.sorted;
        auto s = vp.snapshot();
        std::memcpy(grid, s.data(), sizeof(uint64_t) * s.size());
        return DMM_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

// integer_sort_general on the vp view with an explicit domain on ANY keys (run_algorithm only takes
// generated instances): Machine::steps() and the stats, for the recursion's step meter.
int dmmr_integer_sort_general_steps(uint32_t w, uint32_t m, uint64_t* grid, uint64_t domain, int enforce_pre,
                                    int strict, uint32_t* cleanup_retries, uint32_t* sorted, uint64_t* steps) {
    try {
        Machine mach(MachineConfig::standard(w, m, strict != 0));
        const auto& cfg = mach.config();
        std::vector<u32> rows(w);
        for (u32 r = 0; r < w; ++r)
            rows[r] = r;
        MatrixView vp = MatrixView::make(mach, rows, cfg.work_base(), m, cfg.scratch_a_base(),
                                         cfg.scratch_b_base());
        vp.load(std::vector<word>(grid, grid + u64(w) * m));
        GeneralStats st = integer_sort_general(vp, domain, nullptr, enforce_pre != 0);
        *cleanup_retries = st.cleanup_retries;
        *sorted = st.sorted;
        *steps = mach.steps();
        auto s = vp.snapshot();
        std::memcpy(grid, s.data(), sizeof(uint64_t) * s.size());
        return DMM_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

// partition_general on the full view, as run_algorithm does (instance.hpp:326).
int dmmr_partition_general(uint32_t w, uint32_t m, uint64_t* grid, int strict, uint32_t* cleanup_retries,
                           uint32_t* sorted) {
    try {
        Machine mach(MachineConfig::standard(w, m, strict != 0));
        MatrixView v = MatrixView::full(mach);
        v.load(std::vector<word>(grid, grid + u64(w) * m));
        GeneralStats st = partition_general(v);
        *cleanup_retries = st.cleanup_retries;
        *sorted = st.sorted;
        auto s = v.snapshot();
        std::memcpy(grid, s.data(), sizeof(uint64_t) * s.size());
        return DMM_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

int dmmr_permute(uint32_t w, uint32_t m, const uint64_t* grid, uint64_t seed, uint32_t alpha,
                 uint32_t iter_cap, uint64_t* out, dmmr_permute_report* prep, uint32_t* shifts) {
    try {
        Machine mach(MachineConfig::standard(w, m, true));
        const auto& cfg = mach.config();
        std::vector<u32> rows(w);
        for (u32 r = 0; r < w; ++r)
            rows[r] = r;
        MatrixView vp = MatrixView::make(mach, rows, cfg.work_base(), m, cfg.scratch_a_base(),
                                         cfg.scratch_b_base());
        vp.load(std::vector<word>(grid, grid + u64(w) * m));
        Rng rng(seed);
        PermuteParams params;
        params.alpha = alpha;
        params.iter_cap = iter_cap;
        PermuteReport p = permute(mach, rng, params);
        prep->iterations = p.iterations;
        prep->fallback = p.fallback;
        prep->used_packing = p.used_packing;
        prep->packed_width = p.packed_width;
        prep->threshold = p.threshold;
        prep->random_words = p.random_words;
        prep->cleanup_retries = p.cleanup_retries;
        prep->n_hist = static_cast<uint32_t>(std::min<std::size_t>(64, p.leftover_history.size()));
        for (uint32_t i = 0; i < prep->n_hist; ++i)
            prep->leftover_history[i] = p.leftover_history[i];
        if (shifts)
            for (std::size_t i = 0; i < p.shifts.size(); ++i)
                shifts[i] = p.shifts[i];
        for (u32 i = 0; i < w; ++i)
            for (u32 j = 0; j < m; ++j)
                out[u64(i) * m + j] = mach.peek(i, cfg.out_base() + j);
        return DMM_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

// Layout primitives on a standalone machine (layout.hpp:24, :397, :403).
// op: 0 transpose_square, 1 to_column_major, 2 to_row_major.
int dmmr_layout(int op, uint32_t w, uint32_t m, uint64_t* grid) {
    try {
        Machine mach(MachineConfig::standard(w, m, true));
        MatrixView v = MatrixView::full(mach);
        v.load(std::vector<word>(grid, grid + u64(w) * m));
        if (op == 0)
            transpose_square(v);
        else if (op == 1)
            to_column_major(v);
        else
            to_row_major(v);
        auto s = v.snapshot();
        std::memcpy(grid, s.data(), sizeof(uint64_t) * s.size());
        return DMM_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

int dmmr_general_sort_shape_ok(uint64_t W, uint64_t M) { return general_sort_shape_ok(W, M) ? 1 : 0; }
uint64_t dmmr_permute_threshold(uint32_t w, uint32_t m) { return detail::permute_threshold(w, m); }

// ---------------------------------------------------------------------------
// CPU baseline: the reference's own run_algorithm per instance, fanned over
// host threads with an atomic work index (the acceptance.cpp:39-60 pattern).
// Instances are given explicitly (u32, row-major, count x w x m).  kind of
// work: alg as in Algorithm; for integer_sort_general the domain argument is
// used (run_algorithm hard-codes w*m).  Returns elapsed seconds via *secs.
// ---------------------------------------------------------------------------
int dmmr_cpu_baseline(int alg, uint32_t w, uint32_t m, uint64_t count, const uint32_t* in, const uint64_t* seeds,
                      uint64_t domain, uint32_t nthreads, double* secs, uint64_t* n_correct) {
    const u64 n = u64(w) * m;
    std::atomic<u64> next{0}, good{0};
    std::atomic<int> err{DMM_OK};
    auto worker = [&] {
        for (;;) {
            const u64 k = next.fetch_add(1);
            if (k >= count)
                return;
            try {
                if (alg_of(alg) == Algorithm::integer_sort_general) {
                    Machine mach(MachineConfig::standard(w, m, true));
                    TraceAuditor auditor(w);
                    mach.attach_auditor(&auditor);
                    mach.set_host_threads(1);
                    const auto& cfg = mach.config();
                    std::vector<u32> rows(w);
                    for (u32 r = 0; r < w; ++r)
                        rows[r] = r;
                    MatrixView vp = MatrixView::make(mach, rows, cfg.work_base(), m, cfg.scratch_a_base(),
                                                     cfg.scratch_b_base());
                    std::vector<word> g(in + k * n, in + (k + 1) * n);
                    vp.load(g);
                    integer_sort_general(vp, domain);
                    auto snap = vp.snapshot();
                    std::sort(g.begin(), g.end());
                    if (snap == g)
                        good.fetch_add(1);
                } else {
                    Instance inst;
                    inst.kind = instance_kind_for(alg_of(alg));
                    inst.w = w;
                    inst.m = m;
                    inst.seed = seeds ? seeds[k] : k;
                    inst.grid.assign(in + k * n, in + (k + 1) * n);
                    RunOptions opt;
                    opt.host_threads = 1;
                    RunOutcome o = run_algorithm(alg_of(alg), inst, opt);
                    if (o.report.correct)
                        good.fetch_add(1);
                }
            } catch (...) {
                err.store(status_of_current_exception());
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (u32 t = 0; t < std::max<u32>(1, nthreads); ++t)
        pool.emplace_back(worker);
    for (auto& th : pool)
        th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *secs = std::chrono::duration<double>(t1 - t0).count();
    if (n_correct)
        *n_correct = good.load();
    return err.load();
}

// instance_to_text (instance.hpp:103-115): writes up to cap bytes, returns the full length.
uint64_t dmmr_instance_to_text(int kind, uint32_t w, uint32_t m, uint64_t seed, const uint64_t* grid, char* buf,
                               uint64_t cap) {
    Instance in;
    in.kind = static_cast<InstanceKind>(kind);
    in.w = w;
    in.m = m;
    in.seed = seed;
    in.grid.assign(grid, grid + uint64_t(w) * m);
    const std::string s = instance_to_text(in);
    if (buf && cap)
        std::memcpy(buf, s.data(), std::min<uint64_t>(cap, s.size()));
    return s.size();
}

// instance_from_text (instance.hpp:117-128): header into hdr[kind, w, m, seed], grid into
// grid[0..cap); returns a dmm_status.
int dmmr_instance_from_text(const char* text, uint64_t* hdr, uint64_t* grid, uint64_t cap) {
    try {
        std::istringstream is(text);
        Instance in = instance_from_text(is);
        hdr[0] = static_cast<uint64_t>(in.kind);
        hdr[1] = in.w;
        hdr[2] = in.m;
        hdr[3] = in.seed;
        std::memcpy(grid, in.grid.data(), sizeof(uint64_t) * std::min<uint64_t>(cap, in.grid.size()));
        return 0;
    } catch (...) {
        return status_of_current_exception();
    }
}

// offline_schedule (layout.hpp:207-230): perm as (dst_bank, dst_off) pairs; moves out as
// (src_bank, src_off, dst_bank, dst_off) in round order, round_len[r] = moves in round r.
int dmmr_offline_schedule(uint32_t w, uint32_t m, const uint32_t* perm, uint32_t* moves, uint32_t* round_len,
                          uint32_t* n_rounds) {
    try {
        std::vector<std::pair<u32, u32>> p(uint64_t(w) * m);
        for (uint64_t i = 0; i < p.size(); ++i)
            p[i] = {perm[2 * i], perm[2 * i + 1]};
        Schedule s = offline_schedule(w, m, p);
        uint64_t k = 0;
        *n_rounds = uint32_t(s.rounds.size());
        for (std::size_t r = 0; r < s.rounds.size(); ++r) {
            round_len[r] = uint32_t(s.rounds[r].size());
            for (const Move& mv : s.rounds[r]) {
                moves[4 * k] = mv.src_bank;
                moves[4 * k + 1] = mv.src_off;
                moves[4 * k + 2] = mv.dst_bank;
                moves[4 * k + 3] = mv.dst_off;
                ++k;
            }
        }
        return 0;
    } catch (const NotBijective&) {
        return DMM_NOT_BIJECTIVE;
    } catch (...) {
        return status_of_current_exception();
    }
}

// schedule_to_text (layout.hpp:268-278) of a schedule given as round lengths + moves.
uint64_t dmmr_schedule_to_text(const uint32_t* moves, const uint32_t* round_len, uint32_t n_rounds, char* buf,
                               uint64_t cap) {
    Schedule s;
    uint64_t k = 0;
    for (uint32_t r = 0; r < n_rounds; ++r) {
        std::vector<Move> round;
        for (uint32_t i = 0; i < round_len[r]; ++i, ++k)
            round.push_back({moves[4 * k], moves[4 * k + 1], moves[4 * k + 2], moves[4 * k + 3]});
        s.rounds.push_back(std::move(round));
    }
    const std::string t = schedule_to_text(s);
    if (buf && cap)
        std::memcpy(buf, t.data(), std::min<uint64_t>(cap, t.size()));
    return t.size();
}

// trace_to_text (instance.hpp:369-382) of run_algorithm(alg, gen_instance(kind_for(alg), w, m,
// seed), record_trace); returns the full length, copies up to cap bytes.
uint64_t dmmr_trace_text(int alg, uint32_t w, uint32_t m, uint64_t seed, char* buf, uint64_t cap) {
    try {
        RunOptions opt;
        opt.record_trace = true;
        const Algorithm a = alg_of(alg);
        RunOutcome out = run_algorithm(a, gen_instance(instance_kind_for(a), w, m, seed), opt);
        const std::string t = trace_to_text(out.trace);
        if (buf && cap)
            std::memcpy(buf, t.data(), std::min<uint64_t>(cap, t.size()));
        return t.size();
    } catch (...) {
        return 0;
    }
}

// verify_trace (core.hpp:221-237) of a parsed trace text: number of (step, bank) violations,
// or -1 if the text does not parse
int64_t dmmr_verify_trace_text(const char* text) {
    try {
        std::istringstream is(text);
        return int64_t(verify_trace(trace_from_text(is)).size());
    } catch (...) {
        return -1;
    }
}

}  // extern "C"

// dmm_b200.hpp -- header-only C++ drop-in for the reference's hot path.
//
// Same names, argument meaning and error behaviour as /root/reference/proj/include/dmm/
// (namespace dmm::b200 instead of dmm): a reference user keeps their Machine / MatrixView /
// Rng objects and calls
//
//     dmm::b200::partition_general(view)            // partition.hpp:453
//     dmm::b200::integer_sort_general(view, domain)  // partition.hpp:436
//     dmm::b200::sort_tall(view)                     // sort.hpp:352
//     dmm::b200::partition_square(view) / partition_short_wide(view)   // partition.hpp:189 / :178
//     dmm::b200::sort_square(view, asc) / sort_short_wide(view, asc)   // sort.hpp:337 / :225
//     dmm::b200::transpose_square(view)              // layout.hpp:24 (+ to_column_major / to_row_major)
//     dmm::b200::permute(machine, rng, params)       // permute.hpp:545
//     dmm::b200::run_algorithm(alg, instance, opts)  // instance.hpp:277 (the CLI / acceptance dispatch)
//
// Each call gathers the view's cells (peek), runs the sm_100a kernel through the C ABI
// (include/dmm_gpu.h) on a batch of one, writes the result back (poke) and rethrows the
// reference's exception type for a non-OK status.  permute() continues the caller's
// std::mt19937_64 from its exact state and advances it by report.random_words draws, so
// host code after the call sees the same stream as with the reference.
//
// Not reproduced (GPU kernels have no DMM step meter): Machine::steps()/work() do not
// advance (run_algorithm reports the reference's count where it is modelled: dmm_modelled_steps,
// dmm_leaf_steps, dmm_general_steps); PartitionProbe hooks are replayed from the kernel's snapshots (the caller's
// machine holds the reference's window at each call), ShortWideHook calls likewise; traces
// are unsupported (TraceIncomplete); permute() reproduces
// the output region, the report and the Rng position, not the scratch/counter cells.
// Words must fit in 32 bits (KeyOutOfRange otherwise).  Requires <dmm/dmm.hpp>.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <sstream>
#include <string>
#include <vector>

#include <dmm/dmm.hpp>

#include "dmm_gpu.h"

namespace dmm {
namespace b200 {

[[noreturn]] inline void raise(dmm_status s, const std::string& where) {
    const std::string msg = where + " (B200): " + dmm_last_error();
    switch (s) {
        case DMM_SHAPE_VIOLATION: throw ShapeViolation(msg);
        case DMM_INVALID_INSTANCE: throw InvalidInstance(msg);
        case DMM_KEY_OUT_OF_RANGE: throw KeyOutOfRange(msg);
        case DMM_DIVISIBILITY_VIOLATION: throw DivisibilityViolation(msg);
        case DMM_POSTCONDITION_FAILED: throw PostconditionFailed(msg);
        case DMM_PACKING_OVERFLOW: throw PackingOverflow(msg);
        case DMM_CAPACITY_EXCEEDED: throw CapacityExceeded(msg);
        case DMM_NOT_SQUARE: throw NotSquare(msg);
        case DMM_OUT_OF_BOUNDS: throw OutOfBounds(msg);
        case DMM_OVERLAPPING_VIEWS: throw OverlappingViews(msg);
        case DMM_NOT_BIJECTIVE: throw NotBijective(msg);
        case DMM_CONFLICT_VIOLATION: throw ConflictViolation(msg);
        default: throw Error(msg);
    }
}

inline void check(dmm_status s, const char* where) {
    if (s != DMM_OK)
        raise(s, where);
}

inline void cuda_check(cudaError_t e, const char* where) {
    if (e != cudaSuccess)
        throw Error(std::string(where) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
struct DeviceBuffer {
    void* ptr = nullptr;
    explicit DeviceBuffer(std::size_t bytes) { cuda_check(cudaMalloc(&ptr, bytes ? bytes : 16), "cudaMalloc"); }
    ~DeviceBuffer() { cudaFree(ptr); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(ptr); }
};

template <class T>
inline void to_device(DeviceBuffer& d, const std::vector<T>& h) {
    cuda_check(cudaMemcpy(d.ptr, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice), "H2D");
}
template <class T>
inline void to_host(std::vector<T>& h, const DeviceBuffer& d) {
    cuda_check(cudaMemcpy(h.data(), d.ptr, sizeof(T) * h.size(), cudaMemcpyDeviceToHost), "D2H");
}

// view window -> row-major 32-bit grid (the narrowing of SURVEY 8(b))
inline std::vector<uint32_t> gather(const MatrixView& v) {
    std::vector<uint32_t> g(u64(v.W()) * v.M());
    for (u32 r = 0; r < v.W(); ++r)
        for (u32 c = 0; c < v.M(); ++c) {
            const word x = v.machine().peek(v.bank(r), v.off(c));
            if (x >> 32)
                throw KeyOutOfRange("B200 kernels take 32-bit words");
            g[u64(r) * v.M() + c] = static_cast<uint32_t>(x);
        }
    return g;
}
inline void scatter(const MatrixView& v, const std::vector<uint32_t>& g) {
    for (u32 r = 0; r < v.W(); ++r)
        for (u32 c = 0; c < v.M(); ++c)
            v.machine().poke(v.bank(r), v.off(c), g[u64(r) * v.M() + c]);
}

inline bool wants_probe(const PartitionProbe* probe) {
    return probe && (probe->after_balance || probe->after_divide);
}

// Replays the reference's hook calls (partition.hpp:373-391) from the kernel's snapshots: the
// caller's machine holds, at each call, the window the reference would hold, and the hook gets
// the same list of views (balance level / convert_and_divide row ranges, built host-side).
inline void replay_probe(const MatrixView& v, const PartitionProbe& probe, const std::vector<uint32_t>& snaps,
                         uint32_t nsnaps) {
    const u64 cells = u64(v.W()) * v.M();
    auto show = [&](uint32_t i) {
        if (i < nsnaps)
            scatter(v, std::vector<uint32_t>(snaps.begin() + i * cells, snaps.begin() + (i + 1) * cells));
    };
    std::vector<MatrixView> level{v};
    u32 depth = 0;
    uint32_t i = 0;
    while (level.front().W() > v.M()) {
        show(i++);
        if (probe.after_balance)
            probe.after_balance(depth, level);
        const PartitionParams p = PartitionParams::compute(level.front().W(), v.M());
        std::vector<MatrixView> next;
        for (const MatrixView& lv : level) {
            const u32 h = lv.W() / p.subproblems;
            for (u32 k = 0; k < p.subproblems; ++k)
                next.push_back(lv.row_range(k * h, h));
        }
        level.swap(next);
        ++depth;
        show(i++);
        if (probe.after_divide)
            probe.after_divide(depth, level);
    }
}

inline GeneralStats general_impl(bool partition, const MatrixView& v, u64 domain, bool enforce,
                                 const PartitionProbe* probe) {
    std::vector<uint32_t> g = gather(v);
    const uint64_t bytes = sizeof(uint32_t) * g.size();
    DeviceBuffer d(bytes), st(sizeof(dmm_general_stats)), ss(16);
    to_device(d, g);
    uint32_t flags = 0;
    if (!v.machine().config().strict)
        flags |= DMM_FLAG_NONSTRICT;
    if (!enforce)
        flags |= DMM_FLAG_NO_ENFORCE_PRE;
    const bool probing = wants_probe(probe);
    const uint32_t nsnaps = probing ? dmm_general_probe_snaps(v.W(), v.M(), flags) : 0;
    DeviceBuffer dsnap(sizeof(uint32_t) * (nsnaps ? nsnaps * g.size() : 1));
    const char* where = partition ? "partition_general" : "integer_sort_general";
    dmm_status s;
    if (partition)
        s = dmm_partition_general_probe(d.as<uint32_t>(), d.as<uint32_t>(), v.W(), v.M(), 1, flags,
                                        st.as<dmm_general_stats>(), ss.as<uint8_t>(), dsnap.as<uint32_t>(), nsnaps,
                                        nullptr);
    else
        s = dmm_integer_sort_general_probe(d.as<uint32_t>(), d.as<uint32_t>(), v.W(), v.M(), 1, domain, flags,
                                           st.as<dmm_general_stats>(), ss.as<uint8_t>(), dsnap.as<uint32_t>(),
                                           nsnaps, nullptr);
    check(s, where);
    dmm_general_stats hs{};
    uint8_t status = 0;
    cuda_check(cudaMemcpy(&hs, st.ptr, sizeof(hs), cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(&status, ss.ptr, 1, cudaMemcpyDeviceToHost), "D2H");
    // input validation fails before the recursion (no hook calls); a failed cleanup after it
    if (status == DMM_INVALID_INSTANCE || status == DMM_KEY_OUT_OF_RANGE)
        raise(static_cast<dmm_status>(status), where);
    if (probing && nsnaps) {
        std::vector<uint32_t> snaps(u64(nsnaps) * g.size());
        to_host(snaps, dsnap);
        replay_probe(v, *probe, snaps, nsnaps);
    }
    to_host(g, d);
    scatter(v, g);
    if (status != DMM_OK)
        raise(static_cast<dmm_status>(status), where);
    GeneralStats out;
    out.cleanup_retries = hs.cleanup_retries;
    out.sorted = hs.sorted != 0;
    return out;
}

/// GeneralStats partition_general(const MatrixView&, const PartitionProbe* = nullptr)  partition.hpp:453-456
inline GeneralStats partition_general(const MatrixView& v, const PartitionProbe* probe = nullptr) {
    return general_impl(true, v, v.W(), true, probe);
}

/// GeneralStats integer_sort_general(view, domain, probe, enforce)  partition.hpp:436-449
inline GeneralStats integer_sort_general(const MatrixView& v, u64 domain, const PartitionProbe* probe = nullptr,
                                         bool enforce_analysis_pre = true) {
    return general_impl(false, v, domain, enforce_analysis_pre, probe);
}

namespace detail {
template <class Fn>
inline void simple(const MatrixView& v, Fn&& fn, const char* where) {
    std::vector<uint32_t> g = gather(v);
    DeviceBuffer d(sizeof(uint32_t) * g.size());
    to_device(d, g);
    check(fn(d.as<uint32_t>()), where);
    to_host(g, d);
    scatter(v, g);
}
}  // namespace detail

/// void sort_tall(const MatrixView&)  sort.hpp:352-374
inline void sort_tall(const MatrixView& v) {
    detail::simple(v, [&](uint32_t* p) { return dmm_sort_tall(p, p, v.W(), v.M(), 1, nullptr); }, "sort_tall");
}
namespace detail {
// ShortWideHook replay (sort.hpp:189-218): the kernel's literal skeleton captured the window
// at the three stages; the caller's machine holds each when its hook call happens.
inline void short_wide_hooked(const MatrixView& v, bool partition, bool ascending, const ShortWideHook& hook,
                              const char* where) {
    std::vector<uint32_t> g = gather(v);
    DeviceBuffer d(sizeof(uint32_t) * g.size()), ss(16), dsnap(sizeof(uint32_t) * 3 * g.size());
    to_device(d, g);
    check(dmm_short_wide_probe(d.as<uint32_t>(), d.as<uint32_t>(), v.W(), v.M(), 1, partition ? 1 : 0,
                               ascending ? 1 : 0, ss.as<uint8_t>(), dsnap.as<uint32_t>(), nullptr),
          where);
    uint8_t status = 0;
    cuda_check(cudaMemcpy(&status, ss.ptr, 1, cudaMemcpyDeviceToHost), "D2H");
    if (status != DMM_OK)  // check_partition_instance fails before any stage
        raise(static_cast<dmm_status>(status), where);
    std::vector<uint32_t> snaps(3 * g.size());
    to_host(snaps, dsnap);
    const ShortWideStage stages[3] = {ShortWideStage::after_first_convert, ShortWideStage::after_first_pass,
                                      ShortWideStage::done};
    for (int i = 0; i < 3; ++i) {
        scatter(v, std::vector<uint32_t>(snaps.begin() + i * g.size(), snaps.begin() + (i + 1) * g.size()));
        hook(stages[i]);
    }
    to_host(g, d);
    scatter(v, g);
}
// a partition entry point: per-instance status -> the reference's exception
template <class Fn>
inline void partition_entry(const MatrixView& v, Fn&& fn, const char* where) {
    std::vector<uint32_t> g = gather(v);
    DeviceBuffer d(sizeof(uint32_t) * g.size()), ss(16);
    to_device(d, g);
    check(fn(d.as<uint32_t>(), ss.as<uint8_t>()), where);
    uint8_t status = 0;
    cuda_check(cudaMemcpy(&status, ss.ptr, 1, cudaMemcpyDeviceToHost), "D2H");
    if (status != DMM_OK)
        raise(static_cast<dmm_status>(status), where);
    to_host(g, d);
    scatter(v, g);
}
}  // namespace detail

/// void partition_square(const MatrixView&)  partition.hpp:189-197
inline void partition_square(const MatrixView& v) {
    detail::partition_entry(
        v, [&](uint32_t* p, uint8_t* st) { return dmm_partition_square(p, p, v.W(), v.M(), 1, st, nullptr); },
        "partition_square");
}
/// void partition_short_wide(const MatrixView&, const ShortWideHook& = {})  partition.hpp:178-185
inline void partition_short_wide(const MatrixView& v, const ShortWideHook& hook = {}) {
    if (u64(v.W()) * v.W() > v.M())
        throw ShapeViolation("partition_short_wide needs w^2 <= m");
    if (hook)
        return detail::short_wide_hooked(v, true, true, hook, "partition_short_wide");
    detail::partition_entry(
        v, [&](uint32_t* p, uint8_t* st) { return dmm_partition_short_wide(p, p, v.W(), v.M(), 1, st, nullptr); },
        "partition_short_wide");
}
/// void sort_square(const MatrixView&, bool ascending = true)  sort.hpp:337-346
inline void sort_square(const MatrixView& v, bool ascending = true) {
    detail::simple(v, [&](uint32_t* p) { return dmm_sort_square(p, p, v.W(), v.M(), 1, ascending ? 1 : 0, nullptr); },
                   "sort_square");
}
/// void sort_short_wide(const MatrixView&, bool ascending = true, const ShortWideHook& = {})  sort.hpp:225-230
inline void sort_short_wide(const MatrixView& v, bool ascending = true, const ShortWideHook& hook = {}) {
    if (hook) {
        if (u64(v.W()) * v.W() > v.M())
            throw ShapeViolation("short-wide sort needs w^2 <= m");
        return detail::short_wide_hooked(v, false, ascending, hook, "sort_short_wide");
    }
    detail::simple(v,
                   [&](uint32_t* p) { return dmm_sort_short_wide(p, p, v.W(), v.M(), 1, ascending ? 1 : 0, nullptr); },
                   "sort_short_wide");
}

/// transpose_square layout.hpp:24-61
inline void transpose_square(const MatrixView& v) {
    if (v.W() != v.M())
        throw NotSquare("transpose_square needs a square view");
    detail::simple(v, [&](uint32_t* p) { return dmm_transpose_square(p, p, v.W(), 1, nullptr); },
                   "transpose_square");
}
/// to_column_major layout.hpp:397-399
inline void to_column_major(const MatrixView& v) {
    detail::simple(v, [&](uint32_t* p) { return dmm_to_column_major(p, p, v.W(), v.M(), 1, nullptr); },
                   "to_column_major");
}
/// to_row_major layout.hpp:403-405
inline void to_row_major(const MatrixView& v) {
    detail::simple(v, [&](uint32_t* p) { return dmm_to_row_major(p, p, v.W(), v.M(), 1, nullptr); },
                   "to_row_major");
}

/// Schedule offline_schedule(W, M, perm)  layout.hpp:207-230 -- the host precompute of
/// libdmm_b200.so; the same rounds as the reference, move for move.
inline Schedule offline_schedule(u32 W, u32 M, const std::vector<std::pair<u32, u32>>& perm) {
    if (perm.size() != u64(W) * M)
        throw NotBijective("permutation table has wrong size");
    std::vector<uint32_t> p(2 * perm.size()), mv(4 * perm.size() + 4);
    for (std::size_t i = 0; i < perm.size(); ++i) {
        p[2 * i] = perm[i].first;
        p[2 * i + 1] = perm[i].second;
    }
    check(dmm_offline_schedule(W, M, p.data(), mv.data()), "offline_schedule");
    Schedule s;
    for (u32 r = 0; W && r < M; ++r) {
        std::vector<Move> round(W);
        for (u32 i = 0; i < W; ++i) {
            const uint32_t* x = &mv[4 * (u64(r) * W + i)];
            round[i] = {x[0], x[1], x[2], x[3]};
        }
        s.rounds.push_back(std::move(round));
    }
    return s;
}

/// void apply_schedule(const MatrixView&, const Schedule&, u32 dst_base)  layout.hpp:246-263:
/// moves the view's working window into the window at dst_base on the B200 (one warp, DMM bank
/// = shared-memory bank); cells no move writes keep their contents.  A round reusing a bank
/// raises ConflictViolation, a move outside the shape OutOfBounds -- before any write.
inline void apply_schedule(const MatrixView& v, const Schedule& s, u32 dst_base) {
    const u32 W = v.W(), M = v.M();
    std::vector<uint32_t> src = gather(v), dstw(u64(W) * M);
    for (u32 r = 0; r < W; ++r)
        for (u32 c = 0; c < M; ++c) {
            const word x = v.machine().peek(v.bank(r), dst_base + c);
            if (x >> 32)
                throw KeyOutOfRange("B200 kernels take 32-bit words");
            dstw[u64(r) * M + c] = static_cast<uint32_t>(x);
        }
    std::vector<uint32_t> mv, starts{0};
    for (const auto& round : s.rounds) {
        for (const Move& m : round)
            mv.insert(mv.end(), {m.src_bank, m.src_off, m.dst_bank, m.dst_off});
        starts.push_back(uint32_t(mv.size() / 4));
    }
    DeviceBuffer din(sizeof(uint32_t) * src.size()), dout(sizeof(uint32_t) * dstw.size()),
        dmv(sizeof(uint32_t) * mv.size()), dst(sizeof(uint32_t) * starts.size()), dstatus(16);
    to_device(din, src);
    to_device(dout, dstw);
    if (!mv.empty())
        to_device(dmv, mv);
    to_device(dst, starts);
    check(dmm_apply_schedule(din.as<uint32_t>(), dout.as<uint32_t>(), W, M, 1, dmv.as<uint32_t>(),
                                     dst.as<uint32_t>(), uint32_t(s.rounds.size()), uint32_t(mv.size() / 4),
                                     dstatus.as<uint8_t>(), nullptr),
                  "apply_schedule");
    uint8_t status = 0;
    cuda_check(cudaMemcpy(&status, dstatus.ptr, 1, cudaMemcpyDeviceToHost), "D2H");
    if (status != DMM_OK)
        raise(static_cast<dmm_status>(status), "apply_schedule");
    to_host(dstw, dout);
    for (u32 r = 0; r < W; ++r)
        for (u32 c = 0; c < M; ++c)
            v.machine().poke(v.bank(r), dst_base + c, dstw[u64(r) * M + c]);
}
inline void apply_schedule(const MatrixView& v, const Schedule& s) { b200::apply_schedule(v, s, v.s0_base()); }

/// PermuteReport permute(Machine&, Rng&, const PermuteParams&)  permute.hpp:545-628
inline PermuteReport permute(Machine& mach, Rng& rng, const PermuteParams& params = {}) {
    const u32 w = mach.w(), m = mach.m();
    // permute.hpp:547-553: the shape checks run on the device path too (dmm_permute_from_state
    // returns DMM_SHAPE_VIOLATION); the bank-layout check needs the caller's MachineConfig
    if (!mach.config().has_scratch_b())
        throw CapacityExceeded("permute needs the standard 4m+8 bank layout");
    // the caller's engine, mid-stream: libstdc++ prints _M_x[0..312) then _M_p
    std::vector<uint64_t> state(313);
    {
        std::ostringstream os;
        os << rng;
        std::istringstream is(os.str());
        for (auto& s : state)
            if (!(is >> s))
                throw Error("cannot serialize the Rng state");
    }
    std::vector<uint32_t> g(u64(w) * m);
    for (u32 r = 0; r < w; ++r)
        for (u32 c = 0; c < m; ++c) {
            const word x = mach.peek(r, mach.config().work_base() + c);
            if (x >> 32)
                throw KeyOutOfRange("B200 kernels take 32-bit words");
            g[u64(r) * m + c] = static_cast<uint32_t>(x);
        }
    DeviceBuffer din(sizeof(uint32_t) * g.size()), dout(sizeof(uint32_t) * g.size()),
        dst(sizeof(uint64_t) * state.size()), drep(sizeof(dmm_permute_report)),
        dhist(sizeof(uint64_t) * DMM_PERMUTE_MAX_HIST), dsh(sizeof(uint32_t) * w), dss(16);
    to_device(din, g);
    to_device(dst, state);
    check(dmm_permute_from_state(din.as<uint32_t>(), dout.as<uint32_t>(), w, m, 1, dst.as<uint64_t>(), params.alpha,
                                 params.iter_cap, drep.as<dmm_permute_report>(), dhist.as<uint64_t>(),
                                 dsh.as<uint32_t>(), dss.as<uint8_t>(), nullptr),
          "permute");
    dmm_permute_report hr{};
    std::vector<uint64_t> hist(DMM_PERMUTE_MAX_HIST);
    std::vector<uint32_t> shifts(w);
    cuda_check(cudaMemcpy(&hr, drep.ptr, sizeof(hr), cudaMemcpyDeviceToHost), "D2H");
    to_host(hist, dhist);
    to_host(shifts, dsh);
    // the per-instance status: DMM_INVALID_INSTANCE when a label is out of range or the
    // delivered output is not the identity -- raised before the output region is written
    uint8_t pstatus = DMM_OK;
    cuda_check(cudaMemcpy(&pstatus, dss.ptr, 1, cudaMemcpyDeviceToHost), "D2H");
    if (pstatus != DMM_OK)
        raise(static_cast<dmm_status>(pstatus), "permute");
    to_host(g, dout);
    for (u32 i = 0; i < w; ++i)
        for (u32 j = 0; j < m; ++j)
            mach.poke(i, mach.config().out_base() + j, g[u64(i) * m + j]);
    rng.discard(hr.random_words);
    PermuteReport rep;
    rep.iterations = hr.iterations;
    rep.fallback = hr.fallback != 0;
    rep.used_packing = hr.used_packing != 0;
    rep.packed_width = hr.packed_width;
    rep.threshold = hr.threshold;
    rep.random_words = hr.random_words;
    rep.cleanup_retries = hr.cleanup_retries;
    rep.leftover_history.assign(hist.begin(), hist.begin() + hr.n_hist);
    rep.shifts = shifts;
    return rep;
}

/// RunOutcome run_algorithm(Algorithm, const Instance&, const RunOptions&)  instance.hpp:277-363
/// The dispatcher the reference's CLI and acceptance harness use, over the B200 kernels: the
/// same instance checks, views, verification and report fields.  The GPU has no DMM step
/// meter: report.steps / work are the reference's counts where modelled (dmm_modelled_steps,
/// dmm_leaf_steps, dmm_general_steps, dmm_permute_steps); conflicts counts the model's violations (0: every
/// kernel relayout is checked conflict-free at compile time); record_trace throws
/// TraceIncomplete.
inline RunOutcome run_algorithm(Algorithm alg, const Instance& in, const RunOptions& opt = {}) {
    if (in.kind != instance_kind_for(alg))
        throw InvalidInstance(std::string("algorithm ") + algorithm_name(alg) + " needs a " +
                              kind_name(instance_kind_for(alg)) + " instance");
    validate_instance(in);
    if (opt.record_trace)
        throw TraceIncomplete("B200 kernels record no DMM trace (no step meter)");
    Machine mach(MachineConfig::standard(in.w, in.m, opt.strict));
    const auto& cfg = mach.config();
    std::vector<u32> all_rows(in.w);
    for (u32 r = 0; r < in.w; ++r)
        all_rows[r] = r;
    MatrixView v = MatrixView::full(mach);
    MatrixView vp = MatrixView::make(mach, all_rows, cfg.work_base(), in.m, cfg.scratch_a_base(), cfg.scratch_b_base());
    (alg == Algorithm::permute || alg == Algorithm::integer_sort_general ? vp : v).load(in.grid);

    RunOutcome out;
    out.report.algorithm = algorithm_name(alg);
    out.report.w = in.w;
    out.report.m = in.m;
    out.report.seed = opt.seed.value_or(in.seed);
    switch (alg) {
        case Algorithm::sort_short_wide:
            b200::sort_short_wide(v);
            out.report.correct = verify_sorted_result(in, v.snapshot());
            break;
        case Algorithm::sort_square:
            b200::sort_square(v);
            out.report.correct = verify_sorted_result(in, v.snapshot());
            break;
        case Algorithm::sort_tall:
            b200::sort_tall(v);
            out.report.correct = verify_sorted_result(in, v.snapshot());
            break;
        case Algorithm::partition_short_wide:
            b200::partition_short_wide(v);
            out.report.correct = verify_partition_result(in, v.snapshot());
            break;
        case Algorithm::partition_square:
            b200::partition_square(v);
            out.report.correct = verify_partition_result(in, v.snapshot());
            break;
        case Algorithm::partition_general: {
            auto st = b200::partition_general(v);
            out.report.cleanup_retries = st.cleanup_retries;
            out.report.correct = verify_partition_result(in, v.snapshot());
            break;
        }
        case Algorithm::integer_sort_general: {
            auto st = b200::integer_sort_general(vp, u64(in.w) * in.m);
            out.report.cleanup_retries = st.cleanup_retries;
            out.report.correct = verify_sorted_result(in, vp.snapshot());
            break;
        }
        case Algorithm::permute: {
            Rng rng(out.report.seed);
            PermuteParams params;
            params.alpha = opt.alpha;
            auto rep = b200::permute(mach, rng, params);
            out.report.iterations = rep.iterations;
            out.report.fallback = rep.fallback;
            out.report.cleanup_retries = rep.cleanup_retries;
            out.pipeline = rep;
            std::vector<word> outgrid;
            outgrid.reserve(u64(in.w) * in.m);
            for (u32 i = 0; i < in.w; ++i)
                for (u32 j = 0; j < in.m; ++j)
                    outgrid.push_back(mach.peek(i, cfg.out_base() + j));
            out.report.correct = verify_permute_result(in, outgrid);
            break;
        }
    }
    // the reference's Machine::steps() where it does not depend on the data (0 otherwise)
    out.report.steps = dmm_modelled_steps(algorithm_name(alg), in.w, in.m);
    if (out.report.steps == 0 && (alg == Algorithm::partition_general || alg == Algorithm::integer_sort_general)) {
        // data-dependent leaf (dmm_leaf_steps) or the w > m recursion (dmm_general_steps): replay
        // the reference's states on the device
        std::vector<uint32_t> g(in.grid.begin(), in.grid.end());
        DeviceBuffer dg(sizeof(uint32_t) * g.size()), ds(sizeof(uint64_t));
        to_device(dg, g);
        const uint64_t domain = alg == Algorithm::partition_general ? in.w : u64(in.w) * in.m;
        const dmm_status ms =
            in.w <= in.m ? dmm_leaf_steps(dg.as<uint32_t>(), in.w, in.m, 1, domain, ds.as<uint64_t>(), nullptr)
                         : dmm_general_steps(dg.as<uint32_t>(), in.w, in.m, 1, domain, ds.as<uint64_t>(), nullptr,
                                             nullptr);
        if (ms == DMM_OK) {
            std::vector<uint64_t> st(1);
            to_host(st, ds);
            out.report.steps = st[0];
        }
    } else if (alg == Algorithm::permute) {
        // the permutation kernel's phase replay + the finish sort's meter
        std::vector<uint32_t> g(in.grid.begin(), in.grid.end());
        const uint64_t seed = out.report.seed;
        DeviceBuffer dg(sizeof(uint32_t) * g.size()), dsd(sizeof(uint64_t)), ds(sizeof(uint64_t));
        to_device(dg, g);
        cuda_check(cudaMemcpy(dsd.ptr, &seed, sizeof(seed), cudaMemcpyHostToDevice), "H2D");
        if (dmm_permute_steps(dg.as<uint32_t>(), in.w, in.m, 1, dsd.as<uint64_t>(), opt.alpha, 64,
                              ds.as<uint64_t>(), nullptr) == DMM_OK) {
            std::vector<uint64_t> st(1);
            to_host(st, ds);
            out.report.steps = st[0];
        }
    } else if (alg == Algorithm::sort_short_wide || alg == Algorithm::sort_square || alg == Algorithm::sort_tall) {
        std::vector<uint32_t> g(in.grid.size());
        for (std::size_t i = 0; i < g.size(); ++i)
            g[i] = static_cast<uint32_t>(in.grid[i]);  // 32-bit (checked by the sort above)
        DeviceBuffer dg(sizeof(uint32_t) * g.size()), ds(sizeof(uint64_t));
        to_device(dg, g);
        if (dmm_sort_steps(algorithm_name(alg), dg.as<uint32_t>(), in.w, in.m, 1, ds.as<uint64_t>(), nullptr) ==
            DMM_OK) {
            std::vector<uint64_t> st(1);
            to_host(st, ds);
            out.report.steps = st[0];
        }
    }
    out.report.work = out.report.steps * in.w;
    out.report.conflicts = 0;
    return out;
}

}  // namespace b200
}  // namespace dmm

// test_shim.cpp -- the reference's own API, run side by side on the CPU reference (dmm::)
// and on the B200 drop-in (dmm::b200::), in one process.  Built by tests/cpp/Makefile where
// /root/reference exists; run by tests/test_gpu_shim.py on the GPU box.  Cases follow the
// reference's tests (test_partition.cpp, test_permute.cpp, test_layout.cpp, test_sort.cpp).
#include <cstdio>
#include <cstdlib>
#include <functional>

#include "dmm_b200.hpp"

using namespace dmm;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (cond) {                                                        \
            ++g_pass;                                                      \
        } else {                                                           \
            ++g_fail;                                                      \
            std::fprintf(stderr, "FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
        }                                                                  \
    } while (0)

template <class E, class F>
static bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Machine make_machine(u32 w, u32 m) { return Machine(MachineConfig::standard(w, m)); }

static void partition_cases() {
    for (u32 m : {16u, 32u, 64u}) {
        for (u64 seed = 1; seed <= 6; ++seed) {
            Instance in = gen_instance(InstanceKind::partition, 32, m, seed);
            Machine a = make_machine(32, m), b = make_machine(32, m);
            MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
            va.load(in.grid);
            vb.load(in.grid);
            GeneralStats sa = partition_general(va);
            GeneralStats sb = b200::partition_general(vb);
            CHECK(va.snapshot() == vb.snapshot());
            CHECK(sa.cleanup_retries == sb.cleanup_retries && sa.sorted == sb.sorted);
            CHECK(verify_partition_result(in, vb.snapshot()));
        }
    }
    // shape violations raise the same type (partition.hpp:241-244, 443-445)
    {
        Instance in = gen_instance(InstanceKind::partition, 32, 8, 1);
        Machine b = make_machine(32, 8);
        MatrixView vb = MatrixView::full(b);
        vb.load(in.grid);
        CHECK(throws_as<ShapeViolation>([&] { b200::partition_general(vb); }));
        Machine a = make_machine(32, 8);
        MatrixView va = MatrixView::full(a);
        va.load(in.grid);
        CHECK(throws_as<ShapeViolation>([&] { partition_general(va); }));
    }
    // invalid instance (test_partition.cpp:110-115)
    {
        Instance in = gen_instance(InstanceKind::partition, 32, 16, 2);
        in.grid[0] = in.grid[0] == 3 ? 4 : 3;
        Machine b = make_machine(32, 16);
        MatrixView vb = MatrixView::full(b);
        vb.load(in.grid);
        CHECK(throws_as<InvalidInstance>([&] { b200::partition_general(vb); }));
    }
    // view transparency (test_sort.cpp:388-409): a 32-row view of a 64-row machine
    {
        Instance in = gen_instance(InstanceKind::partition, 32, 32, 9);
        Machine a = make_machine(64, 32), b = make_machine(64, 32);
        std::vector<u32> rows;
        for (u32 r = 0; r < 32; ++r)
            rows.push_back(2 * r + 1);  // odd banks
        MatrixView va = make_view(a, rows, 0, 32), vb = make_view(b, rows, 0, 32);
        va.load(in.grid);
        vb.load(in.grid);
        partition_general(va);
        b200::partition_general(vb);
        CHECK(va.snapshot() == vb.snapshot());
    }
}

static void integer_sort_cases() {
    for (u32 m : {16u, 32u, 128u}) {
        Instance in = gen_instance(InstanceKind::permute, 32, m, 5);
        Machine a = make_machine(32, m), b = make_machine(32, m);
        MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
        va.load(in.grid);
        vb.load(in.grid);
        GeneralStats sa = integer_sort_general(va, u64(32) * m);
        GeneralStats sb = b200::integer_sort_general(vb, u64(32) * m);
        CHECK(va.snapshot() == vb.snapshot());
        CHECK(sa.cleanup_retries == sb.cleanup_retries);
    }
    {  // uint32 keys, domain 2^32 (cfg3 path)
        Rng rng(77);
        std::vector<word> g(32 * 128);
        for (auto& x : g)
            x = rng() >> 32;
        Machine a = make_machine(32, 128), b = make_machine(32, 128);
        MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
        va.load(g);
        vb.load(g);
        integer_sort_general(va, u64(1) << 32);
        b200::integer_sort_general(vb, u64(1) << 32);
        CHECK(va.snapshot() == vb.snapshot());
    }
    {  // key outside the domain (test_partition.cpp:57-61)
        Instance in = gen_instance(InstanceKind::permute, 32, 16, 5);
        in.grid[7] = 9999;
        Machine b = make_machine(32, 16);
        MatrixView vb = MatrixView::full(b);
        vb.load(in.grid);
        CHECK(throws_as<KeyOutOfRange>([&] { b200::integer_sort_general(vb, 512); }));
    }
}

static void layout_and_sort_cases() {
    Rng rng(11);
    for (u32 m : {8u, 16u, 32u}) {
        std::vector<word> g(32 * m);
        for (auto& x : g)
            x = rng() >> 40;
        Machine a = make_machine(32, m), b = make_machine(32, m);
        MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
        va.load(g);
        vb.load(g);
        to_column_major(va);
        b200::to_column_major(vb);
        CHECK(va.snapshot() == vb.snapshot());
        to_row_major(va);
        b200::to_row_major(vb);
        CHECK(va.snapshot() == vb.snapshot() && vb.snapshot() == g);
        sort_tall(va);
        b200::sort_tall(vb);
        CHECK(va.snapshot() == vb.snapshot());
    }
    {
        std::vector<word> g(32 * 32);
        for (auto& x : g)
            x = rng() >> 40;
        Machine a = make_machine(32, 32), b = make_machine(32, 32);
        MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
        va.load(g);
        vb.load(g);
        transpose_square(va);
        b200::transpose_square(vb);
        CHECK(va.snapshot() == vb.snapshot());
    }
}

static void permute_cases() {
    for (u32 m : {32u, 16u, 4u, 2u}) {
        for (u64 seed = 1; seed <= 6; ++seed) {
            Instance in = gen_instance(InstanceKind::permute, 32, m, seed);
            Machine a = make_machine(32, m), b = make_machine(32, m);
            MatrixView va = MatrixView::make(a, [] { std::vector<u32> r(32); for (u32 i = 0; i < 32; ++i) r[i] = i; return r; }(),
                                             0, m, 2 * m, 3 * m);
            MatrixView vb = MatrixView::make(b, va.rows(), 0, m, 2 * m, 3 * m);
            va.load(in.grid);
            vb.load(in.grid);
            Rng ra(seed), rb(seed);
            // a caller that already consumed some draws: the drop-in must continue the stream
            for (u64 i = 0; i < seed; ++i) {
                ra();
                rb();
            }
            PermuteReport pa = permute(a, ra);
            PermuteReport pb = b200::permute(b, rb);
            CHECK(permute_output_correct(b));
            CHECK(pa.iterations == pb.iterations && pa.fallback == pb.fallback);
            CHECK(pa.used_packing == pb.used_packing && pa.packed_width == pb.packed_width);
            CHECK(pa.threshold == pb.threshold && pa.random_words == pb.random_words);
            CHECK(pa.cleanup_retries == pb.cleanup_retries);
            CHECK(pa.leftover_history == pb.leftover_history && pa.shifts == pb.shifts);
            CHECK(ra() == rb());  // the caller's Rng continues identically
            for (u32 i = 0; i < 32; ++i)
                for (u32 j = 0; j < m; ++j)
                    CHECK(a.peek(i, m + j) == b.peek(i, m + j));
        }
    }
    Machine bad = make_machine(32, 8);
    Rng r(1);
    CHECK(throws_as<ShapeViolation>([&] { b200::permute(bad, r); }));
}

// sub-warp machines (w < 32): the square / short-wide entry points exist only there
static void subwarp_cases() {
    // partition_square / partition_short_wide (partition.hpp:178-197); 64 x 64 is a two-warp machine
    for (auto [w, m] : {std::pair<u32, u32>{16, 16}, {4, 4}, {64, 64}, {8, 64}, {4, 16}, {2, 4}, {3, 9}}) {
        for (u64 seed = 1; seed <= 3; ++seed) {
            Instance in = gen_instance(InstanceKind::partition, w, m, seed);
            Machine a = make_machine(w, m), b = make_machine(w, m);
            MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
            va.load(in.grid);
            vb.load(in.grid);
            if (w == m) {
                partition_square(va);
                b200::partition_square(vb);
            } else {
                partition_short_wide(va);
                b200::partition_short_wide(vb);
            }
            CHECK(va.snapshot() == vb.snapshot());
        }
    }
    // general partition and integer sort at w in {16, 8, 4} with GeneralStats
    for (auto [w, m] : {std::pair<u32, u32>{16, 8}, {16, 32}, {8, 16}, {4, 8}, {64, 8}, {128, 64}}) {
        for (u64 seed = 1; seed <= 3; ++seed) {
            Instance in = gen_instance(InstanceKind::partition, w, m, seed);
            Machine a = make_machine(w, m), b = make_machine(w, m);
            MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
            va.load(in.grid);
            vb.load(in.grid);
            GeneralStats sa = partition_general(va);
            GeneralStats sb = b200::partition_general(vb);
            CHECK(va.snapshot() == vb.snapshot());
            CHECK(sa.cleanup_retries == sb.cleanup_retries && sa.sorted == sb.sorted);
        }
    }
    // comparison sorts: sort_square 16 x 16 / 4 x 4, sort_short_wide 8 x 64 / 4 x 16, both directions
    Rng rng(29);
    for (auto [w, m] : {std::pair<u32, u32>{16, 16}, {4, 4}, {64, 64}, {8, 64}, {4, 16}}) {
        for (bool asc : {true, false}) {
            std::vector<word> g(u64(w) * m);
            for (auto& x : g)
                x = rng() >> 40;
            Machine a = make_machine(w, m), b = make_machine(w, m);
            MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
            va.load(g);
            vb.load(g);
            if (w == m) {
                sort_square(va, asc);
                b200::sort_square(vb, asc);
            } else {
                sort_short_wide(va, asc);
                b200::sort_short_wide(vb, asc);
            }
            CHECK(va.snapshot() == vb.snapshot());
        }
    }
    // the same error types: bad label counts, w^2 > m
    {
        Instance in = gen_instance(InstanceKind::partition, 16, 16, 2);
        in.grid[0] = in.grid[0] == 15 ? 14 : 15;
        Machine b = make_machine(16, 16);
        MatrixView vb = MatrixView::full(b);
        vb.load(in.grid);
        CHECK(throws_as<InvalidInstance>([&] { b200::partition_square(vb); }));
        Machine c = make_machine(8, 32);
        MatrixView vc = MatrixView::full(c);
        CHECK(throws_as<ShapeViolation>([&] { b200::partition_short_wide(vc); }));
    }
}

// PartitionProbe hooks (partition.hpp:298-301): the same calls, depths, view shapes and
// machine contents at every call (modelled on test_partition.cpp:344-368)
static void probe_cases() {
    struct Event {
        int kind;
        u32 depth, nviews, view_w;
        std::vector<word> snap;
        bool operator==(const Event&) const = default;
    };
    for (auto [w, m] : {std::pair<u32, u32>{32, 16}, {16, 8}, {64, 16}, {256, 16}}) {
        for (u64 seed = 1; seed <= 4; ++seed) {
            Instance in = gen_instance(InstanceKind::partition, w, m, seed);
            std::vector<Event> ea, eb;
            Machine a = make_machine(w, m), b = make_machine(w, m);
            MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
            va.load(in.grid);
            vb.load(in.grid);
            auto probe_for = [](std::vector<Event>& ev, const MatrixView& whole) {
                PartitionProbe p;
                p.after_balance = [&ev, whole](u32 d, const std::vector<MatrixView>& lv) {
                    ev.push_back({0, d, u32(lv.size()), lv.front().W(), whole.snapshot()});
                };
                p.after_divide = [&ev, whole](u32 d, const std::vector<MatrixView>& lv) {
                    ev.push_back({1, d, u32(lv.size()), lv.front().W(), whole.snapshot()});
                };
                return p;
            };
            PartitionProbe pa = probe_for(ea, va), pb = probe_for(eb, vb);
            GeneralStats sa = partition_general(va, &pa);
            GeneralStats sb = b200::partition_general(vb, &pb);
            CHECK(!ea.empty() && ea == eb);
            CHECK(va.snapshot() == vb.snapshot());
            CHECK(sa.cleanup_retries == sb.cleanup_retries);
        }
    }
}

// run_algorithm (instance.hpp:277-363): the CLI / acceptance dispatch, every algorithm on a
// shape it accepts; the same report fields (steps: every meter but the permutation's)
static void run_algorithm_cases() {
    struct Case {
        Algorithm a;
        u32 w, m;
    };
    const Case cases[] = {{Algorithm::partition_general, 32, 16}, {Algorithm::partition_general, 64, 16},
                          {Algorithm::integer_sort_general, 32, 32}, {Algorithm::partition_square, 16, 16},
                          {Algorithm::partition_short_wide, 8, 64}, {Algorithm::partition_short_wide, 3, 9},
                          {Algorithm::sort_square, 16, 16}, {Algorithm::partition_general, 16, 16},
                          {Algorithm::integer_sort_general, 8, 64}, {Algorithm::partition_general, 32, 32},
                          {Algorithm::partition_general, 32, 64}, {Algorithm::integer_sort_general, 32, 128},
                          {Algorithm::sort_short_wide, 4, 16}, {Algorithm::sort_tall, 128, 32},
                          {Algorithm::permute, 32, 32}, {Algorithm::permute, 128, 64},
                          {Algorithm::partition_general, 64, 32}, {Algorithm::integer_sort_general, 64, 8},
                          // the w = 32 short-wide machine (32 x 1024: the CTA kernel, short_wide32.cu)
                          {Algorithm::partition_short_wide, 32, 1024}, {Algorithm::partition_general, 32, 1024},
                          {Algorithm::integer_sort_general, 32, 1024}};
    for (const Case& c : cases) {
        for (u64 seed = 1; seed <= 3; ++seed) {
            Instance in = gen_instance(instance_kind_for(c.a), c.w, c.m, seed);
            if (in.kind == InstanceKind::sort)
                for (auto& x : in.grid)
                    x >>= 32;  // the B200 layout narrows words to 32 bits (KeyOutOfRange otherwise)
            RunOutcome ra = run_algorithm(c.a, in), rb = b200::run_algorithm(c.a, in);
            CHECK(rb.report.correct && ra.report.correct);
            CHECK(ra.report.algorithm == rb.report.algorithm && ra.report.seed == rb.report.seed);
            CHECK(ra.report.cleanup_retries == rb.report.cleanup_retries);
            CHECK(ra.report.iterations == rb.report.iterations && ra.report.fallback == rb.report.fallback);
            if (dmm_modelled_steps(algorithm_name(c.a), c.w, c.m) || c.a == Algorithm::sort_short_wide ||
                c.a == Algorithm::permute ||
                c.a == Algorithm::sort_square || c.a == Algorithm::sort_tall ||
                c.a == Algorithm::partition_general || c.a == Algorithm::integer_sort_general)
                // modelled / replayed meters (w > m: dmm_general_steps)
                CHECK(ra.report.steps == rb.report.steps && ra.report.work == rb.report.work);
            if (c.a == Algorithm::permute) {
                CHECK(ra.pipeline.random_words == rb.pipeline.random_words);
                CHECK(ra.pipeline.leftover_history == rb.pipeline.leftover_history);
                CHECK(ra.pipeline.shifts == rb.pipeline.shifts);
            }
        }
    }
    CHECK(throws_as<KeyOutOfRange>(
        [&] { b200::run_algorithm(Algorithm::sort_tall, gen_instance(InstanceKind::sort, 128, 32, 1)); }));
    RunOptions tr;
    tr.record_trace = true;
    CHECK(throws_as<TraceIncomplete>(
        [&] { b200::run_algorithm(Algorithm::partition_general, gen_instance(InstanceKind::partition, 32, 16, 1), tr); }));
    CHECK(throws_as<InvalidInstance>(
        [&] { b200::run_algorithm(Algorithm::permute, gen_instance(InstanceKind::partition, 32, 16, 1)); }));
}

// ShortWideHook (sort.hpp:189-218): the same three calls with the same machine contents
static void short_wide_hook_cases() {
    for (auto [w, m] : {std::pair<u32, u32>{8, 64}, {4, 16}, {2, 8}, {3, 9}, {32, 1024}}) {
        for (int part = 0; part < 2; ++part) {
            for (bool asc : {true, false}) {
                if (part && !asc)
                    continue;
                Instance in = part ? gen_instance(InstanceKind::partition, w, m, 3)
                                   : gen_instance(InstanceKind::sort, w, m, 3);
                if (!part)
                    for (auto& x : in.grid)
                        x >>= 40;
                Machine a = make_machine(w, m), b = make_machine(w, m);
                MatrixView va = MatrixView::full(a), vb = MatrixView::full(b);
                va.load(in.grid);
                vb.load(in.grid);
                std::vector<std::pair<int, std::vector<word>>> ea, eb;
                ShortWideHook ha = [&](ShortWideStage st) { ea.push_back({int(st), va.snapshot()}); };
                ShortWideHook hb = [&](ShortWideStage st) { eb.push_back({int(st), vb.snapshot()}); };
                if (part) {
                    partition_short_wide(va, ha);
                    b200::partition_short_wide(vb, hb);
                } else {
                    sort_short_wide(va, asc, ha);
                    b200::sort_short_wide(vb, asc, hb);
                }
                CHECK(ea.size() == 3 && ea == eb);
                CHECK(va.snapshot() == vb.snapshot());
            }
        }
    }
}

static void schedule_cases() {
    // offline_schedule move for move, apply_schedule into the s0 window cell for cell
    Rng rng(19);
    for (auto [W, M] : {std::pair<u32, u32>{16, 8}, {32, 32}, {5, 7}, {4, 3}, {32, 64}}) {
        for (int t = 0; t < 4; ++t) {
            auto lin = random_permutation(rng, u64(W) * M);
            std::vector<std::pair<u32, u32>> perm(lin.size());
            for (std::size_t i = 0; i < lin.size(); ++i)
                perm[i] = {u32(lin[i] / M), u32(lin[i] % M)};
            Schedule a = offline_schedule(W, M, perm), b = b200::offline_schedule(W, M, perm);
            CHECK(schedule_to_text(a) == schedule_to_text(b));
            Machine ma = make_machine(W, M), mb = make_machine(W, M);
            MatrixView va = MatrixView::full(ma), vb = MatrixView::full(mb);
            std::vector<word> g(u64(W) * M);
            for (auto& x : g)
                x = rng() >> 33;
            va.load(g);
            vb.load(g);
            apply_schedule(va, a);
            b200::apply_schedule(vb, b);
            bool same = true;
            for (u32 r = 0; r < W; ++r)
                for (u32 c = 0; c < M; ++c)
                    same = same && ma.peek(r, va.s0(c)) == mb.peek(r, vb.s0(c));
            CHECK(same);
        }
    }
    {
        std::vector<std::pair<u32, u32>> bad(8, {0, 0});
        CHECK(throws_as<NotBijective>([&] { b200::offline_schedule(4, 2, bad); }));
        Machine mb = make_machine(4, 2);
        MatrixView vb = MatrixView::full(mb);
        Schedule clash;
        clash.rounds.push_back({{0, 0, 1, 0}, {0, 1, 2, 0}});
        CHECK(throws_as<ConflictViolation>([&] { b200::apply_schedule(vb, clash); }));
    }
}

int main() {
    partition_cases();
    integer_sort_cases();
    layout_and_sort_cases();
    subwarp_cases();
    probe_cases();
    run_algorithm_cases();
    short_wide_hook_cases();
    permute_cases();
    schedule_cases();
    std::printf("shim parity: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}

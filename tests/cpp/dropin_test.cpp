// dropin_test.cpp — exercises the C++ loadsched drop-in (include/loadsched_gpu.hpp)
// the way a reference caller would, against the reference's published answers
// (README demo, test goldens) and, in `dump` mode, writes the flat plan for the
// pytest driver (tests/test_gpu_cpp.py) to compare with the oracle.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "loadsched_gpu.hpp"

using namespace loadsched;

static int fails = 0, passes = 0;
#define EXPECT(cond)                                                        \
    do {                                                                    \
        if (cond) ++passes;                                                 \
        else { ++fails; std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); } \
    } while (0)

template <typename E, typename F>
static bool throws(F f) {
    try { f(); } catch (const E&) { return true; } catch (...) { return false; }
    return false;
}

static PipelineConfig demo() {
    PipelineConfig c;
    c.trace = {1024, 6, 4, 8, 7, true};  // README.md:74-87
    c.buffer_capacity = 64;
    return c;
}

static int run_checks() {
    // trace goldens (tests/test_trace.cpp:29-34)
    AccessTrace t = generate_trace({8, 2, 2, 2, 42, true});
    EXPECT(t.epochs.size() == 2);
    EXPECT((t.epochs[0] == std::vector<SampleId>{7, 4, 1, 2, 5, 6, 0, 3}));
    EXPECT((t.epochs[1] == std::vector<SampleId>{0, 5, 2, 6, 4, 1, 7, 3}));
    EXPECT(slice(t, 0, 0, 1) == (std::vector<SampleId>{1, 2}));
    EXPECT(throws<ConfigError>([] { generate_trace({3, 1, 2, 2, 0, true}); }));
    EXPECT(throws<ValidationError>([&] { slice(t, 2, 0, 0); }));
    // reuse graph golden (tests/test_reuse_graph.cpp:87-94)
    ReuseGraph g = build_reuse_graph(generate_trace({6, 3, 1, 2, 42, true}), 3, WindowMode::Global);
    EXPECT((g.weights == std::vector<std::uint64_t>{0, 1, 1, 1, 0, 2, 1, 2, 0}));
    AccessTrace t2 = generate_trace({6, 2, 2, 1, 42, true});
    EXPECT(build_reuse_graph(t2, 2, WindowMode::PerNode).weight(0, 1) == 4);
    // epoch order (tests/test_epoch_order.cpp:55-66)
    ReuseGraph ks;
    ks.num_epochs = 3;
    ks.weights = {0, 2, 5, 1, 0, 3, 4, 2, 0};
    EXPECT(path_cost(ks, {1, 2, 0}) == 7);
    EXPECT(throws<ValidationError>([&] { path_cost(ks, {0, 1, 1}); }));
    PsoParams bad;
    bad.inertia = 1.0;
    EXPECT(throws<ValidationError>([&] { pso_order(ks, bad); }));
    PsoResult pr = pso_order(ks, PsoParams{});
    EXPECT(pr.best.cost == 3 && (pr.best.order == std::vector<std::uint32_t>{2, 1, 0}));
    // the README demo end to end: order, plan, replay totals
    PipelineConfig c = demo();
    PlanOutput out = plan_schedule(c);
    EXPECT((out.plan.order.order == std::vector<std::uint32_t>{5, 2, 3, 0, 1, 4}));
    EXPECT(out.plan.order.cost == 939);
    EXPECT(out.pso.has_value());
    bool ms = true;
    for (const EpochPlan& ep : out.plan.epochs)
        for (std::size_t s = 0; s < ep.steps.size(); ++s)
            ms = ms && same_multiset(ep.steps[s].assignment, global_batch(out.trace, ep.epoch, s));
    EXPECT(ms);
    SimResult sim = simulate_plan(out.plan, 64, Policy::Clairvoyant);
    EXPECT(sim.total_misses == 4864 && sim.total_hits == 1280);
    EXPECT(sim.rows.size() == 6 * 32 * 4);
    // the README demo's baseline pass: LRU, identity order, slicing (README.md:87)
    const PipelineConfig base = baseline_config(c);
    EXPECT(base.policy == Policy::Lru && !base.optim_order && !base.optim_remap && !base.optim_balance);
    SimResult bs = simulate_plan(plan_schedule(base).plan, 64, Policy::Lru);
    EXPECT(bs.total_misses == 6109);
    // a buffer holding the whole dataset only cold-misses (tests/test_pipeline.cpp:164-173)
    PipelineConfig w;
    w.trace = {64, 3, 1, 8, 5, true};
    w.buffer_capacity = 64;
    SimResult ws = simulate_plan(plan_schedule(w).plan, 64, Policy::Clairvoyant);
    EXPECT(ws.total_misses == 64 && ws.total_hits == 3 * 64 - 64);
    // text artifacts: write -> read round trips (plan.cpp:44-214, trace.cpp:72-147)
    {
        const std::string pp = "/tmp/lsg_dropin_plan.txt", tp = "/tmp/lsg_dropin_trace.txt";
        write_plan_file(pp, out.plan);
        const SchedulePlan back = read_plan_file(pp);
        SimResult s2 = simulate_plan(back, 64, Policy::Clairvoyant);
        EXPECT(s2.total_misses == 4864 && s2.total_hits == 1280);
        EXPECT(back.order.order == out.plan.order.order && back.epochs.size() == out.plan.epochs.size());
        write_trace_file(tp, out.trace);
        const AccessTrace tb = read_trace_file(tp);
        EXPECT(tb.epochs == out.trace.epochs && tb.config.seed == 7);
        std::remove(pp.c_str());
        std::remove(tp.c_str());
        EXPECT(throws<StorageError>([&] { read_plan_file("/nonexistent/plan.txt"); }));
    }
    // the Store (tests/test_store.cpp:63-65 golden; :73-91 chunk == singles)
    {
        const std::string sp = "/tmp/lsg_dropin_store.bin";
        create_store(sp, 8, 16, 1);
        Store st(sp);
        EXPECT(st.sample_count() == 8 && st.sample_size() == 16 && st.header().version == 1);
        auto a = st.read_one(0), b2 = st.read_one(1);
        static const unsigned char gold[32] = {0xc1, 0x5c, 0x02, 0x89, 0xec, 0x2d, 0x0a, 0x91, 0x67, 0xec, 0x8e,
                                               0x65, 0xa1, 0x8d, 0xeb, 0xbe, 0x5e, 0x55, 0x32, 0xfb, 0xee, 0xa2,
                                               0x93, 0xf8, 0x0b, 0xc9, 0x42, 0xee, 0x90, 0x86, 0xc1, 0x71};
        EXPECT(std::memcmp(a.data(), gold, 16) == 0 && std::memcmp(b2.data(), gold + 16, 16) == 0);
        auto ch = st.read_chunk(2, 5);
        bool same = true;
        for (std::uint64_t i = 0; i < 5; ++i) {
            auto one = st.read_one(2 + i);
            same = same && std::memcmp(ch.data() + i * 16, one.data(), 16) == 0;
        }
        EXPECT(same);
        EXPECT(throws<ValidationError>([&] { st.read_one(8); }));
        EXPECT(throws<ValidationError>([&] { st.read_chunk(0, 0); }));
        EXPECT(throws<StorageError>([&] { Store bad("/nonexistent/lsg.bin"); }));
        EXPECT(throws<StorageError>([&] { create_store(sp, 0, 4, 1); }));
        std::remove(sp.c_str());
    }
    // chunk_insert_redundant with the LRU policy (silent touch_or_insert, buffer.cpp:88-91)
    PipelineConfig red = demo();
    red.chunk_insert_redundant = true;
    red.policy = Policy::Lru;
    PlanOutput lro = plan_schedule(red);
    SimResult lsim = simulate_plan(lro.plan, 64, Policy::Lru, true);
    EXPECT(lsim.total_hits + lsim.total_misses == 6 * 1024);
    // chunk_insert_redundant (pipeline.cpp:103-114) with the clairvoyant policy
    red.policy = Policy::Clairvoyant;
    PlanOutput ro = plan_schedule(red);
    SimResult rsim = simulate_plan(ro.plan, 64, Policy::Clairvoyant, true);
    EXPECT(rsim.total_hits + rsim.total_misses == 6 * 1024);
    std::printf("dropin_test: %d passed, %d failed\n", passes, fails);
    return fails ? 1 : 0;
}

// dump <dir> D E N b seed C drop_last optim_order optim_remap optim_balance graph_mode
static int dump(int argc, char** argv) {
    if (argc < 14) return 2;
    PipelineConfig c;
    c.trace = {std::stoull(argv[3]), std::uint32_t(std::stoul(argv[4])), std::uint32_t(std::stoul(argv[5])),
               std::stoull(argv[6]), std::stoull(argv[7]), std::stoi(argv[9]) != 0};
    c.buffer_capacity = std::stoull(argv[8]);
    c.optim_order = std::stoi(argv[10]) != 0;
    c.optim_remap = std::stoi(argv[11]) != 0;
    c.optim_balance = std::stoi(argv[12]) != 0;
    c.graph_mode = std::string(argv[13]) == "pernode" ? WindowMode::PerNode : WindowMode::Global;
    c.pso.max_iters = 50;
    PlanOutput out = plan_schedule(c);
    SimResult sim = simulate_plan(out.plan, c.buffer_capacity, Policy::Clairvoyant);
    const std::string dir = argv[2];
    std::ofstream items(dir + "/items.u32", std::ios::binary), off(dir + "/nodeoff.u32", std::ios::binary),
        rows(dir + "/rows.u32", std::ios::binary), ord(dir + "/order.u32", std::ios::binary);
    for (const EpochPlan& ep : out.plan.epochs)
        for (const StepPlan& st : ep.steps) {
            std::uint32_t o = 0;
            for (const auto& l : st.assignment.nodes) {
                off.write(reinterpret_cast<const char*>(&o), 4);
                for (const Assigned& a : l) {
                    const std::uint32_t v = std::uint32_t(a.id) | (a.source == Source::BufferHit ? 0x80000000u : 0u);
                    items.write(reinterpret_cast<const char*>(&v), 4);
                    ++o;
                }
            }
            off.write(reinterpret_cast<const char*>(&o), 4);
        }
    for (const StepNodeStats& r : sim.rows) {
        const std::uint32_t hm[2] = {std::uint32_t(r.hits), std::uint32_t(r.misses)};
        rows.write(reinterpret_cast<const char*>(hm), 8);
    }
    ord.write(reinterpret_cast<const char*>(out.plan.order.order.data()), 4 * out.plan.order.order.size());
    std::ofstream met(dir + "/metrics.csv");
    write_metrics(met, out.plan, sim, CostModel{});
    std::FILE* f = std::fopen((dir + "/costs.txt").c_str(), "w");
    std::fprintf(f, "%.6f %.6f\n", total_barrier_cost(out.plan, CostModel{}), total_io_cost(out.plan, CostModel{}));
    std::fclose(f);
    return 0;
}

// run_pipeline (pipeline.cpp:266-311) of the test_pipeline small config into
// argv[2]; the exit code is the error class (4 = CapabilityError for the
// out-of-scope summary.txt)
int run_pipeline_mode(char** argv) {
    PipelineConfig c;
    c.trace = {48, 4, 2, 4, 11, true};
    c.buffer_capacity = 8;
    try {
        (void)run_pipeline(c, argv[2]);
    } catch (const Error& e) {
        std::printf("%s\n", e.what());
        return int(e.error_class());
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 2 && std::strcmp(argv[1], "run_pipeline") == 0) return run_pipeline_mode(argv);
    try {
        if (argc > 1 && std::strcmp(argv[1], "dump") == 0) return dump(argc, argv);
        return run_checks();
    } catch (const Error& e) {
        std::fprintf(stderr, "loadsched error (class %d): %s\n", e.exit_code(), e.what());
        return e.exit_code();
    }
}

// oracle/ref_dump.cpp — TEST INFRASTRUCTURE ONLY.
//
// A driver linked against the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It runs the
// reference's own public API and dumps its outputs as raw little-endian arrays
// so tests can compare the CUDA path (and the C restatement) bit for bit, and
// so bench.py's reference arm can time the reference planner on host cores.
//
//   ref_dump plan     <outdir> key=value...   plan_schedule + simulate_plan
//   ref_dump simulate <indir>  C policy       simulate_plan over a dumped plan
//   ref_dump time     <samples> key=value...  stage timings (JSON on stdout)
//   ref_dump store    <out> count size seed   Store payload bytes (no header)
//   ref_dump storefile <path> count size seed  the reference's store file
//   ref_dump text <outdir> key=value...        trace.txt, graph.txt, plan.txt
//   ref_dump gather   <dir> count size n thr  Store::read_one batch-fetch timing
//
// key=value pairs go through the reference's apply_config_entry
// (proj/src/config.cpp) so their meaning is exactly the reference's.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <thread>
#include <vector>

#include "loadsched/buffer.hpp"
#include "loadsched/config.hpp"
#include "loadsched/errors.hpp"
#include "loadsched/pipeline.hpp"
#include "loadsched/prng.hpp"
#include "loadsched/store.hpp"

using namespace loadsched;

namespace {

template <typename T>
void dump(const std::string& path, const std::vector<T>& v) {
    std::ofstream out(path, std::ios::binary);
    out.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(T)));
    if (!out) throw StorageError("ref_dump: write failed " + path);
}

template <typename T>
std::vector<T> load(const std::string& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw StorageError("ref_dump: cannot open " + path);
    const std::streamsize n = in.tellg();
    in.seekg(0);
    std::vector<T> v(std::size_t(n) / sizeof(T));
    in.read(reinterpret_cast<char*>(v.data()), n);
    return v;
}

PipelineConfig parse_kv(int argc, char** argv, int first) {
    PipelineConfig cfg;
    for (int i = first; i < argc; ++i) {
        const std::string kv = argv[i];
        const auto eq = kv.find('=');
        if (eq == std::string::npos) throw ConfigError("ref_dump: expected key=value: " + kv);
        apply_config_entry(cfg, kv.substr(0, eq), kv.substr(eq + 1));
    }
    return cfg;
}

// Flatten a SchedulePlan into the CSR layout the CUDA path emits.
void dump_plan(const std::string& dir, const SchedulePlan& plan) {
    const std::uint32_t N = plan.num_nodes;
    std::vector<std::uint32_t> items, nodeoff, fb, fa, order(plan.order.order.begin(),
                                                             plan.order.order.end());
    for (const EpochPlan& ep : plan.epochs) {
        for (const StepPlan& st : ep.steps) {
            std::uint32_t off = 0;
            for (std::uint32_t k = 0; k < N; ++k) {
                nodeoff.push_back(off);
                for (const Assigned& a : st.assignment.nodes[k]) {
                    items.push_back(std::uint32_t(a.id) |
                                    (a.source == Source::BufferHit ? 0x80000000u : 0u));
                    ++off;
                }
            }
            nodeoff.push_back(off);
            for (std::uint32_t k = 0; k < N; ++k) {
                fb.push_back(std::uint32_t(st.fetches_before[k]));
                fa.push_back(std::uint32_t(st.fetches_after[k]));
            }
        }
    }
    // StepPlan::reads (chunking.cpp / pipeline.cpp:83-88) in the same layout:
    // list (g, k)'s reads at its item offsets
    std::vector<std::uint32_t> rstart(items.size(), 0), rend(items.size(), 0), rcount, rneed, rred;
    std::size_t base = 0, g = 0;
    for (const EpochPlan& ep : plan.epochs)
        for (const StepPlan& st : ep.steps) {
            for (std::uint32_t k = 0; k < N; ++k) {
                const std::size_t lo = base + nodeoff[g * (N + 1) + k];
                const ChunkPlan& cp = st.reads[k];
                for (std::size_t r = 0; r < cp.reads.size(); ++r) {
                    rstart[lo + r] = std::uint32_t(cp.reads[r].start);
                    rend[lo + r] = std::uint32_t(cp.reads[r].end);
                }
                rcount.push_back(std::uint32_t(cp.reads.size()));
                rneed.push_back(std::uint32_t(cp.needed));
                rred.push_back(std::uint32_t(cp.redundant));
            }
            base += nodeoff[g * (N + 1) + N];
            ++g;
        }
    dump(dir + "/rstart.u32", rstart);
    dump(dir + "/rend.u32", rend);
    dump(dir + "/rcount.u32", rcount);
    dump(dir + "/rneed.u32", rneed);
    dump(dir + "/rred.u32", rred);
    dump(dir + "/items.u32", items);
    dump(dir + "/nodeoff.u32", nodeoff);
    dump(dir + "/fb.u32", fb);
    dump(dir + "/fa.u32", fa);
    dump(dir + "/order.u32", order);
    dump(dir + "/cost.u64", std::vector<std::uint64_t>{plan.order.cost});
}

void dump_sim(const std::string& dir, const SimResult& sim) {
    std::vector<std::uint32_t> hits, misses;
    for (const StepNodeStats& r : sim.rows) {
        hits.push_back(std::uint32_t(r.hits));
        misses.push_back(std::uint32_t(r.misses));
    }
    dump(dir + "/hits.u32", hits);
    dump(dir + "/misses.u32", misses);
    dump(dir + "/simtot.u64", std::vector<std::uint64_t>{sim.total_hits, sim.total_misses});
}

// Shadow of the planner's residency (pipeline.cpp:90-102): replay the final
// plan through the reference Buffer with step-granular next-use keys and
// record, after every step, each node's resident count and an order-free
// digest (sum and xor of mix(id)). Valid when chunk_insert_redundant is off.
void dump_residency(const std::string& dir, const PipelineConfig& cfg, const PlanOutput& out) {
    const SchedulePlan& plan = out.plan;
    const std::uint32_t N = plan.num_nodes;
    std::vector<std::vector<std::uint64_t>> occ(plan.dataset_size);
    std::uint64_t g = 0;
    for (const EpochPlan& ep : plan.epochs)
        for (std::size_t t = 0; t < ep.steps.size(); ++t, ++g)
            for (const auto& list : ep.steps[t].assignment.nodes)
                for (const Assigned& a : list) occ[a.id].push_back(g);
    std::vector<std::size_t> cur(plan.dataset_size, 0);
    std::vector<std::unique_ptr<Buffer>> bufs;
    for (std::uint32_t k = 0; k < N; ++k) bufs.push_back(make_buffer(cfg.policy, cfg.buffer_capacity));
    std::vector<std::uint64_t> digest;
    g = 0;
    for (const EpochPlan& ep : plan.epochs) {
        for (std::size_t t = 0; t < ep.steps.size(); ++t, ++g) {
            for (std::uint32_t k = 0; k < N; ++k) {
                for (const Assigned& a : ep.steps[t].assignment.nodes[k]) {
                    auto& c = cur[a.id];
                    const std::uint64_t nu = c + 1 < occ[a.id].size() ? occ[a.id][c + 1] : kNeverUsed;
                    ++c;
                    bufs[k]->access(a.id, nu);
                }
            }
            for (std::uint32_t k = 0; k < N; ++k) {
                std::uint64_t sum = 0, x = 0;
                for (SampleId id : bufs[k]->resident()) {
                    std::uint64_t z = id + 0x9E3779B97F4A7C15ULL;
                    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
                    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
                    z ^= z >> 31;
                    sum += z;
                    x ^= z;
                }
                digest.push_back(bufs[k]->resident().size());
                digest.push_back(sum);
                digest.push_back(x);
            }
        }
    }
    dump(dir + "/residency.u64", digest);
}

int cmd_plan(int argc, char** argv) {
    const std::string dir = argv[2];
    const PipelineConfig cfg = parse_kv(argc, argv, 3);
    const PlanOutput out = plan_schedule(cfg);
    std::vector<std::uint32_t> trace;
    for (const auto& ep : out.trace.epochs)
        for (SampleId id : ep) trace.push_back(std::uint32_t(id));
    dump(dir + "/trace.u32", trace);
    dump(dir + "/graph.u64", out.graph.weights);
    if (out.pso) {
        dump(dir + "/hist.u64", out.pso->history);
        dump(dir + "/iters.u32", std::vector<std::uint32_t>{out.pso->iterations});
    }
    dump_plan(dir, out.plan);
    const bool redundant = cfg.chunk_insert_redundant && cfg.optim_chunk;
    dump_sim(dir, simulate_plan(out.plan, cfg.buffer_capacity, cfg.policy, redundant));
    // REF_DUMP_NO_RESIDENCY=1 skips the shadow replay (full-size golden runs)
    const char* nores = std::getenv("REF_DUMP_NO_RESIDENCY");
    if (!redundant && !(nores && nores[0] == '1')) dump_residency(dir, cfg, out);
    return 0;
}

// Rebuild a SchedulePlan from CSR arrays (steps listed in execution order,
// `spe` steps per epoch) and replay it.
int cmd_simulate(int argc, char** argv) {
    if (argc < 8) throw ValidationError("simulate <dir> N D spe C clairvoyant|lru");
    const std::string dir = argv[2];
    const std::uint32_t N = std::uint32_t(std::stoul(argv[3]));
    const std::uint64_t D = std::stoull(argv[4]);
    const std::uint64_t spe = std::stoull(argv[5]);
    const std::uint64_t C = std::stoull(argv[6]);
    const Policy policy = std::string(argv[7]) == "lru" ? Policy::Lru : Policy::Clairvoyant;
    const auto items = load<std::uint32_t>(dir + "/items.u32");
    const auto nodeoff = load<std::uint32_t>(dir + "/nodeoff.u32");
    const std::size_t T = nodeoff.size() / (N + 1);
    SchedulePlan plan;
    plan.dataset_size = D;
    plan.num_nodes = N;
    std::size_t base = 0;
    for (std::size_t g = 0; g < T; ++g) {
        if (g % spe == 0) plan.epochs.push_back(EpochPlan{std::uint32_t(g / spe), {}});
        StepPlan st;
        st.assignment.nodes.resize(N);
        for (std::uint32_t k = 0; k < N; ++k)
            for (std::uint32_t i = nodeoff[g * (N + 1) + k]; i < nodeoff[g * (N + 1) + k + 1]; ++i) {
                const std::uint32_t v = items[base + i];
                st.assignment.nodes[k].push_back(
                    {v & 0x7FFFFFFFu, (v >> 31) ? Source::BufferHit : Source::PfsFetch});
            }
        base += nodeoff[g * (N + 1) + N];
        plan.epochs.back().steps.push_back(std::move(st));
    }
    dump_sim(dir, simulate_plan(plan, C, policy, false));
    return 0;
}

double secs(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Stage timings of the reference planner on one host core (bench.py's
// reference arm and cpu_baseline). `samples` repeats the whole plan.
int cmd_time(int argc, char** argv) {
    const int reps = std::stoi(argv[2]);
    const PipelineConfig cfg = parse_kv(argc, argv, 3);
    double t_trace = 0, t_graph = 0, t_pso = 0, t_plan = 0, t_sim = 0;
    std::uint64_t accesses = 0, misses = 0;
    // REF_DUMP_STAGES=0: time plan_schedule + simulate_plan only (the stage
    // split re-runs trace, graph and PSO outside plan_schedule)
    const char* stg = std::getenv("REF_DUMP_STAGES");
    const bool stages = !(stg && stg[0] == '0');
    for (int r = 0; r < reps; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        if (stages) {
            const AccessTrace trace = generate_trace(cfg.trace);
            t_trace += secs(t0);
            t0 = std::chrono::steady_clock::now();
            const ReuseGraph graph = build_reuse_graph(trace, cfg.buffer_capacity, cfg.graph_mode);
            t_graph += secs(t0);
            if (cfg.optim_order) {
                PsoParams p = cfg.pso;
                p.seed = cfg.trace.seed;
                t0 = std::chrono::steady_clock::now();
                (void)pso_order(graph, p);
                t_pso += secs(t0);
            }
        }
        t0 = std::chrono::steady_clock::now();
        const PlanOutput out = plan_schedule(cfg); // repeats trace/graph/pso internally
        t_plan += secs(t0);
        t0 = std::chrono::steady_clock::now();
        const SimResult sim = simulate_plan(out.plan, cfg.buffer_capacity, cfg.policy,
                                            cfg.chunk_insert_redundant && cfg.optim_chunk);
        t_sim += secs(t0);
        accesses += sim.total_hits + sim.total_misses;
        misses += sim.total_misses;
    }
    std::printf("{\"reps\": %d, \"trace_s\": %.6f, \"graph_s\": %.6f, \"pso_s\": %.6f, "
                "\"plan_schedule_s\": %.6f, \"simulate_s\": %.6f, \"accesses\": %llu, "
                "\"misses\": %llu}\n",
                reps, t_trace, t_graph, t_pso, t_plan, t_sim, (unsigned long long)accesses,
                (unsigned long long)misses);
    return 0;
}

// Batch fetch through the reference's own Store::read_one (store.cpp:134-139)
// from a page-cached store file: `reps` rounds of `nreads` random samples
// split over `threads` host threads (Store is documented safe for concurrent
// reads, store.hpp:29-30). Prints JSON with every round's seconds.
int cmd_gather(int argc, char** argv) {
    if (argc < 7) throw ValidationError("gather <dir> count size nreads threads [reps]");
    const std::string path = std::string(argv[2]) + "/ref_gather_store.bin";
    const std::uint64_t count = std::stoull(argv[3]), size = std::stoull(argv[4]);
    const std::uint64_t nreads = std::stoull(argv[5]);
    const unsigned threads = unsigned(std::stoul(argv[6]));
    const int reps = argc > 7 ? std::stoi(argv[7]) : 1;
    create_store(path, count, size, 1, ~0ULL);
    Store store(path);
    for (std::uint64_t i = 0; i < count; ++i) (void)store.read_one(i);  // page-cache warm
    SplitMix64 rng(7);
    std::vector<double> secs_per_rep;
    std::uint64_t chk = 0;
    for (int r = 0; r < reps; ++r) {
        std::vector<std::uint64_t> ids(nreads);
        for (auto& v : ids) v = rng.next_below(count);
        std::vector<std::thread> pool;
        std::vector<std::uint64_t> sink(threads, 0);
        const auto t0 = std::chrono::steady_clock::now();
        for (unsigned t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                for (std::uint64_t i = t; i < nreads; i += threads) {
                    const auto bytes = store.read_one(ids[i]);
                    sink[t] += std::to_integer<unsigned>(bytes[i % bytes.size()]);
                }
            });
        for (auto& th : pool) th.join();
        secs_per_rep.push_back(secs(t0));
        for (auto v : sink) chk += v;
    }
    std::remove(path.c_str());
    std::printf("{\"seconds\": %.6f, \"samples\": %llu, \"bytes\": %llu, \"threads\": %u, \"chk\": %llu, \"reps\": [",
                secs_per_rep.back(), (unsigned long long)nreads, (unsigned long long)(nreads * size), threads,
                (unsigned long long)chk);
    for (std::size_t i = 0; i < secs_per_rep.size(); ++i) std::printf("%s%.6f", i ? ", " : "", secs_per_rep[i]);
    std::printf("]}\n");
    return 0;
}

int cmd_store(int argc, char** argv) {
    if (argc < 6) throw ValidationError("store <out> count size seed");
    const std::string path = std::string(argv[2]) + ".store";
    create_store(path, std::stoull(argv[3]), std::stoull(argv[4]), std::stoull(argv[5]), ~0ULL);
    Store s(path);
    std::vector<std::uint8_t> all;
    for (std::uint64_t i = 0; i < s.sample_count(); ++i) {
        auto one = s.read_one(i);
        for (std::byte b : one) all.push_back(std::uint8_t(b));
    }
    dump(std::string(argv[2]), all);
    std::remove(path.c_str());
    return 0;
}

// run the reference's reader on a file: prints "ok ..." or "error <class> <msg>"
int cmd_read(int argc, char** argv) {
    const std::string kind = argv[2], path = argv[3];
    try {
        if (kind == "trace") {
            const AccessTrace t = read_trace_file(path);
            std::printf("ok %zu\n", t.epochs.size());
        } else if (kind == "graph") {
            const ReuseGraph g = read_graph_file(path);
            std::printf("ok %u\n", g.num_epochs);
        } else {
            const SchedulePlan p = read_plan_file(path);
            std::printf("ok %zu\n", p.epochs.size());
        }
    } catch (const Error& e) {
        std::printf("error %d %s\n", e.exit_code(), e.what());
    } catch (const std::exception& e) {
        std::printf("error 7 %s\n", e.what());
    }
    return 0;
}

// the reference's own text artifacts of a plan_schedule run:
// <dir>/trace.txt, graph.txt, plan.txt (write_*_file)
int cmd_text(int argc, char** argv) {
    const std::string dir = argv[2];
    const PipelineConfig cfg = parse_kv(argc, argv, 3);
    const PlanOutput out = plan_schedule(cfg);
    write_trace_file(dir + "/trace.txt", out.trace);
    write_graph_file(dir + "/graph.txt", out.graph);
    write_plan_file(dir + "/plan.txt", out.plan);
    // metrics.csv as run_pipeline writes it (pipeline.cpp:153-179, 193-196)
    const SimResult sim = simulate_plan(out.plan, cfg.buffer_capacity, cfg.policy,
                                        cfg.chunk_insert_redundant && cfg.optim_chunk);
    std::ofstream m(dir + "/metrics.csv");
    write_metrics(m, out.plan, sim, CostModel{});
    std::FILE* f = std::fopen((dir + "/costs.txt").c_str(), "w");
    std::fprintf(f, "%.6f %.6f\n", total_barrier_cost(out.plan, CostModel{}), total_io_cost(out.plan, CostModel{}));
    std::fclose(f);
    // the same totals under the config's cost model, every bit (%a)
    f = std::fopen((dir + "/costs_exact.txt").c_str(), "w");
    std::fprintf(f, "%a %a\n", total_barrier_cost(out.plan, cfg.model), total_io_cost(out.plan, cfg.model));
    std::fclose(f);
    return 0;
}

// run_pipeline (pipeline.cpp:266-311) of test_pipeline.cpp's small config
// into <dir> (every artifact, summary.txt included)
int cmd_runpipe(int argc, char** argv) {
    if (argc < 3) throw ValidationError("runpipe <dir>");
    PipelineConfig c;
    c.trace = {48, 4, 2, 4, 11, true};
    c.buffer_capacity = 8;
    (void)run_pipeline(c, argv[2]);
    return 0;
}

// the reference's create_store output itself (header + payload) at <path>
int cmd_storefile(int argc, char** argv) {
    if (argc < 6) throw ValidationError("storefile <path> count size seed");
    create_store(argv[2], std::stoull(argv[3]), std::stoull(argv[4]), std::stoull(argv[5]), ~0ULL);
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: ref_dump plan|simulate|time|store ...\n");
        return 1;
    }
    try {
        const std::string cmd = argv[1];
        if (cmd == "plan") return cmd_plan(argc, argv);
        if (cmd == "simulate") return cmd_simulate(argc, argv);
        if (cmd == "time") return cmd_time(argc, argv);
        if (cmd == "store") return cmd_store(argc, argv);
        if (cmd == "storefile") return cmd_storefile(argc, argv);
        if (cmd == "text") return cmd_text(argc, argv);
        if (cmd == "read") return cmd_read(argc, argv);
        if (cmd == "gather") return cmd_gather(argc, argv);
        if (cmd == "runpipe") return cmd_runpipe(argc, argv);
        std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
        return 1;
    } catch (const Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return e.exit_code();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 7;
    }
}

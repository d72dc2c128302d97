// loadsched_gpu.cpp — the C++ `loadsched` API (include/loadsched_gpu.hpp) over
// the lsg C ABI. Host code here only converts layouts (uint64 vectors <-> the
// flat uint32 device layout), moves data, and maps status codes to the
// reference's exception classes (errors.hpp:10-46); every computation on the
// planner path runs in the CUDA library.
#include "loadsched_gpu.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <memory>
#include <numeric>
#include <unordered_map>
#include <unordered_set>
#include <iterator>

#include "lsg.h"

namespace loadsched {

namespace {

[[noreturn]] void throw_class(int rc, const std::string& msg) {
    switch (rc) {
        case 2: throw ConfigError(msg);
        case 3: throw ValidationError(msg);
        case 4: throw CapabilityError(msg);
        case 6: throw StorageError(msg);
        default: throw InternalError(msg);
    }
}

void check(int rc) {
    if (rc != 0) throw_class(rc, lsg_last_error());
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw InternalError(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
template <typename T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(std::size_t n) { cuda_check(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void upload(const T* h, std::size_t n) { cuda_check(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D"); }
    void download(T* h, std::size_t n) const { cuda_check(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H"); }
};

lsg_config to_c(const PipelineConfig& c) {
    lsg_config o{};
    o.dataset_size = c.trace.dataset_size;
    o.num_epochs = c.trace.num_epochs;
    o.num_nodes = c.trace.num_nodes;
    o.local_batch = c.trace.local_batch;
    o.seed = c.trace.seed;
    o.drop_last = c.trace.drop_last ? 1 : 0;
    o.policy = c.policy == Policy::Clairvoyant ? 0 : 1;
    o.buffer_capacity = c.buffer_capacity;
    o.graph_mode = c.graph_mode == WindowMode::Global ? 0 : 1;
    o.insert_redundant = c.chunk_insert_redundant ? 1 : 0;
    o.chunk_threshold = c.chunk_threshold;
    o.optim_order = c.optim_order;
    o.optim_remap = c.optim_remap;
    o.optim_balance = c.optim_balance;
    o.optim_chunk = c.optim_chunk;
    o.pso_swarm = c.pso.swarm_size;
    o.pso_iters = c.pso.max_iters;
    o.pso_stagnation = c.pso.stagnation_limit;
    o.pso_restart = c.pso.restart_limit;
    o.pso_p_personal = c.pso.p_personal;
    o.pso_p_global = c.pso.p_global;
    o.pso_inertia = c.pso.inertia;
    o.pso_kick = c.pso.kick;
    return o;
}

std::uint64_t keep_of(const TraceConfig& t) {
    return t.drop_last ? t.steps_per_epoch() * t.global_batch() : t.dataset_size;
}

}  // namespace

// trace.cpp:12-24 semantics
std::uint64_t TraceConfig::steps_per_epoch() const {
    const std::uint64_t B = global_batch();
    if (B == 0) return 0;
    return drop_last ? dataset_size / B : (dataset_size + B - 1) / B;
}

void TraceConfig::validate() const {
    PipelineConfig p;
    p.trace = *this;
    p.buffer_capacity = 1;
    const lsg_config c = to_c(p);
    lsg_shape sh;
    check(lsg_shape_of(&c, &sh));
}

void PipelineConfig::validate() const {
    // config.cpp:11-23 order: trace, buffer, chunk threshold, cost model, PSO
    PipelineConfig head = *this;
    head.pso = PsoParams{};
    const lsg_config c0 = to_c(head);
    lsg_shape sh;
    check(lsg_shape_of(&c0, &sh));
    if (model.seek_cost < 0.0 || model.stream_cost < 0.0) throw ConfigError("seek_cost and stream_cost must be >= 0");
    const lsg_config c = to_c(*this);
    check(lsg_shape_of(&c, &sh));
}

AccessTrace generate_trace(const TraceConfig& config) {
    PipelineConfig p;
    p.trace = config;
    p.buffer_capacity = 1;
    const lsg_config c = to_c(p);
    if (config.num_nodes == 0 || config.local_batch == 0 || config.num_epochs == 0 ||
        config.dataset_size < config.global_batch())
        check(lsg_generate_trace(&c, nullptr, nullptr));  // reports the ConfigError
    const std::uint64_t keep = keep_of(config), E = config.num_epochs;
    DevBuf<std::uint32_t> d(E * keep);
    check(lsg_generate_trace(&c, d.p, nullptr));
    std::vector<std::uint32_t> h(E * keep);
    d.download(h.data(), h.size());
    AccessTrace t;
    t.config = config;
    t.epochs.resize(E);
    for (std::uint64_t e = 0; e < E; ++e) t.epochs[e].assign(h.begin() + e * keep, h.begin() + (e + 1) * keep);
    return t;
}

// trace.cpp:45-70 (views of host data)
std::vector<SampleId> slice(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t step, std::uint32_t node) {
    const TraceConfig& c = trace.config;
    if (epoch >= trace.epochs.size()) throw ValidationError("slice: epoch out of range");
    if (step >= c.steps_per_epoch()) throw ValidationError("slice: step out of range");
    if (node >= c.num_nodes) throw ValidationError("slice: node out of range");
    const auto& seq = trace.epochs[epoch];
    const std::uint64_t lo = std::min<std::uint64_t>(step * c.global_batch() + std::uint64_t(node) * c.local_batch, seq.size());
    const std::uint64_t hi = std::min<std::uint64_t>(lo + c.local_batch, seq.size());
    return std::vector<SampleId>(seq.begin() + lo, seq.begin() + std::max(lo, hi));
}

std::vector<SampleId> global_batch(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t step) {
    const TraceConfig& c = trace.config;
    if (epoch >= trace.epochs.size()) throw ValidationError("global_batch: epoch out of range");
    if (step >= c.steps_per_epoch()) throw ValidationError("global_batch: step out of range");
    const auto& seq = trace.epochs[epoch];
    const std::uint64_t lo = std::min<std::uint64_t>(step * c.global_batch(), seq.size());
    const std::uint64_t hi = std::min<std::uint64_t>(lo + c.global_batch(), seq.size());
    return std::vector<SampleId>(seq.begin() + lo, seq.begin() + hi);
}

ReuseGraph build_reuse_graph(const AccessTrace& trace, std::uint64_t buffer_size, WindowMode mode) {
    const std::uint32_t E = std::uint32_t(trace.epochs.size());
    const std::uint64_t len = trace.epoch_length();
    std::vector<std::uint32_t> flat(std::size_t(E) * len);
    for (std::uint32_t e = 0; e < E; ++e) {
        if (trace.epochs[e].size() != len) throw ValidationError("build_reuse_graph: ragged trace");
        for (std::uint64_t i = 0; i < len; ++i) {
            const SampleId x = trace.epochs[e][i];
            if (x >= trace.config.dataset_size) throw ValidationError("build_reuse_graph: id out of range");
            flat[std::size_t(e) * len + i] = std::uint32_t(x);
        }
    }
    DevBuf<std::uint32_t> dt(flat.size());
    dt.upload(flat.data(), flat.size());
    DevBuf<std::uint64_t> dw(std::size_t(E) * E);
    check(lsg_build_reuse_graph(dt.p, E, len, trace.config.dataset_size, trace.config.num_nodes,
                                trace.config.local_batch, trace.config.drop_last ? 1 : 0, buffer_size,
                                mode == WindowMode::Global ? 0 : 1, dw.p, nullptr));
    ReuseGraph g;
    g.num_epochs = E;
    g.buffer_size = buffer_size;
    g.mode = mode;
    g.weights.resize(std::size_t(E) * E);
    cuda_check(cudaDeviceSynchronize(), "sync");
    dw.download(g.weights.data(), g.weights.size());
    return g;
}

namespace {
// K2 windows of `epoch` as id sets (reuse_graph.cpp:43-56)
std::vector<IdSet> buffer_window(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t buffer_size,
                                 WindowMode mode, bool first) {
    if (epoch >= trace.epochs.size()) throw ValidationError("buffer window: epoch out of range");
    if (buffer_size == 0) throw ValidationError("buffer window: buffer_size must be >= 1");
    const TraceConfig& c = trace.config;
    const std::uint64_t len = trace.epochs[epoch].size();
    std::vector<std::uint32_t> flat(std::max<std::uint64_t>(len, 1));
    for (std::uint64_t i = 0; i < len; ++i) {
        const SampleId x = trace.epochs[epoch][i];
        if (x >= (1ull << 31) || x >= c.dataset_size) throw CapabilityError("buffer window: ids must be < dataset_size");
        flat[i] = std::uint32_t(x);
    }
    const std::uint32_t W = mode == WindowMode::Global ? 1u : c.num_nodes;
    const std::uint64_t words = (c.dataset_size + 31) / 32;
    DevBuf<std::uint32_t> dt(flat.size()), df(W * words), dl(W * words);
    dt.upload(flat.data(), flat.size());
    check(lsg_buffer_windows(dt.p, 1, len, c.dataset_size, c.num_nodes, c.local_batch, c.drop_last ? 1 : 0,
                             buffer_size, mode == WindowMode::Global ? 0 : 1, df.p, dl.p, nullptr));
    std::vector<std::uint32_t> bits(W * words);
    cuda_check(cudaDeviceSynchronize(), "sync");
    (first ? df : dl).download(bits.data(), bits.size());
    std::vector<IdSet> out(W);
    for (std::uint32_t k = 0; k < W; ++k)
        for (std::uint64_t w = 0; w < words; ++w)
            for (std::uint32_t v = bits[k * words + w]; v; v &= v - 1) out[k].insert(w * 32 + __builtin_ctz(v));
    return out;
}
}  // namespace

std::vector<IdSet> last_buffer_window(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t buffer_size,
                                      WindowMode mode) {
    return buffer_window(trace, epoch, buffer_size, mode, false);
}

std::vector<IdSet> first_buffer_window(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t buffer_size,
                                       WindowMode mode) {
    return buffer_window(trace, epoch, buffer_size, mode, true);
}

// epoch_order.cpp:32-52 on the device (all E! paths, E <= 10)
EpochOrder brute_force_order(const ReuseGraph& graph) {
    const std::uint32_t E = graph.num_epochs;
    DevBuf<std::uint64_t> dw(std::size_t(E) * E + 1), dc(1);
    DevBuf<std::uint32_t> dord(E + 1);
    if (E) dw.upload(graph.weights.data(), std::size_t(E) * E);
    check(lsg_brute_force_order(dw.p, E, dord.p, dc.p, nullptr));
    EpochOrder r;
    r.order.resize(E);
    cuda_check(cudaDeviceSynchronize(), "sync");
    dord.download(r.order.data(), E);
    dc.download(&r.cost, 1);
    return r;
}

// chunking.cpp:9-33 through the device read planner
ChunkPlan plan_chunks(const std::vector<SampleId>& fetch_ids, std::uint64_t threshold) {
    std::vector<std::uint32_t> ids(fetch_ids.size());
    for (std::size_t i = 0; i < ids.size(); ++i) {
        if (fetch_ids[i] >= (1ull << 31)) throw CapabilityError("plan_chunks: sample ids must be < 2^31 on device");
        ids[i] = std::uint32_t(fetch_ids[i]);
    }
    std::vector<std::uint32_t> rs(ids.size() + 1), re(ids.size() + 1);
    std::uint64_t meta[3];
    check(lsg_plan_chunks(ids.data(), ids.size(), threshold, rs.data(), re.data(), meta, nullptr));
    ChunkPlan p;
    for (std::uint64_t i = 0; i < meta[0]; ++i)
        p.reads.push_back({rs[i] == re[i] ? Read::Kind::Single : Read::Kind::Chunk, rs[i], re[i]});
    p.needed = meta[1];
    p.redundant = meta[2];
    return p;
}

namespace {

StepAssignment step_from_lists(const std::vector<std::uint32_t>& items, const std::vector<std::uint32_t>& off,
                               std::size_t N) {
    StepAssignment step;
    step.nodes.resize(N);
    for (std::size_t k = 0; k < N; ++k)
        for (std::uint32_t p = off[k]; p < off[k + 1]; ++p)
            step.nodes[k].push_back({items[p] & ~LSG_HIT_BIT, (items[p] & LSG_HIT_BIT) ? Source::BufferHit : Source::PfsFetch});
    return step;
}

StepAssignment locality_step(const std::vector<const IdSet*>& buffers, const std::vector<SampleId>& batch,
                             std::uint64_t local_batch, bool slice) {
    const char* who = slice ? "slice_step" : "remap_step";
    const std::size_t N = buffers.size();
    std::vector<std::uint64_t> roff(N + 1, 0);
    std::vector<std::uint32_t> rids;
    for (std::size_t k = 0; k < N; ++k) {
        for (SampleId id : *buffers[k]) {
            if (id >= (1ull << 31)) throw CapabilityError(std::string(who) + ": sample ids must be < 2^31 on device");
            rids.push_back(std::uint32_t(id));
        }
        roff[k + 1] = rids.size();
    }
    std::vector<std::uint32_t> ids(batch.size());
    for (std::size_t i = 0; i < batch.size(); ++i) {
        if (batch[i] >= (1ull << 31)) throw CapabilityError(std::string(who) + ": sample ids must be < 2^31 on device");
        ids[i] = std::uint32_t(batch[i]);
    }
    std::vector<std::uint32_t> items(ids.size() + 1), off(N + 1, 0);
    check(lsg_remap_step(roff.data(), rids.data(), std::uint32_t(N), ids.data(), ids.size(), local_batch,
                         slice ? 1 : 0, items.data(), off.data(), nullptr));
    StepAssignment step = step_from_lists(items, off, N);
    if (!slice && !same_multiset(step, batch)) throw InternalError("remap_step: assignment multiset mismatch");
    return step;
}

}  // namespace

// locality.cpp:7-39
StepAssignment remap_step(const std::vector<const IdSet*>& buffers, const std::vector<SampleId>& batch,
                          std::uint64_t local_batch) {
    return locality_step(buffers, batch, local_batch, false);
}

// locality.cpp:41-54: every step against one fixed residency snapshot
std::vector<StepAssignment> remap_epoch(const std::vector<IdSet>& prev_buffers,
                                        const std::vector<std::vector<SampleId>>& epoch_batches,
                                        std::uint64_t local_batch) {
    std::vector<const IdSet*> views;
    for (const IdSet& s : prev_buffers) views.push_back(&s);
    std::vector<StepAssignment> out;
    out.reserve(epoch_batches.size());
    for (const auto& batch : epoch_batches) out.push_back(remap_step(views, batch, local_batch));
    return out;
}

// locality.cpp:56-73
StepAssignment slice_step(const std::vector<const IdSet*>& buffers, const std::vector<SampleId>& batch,
                          std::uint64_t local_batch) {
    return locality_step(buffers, batch, local_batch, true);
}

// balance.cpp:10-39
std::uint64_t balance_step(StepAssignment& step) {
    const std::size_t N = step.nodes.size();
    if (N == 0) throw ValidationError("balance_step: no nodes");
    std::vector<std::uint32_t> items, off(N + 1, 0);
    for (std::size_t k = 0; k < N; ++k) {
        for (const Assigned& a : step.nodes[k]) {
            if (a.id >= (1ull << 31)) throw CapabilityError("balance_step: sample ids must be < 2^31 on device");
            items.push_back(std::uint32_t(a.id) | (a.source == Source::BufferHit ? LSG_HIT_BIT : 0u));
        }
        off[k + 1] = std::uint32_t(items.size());
    }
    std::uint64_t moves = 0;
    items.push_back(0);
    check(lsg_balance_step(items.data(), off.data(), std::uint32_t(N), &moves, nullptr));
    step = step_from_lists(items, off, N);
    return moves;
}

// barrier_time (balance.cpp:41-47): the step waits for its most loaded node.
// Costs are monotone in the count (per_fetch >= 0 for any model the
// reference accepts), so the slowest node is the one with the most fetches.
double barrier_time(const StepAssignment& step, const CostModel& model) {
    const auto counts = step.fetch_counts();
    if (counts.empty()) return 0.0;
    const std::uint64_t most = *std::max_element(counts.begin(), counts.end());
    return std::max(0.0, double(most) * (model.seek_cost + model.stream_cost));
}

// batch_size_stats (balance.cpp:51-72): population standard deviation of the
// per-node list lengths of every step (left-to-right sums, as the reference)
std::vector<StepSizes> batch_size_stats(const SchedulePlan& plan) {
    std::vector<StepSizes> stats;
    for (const EpochPlan& ep : plan.epochs) {
        std::uint64_t t = 0;
        for (const StepPlan& sp : ep.steps) {
            StepSizes s{ep.epoch, t++, {}, 0.0};
            std::transform(sp.assignment.nodes.begin(), sp.assignment.nodes.end(), std::back_inserter(s.sizes),
                           [](const auto& list) { return std::uint64_t(list.size()); });
            const double n = double(s.sizes.size());
            const double mu = std::accumulate(s.sizes.begin(), s.sizes.end(), 0.0,
                                              [](double acc, std::uint64_t v) { return acc + double(v); }) / n;
            const double ss = std::accumulate(s.sizes.begin(), s.sizes.end(), 0.0, [mu](double acc, std::uint64_t v) {
                const double d = double(v) - mu;
                return acc + d * d;
            });
            s.stddev = std::sqrt(ss / n);
            stats.push_back(std::move(s));
        }
    }
    return stats;
}

// ---- buffer.cpp:10-98 on the device (buffer_api.cu) ------------------------
Buffer::Buffer(Policy policy, std::uint64_t capacity) : capacity_(capacity) {
    if (capacity == 0) throw ValidationError("buffer capacity must be >= 1");
    lsg_buffer* h = nullptr;
    check(lsg_buffer_create(policy == Policy::Lru ? 1 : 0, capacity, &h));
    handle_ = h;
}

Buffer::~Buffer() { lsg_buffer_destroy(static_cast<lsg_buffer*>(handle_)); }

bool Buffer::access(SampleId id, std::uint64_t next_use) {
    std::uint8_t hit = 0;
    check(lsg_buffer_access(static_cast<lsg_buffer*>(handle_), &id, &next_use, 1, 0, &hit, nullptr));
    stale_ = true;
    return hit != 0;
}

std::vector<bool> Buffer::access_batch(const std::vector<SampleId>& ids, const std::vector<std::uint64_t>& next_use) {
    if (ids.size() != next_use.size()) throw ValidationError("access_batch: ids and next_use differ in length");
    std::vector<std::uint8_t> hit(ids.size());
    check(lsg_buffer_access(static_cast<lsg_buffer*>(handle_), ids.data(), next_use.data(), ids.size(), 0,
                            hit.data(), nullptr));
    stale_ = true;
    return std::vector<bool>(hit.begin(), hit.end());
}

void Buffer::insert_silent(SampleId id, std::uint64_t next_use) {
    check(lsg_buffer_access(static_cast<lsg_buffer*>(handle_), &id, &next_use, 1, 1, nullptr, nullptr));
    stale_ = true;
}

void Buffer::clear() {
    check(lsg_buffer_clear(static_cast<lsg_buffer*>(handle_)));
    stale_ = true;
}

const IdSet& Buffer::resident() const {
    if (stale_) {
        std::uint64_t n = 0;
        check(lsg_buffer_resident(static_cast<lsg_buffer*>(handle_), nullptr, 0, &n));
        std::vector<std::uint64_t> ids(n);
        check(lsg_buffer_resident(static_cast<lsg_buffer*>(handle_), ids.data(), n, &n));
        resident_ = IdSet(ids.begin(), ids.end());
        stale_ = false;
    }
    return resident_;
}

std::unique_ptr<Buffer> make_buffer(Policy policy, std::uint64_t capacity) {
    if (policy == Policy::Clairvoyant) return std::make_unique<ClairvoyantBuffer>(capacity);
    return std::make_unique<LruBuffer>(capacity);
}

// buffer.cpp:116-125 through the K7 replay
std::uint64_t simulate_sequence(const std::vector<SampleId>& seq, std::uint64_t capacity, Policy policy) {
    std::vector<std::uint32_t> ids(seq.size());
    for (std::size_t i = 0; i < seq.size(); ++i) {
        if (seq[i] >= (1ull << 31)) throw CapabilityError("simulate_sequence: sample ids must be < 2^31 on device");
        ids[i] = std::uint32_t(seq[i]);
    }
    std::uint64_t misses = 0;
    check(lsg_simulate_sequence(ids.data(), ids.size(), capacity, policy == Policy::Lru ? 1 : 0, &misses, nullptr));
    return misses;
}

std::uint64_t optimal_miss_oracle(const std::vector<SampleId>& seq, std::uint64_t capacity) {
    std::uint64_t misses = 0;
    check(lsg_optimal_miss_oracle(seq.data(), seq.size(), capacity, &misses, nullptr));
    return misses;
}

std::uint64_t optimal_miss_oracle(const std::vector<SampleId>& seq, std::uint64_t capacity, OracleWorkspace&) {
    return optimal_miss_oracle(seq, capacity);
}

// read_cost (cost_model.cpp:9-18): one seek plus the span streamed per read
double read_cost(const std::vector<Read>& reads, const CostModel& model) {
    return std::accumulate(reads.begin(), reads.end(), 0.0, [&model](double acc, const Read& r) {
        return acc + (model.seek_cost + double(r.span()) * model.stream_cost);
    });
}
double read_cost(const ChunkPlan& plan, const CostModel& model) { return read_cost(plan.reads, model); }

// derive_threshold (cost_model.cpp:64-71): a chunk read of span s beats s
// single reads while (s - 1) * stream < (s - 1) * seek, i.e. spans up to
// seek/stream + 2 (floored), never beyond max_threshold
std::uint64_t derive_threshold(const CostModel& model, std::uint64_t max_threshold) {
    if (model.seek_cost < 0.0 || model.stream_cost < 0.0)
        throw ValidationError("derive_threshold: negative model parameters");
    if (model.stream_cost == 0.0) return max_threshold;
    const double limit = std::floor(model.seek_cost / model.stream_cost + 2.0);
    return limit >= double(max_threshold) ? max_threshold : std::uint64_t(limit);
}

// redundant_ids (chunking.cpp:35-45): ids a chunk read brings in that the
// list did not ask for, in read order
std::vector<SampleId> redundant_ids(const ChunkPlan& plan, const std::vector<SampleId>& fetch_ids) {
    const std::unordered_set<SampleId> wanted(fetch_ids.begin(), fetch_ids.end());
    std::vector<SampleId> extra;
    for (const Read& r : plan.reads)
        if (r.kind == Read::Kind::Chunk)
            for (SampleId x = r.start; x <= r.end; ++x)
                if (!wanted.count(x)) extra.push_back(x);
    return extra;
}

// chunked_fraction (chunking.cpp:49-69): percent of needed samples that
// arrive inside chunk reads (a chunk's redundant ids do not count)
double chunked_fraction(const std::vector<ChunkPlan>& plans) {
    std::uint64_t needed = 0, chunked = 0;
    for (const ChunkPlan& p : plans) {
        needed += p.needed;
        chunked += std::accumulate(p.reads.begin(), p.reads.end(), std::uint64_t(0),
                                   [](std::uint64_t acc, const Read& r) {
                                       return acc + (r.kind == Read::Kind::Chunk ? r.span() : 0);
                                   }) -
                   p.redundant;
    }
    return needed ? 100.0 * double(chunked) / double(needed) : 0.0;
}

double chunked_fraction(const ChunkPlan& plan) { return chunked_fraction(std::vector<ChunkPlan>{plan}); }

// path_cost (epoch_order.cpp:11-22): the open path's weight; the order must
// be a permutation of the epochs
std::uint64_t path_cost(const ReuseGraph& graph, const std::vector<std::uint32_t>& order) {
    if (order.size() != graph.num_epochs) throw ValidationError("path_cost: order length != num_epochs");
    std::vector<std::uint32_t> sorted(order);
    std::sort(sorted.begin(), sorted.end());
    for (std::uint32_t i = 0; i < sorted.size(); ++i)
        if (sorted[i] != i) throw ValidationError("path_cost: order is not a permutation");
    std::uint64_t c = 0;
    for (auto it = order.begin(); it != order.end() && std::next(it) != order.end(); ++it)
        c += graph.weight(*it, *std::next(it));
    return c;
}

// identity_order (epoch_order.cpp:24-30)
EpochOrder identity_order(const ReuseGraph& graph) {
    std::vector<std::uint32_t> ids(graph.num_epochs);
    std::iota(ids.begin(), ids.end(), 0u);
    const std::uint64_t c = path_cost(graph, ids);
    return EpochOrder{std::move(ids), c};
}

PsoResult pso_order(const ReuseGraph& graph, const PsoParams& p) {
    const std::uint32_t E = graph.num_epochs;
    if (E == 0) throw ValidationError("pso_order: empty graph");
    DevBuf<std::uint64_t> dw(std::size_t(E) * E);
    dw.upload(graph.weights.data(), graph.weights.size());
    DevBuf<std::uint32_t> dord(E), diters(1);
    DevBuf<std::uint64_t> dcost(1), dhist(p.max_iters);
    check(lsg_pso_order(dw.p, E, p.swarm_size, p.max_iters, p.p_personal, p.p_global, p.inertia, p.kick,
                        p.stagnation_limit, p.restart_limit, p.seed, dord.p, dcost.p, dhist.p, diters.p, nullptr));
    PsoResult r;
    r.best.order.resize(E);
    dord.download(r.best.order.data(), E);
    dcost.download(&r.best.cost, 1);
    diters.download(&r.iterations, 1);
    r.history.resize(r.iterations);
    dhist.download(r.history.data(), r.iterations);
    return r;
}

// StepAssignment accessors and same_multiset (plan.cpp:11-42)
std::vector<std::uint64_t> StepAssignment::fetch_counts() const {
    std::vector<std::uint64_t> counts;
    counts.reserve(nodes.size());
    for (const auto& list : nodes)
        counts.push_back(std::uint64_t(std::count_if(list.begin(), list.end(), [](const Assigned& a) {
            return a.source == Source::PfsFetch;
        })));
    return counts;
}
std::vector<SampleId> StepAssignment::fetch_ids(std::uint32_t node) const {
    const auto& list = nodes.at(node);
    std::vector<SampleId> ids;
    for (const Assigned& a : list)
        if (a.source == Source::PfsFetch) ids.push_back(a.id);
    return ids;
}
std::uint64_t StepAssignment::total_assigned() const {
    return std::accumulate(nodes.begin(), nodes.end(), std::uint64_t(0),
                           [](std::uint64_t acc, const auto& list) { return acc + list.size(); });
}
bool same_multiset(const StepAssignment& step, const std::vector<SampleId>& batch) {
    if (step.total_assigned() != batch.size()) return false;
    std::unordered_map<SampleId, std::int64_t> balance;
    for (SampleId x : batch) ++balance[x];
    for (const auto& list : step.nodes)
        for (const Assigned& a : list)
            if (--balance[a.id] < 0) return false;
    return true;  // equal sizes and no id over-used: every count is zero
}

// ---- text artifacts ----------------------------------------------------
namespace {

std::string slurp(std::istream& in) {
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

template <class Fn>
std::string two_call(Fn fn) {
    std::uint64_t n = 0;
    check(fn(nullptr, 0, &n));
    std::string s(n, '\0');
    check(fn(s.data(), n, &n));
    return s;
}

void write_all(const std::string& path, const std::string& data) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw StorageError("cannot open for writing: " + path);
    out.write(data.data(), std::streamsize(data.size()));
    if (!out) throw StorageError("write failed: " + path);
}

std::string read_all(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw StorageError("cannot open for reading: " + path);
    return slurp(in);
}

}  // namespace

void write_trace(std::ostream& out, const AccessTrace& trace) {
    const TraceConfig& c = trace.config;
    const std::uint64_t keep = trace.epoch_length();
    std::vector<std::uint32_t> ids;
    ids.reserve(trace.epochs.size() * keep);
    for (const auto& ep : trace.epochs) {
        if (ep.size() != keep) throw CapabilityError("write_trace: ragged epochs are not on the device path");
        for (SampleId x : ep) {
            if (x >= (1ull << 31)) throw CapabilityError("write_trace: sample ids must be < 2^31 on device");
            ids.push_back(std::uint32_t(x));
        }
    }
    DevBuf<std::uint32_t> d(ids.size());
    d.upload(ids.data(), ids.size());
    out << two_call([&](char* h, std::uint64_t cap, std::uint64_t* n) {
        return lsg_format_trace(d.p, c.dataset_size, std::uint32_t(trace.epochs.size()), c.num_nodes, c.local_batch,
                                c.seed, c.drop_last ? 1 : 0, keep, h, cap, n, nullptr);
    });
}

AccessTrace read_trace(std::istream& in) {
    const std::string s = slurp(in);
    lsg_trace_text h{};
    check(lsg_parse_trace(s.data(), s.size(), &h, nullptr, 0));
    std::vector<std::uint32_t> ids(std::size_t(h.num_epochs) * h.keep);
    check(lsg_parse_trace(s.data(), s.size(), &h, ids.data(), ids.size()));
    AccessTrace t;
    t.config = {h.dataset_size, h.num_epochs, h.num_nodes, h.local_batch, h.seed, h.drop_last != 0};
    t.epochs.assign(h.num_epochs, std::vector<SampleId>(h.keep));
    for (std::uint32_t e = 0; e < h.num_epochs; ++e)
        for (std::uint64_t i = 0; i < h.keep; ++i) t.epochs[e][i] = ids[e * h.keep + i];
    return t;
}

void write_trace_file(const std::string& path, const AccessTrace& trace) {
    std::ostringstream ss;
    write_trace(ss, trace);
    write_all(path, ss.str());
}

AccessTrace read_trace_file(const std::string& path) {
    std::istringstream in(read_all(path));
    return read_trace(in);
}

void write_graph(std::ostream& out, const ReuseGraph& graph) {
    DevBuf<std::uint64_t> d(graph.weights.size());
    d.upload(graph.weights.data(), graph.weights.size());
    out << two_call([&](char* h, std::uint64_t cap, std::uint64_t* n) {
        return lsg_format_graph(d.p, graph.num_epochs, h, cap, n, nullptr);
    });
}

ReuseGraph read_graph(std::istream& in) {
    const std::string s = slurp(in);
    std::uint32_t E = 0;
    check(lsg_parse_graph(s.data(), s.size(), &E, nullptr, 0));
    ReuseGraph g;
    g.num_epochs = E;
    g.weights.assign(std::size_t(E) * E, 0);
    check(lsg_parse_graph(s.data(), s.size(), &E, g.weights.data(), g.weights.size()));
    return g;
}

void write_graph_file(const std::string& path, const ReuseGraph& graph) {
    std::ostringstream ss;
    write_graph(ss, graph);
    write_all(path, ss.str());
}

ReuseGraph read_graph_file(const std::string& path) {
    std::istringstream in(read_all(path));
    return read_graph(in);
}

void write_plan(std::ostream& out, const SchedulePlan& plan) {
    const std::uint32_t N = plan.num_nodes, E = std::uint32_t(plan.epochs.size());
    const std::uint64_t S = E ? plan.epochs.front().steps.size() : 0;
    std::vector<std::uint32_t> items, off, fb, fa, rs, re, rc, order;
    for (std::uint32_t i = 0; i < E; ++i) {
        const EpochPlan& ep = plan.epochs[i];
        if (ep.steps.size() != S || i >= plan.order.order.size() || plan.order.order[i] != ep.epoch)
            throw CapabilityError("write_plan: the device writer needs uniform steps in schedule order");
        order.push_back(ep.epoch);
        for (const StepPlan& st : ep.steps) {
            std::uint32_t o = 0;
            for (std::uint32_t k = 0; k < N; ++k) {
                off.push_back(o);
                fb.push_back(std::uint32_t(st.fetches_before.at(k)));
                fa.push_back(std::uint32_t(st.fetches_after.at(k)));
                const auto& list = st.assignment.nodes.at(k);
                const auto& reads = st.reads.size() == N ? st.reads[k].reads : std::vector<Read>{};
                if (reads.size() > list.size()) throw CapabilityError("write_plan: more reads than samples in a list");
                for (std::size_t j = 0; j < list.size(); ++j) {
                    items.push_back(std::uint32_t(list[j].id) | (list[j].source == Source::BufferHit ? LSG_HIT_BIT : 0u));
                    const bool has = j < reads.size();
                    if (has && (reads[j].kind == Read::Kind::Single) != (reads[j].start == reads[j].end))
                        throw CapabilityError("write_plan: read kind differs from its span");
                    rs.push_back(has ? std::uint32_t(reads[j].start) : 0u);
                    re.push_back(has ? std::uint32_t(reads[j].end) : 0u);
                    ++o;
                }
                rc.push_back(std::uint32_t(reads.size()));
            }
            off.push_back(o);
        }
    }
    const std::uint64_t T = std::uint64_t(E) * S;
    DevBuf<std::uint32_t> di(items.size()), doff(off.size()), dfb(fb.size()), dfa(fa.size()), drs(rs.size()),
        dre(re.size()), drc(rc.size()), dord(order.size());
    di.upload(items.data(), items.size());
    doff.upload(off.data(), off.size());
    dfb.upload(fb.data(), fb.size());
    dfa.upload(fa.data(), fa.size());
    drs.upload(rs.data(), rs.size());
    dre.upload(re.data(), re.size());
    drc.upload(rc.data(), rc.size());
    dord.upload(order.data(), order.size());
    out << two_call([&](char* h, std::uint64_t cap, std::uint64_t* n) {
        return lsg_format_plan(di.p, doff.p, dfb.p, dfa.p, drs.p, dre.p, drc.p, dord.p, plan.order.cost, E, T, N,
                               S ? S : 1, plan.dataset_size, plan.local_batch, plan.chunk_threshold, h, cap, n,
                               nullptr);
    });
}

SchedulePlan read_plan(std::istream& in) {
    const std::string s = slurp(in);
    lsg_parsed_plan* h = nullptr;
    lsg_plan_view v{};
    check(lsg_parse_plan(s.data(), s.size(), &h, &v));
    std::unique_ptr<lsg_parsed_plan, void (*)(lsg_parsed_plan*)> guard(h, lsg_free_plan);
    SchedulePlan p;
    p.dataset_size = v.dataset_size;
    p.num_nodes = v.num_nodes;
    p.local_batch = v.local_batch;
    p.chunk_threshold = v.chunk_threshold;
    p.order.order.assign(v.order, v.order + v.num_epochs);
    p.order.cost = v.cost;
    const std::uint32_t N = v.num_nodes;
    std::uint64_t g = 0, base = 0;
    for (std::uint32_t e = 0; e < v.num_epochs; ++e) {
        EpochPlan ep;
        ep.epoch = v.epoch_ids[e];
        for (std::uint64_t t = 0; t < v.epoch_steps[e]; ++t, ++g) {
            StepPlan st;
            st.assignment.nodes.resize(N);
            st.reads.resize(N);
            const std::uint32_t* off = v.node_off + g * (N + 1);
            for (std::uint32_t k = 0; k < N; ++k) {
                for (std::uint32_t i = off[k]; i < off[k + 1]; ++i) {
                    const std::uint32_t it = v.items[base + i];
                    st.assignment.nodes[k].push_back(
                        {it & ~LSG_HIT_BIT, (it & LSG_HIT_BIT) ? Source::BufferHit : Source::PfsFetch});
                }
                st.fetches_before.push_back(v.fetch_before[g * N + k]);
                st.fetches_after.push_back(v.fetch_after[g * N + k]);
                ChunkPlan& cp = st.reads[k];
                for (std::uint64_t q = v.read_off[g * N + k]; q < v.read_off[g * N + k + 1]; ++q)
                    cp.reads.push_back({v.read_chunk[q] ? Read::Kind::Chunk : Read::Kind::Single, v.read_start[q],
                                        v.read_end[q]});
                cp.needed = v.needed[g * N + k];
                cp.redundant = v.redundant[g * N + k];
            }
            base += off[N];
            ep.steps.push_back(std::move(st));
        }
        p.epochs.push_back(std::move(ep));
    }
    return p;
}

void write_plan_file(const std::string& path, const SchedulePlan& plan) {
    std::ostringstream ss;
    write_plan(ss, plan);
    write_all(path, ss.str());
}

SchedulePlan read_plan_file(const std::string& path) {
    std::istringstream in(read_all(path));
    return read_plan(in);
}

void create_store(const std::string& path, std::uint64_t sample_count, std::uint64_t sample_size,
                  std::uint64_t fill_seed, std::uint64_t max_bytes) {
    check(lsg_store_create(path.c_str(), sample_count, sample_size, fill_seed, max_bytes, nullptr));
}

Store::Store(const std::string& path) {
    lsg_store* h = nullptr;
    check(lsg_store_open(path.c_str(), &h));
    h_ = h;
    check(lsg_store_info(h, &header_.sample_count, &header_.sample_size));
}

Store::~Store() { lsg_store_close(static_cast<lsg_store*>(h_)); }

std::vector<std::byte> Store::read_chunk(std::uint64_t start, std::uint64_t count) const {
    std::vector<std::byte> out(std::max<std::uint64_t>(count, 1) * header_.sample_size);
    check(lsg_store_read(static_cast<lsg_store*>(h_), start, count, out.data()));
    out.resize(count * header_.sample_size);
    return out;
}

std::vector<std::byte> Store::read_one(std::uint64_t index) const { return read_chunk(index, 1); }

void Store::read_rows_device(const std::vector<SampleId>& ids, void* d_rows, std::uint64_t threshold,
                             void* stream) const {
    std::vector<std::uint32_t> v(ids.size());
    for (std::size_t i = 0; i < ids.size(); ++i) {
        if (ids[i] >= header_.sample_count) throw ValidationError("store: sample index out of range");
        v[i] = std::uint32_t(ids[i]);
    }
    check(lsg_store_read_rows(static_cast<lsg_store*>(h_), v.data(), v.size(), threshold, d_rows, stream));
}

PipelineConfig baseline_config(const PipelineConfig& config) {
    PipelineConfig base = config;
    base.policy = Policy::Lru;
    base.optim_order = false;
    base.optim_remap = false;
    base.optim_balance = false;
    base.optim_chunk = false;
    base.chunk_insert_redundant = false;
    return base;
}

PlanOutput plan_schedule(const PipelineConfig& config) {
    const lsg_config c = to_c(config);
    lsg_shape sh;
    check(lsg_shape_of(&c, &sh));
    const std::uint32_t E = config.trace.num_epochs, N = config.trace.num_nodes;
    const std::uint64_t keep = sh.keep, S = sh.steps_per_epoch, T = sh.total_steps;
    std::vector<std::uint32_t> trace(sh.total_items), order(E), items(sh.total_items), off(T * (N + 1)),
        fb(T * N), fa(T * N), rs(sh.total_items), re(sh.total_items), rc(T * N), rn(T * N), rr(T * N);
    std::vector<std::uint64_t> graph(std::size_t(E) * E), hist(config.pso.max_iters);
    std::uint64_t cost = 0;
    std::uint32_t iters = 0;
    lsg_plan_out h{trace.data(), graph.data(), order.data(), &cost, hist.data(), &iters, items.data(),
                   off.data(), fb.data(), fa.data(), rs.data(), re.data(), rc.data(), rn.data(), rr.data()};
    check(lsg_plan_host(&c, &h, nullptr));

    PlanOutput out;
    out.trace.config = config.trace;
    out.trace.epochs.resize(E);
    for (std::uint32_t e = 0; e < E; ++e)
        out.trace.epochs[e].assign(trace.begin() + std::size_t(e) * keep, trace.begin() + std::size_t(e + 1) * keep);
    out.graph.num_epochs = E;
    out.graph.buffer_size = config.buffer_capacity;
    out.graph.mode = config.graph_mode;
    out.graph.weights = graph;
    SchedulePlan& p = out.plan;
    p.dataset_size = config.trace.dataset_size;
    p.num_nodes = N;
    p.local_batch = config.trace.local_batch;
    p.chunk_threshold = config.optim_chunk ? config.chunk_threshold : 0;  // pipeline.cpp:52
    p.order.order = order;
    p.order.cost = cost;
    if (config.optim_order) {
        PsoResult r;
        r.best = p.order;
        r.history.assign(hist.begin(), hist.begin() + iters);
        r.iterations = iters;
        out.pso = r;
    }
    std::uint64_t base = 0;
    for (std::uint32_t i = 0; i < E; ++i) {
        EpochPlan ep;
        ep.epoch = order[i];
        for (std::uint64_t t = 0; t < S; ++t) {
            const std::uint64_t g = std::uint64_t(i) * S + t;
            const std::uint32_t* o = off.data() + g * (N + 1);
            StepPlan st;
            st.assignment.nodes.resize(N);
            for (std::uint32_t k = 0; k < N; ++k) {
                auto& list = st.assignment.nodes[k];
                list.reserve(o[k + 1] - o[k]);
                for (std::uint32_t q = o[k]; q < o[k + 1]; ++q) {
                    const std::uint32_t v = items[base + q];
                    list.push_back({SampleId(v & ~LSG_HIT_BIT), (v & LSG_HIT_BIT) ? Source::BufferHit : Source::PfsFetch});
                }
                st.fetches_before.push_back(fb[g * N + k]);
                st.fetches_after.push_back(fa[g * N + k]);
                ChunkPlan cp;  // chunking.hpp:24-28
                for (std::uint32_t r = 0; r < rc[g * N + k]; ++r) {
                    const std::size_t at = base + o[k] + r;
                    cp.reads.push_back({rs[at] == re[at] ? Read::Kind::Single : Read::Kind::Chunk, rs[at], re[at]});
                }
                cp.needed = rn[g * N + k];
                cp.redundant = rr[g * N + k];
                st.reads.push_back(std::move(cp));
            }
            base += o[N];
            ep.steps.push_back(std::move(st));
        }
        p.epochs.push_back(std::move(ep));
    }
    return out;
}

SimResult simulate_plan(const SchedulePlan& plan, std::uint64_t capacity, Policy policy, bool insert_redundant) {
    const std::uint32_t N = plan.num_nodes;
    std::vector<std::uint32_t> items, off, rs, re, rc;
    std::uint64_t T = 0;
    for (const EpochPlan& ep : plan.epochs)
        for (const StepPlan& st : ep.steps) {
            if (st.assignment.nodes.size() != N) throw ValidationError("simulate_plan: node count mismatch");
            if (insert_redundant && st.reads.size() != N) throw ValidationError("simulate_plan: step without reads");
            std::uint32_t o = 0;
            for (std::uint32_t k = 0; k < N; ++k) {
                const auto& list = st.assignment.nodes[k];
                off.push_back(o);
                for (const Assigned& a : list) {
                    if (a.id >= (1ull << 31)) throw CapabilityError("simulate_plan: sample ids must be < 2^31 on device");
                    items.push_back(std::uint32_t(a.id) | (a.source == Source::BufferHit ? LSG_HIT_BIT : 0u));
                    ++o;
                }
                if (insert_redundant) {  // reads at the list's item offsets (lsg_plan_out layout)
                    const auto& reads = st.reads[k].reads;
                    if (reads.size() > list.size()) throw ValidationError("simulate_plan: more reads than samples");
                    for (std::size_t i = 0; i < list.size(); ++i) {
                        rs.push_back(i < reads.size() ? std::uint32_t(reads[i].start) : 0u);
                        re.push_back(i < reads.size() ? std::uint32_t(reads[i].end) : 0u);
                    }
                    rc.push_back(std::uint32_t(reads.size()));
                }
            }
            off.push_back(o);
            ++T;
        }
    SimResult r;
    r.policy = policy;
    if (T == 0) return r;
    DevBuf<std::uint32_t> di(items.size()), doff(off.size()), dh(T * N), dm(T * N);
    di.upload(items.data(), items.size());
    doff.upload(off.data(), off.size());
    if (insert_redundant) {
        DevBuf<std::uint32_t> drs(rs.size()), dre(re.size()), drc(rc.size());
        drs.upload(rs.data(), rs.size());
        dre.upload(re.data(), re.size());
        drc.upload(rc.data(), rc.size());
        check(lsg_simulate_ex(di.p, doff.p, T, N, plan.dataset_size, capacity, policy == Policy::Clairvoyant ? 0 : 1,
                              1, drs.p, dre.p, drc.p, 0, N, dh.p, dm.p, nullptr, nullptr));
    } else {
        check(lsg_simulate(di.p, doff.p, T, N, plan.dataset_size, capacity, policy == Policy::Clairvoyant ? 0 : 1, 0,
                           N, dh.p, dm.p, nullptr, nullptr));
    }
    std::vector<std::uint32_t> h(T * N), m(T * N);
    dh.download(h.data(), h.size());
    dm.download(m.data(), m.size());
    std::uint64_t g = 0;
    for (const EpochPlan& ep : plan.epochs)
        for (std::size_t t = 0; t < ep.steps.size(); ++t, ++g)
            for (std::uint32_t k = 0; k < N; ++k) {
                r.rows.push_back({ep.epoch, t, k, h[g * N + k], m[g * N + k]});
                r.total_hits += h[g * N + k];
                r.total_misses += m[g * N + k];
            }
    return r;
}

// ---- run reporting (config.cpp:157-159, pipeline.cpp:133-179) -------------
const char* policy_name(Policy policy) { return policy == Policy::Clairvoyant ? "clairvoyant" : "lru"; }

namespace {
// the plan's fetch_after counts, node offsets and reads in the flat device
// layout (lsg_plan_out) for lsg_plan_costs
struct FlatCosts {
    std::uint64_t T = 0;
    std::uint32_t N = 0;
    std::vector<std::uint32_t> fa, off, rs, re, rc;
};
FlatCosts flatten_costs(const SchedulePlan& plan, bool reads) {
    FlatCosts f;
    f.N = plan.num_nodes;
    for (const EpochPlan& ep : plan.epochs)
        for (const StepPlan& sp : ep.steps) {
            ++f.T;
            std::uint32_t o = 0;
            for (std::uint32_t k = 0; k < f.N; ++k) {
                f.fa.push_back(k < sp.assignment.nodes.size()
                                   ? std::uint32_t(std::count_if(sp.assignment.nodes[k].begin(),
                                                                 sp.assignment.nodes[k].end(),
                                                                 [](const Assigned& a) {
                                                                     return a.source == Source::PfsFetch;
                                                                 }))
                                   : 0u);
                f.off.push_back(o);
                const std::size_t len = k < sp.assignment.nodes.size() ? sp.assignment.nodes[k].size() : 0;
                if (reads) {
                    static const std::vector<Read> none;
                    const auto& rd = k < sp.reads.size() ? sp.reads[k].reads : none;
                    // reads sit at their list's item offsets; a list may hold
                    // fewer items than reads only in a hand-made plan
                    const std::size_t slots = std::max(len, rd.size());
                    for (std::size_t i = 0; i < slots; ++i) {
                        f.rs.push_back(i < rd.size() ? std::uint32_t(rd[i].start) : 0u);
                        f.re.push_back(i < rd.size() ? std::uint32_t(rd[i].end) : 0u);
                    }
                    f.rc.push_back(std::uint32_t(rd.size()));
                    o += std::uint32_t(slots);
                } else {
                    o += std::uint32_t(len);
                }
            }
            f.off.push_back(o);
        }
    return f;
}

std::pair<double, double> device_costs(const SchedulePlan& plan, const CostModel& model, bool reads) {
    const FlatCosts f = flatten_costs(plan, reads);
    if (f.T == 0) return {0.0, 0.0};
    DevBuf<std::uint32_t> fa(f.fa.size()), off(f.off.size()), rs(f.rs.size()), re(f.re.size()), rc(f.rc.size());
    fa.upload(f.fa.data(), f.fa.size());
    off.upload(f.off.data(), f.off.size());
    if (reads) {
        rs.upload(f.rs.data(), f.rs.size());
        re.upload(f.re.data(), f.re.size());
        rc.upload(f.rc.data(), f.rc.size());
    }
    double bar = 0.0, io = 0.0;
    check(lsg_plan_costs(nullptr, fa.p, off.p, reads ? rs.p : nullptr, reads ? re.p : nullptr, reads ? rc.p : nullptr, f.T,
                         f.N, model.seek_cost, model.stream_cost, &bar, &io, nullptr));
    return {bar, io};
}
}  // namespace

// total_barrier_cost / total_io_cost (pipeline.cpp:133-151): summed on the
// device over the flat plan (lsg_plan_costs)
double total_barrier_cost(const SchedulePlan& plan, const CostModel& model) {
    return device_costs(plan, model, false).first;
}

double total_io_cost(const SchedulePlan& plan, const CostModel& model) {
    return device_costs(plan, model, true).second;
}

// write_metrics (pipeline.cpp:153-179): one CSV row per (epoch, step, node)
// in execution order; a step's barrier columns are its most loaded node's
// fetch count before / after balancing x (seek + stream), "%.6f"
void write_metrics(std::ostream& out, const SchedulePlan& plan, const SimResult& sim, const CostModel& model) {
    out << "epoch,step,node,hits,misses,policy,fetches_before,fetches_after,barrier_before,barrier_after\n";
    const double per_fetch = model.seek_cost + model.stream_cost;
    const char* pol = policy_name(sim.policy);
    auto barrier = [per_fetch](const std::vector<std::uint64_t>& counts, char* buf, std::size_t n) {
        const std::uint64_t most = counts.empty() ? 0 : *std::max_element(counts.begin(), counts.end());
        std::snprintf(buf, n, "%.6f", double(most) * per_fetch);
    };
    auto row = sim.rows.begin();
    char bb[64], ba[64], line[256];
    for (const EpochPlan& ep : plan.epochs) {
        std::uint64_t t = 0;
        for (const StepPlan& sp : ep.steps) {
            barrier(sp.fetches_before, bb, sizeof bb);
            barrier(sp.fetches_after, ba, sizeof ba);
            for (std::uint32_t k = 0; k < plan.num_nodes; ++k, ++row) {
                if (row == sim.rows.end() || row->epoch != ep.epoch || row->step != t || row->node != k)
                    throw InternalError("write_metrics: simulation rows out of order");
                std::snprintf(line, sizeof line, "%u,%llu,%u,%llu,%llu,%s,%llu,%llu,%s,%s\n", ep.epoch,
                              (unsigned long long)t, k, (unsigned long long)row->hits,
                              (unsigned long long)row->misses, pol, (unsigned long long)sp.fetches_before.at(k),
                              (unsigned long long)sp.fetches_after.at(k), bb, ba);
                out << line;
            }
            ++t;
        }
    }
}

PipelineResult run_pipeline(const PipelineConfig& config, const std::string& out_dir) {
    config.validate();
    PipelineResult r;
    r.output = plan_schedule(config);
    r.sim = simulate_plan(r.output.plan, config.buffer_capacity, config.policy,
                          config.chunk_insert_redundant && config.optim_chunk);
    const PipelineConfig base = baseline_config(config);
    r.baseline_plan = plan_schedule(base).plan;
    r.baseline_sim = simulate_plan(r.baseline_plan, base.buffer_capacity, base.policy, false);
    if (out_dir.empty()) return r;
    namespace fs = std::filesystem;
    std::error_code ec;
    fs::create_directories(out_dir, ec);
    if (ec) throw StorageError("cannot create output directory: " + out_dir);
    const fs::path dir(out_dir);
    auto open = [&dir](const char* name) {
        std::ofstream f(dir / name, std::ios::binary);
        if (!f) throw StorageError(std::string("cannot write ") + name);
        return f;
    };
    write_trace_file((dir / "trace.txt").string(), r.output.trace);
    write_graph_file((dir / "graph.txt").string(), r.output.graph);
    {
        std::ofstream f = open("order.txt");
        f << "order:";
        for (std::uint32_t e : r.output.plan.order.order) f << ' ' << e;
        f << "\ncost: " << r.output.plan.order.cost << "\n";
    }
    write_plan_file((dir / "plan.txt").string(), r.output.plan);
    {
        std::ofstream f = open("metrics.csv");
        write_metrics(f, r.output.plan, r.sim, config.model);
    }
    {
        std::ofstream f = open("baseline_metrics.csv");
        write_metrics(f, r.baseline_plan, r.baseline_sim, config.model);
    }
    throw CapabilityError("run_pipeline: summary.txt is the ablation-ladder report, out of scope for the B200 "
                          "drop-in (the other artifacts were written)");
}

}  // namespace loadsched

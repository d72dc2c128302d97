// include/loadsched_gpu.hpp — C++ drop-in for the hot path of the reference
// `loadsched` library (/root/reference/proj/include/loadsched), backed by the
// sm_100a kernels through the C ABI (lsg.h).
//
// A caller of the reference keeps its code: the namespace, value types, field
// names, function signatures and exception classes below follow the reference
// API for the planner path (cited per declaration); results are bit-identical.
// Everything is computed on the current CUDA device; inputs are uploaded and
// outputs returned by value as the reference does. Both buffer policies
// (Clairvoyant, Lru) run on device, chunk_insert_redundant included; Store
// files, the text artifacts (trace / graph / plan files) and the run reports
// (metrics.csv, cost totals) are read and written in the reference's formats.
// Out of this header (and out of scope): the CLI, config
// files, cost-model calibration, the ablation ladder and summary report.
#pragma once

#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <memory>
#include <vector>

namespace loadsched {

// ---- errors.hpp:10-46 ----------------------------------------------------
enum class ErrorClass { Config = 2, Validation = 3, Capability = 4, Calibration = 5, Storage = 6, Internal = 7 };

class Error : public std::runtime_error {
  public:
    Error(ErrorClass c, const std::string& what) : std::runtime_error(what), cls_(c) {}
    ErrorClass error_class() const { return cls_; }
    int exit_code() const { return static_cast<int>(cls_); }

  private:
    ErrorClass cls_;
};
#define LOADSCHED_GPU_ERROR(Name, Cls)                                   \
    struct Name : Error {                                                \
        explicit Name(const std::string& w) : Error(ErrorClass::Cls, w) {} \
    };
LOADSCHED_GPU_ERROR(ConfigError, Config)
LOADSCHED_GPU_ERROR(ValidationError, Validation)
LOADSCHED_GPU_ERROR(CapabilityError, Capability)
LOADSCHED_GPU_ERROR(StorageError, Storage)
LOADSCHED_GPU_ERROR(InternalError, Internal)
#undef LOADSCHED_GPU_ERROR

using SampleId = std::uint64_t;  // trace.hpp:11 (device ids are 32-bit)
using IdSet = std::unordered_set<SampleId>;

// ---- prng.hpp:12-53: the splitmix64 stream every random choice draws from
// (host side of the counter-based draws the kernels compute in parallel) ----
inline constexpr std::uint64_t kGoldenGamma = 0x9E3779B97F4A7C15ULL;

class SplitMix64 {
  public:
    using result_type = std::uint64_t;
    explicit constexpr SplitMix64(std::uint64_t seed) : state_(seed) {}
    constexpr std::uint64_t next() {
        std::uint64_t z = (state_ += kGoldenGamma);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    constexpr std::uint64_t operator()() { return next(); }
    constexpr std::uint64_t next_below(std::uint64_t bound) { return next() % bound; }
    constexpr double next_double() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
    static constexpr std::uint64_t min() { return 0; }
    static constexpr std::uint64_t max() { return ~0ULL; }

  private:
    std::uint64_t state_;
};

// in-place Fisher-Yates, i = n .. 2 swapping a[i-1] with a[next_below(i)]
template <typename T>
void fisher_yates_shuffle(std::vector<T>& a, SplitMix64& rng) {
    for (std::size_t i = a.size(); i > 1; --i) {
        const std::size_t j = std::size_t(rng.next_below(i));
        T t = a[i - 1];
        a[i - 1] = a[j];
        a[j] = t;
    }
}

// ---- trace.hpp:15-57 -------------------------------------------------------
struct TraceConfig {
    std::uint64_t dataset_size = 0;
    std::uint32_t num_epochs = 0;
    std::uint32_t num_nodes = 0;
    std::uint64_t local_batch = 0;
    std::uint64_t seed = 0;
    bool drop_last = true;

    std::uint64_t global_batch() const { return std::uint64_t(num_nodes) * local_batch; }
    std::uint64_t steps_per_epoch() const;
    void validate() const;
};

struct AccessTrace {
    TraceConfig config;
    std::vector<std::vector<SampleId>> epochs;
    std::uint64_t epoch_length() const { return epochs.empty() ? 0 : epochs.front().size(); }
};

AccessTrace generate_trace(const TraceConfig& config);
std::vector<SampleId> slice(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t step,
                            std::uint32_t node);
std::vector<SampleId> global_batch(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t step);

// ---- reuse_graph.hpp:15-53 -------------------------------------------------
enum class WindowMode { Global, PerNode };

struct ReuseGraph {
    std::uint32_t num_epochs = 0;
    std::uint64_t buffer_size = 0;
    WindowMode mode = WindowMode::Global;
    std::vector<std::uint64_t> weights;  // row-major E x E
    std::uint64_t weight(std::uint32_t u, std::uint32_t v) const { return weights[std::size_t(u) * num_epochs + v]; }
    std::uint64_t& weight(std::uint32_t u, std::uint32_t v) { return weights[std::size_t(u) * num_epochs + v]; }
};

ReuseGraph build_reuse_graph(const AccessTrace& trace, std::uint64_t buffer_size, WindowMode mode);
// the K2 window bitsets of one epoch as id sets (reuse_graph.hpp:38-48)
std::vector<IdSet> last_buffer_window(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t buffer_size,
                                      WindowMode mode);
std::vector<IdSet> first_buffer_window(const AccessTrace& trace, std::uint32_t epoch, std::uint64_t buffer_size,
                                       WindowMode mode);

// ---- epoch_order.hpp:13-63 -------------------------------------------------
struct EpochOrder {
    std::vector<std::uint32_t> order;
    std::uint64_t cost = 0;
};

struct PsoParams {
    std::uint32_t swarm_size = 32;
    std::uint32_t max_iters = 500;
    double p_personal = 0.5;
    double p_global = 0.5;
    double inertia = 0.5;
    double kick = 1.0;
    std::uint32_t stagnation_limit = 100;
    std::uint32_t restart_limit = 20;
    std::uint64_t seed = 0;
};

struct PsoResult {
    EpochOrder best;
    std::vector<std::uint64_t> history;
    std::uint32_t iterations = 0;
};

std::uint64_t path_cost(const ReuseGraph& graph, const std::vector<std::uint32_t>& order);
PsoResult pso_order(const ReuseGraph& graph, const PsoParams& params);
EpochOrder identity_order(const ReuseGraph& graph);
EpochOrder brute_force_order(const ReuseGraph& graph);  // epoch_order.hpp:35-38, E <= 10 on device

// ---- plan.hpp:16-53 --------------------------------------------------------
enum class Source { BufferHit, PfsFetch };

struct Assigned {
    SampleId id = 0;
    Source source = Source::PfsFetch;
    friend bool operator==(const Assigned&, const Assigned&) = default;
};

struct StepAssignment {
    std::vector<std::vector<Assigned>> nodes;
    std::vector<std::uint64_t> fetch_counts() const;
    std::vector<SampleId> fetch_ids(std::uint32_t node) const;
    std::uint64_t total_assigned() const;
};

struct Read {  // chunking.hpp:13-22
    enum class Kind { Single, Chunk };
    Kind kind = Kind::Single;
    SampleId start = 0, end = 0;
    std::uint64_t span() const { return end - start + 1; }
    friend bool operator==(const Read&, const Read&) = default;
};
struct ChunkPlan {
    std::vector<Read> reads;
    std::uint64_t needed = 0, redundant = 0;
};

struct StepPlan {
    StepAssignment assignment;
    std::vector<std::uint64_t> fetches_before;
    std::vector<std::uint64_t> fetches_after;
    std::vector<ChunkPlan> reads;  // per node read plan (chunking.cpp / pipeline.cpp:83-88)
};

struct EpochPlan {
    std::uint32_t epoch = 0;
    std::vector<StepPlan> steps;
};

struct SchedulePlan {
    std::uint64_t dataset_size = 0;
    std::uint32_t num_nodes = 0;
    std::uint64_t local_batch = 0;
    std::uint64_t chunk_threshold = 0;
    EpochOrder order;
    std::vector<EpochPlan> epochs;
};

bool same_multiset(const StepAssignment& step, const std::vector<SampleId>& batch);

// ---- locality.hpp:23-39 / balance.hpp:13-32: one step against explicit
// residency sets, on the device (lsg_remap_step / lsg_balance_step)
StepAssignment remap_step(const std::vector<const IdSet*>& buffers, const std::vector<SampleId>& batch,
                          std::uint64_t local_batch);
std::vector<StepAssignment> remap_epoch(const std::vector<IdSet>& prev_buffers,
                                        const std::vector<std::vector<SampleId>>& epoch_batches,
                                        std::uint64_t local_batch);
StepAssignment slice_step(const std::vector<const IdSet*>& buffers, const std::vector<SampleId>& batch,
                          std::uint64_t local_batch);
std::uint64_t balance_step(StepAssignment& step);

struct CostModel {  // cost_model.hpp:13-16
    double seek_cost = 13.0;
    double stream_cost = 1.0;
};
double barrier_time(const StepAssignment& step, const CostModel& model);
struct StepSizes {
    std::uint32_t epoch = 0;
    std::uint64_t step = 0;
    std::vector<std::uint64_t> sizes;
    double stddev = 0.0;
};
// host reporting helper over a finished plan (balance.cpp:52-72)
std::vector<StepSizes> batch_size_stats(const SchedulePlan& plan);

// ---- chunking.hpp:23-39: plan_chunks runs the device read planner on one
// list; redundant_ids / chunked_fraction are host-side accessors of a plan
ChunkPlan plan_chunks(const std::vector<SampleId>& fetch_ids, std::uint64_t threshold);
std::vector<SampleId> redundant_ids(const ChunkPlan& plan, const std::vector<SampleId>& fetch_ids);
double chunked_fraction(const ChunkPlan& plan);
double chunked_fraction(const std::vector<ChunkPlan>& plans);
// cost_model.hpp:24-27, 45-48: host formulas that price a read plan and set
// the chunk threshold the device read planner uses
double read_cost(const ChunkPlan& plan, const CostModel& model);
double read_cost(const std::vector<Read>& reads, const CostModel& model);
std::uint64_t derive_threshold(const CostModel& model, std::uint64_t max_threshold);

// ---- buffer.hpp:16-118 (simulation results) --------------------------------
enum class Policy { Clairvoyant, Lru };

struct StepNodeStats {
    std::uint32_t epoch = 0;
    std::uint64_t step = 0;
    std::uint32_t node = 0;
    std::uint64_t hits = 0;
    std::uint64_t misses = 0;
};

struct SimResult {
    Policy policy = Policy::Clairvoyant;
    std::vector<StepNodeStats> rows;
    std::uint64_t total_hits = 0;
    std::uint64_t total_misses = 0;
};

SimResult simulate_plan(const SchedulePlan& plan, std::uint64_t capacity, Policy policy,
                        bool insert_redundant = false);

// ---- buffer.hpp:19-96: one node's buffer as device-resident state
// (lsg_buffer_*); every call applies its accesses on the GPU in order.
inline constexpr std::uint64_t kNeverUsed = ~std::uint64_t{0};

class Buffer {
  public:
    explicit Buffer(std::uint64_t capacity) : Buffer(Policy::Clairvoyant, capacity) {}
    virtual ~Buffer();
    Buffer(const Buffer&) = delete;
    Buffer& operator=(const Buffer&) = delete;

    virtual bool access(SampleId id, std::uint64_t next_use);
    virtual void insert_silent(SampleId id, std::uint64_t next_use);
    virtual void clear();
    // batched Buffer::access over a sequence, one device launch
    std::vector<bool> access_batch(const std::vector<SampleId>& ids, const std::vector<std::uint64_t>& next_use);

    const IdSet& resident() const;
    std::uint64_t capacity() const { return capacity_; }

  protected:
    Buffer(Policy policy, std::uint64_t capacity);
    std::uint64_t capacity_;

  private:
    void* handle_ = nullptr;
    mutable IdSet resident_;
    mutable bool stale_ = true;
};

class ClairvoyantBuffer : public Buffer {
  public:
    explicit ClairvoyantBuffer(std::uint64_t capacity) : Buffer(Policy::Clairvoyant, capacity) {}
};

class LruBuffer : public Buffer {
  public:
    explicit LruBuffer(std::uint64_t capacity) : Buffer(Policy::Lru, capacity) {}
};

std::unique_ptr<Buffer> make_buffer(Policy policy, std::uint64_t capacity);
std::uint64_t simulate_sequence(const std::vector<SampleId>& seq, std::uint64_t capacity, Policy policy);

struct OracleWorkspace {  // kept for signature parity; the device DP needs no host scratch
    std::vector<std::int8_t> memo;
    std::vector<std::uint8_t> labels;
};
std::uint64_t optimal_miss_oracle(const std::vector<SampleId>& seq, std::uint64_t capacity);
std::uint64_t optimal_miss_oracle(const std::vector<SampleId>& seq, std::uint64_t capacity, OracleWorkspace& ws);

// ---- config.hpp:17-36 / pipeline.hpp:17-27 ---------------------------------
struct PipelineConfig {
    TraceConfig trace;
    std::uint64_t buffer_capacity = 0;
    Policy policy = Policy::Clairvoyant;
    WindowMode graph_mode = WindowMode::Global;
    std::uint64_t chunk_threshold = 15;
    bool chunk_insert_redundant = false;
    CostModel model{};  // config.hpp:25 (the run reports' cost model)
    PsoParams pso{};
    bool optim_order = true;
    bool optim_remap = true;
    bool optim_balance = true;
    bool optim_chunk = true;
    void validate() const;
};

struct PlanOutput {
    AccessTrace trace;
    ReuseGraph graph;
    std::optional<PsoResult> pso;
    SchedulePlan plan;
};

PlanOutput plan_schedule(const PipelineConfig& config);

// ---- run reporting over a finished plan (config.cpp:157-159,
// pipeline.hpp:43-44, 62-63): host formulas/formatters over the device
// planner's and replay's outputs, byte-identical to the reference's
const char* policy_name(Policy policy);
double total_barrier_cost(const SchedulePlan& plan, const CostModel& model);
double total_io_cost(const SchedulePlan& plan, const CostModel& model);
// metrics.csv: one row per (epoch, step, node) in execution order
void write_metrics(std::ostream& out, const SchedulePlan& plan, const SimResult& sim, const CostModel& model);

// ---- text artifacts (trace.hpp:42-47, reuse_graph.hpp:55-60, plan.hpp:55-68)
// Writers format on the GPU (byte-identical to the reference's); readers
// accept the reference's grammar with its error classes and messages.
void write_trace(std::ostream& out, const AccessTrace& trace);
AccessTrace read_trace(std::istream& in);
void write_trace_file(const std::string& path, const AccessTrace& trace);
AccessTrace read_trace_file(const std::string& path);
void write_graph(std::ostream& out, const ReuseGraph& graph);
ReuseGraph read_graph(std::istream& in);
void write_graph_file(const std::string& path, const ReuseGraph& graph);
ReuseGraph read_graph_file(const std::string& path);
void write_plan(std::ostream& out, const SchedulePlan& plan);
SchedulePlan read_plan(std::istream& in);
void write_plan_file(const std::string& path, const SchedulePlan& plan);
SchedulePlan read_plan_file(const std::string& path);

// ---- store.hpp:13-50 --------------------------------------------------------
// SLRD sample files; create_store computes the splitmix64 payload on the GPU
// and writes a file byte-identical to the reference's. Store::read_one /
// read_chunk return host bytes like the reference; read_rows_device() moves
// a set of samples straight into HBM (chunked parallel reads).
struct StoreHeader {
    std::uint16_t version = 1;
    std::uint64_t sample_count = 0;
    std::uint64_t sample_size = 0;
};

inline constexpr std::size_t kStoreHeaderBytes = 4 + 2 + 8 + 8;
inline constexpr std::uint64_t kDefaultStoreBudget = 1ULL << 30;  // 1 GiB

void create_store(const std::string& path, std::uint64_t sample_count, std::uint64_t sample_size,
                  std::uint64_t fill_seed, std::uint64_t max_bytes = kDefaultStoreBudget);

class Store {
  public:
    explicit Store(const std::string& path);
    ~Store();
    Store(const Store&) = delete;
    Store& operator=(const Store&) = delete;

    const StoreHeader& header() const { return header_; }
    std::uint64_t sample_count() const { return header_.sample_count; }
    std::uint64_t sample_size() const { return header_.sample_size; }

    std::vector<std::byte> read_one(std::uint64_t index) const;
    std::vector<std::byte> read_chunk(std::uint64_t start, std::uint64_t count) const;
    // B200 extension: samples ids into device rows (pitch = sample size)
    void read_rows_device(const std::vector<SampleId>& ids, void* d_rows, std::uint64_t threshold = 15,
                          void* stream = nullptr) const;

  private:
    void* h_ = nullptr;  // lsg_store*
    StoreHeader header_;
};

// pipeline.cpp:122-131: the comparison pass of run_pipeline (LRU buffers,
// identity order, slicing, no balance, no chunking).
PipelineConfig baseline_config(const PipelineConfig& config);

// pipeline.hpp:33-40 (the ablation ladder's row type; the ladder itself is
// out of scope)
struct PassTotals {
    std::string name;
    std::uint64_t misses = 0;
    std::uint64_t hits = 0;
    double hit_rate = 0.0;
    double barrier_cost = 0.0;
    double io_cost = 0.0;
};

// pipeline.hpp:46-57 / pipeline.cpp:266-311: the configured pass plus the LRU
// baseline pass, all planned and replayed on the device. With an out_dir the
// run's artifacts are written in the reference's formats (trace.txt,
// graph.txt, order.txt, plan.txt, metrics.csv, baseline_metrics.csv); the
// reference's summary.txt is the ablation-ladder report, out of scope here:
// after writing the others run_pipeline throws CapabilityError for it.
struct PipelineResult {
    PlanOutput output;
    SimResult sim;
    SchedulePlan baseline_plan;
    SimResult baseline_sim;
};
PipelineResult run_pipeline(const PipelineConfig& config, const std::string& out_dir);

}  // namespace loadsched

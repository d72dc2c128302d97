// capi.cu — the extern "C" boundary (include/lsg.h). Validation mirrors the
// reference's own checks so error classes match (errors.hpp:11-18):
// TraceConfig::validate (trace.cpp:18-24), PipelineConfig::validate
// (config.cpp:11-22), pso_order's guards (epoch_order.cpp:123-128).
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"

namespace lsg {

// kernel entry points (one per .cu file)
int generate_trace_device(uint64_t D, uint32_t E, uint64_t keep, uint64_t seed, uint32_t* d_trace,
                          uint32_t* d_inv, cudaStream_t st);
int build_reuse_graph_device(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D,
                             uint32_t N, uint64_t b, bool drop_last, uint64_t buffer_size, int mode,
                             bool rows_distinct_known, uint64_t* d_w, cudaStream_t st, uint32_t r0 = 0,
                             uint32_t r1 = kNone);
int pso_order_device(const uint64_t* d_w, uint32_t E, uint32_t swarm, uint32_t iters, double pp,
                     double pg, double inertia, double kick, uint32_t stagnation, uint32_t restart,
                     uint64_t seed, uint32_t* d_order, uint64_t* d_cost, uint64_t* d_hist,
                     uint32_t* d_iters, uint32_t* d_status, cudaStream_t st);
int plan_loop_device(const PlanDims& dm, uint64_t C, int policy, int remap, int balance, int insred, uint64_t thr,
                     const uint32_t* d_trace,
                     const uint32_t* d_order, const uint32_t* d_inv, uint32_t* d_items,
                     uint32_t* d_node_off, uint32_t* d_fb, uint32_t* d_fa, uint32_t* d_status,
                     cudaStream_t st);
int simulate_device(const uint32_t* d_items, const uint32_t* d_node_off, uint64_t T, uint32_t N,
                    uint64_t D, uint64_t C, int policy, uint32_t k0, uint32_t k1, uint32_t* d_hits,
                    uint32_t* d_misses, uint32_t* d_slot, const uint32_t* d_rstart, const uint32_t* d_rend,
                    const uint32_t* d_rcount, int insred, uint32_t* d_status, cudaStream_t st);
int plan_reads_device(const uint32_t* d_items, const uint32_t* d_node_off, uint32_t T, uint32_t N,
                      uint32_t S, uint32_t B, uint32_t keep, int chunked, uint64_t thr, uint32_t* rstart,
                      uint32_t* rend, uint32_t* rcount, uint32_t* needed, uint32_t* redundant,
                      cudaStream_t st);
int gather_device(const void* d_buf, const uint32_t* d_slots, uint64_t n, uint64_t sample_bytes,
                  void* d_out, cudaStream_t st);
int store_fill_device(const uint32_t* d_ids, uint64_t n, uint64_t sample_bytes, uint64_t seed,
                      void* d_dst, cudaStream_t st);
int batch_fetch_device(void* d_buf, const uint32_t* d_ids, const uint32_t* d_slots, uint64_t n,
                       uint64_t sample_bytes, uint64_t seed, void* d_out, cudaStream_t st);
int fetch_step_device(void* const* d_bufs, void* const* d_outs, const uint32_t* d_items,
                      const uint32_t* d_slots, const uint32_t* d_node_off, uint32_t k0, uint32_t k1,
                      uint64_t rows_hint, uint64_t sample_bytes, uint64_t seed, cudaStream_t st);

namespace {
thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

__global__ void k_identity_order(const uint64_t* __restrict__ w, uint32_t E, uint32_t* order,
                                 uint64_t* cost) {
    uint64_t c = 0;
    for (uint32_t i = threadIdx.x; i < E; i += blockDim.x) {
        order[i] = i;
        if (i + 1 < E) c += w[size_t(i) * E + i + 1];
    }
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, s);
    __shared__ uint64_t part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (uint32_t i = 0; i < (blockDim.x >> 5); ++i) t += part[i];
        *cost = t;
    }
}
}  // namespace

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_error(cudaError_t e, const char* where) {
    g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return kInternal;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void keep_pool() {
    static std::atomic<uint64_t> done_mask{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
    const uint64_t bit = 1ull << dev;
    if (done_mask.load() & bit) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // no cross-stream reuse that would insert a wait: the planner frees
        // its step-loop scratch right after launching the persistent kernel,
        // and a replay on another stream reusing that block would wait for
        // the whole plan (measured: the replay ended exactly with the
        // concurrent plan). Opportunistic reuse (already-completed frees)
        // stays on.
        int no = 0;
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
    }
    done_mask.fetch_or(bit);
}

bool l2_pin(cudaStream_t st, const void* p, size_t bytes) {
    static int on = -1;
    if (on < 0) {
        // measured (tools/replay_probe.py): pinning the replay's state made
        // both the replay and a planner beside a streaming fetch slower
        // (replay 232 -> 450 ms), so the window is opt-in
        const char* e = std::getenv("LSG_L2PIN");
        on = (e && e[0] == '1') ? 1 : 0;
    }
    if (!on || !p || bytes == 0) return false;
    int dev = 0, maxp = 0, maxw = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (maxp <= 0 || maxw <= 0) return false;
    static std::atomic<uint64_t> limit_set{0};  // per device: set-aside configured once
    const uint64_t bit = 1ull << (dev & 63);
    if (!(limit_set.load() & bit)) {
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(maxp)) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        limit_set.fetch_or(bit);
    }
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = const_cast<void*>(p);
    v.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, size_t(maxw));
    v.accessPolicyWindow.hitRatio = float(std::min<double>(1.0, double(maxp) / double(v.accessPolicyWindow.num_bytes)));
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

void l2_unpin(cudaStream_t st) {
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaGetLastError();
}

int d2h_small(void* h, const void* d, size_t bytes, cudaStream_t st) {
    static thread_local void* stage = nullptr;
    if (bytes > 64) return set_error(kInternal, "d2h_small: readback larger than 64 bytes");
    if (!stage) LSG_CUDA(cudaMallocHost(&stage, 64));
    LSG_CUDA(cudaMemcpyAsync(stage, d, bytes, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    std::memcpy(h, stage, bytes);
    return kOk;
}

size_t exclusive_smem(size_t need) {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("LSG_EXCLUSIVE_SM");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    constexpr size_t kWhole = 200 * 1024;  // > half an SM's 228 KB: no second CTA of this size or a fetch CTA fits
    return on ? std::max(need, kWhole) : need;
}

bool profiling() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("LSG_PROFILE");
        on = (e && e[0] && e[0] != '0') ? 1 : 0;
    }
    return on == 1;
}

static int validate(const lsg_config* c, lsg_shape* sh) {
    if (!c) return set_error(kValidation, "null config");
    if (c->num_nodes == 0) return set_error(kConfig, "num_nodes must be >= 1");
    if (c->local_batch == 0) return set_error(kConfig, "local_batch must be >= 1");
    if (c->num_epochs == 0) return set_error(kConfig, "num_epochs must be >= 1");
    const uint64_t B = uint64_t(c->num_nodes) * c->local_batch;
    if (c->dataset_size < B) return set_error(kConfig, "dataset_size must be >= num_nodes * local_batch");
    if (c->buffer_capacity == 0) return set_error(kConfig, "buffer_capacity must be >= 1");
    if (c->chunk_threshold == 0) return set_error(kConfig, "chunk_threshold must be >= 1");
    if (c->pso_swarm == 0) return set_error(kConfig, "pso_swarm must be >= 1");
    if (c->pso_iters == 0) return set_error(kConfig, "pso_iters must be >= 1");
    if (c->pso_p_personal < 0.0 || c->pso_p_personal > 1.0 || c->pso_p_global < 0.0 || c->pso_p_global > 1.0)
        return set_error(kConfig, "pso pull probabilities must lie in [0, 1]");
    if (c->pso_inertia < 0.0 || c->pso_inertia >= 1.0) return set_error(kConfig, "pso_inertia must lie in [0, 1)");
    if (c->pso_kick < 0.0 || c->pso_kick > 1.0) return set_error(kConfig, "pso_kick must lie in [0, 1]");
    if (c->dataset_size >= (1ull << 31)) return set_error(kCapability, "dataset_size must be < 2^31 on device");
    if (sh) {
        sh->global_batch = B;
        sh->steps_per_epoch = c->drop_last ? c->dataset_size / B : (c->dataset_size + B - 1) / B;
        sh->keep = c->drop_last ? sh->steps_per_epoch * B : c->dataset_size;
        sh->total_steps = uint64_t(c->num_epochs) * sh->steps_per_epoch;
        sh->total_items = uint64_t(c->num_epochs) * sh->keep;
    }
    return kOk;
}

}  // namespace lsg

using namespace lsg;

extern "C" {

int lsg_version(void) { return 1; }
const char* lsg_last_error(void) { return g_err.c_str(); }
uint64_t lsg_launch_count(void) { return g_launches.load(); }

int lsg_shape_of(const lsg_config* cfg, lsg_shape* out) { return validate(cfg, out); }

int lsg_generate_trace(const lsg_config* cfg, uint32_t* d_trace, void* stream) {
    // only the trace fields are validated here (trace.cpp:18-24)
    if (!cfg) return set_error(kValidation, "null config");
    if (cfg->num_nodes == 0) return set_error(kConfig, "num_nodes must be >= 1");
    if (cfg->local_batch == 0) return set_error(kConfig, "local_batch must be >= 1");
    if (cfg->num_epochs == 0) return set_error(kConfig, "num_epochs must be >= 1");
    const uint64_t B = uint64_t(cfg->num_nodes) * cfg->local_batch;
    if (cfg->dataset_size < B) return set_error(kConfig, "dataset_size must be >= num_nodes * local_batch");
    if (cfg->dataset_size >= (1ull << 31)) return set_error(kCapability, "dataset_size must be < 2^31 on device");
    const uint64_t S = cfg->drop_last ? cfg->dataset_size / B : (cfg->dataset_size + B - 1) / B;
    const uint64_t keep = cfg->drop_last ? S * B : cfg->dataset_size;
    return generate_trace_device(cfg->dataset_size, cfg->num_epochs, keep, cfg->seed, d_trace, nullptr,
                                 static_cast<cudaStream_t>(stream));
}

int lsg_build_reuse_graph(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D, uint32_t N,
                          uint64_t b, int32_t drop_last, uint64_t buffer_size, int32_t mode,
                          uint64_t* d_w, void* stream) {
    if (N == 0 || b == 0) return set_error(kConfig, "num_nodes and local_batch must be >= 1");
    if (D >= (1ull << 31) || len >= (1ull << 31)) return set_error(kCapability, "trace too large for device ids");
    return build_reuse_graph_device(d_trace, E, len, D, N, b, drop_last != 0, buffer_size, mode, false,
                                    d_w, static_cast<cudaStream_t>(stream));
}

int lsg_build_reuse_graph_rows(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D, uint32_t N,
                               uint64_t b, int32_t drop_last, uint64_t buffer_size, int32_t mode,
                               uint32_t row_begin, uint32_t row_end, uint64_t* d_w_rows, void* stream) {
    if (N == 0 || b == 0) return set_error(kConfig, "num_nodes and local_batch must be >= 1");
    if (D >= (1ull << 31) || len >= (1ull << 31)) return set_error(kCapability, "trace too large for device ids");
    if (row_begin > row_end || row_end > E) return set_error(kValidation, "build_reuse_graph_rows: bad row range");
    return build_reuse_graph_device(d_trace, E, len, D, N, b, drop_last != 0, buffer_size, mode, false,
                                    d_w_rows, static_cast<cudaStream_t>(stream), row_begin, row_end);
}

int lsg_pso_order(const uint64_t* d_w, uint32_t E, uint32_t swarm, uint32_t iters, double p_personal,
                  double p_global, double inertia, double kick, uint32_t stagnation, uint32_t restart,
                  uint64_t seed, uint32_t* d_order, uint64_t* d_cost, uint64_t* d_hist, uint32_t* d_iters,
                  void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    uint32_t* status = sc.get<uint32_t>(1);
    if (!status) return set_error(kInternal, "pso: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(status, 0, 4, st));
    int rc = pso_order_device(d_w, E, swarm, iters, p_personal, p_global, inertia, kick, stagnation,
                              restart, seed, d_order, d_cost, d_hist, d_iters, status, st);
    if (rc) return rc;
    uint32_t h = 0;
    if (int _rc = d2h_small(&h, status, 4, st)) return _rc;
    LSG_CUDA(cudaStreamSynchronize(st));
    if (h) return set_error(kInternal, "pso_order: velocity capacity exceeded");
    return kOk;
}

int lsg_plan(const lsg_config* cfg, const lsg_plan_out* out, void* stream) {
    lsg_shape sh;
    int rc = validate(cfg, &sh);
    if (rc) return rc;
    if (!out || !out->items || !out->node_off) return set_error(kValidation, "plan: items and node_off are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t E = cfg->num_epochs, N = cfg->num_nodes;
    const uint64_t D = cfg->dataset_size;
    Scratch sc(st);
    uint32_t* trace = out->trace ? out->trace : sc.get<uint32_t>(sh.total_items);
    uint32_t* inv = sc.get<uint32_t>(size_t(E) * D);
    uint64_t* graph = out->graph ? out->graph : sc.get<uint64_t>(size_t(E) * E);
    uint32_t* order = out->order ? out->order : sc.get<uint32_t>(E);
    uint64_t* cost = out->cost ? out->cost : sc.get<uint64_t>(1);
    uint32_t* status = sc.get<uint32_t>(1);
    if (!trace || !inv || !graph || !order || !cost || !status)
        return set_error(kInternal, "plan: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(status, 0, 4, st));
    if ((rc = generate_trace_device(D, E, sh.keep, cfg->seed, trace, inv, st))) return rc;
    if ((rc = build_reuse_graph_device(trace, E, sh.keep, D, N, cfg->local_batch, cfg->drop_last != 0,
                                       cfg->buffer_capacity, cfg->graph_mode, true, graph, st)))
        return rc;
    if (cfg->optim_order) {
        rc = pso_order_device(graph, E, cfg->pso_swarm, cfg->pso_iters, cfg->pso_p_personal,
                              cfg->pso_p_global, cfg->pso_inertia, cfg->pso_kick, cfg->pso_stagnation,
                              cfg->pso_restart, cfg->seed, order, cost, out->hist, out->iters, status, st);
        if (rc) return rc;
    } else {
        k_identity_order<<<1, 256, 0, st>>>(graph, E, order, cost);
        LSG_LAUNCH_CHECK("k_identity_order");
        if (out->iters) LSG_CUDA(cudaMemsetAsync(out->iters, 0, 4, st));
    }
    PlanDims dm{D, sh.global_batch, sh.steps_per_epoch, sh.keep, sh.total_steps, N, E,
                uint32_t(cfg->local_batch)};
    if ((rc = plan_loop_device(dm, cfg->buffer_capacity, cfg->policy, cfg->optim_remap, cfg->optim_balance,
                               cfg->insert_redundant && cfg->optim_chunk, cfg->chunk_threshold, trace,
                               order, inv, out->items, out->node_off, out->fetch_before,
                               out->fetch_after, status, st)))
        return rc;
    // StepPlan.reads: plan_chunks when optim_chunk, singles otherwise (pipeline.cpp:83-88)
    if ((rc = plan_reads_device(out->items, out->node_off, uint32_t(sh.total_steps), N,
                                uint32_t(sh.steps_per_epoch), uint32_t(sh.global_batch), uint32_t(sh.keep),
                                cfg->optim_chunk, cfg->chunk_threshold, out->read_start, out->read_end,
                                out->read_count, out->read_needed, out->read_redundant, st)))
        return rc;
    uint32_t h = 0;
    if (int _rc = d2h_small(&h, status, 4, st)) return _rc;
    LSG_CUDA(cudaStreamSynchronize(st));
    if (h & (1u << 20))
        return set_error(kCapability, "plan: the LRU planner's redundant ids exceed its device store (2 GiB)");
    if (h) return set_error(kInternal, "plan: device invariant violated (status " + std::to_string(h) + ")");
    return kOk;
}

int lsg_plan_host(const lsg_config* cfg, const lsg_plan_out* h, void* stream) {
    lsg_shape sh;
    int rc = validate(cfg, &sh);
    if (rc) return rc;
    if (!h || !h->items || !h->node_off) return set_error(kValidation, "plan: items and node_off are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t E = cfg->num_epochs, N = cfg->num_nodes;
    const size_t T = sh.total_steps;
    struct Arr { void* host; size_t bytes; void** dev; };
    lsg_plan_out d{};
    Arr arrs[] = {
        {h->trace, sh.total_items * 4, reinterpret_cast<void**>(&d.trace)},
        {h->graph, size_t(E) * E * 8, reinterpret_cast<void**>(&d.graph)},
        {h->order, size_t(E) * 4, reinterpret_cast<void**>(&d.order)},
        {h->cost, 8, reinterpret_cast<void**>(&d.cost)},
        {h->hist, size_t(cfg->pso_iters) * 8, reinterpret_cast<void**>(&d.hist)},
        {h->iters, 4, reinterpret_cast<void**>(&d.iters)},
        {h->items, sh.total_items * 4, reinterpret_cast<void**>(&d.items)},
        {h->node_off, T * (N + 1) * 4, reinterpret_cast<void**>(&d.node_off)},
        {h->fetch_before, T * N * 4, reinterpret_cast<void**>(&d.fetch_before)},
        {h->fetch_after, T * N * 4, reinterpret_cast<void**>(&d.fetch_after)},
        {h->read_start, sh.total_items * 4, reinterpret_cast<void**>(&d.read_start)},
        {h->read_end, sh.total_items * 4, reinterpret_cast<void**>(&d.read_end)},
        {h->read_count, T * N * 4, reinterpret_cast<void**>(&d.read_count)},
        {h->read_needed, T * N * 4, reinterpret_cast<void**>(&d.read_needed)},
        {h->read_redundant, T * N * 4, reinterpret_cast<void**>(&d.read_redundant)},
    };
    Scratch sc(st);
    for (Arr& a : arrs)
        if (a.host) {
            *a.dev = sc.get<unsigned char>(a.bytes);
            if (!*a.dev) return set_error(kInternal, "plan_host: device allocation failed");
        }
    if ((rc = lsg_plan(cfg, &d, stream))) return rc;
    for (Arr& a : arrs)
        if (a.host) LSG_CUDA(cudaMemcpyAsync(a.host, *a.dev, a.bytes, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    return kOk;
}

int lsg_simulate(const uint32_t* d_items, const uint32_t* d_node_off, uint64_t T, uint32_t N, uint64_t D,
                 uint64_t capacity, int32_t policy, uint32_t node_begin, uint32_t node_end,
                 uint32_t* d_hits, uint32_t* d_misses, uint32_t* d_slot, void* stream) {
    return lsg_simulate_ex(d_items, d_node_off, T, N, D, capacity, policy, 0, nullptr, nullptr, nullptr,
                           node_begin, node_end, d_hits, d_misses, d_slot, stream);
}

int lsg_simulate_ex(const uint32_t* d_items, const uint32_t* d_node_off, uint64_t T, uint32_t N, uint64_t D,
                    uint64_t capacity, int32_t policy, int32_t insert_redundant, const uint32_t* d_read_start,
                    const uint32_t* d_read_end, const uint32_t* d_read_count, uint32_t node_begin,
                    uint32_t node_end, uint32_t* d_hits, uint32_t* d_misses, uint32_t* d_slot, void* stream) {
    if (capacity == 0) return set_error(kValidation, "buffer capacity must be >= 1");
    if (policy != 0 && policy != 1) return set_error(kConfig, "simulate: policy must be clairvoyant (0) or lru (1)");
    if (N == 0) return set_error(kValidation, "simulate: num_nodes must be >= 1");
    if (node_end > N || node_begin > node_end) return set_error(kValidation, "simulate: bad node range");
    if (D >= (1ull << 31)) return set_error(kCapability, "simulate: dataset_size must be < 2^31 on device");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    uint32_t* status = sc.get<uint32_t>(1);
    if (!status) return set_error(kInternal, "simulate: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(status, 0, 4, st));
    int rc = simulate_device(d_items, d_node_off, T, N, D, capacity, policy, node_begin, node_end, d_hits,
                             d_misses, d_slot, d_read_start, d_read_end, d_read_count, insert_redundant != 0,
                             status, st);
    if (rc) return rc;
    uint32_t h = 0;
    if (int _rc = d2h_small(&h, status, 4, st)) return _rc;
    LSG_CUDA(cudaStreamSynchronize(st));
    if (h) return set_error(kInternal, "simulate: device invariant violated (status " + std::to_string(h) + ")");
    return kOk;
}

int lsg_store_fill(const uint32_t* d_ids, uint64_t n, uint64_t sample_bytes, uint64_t fill_seed,
                   void* d_dst, void* stream) {
    return store_fill_device(d_ids, n, sample_bytes, fill_seed, d_dst, static_cast<cudaStream_t>(stream));
}

int lsg_gather(const void* d_buf, const uint32_t* d_slots, uint64_t n, uint64_t sample_bytes,
               void* d_out, void* stream) {
    return gather_device(d_buf, d_slots, n, sample_bytes, d_out, static_cast<cudaStream_t>(stream));
}

int lsg_batch_fetch(void* d_buf, const uint32_t* d_ids, const uint32_t* d_slots, uint64_t n,
                    uint64_t sample_bytes, uint64_t fill_seed, void* d_out, void* stream) {
    return batch_fetch_device(d_buf, d_ids, d_slots, n, sample_bytes, fill_seed, d_out,
                              static_cast<cudaStream_t>(stream));
}

int lsg_fetch_step(void* const* d_bufs, void* const* d_outs, const uint32_t* d_items,
                   const uint32_t* d_slots, const uint32_t* d_node_off, uint32_t node_begin,
                   uint32_t node_end, uint64_t rows_hint, uint64_t sample_bytes, uint64_t fill_seed,
                   void* stream) {
    return fetch_step_device(d_bufs, d_outs, d_items, d_slots, d_node_off, node_begin, node_end,
                             rows_hint, sample_bytes, fill_seed, static_cast<cudaStream_t>(stream));
}

int lsg_fetch_steps(void* const* d_bufs, void* const* d_outs, const uint32_t* d_items, const uint32_t* d_slots,
                    const uint32_t* d_node_off, const uint32_t* h_node_off, uint64_t step_begin,
                    uint64_t step_end, uint32_t N, uint32_t node_begin, uint32_t node_end,
                    uint64_t sample_bytes, uint64_t fill_seed, void* stream) {
    // a job without a host tier: misses synthesised on device (lsg_fetch_job)
    lsg_fetch_job_desc d{d_bufs, d_outs, d_items, d_slots, d_node_off, h_node_off, step_begin, step_end,
                         N, node_begin, node_end, sample_bytes, fill_seed, nullptr, 0, nullptr};
    lsg_fetch_job* j = nullptr;
    if (int rc = lsg_fetch_job_create(&d, &j, stream)) return rc;
    const int rc = lsg_fetch_job_run(j, stream);
    lsg_fetch_job_destroy(j, stream);
    return rc;
}

}  // extern "C"

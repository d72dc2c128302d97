/* include/lsg.h — C ABI of the B200-native SOLAR loading planner ("lsg").
 *
 * This is the drop-in boundary for the reference library's hot path
 * (/root/reference/proj, namespace loadsched). Every entry point is plain C:
 * integers, plain pointers and sizes, no torch or STL types. Each function
 * cites the reference interface it replaces. The host C++ layer
 * (include/loadsched_gpu.hpp, implemented in
 * paper_2211_00224_b200/host/loadsched_gpu.cpp -> libloadsched_gpu.so)
 * re-exposes the reference's own C++ signatures on top of these calls;
 * INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Return value: 0 on success, else the reference ErrorClass code
 *    (errors.hpp:11-18): 2 Config, 3 Validation, 4 Capability, 6 Storage,
 *    7 Internal. lsg_last_error() returns a thread-local message.
 *  - "d_" pointers are device (HBM) pointers; "h_" pointers are host memory.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Device-pointer
 *    calls are asynchronous on the stream unless stated; calls that must
 *    report a device-detected invariant failure synchronise the stream once.
 *  - Sample ids are uint32 on the device (the reference SampleId is uint64,
 *    trace.hpp:11; D < 2^31 is enforced, widening happens in the host layer).
 *  - Hit tags travel in bit 31 of an item: item = id | (hit ? LSG_HIT_BIT : 0).
 *  - Keys/next-use values: LSG_NEVER means "never used again" (buffer.hpp:19).
 */
#ifndef LSG_H
#define LSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSG_HIT_BIT 0x80000000u
#define LSG_NEVER 0xFFFFFFFEu

/* Mirrors PipelineConfig (config.hpp:17-36) minus the cost-model fields,
 * which do not reach the hot path. Field order is ABI. */
typedef struct lsg_config {
    uint64_t dataset_size;    /* D  (TraceConfig::dataset_size) */
    uint32_t num_epochs;      /* E */
    uint32_t num_nodes;       /* N */
    uint64_t local_batch;     /* b */
    uint64_t seed;
    int32_t drop_last;
    int32_t policy;           /* 0 clairvoyant, 1 lru (Policy, buffer.hpp:16) */
    uint64_t buffer_capacity; /* C per node */
    int32_t graph_mode;       /* 0 global, 1 pernode (WindowMode) */
    int32_t insert_redundant; /* chunk_insert_redundant */
    uint64_t chunk_threshold;
    int32_t optim_order, optim_remap, optim_balance, optim_chunk;
    uint32_t pso_swarm, pso_iters, pso_stagnation, pso_restart;
    double pso_p_personal, pso_p_global, pso_inertia, pso_kick;
} lsg_config;

/* Derived plan shape (TraceConfig::steps_per_epoch, trace.cpp:12-16). */
typedef struct lsg_shape {
    uint64_t global_batch;    /* B = N*b */
    uint64_t steps_per_epoch; /* S */
    uint64_t keep;            /* ids kept per epoch (S*B under drop_last, else D) */
    uint64_t total_steps;     /* T = E*S */
    uint64_t total_items;     /* E*keep */
} lsg_shape;

/* Device outputs of lsg_plan (PlanOutput, pipeline.hpp:17-22 flattened).
 * Any pointer may be NULL except items/node_off, which the planner needs. */
typedef struct lsg_plan_out {
    uint32_t* trace;        /* [E][keep]  AccessTrace.epochs */
    uint64_t* graph;        /* [E][E]     ReuseGraph.weights */
    uint32_t* order;        /* [E]        SchedulePlan.order.order */
    uint64_t* cost;         /* [1]        SchedulePlan.order.cost */
    uint64_t* hist;         /* [pso_iters] PsoResult.history */
    uint32_t* iters;        /* [1]        PsoResult.iterations */
    uint32_t* items;        /* [E*keep]   node lists, steps in execution order */
    uint32_t* node_off;     /* [T][N+1]   per-step list offsets */
    uint32_t* fetch_before; /* [T][N]     StepPlan.fetches_before */
    uint32_t* fetch_after;  /* [T][N]     StepPlan.fetches_after */
    /* StepPlan.reads (pipeline.cpp:83-88): reads of list (g, k) at its item
     * offsets, start == end for a Single read; counts and ChunkPlan.needed /
     * .redundant per (g, k). NULL read_start skips chunk planning. */
    uint32_t* read_start;   /* [E*keep] */
    uint32_t* read_end;     /* [E*keep] */
    uint32_t* read_count;   /* [T][N] */
    uint32_t* read_needed;  /* [T][N] */
    uint32_t* read_redundant; /* [T][N] */
} lsg_plan_out;

int lsg_version(void);
const char* lsg_last_error(void);

/* Validation + derived shape; Config errors as TraceConfig::validate
 * (trace.cpp:18-24) and PipelineConfig::validate (config.cpp:11-22). */
int lsg_shape_of(const lsg_config* cfg, lsg_shape* out);

/* ---- K1: generate_trace(const TraceConfig&) -> AccessTrace
 *      (trace.hpp:40, trace.cpp:26-43). d_trace: [E][keep] uint32. */
int lsg_generate_trace(const lsg_config* cfg, uint32_t* d_trace, void* stream);

/* ---- K2/K3: build_reuse_graph(trace, buffer_size, mode) -> ReuseGraph
 *      (reuse_graph.hpp:53, reuse_graph.cpp:77-101). d_trace: [E][len]
 *      (any ids < D, repeats allowed, as read_trace admits); d_w: [E][E]. */
int lsg_build_reuse_graph(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D,
                          uint32_t N, uint64_t b, int32_t drop_last, uint64_t buffer_size,
                          int32_t mode, uint64_t* d_w, void* stream);

/* Rows [row_begin, row_end) of the same matrix into d_w_rows
 * ([row_end - row_begin][E], row-major): the multi-GPU row sharding of K3
 * (each GPU builds all window bitsets and its row block; an all-gather of the
 * blocks yields build_reuse_graph's weights on every GPU). */
int lsg_build_reuse_graph_rows(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D,
                               uint32_t N, uint64_t b, int32_t drop_last, uint64_t buffer_size,
                               int32_t mode, uint32_t row_begin, uint32_t row_end, uint64_t* d_w_rows,
                               void* stream);

/* ---- K4: pso_order(graph, PsoParams) -> PsoResult
 *      (epoch_order.hpp:60, epoch_order.cpp:121-221). Bit-exact. */
int lsg_pso_order(const uint64_t* d_w, uint32_t E, uint32_t swarm, uint32_t iters,
                  double p_personal, double p_global, double inertia, double kick,
                  uint32_t stagnation, uint32_t restart, uint64_t seed, uint32_t* d_order,
                  uint64_t* d_cost, uint64_t* d_hist, uint32_t* d_iters, void* stream);

/* ---- K1..K6: plan_schedule(const PipelineConfig&) -> PlanOutput
 *      (pipeline.hpp:27, pipeline.cpp:32-120). Synchronises `stream` once to
 *      report device-side invariant failures (InternalError). */
int lsg_plan(const lsg_config* cfg, const lsg_plan_out* out, void* stream);

/* Same, with host outputs (pinned or pageable): the e2e path. Host arrays
 * follow lsg_plan_out layout; NULL members are skipped. */
int lsg_plan_host(const lsg_config* cfg, const lsg_plan_out* h_out, void* stream);

/* ---- K7: simulate_plan(plan, capacity, policy, false) -> SimResult
 *      (buffer.hpp:117-118, buffer.cpp:183-247). The plan is given in the
 *      lsg_plan_out item/offset layout with `T` steps of N nodes. Replays
 *      nodes [node_begin, node_end) only (per-rank sharding); rows of other
 *      nodes are left untouched. d_hits/d_misses: [T][N]. Optional d_slot
 *      ([total items]) receives, per access, the HBM buffer slot the sample
 *      occupies after its access (LSG_NEVER when it was bypassed). */
int lsg_simulate(const uint32_t* d_items, const uint32_t* d_node_off, uint64_t T, uint32_t N,
                 uint64_t D, uint64_t capacity, int32_t policy, uint32_t node_begin,
                 uint32_t node_end, uint32_t* d_hits, uint32_t* d_misses, uint32_t* d_slot,
                 void* stream);

/* Same with simulate_plan's insert_redundant (buffer.cpp:224-238): after each
 * (step, node) list, the ids its chunk reads stream without requesting them
 * (redundant_ids, chunking.cpp:35-45) are inserted silently with their next
 * position on the node. d_read_*: the plan's reads at its item offsets
 * (lsg_plan_out.read_start / read_end / read_count). Clairvoyant policy;
 * d_slot must be NULL when insert_redundant is set. */
int lsg_simulate_ex(const uint32_t* d_items, const uint32_t* d_node_off, uint64_t T, uint32_t N, uint64_t D,
                    uint64_t capacity, int32_t policy, int32_t insert_redundant, const uint32_t* d_read_start,
                    const uint32_t* d_read_end, const uint32_t* d_read_count, uint32_t node_begin,
                    uint32_t node_end, uint32_t* d_hits, uint32_t* d_misses, uint32_t* d_slot, void* stream);

/* ---- K9: Store payload (store.cpp:70-80) of samples ids[0..n) written to
 *      dst rows: row r of `dst` (row pitch sample_bytes) receives the bytes
 *      Store::read_one(ids[r]) would return for fill_seed. */
int lsg_store_fill(const uint32_t* d_ids, uint64_t n, uint64_t sample_bytes, uint64_t fill_seed,
                   void* d_dst, void* stream);

/* ---- K8: batch gather from an HBM-resident sample buffer
 *      (replaces Store::read_one/read_chunk, store.hpp:42-44, for buffered
 *      samples). out row r = buf row slots[r]; rows are sample_bytes long and
 *      16-byte aligned. */
int lsg_gather(const void* d_buf, const uint32_t* d_slots, uint64_t n, uint64_t sample_bytes,
               void* d_out, void* stream);

/* ---- K8+K9: fetch one node's batch for one step (the loading phase of a
 *      training step on that rank): rows whose replay slot (lsg_simulate
 *      d_slot, bit 31 = resident at step start) is a hit are gathered from
 *      their HBM slot; all other rows receive the sample's Store payload
 *      (the storage read, synthesised on device) in the batch and, unless the
 *      replay bypassed the sample (LSG_NEVER), in its new HBM slot. Hits are
 *      copied before any miss is written, so a slot freed and re-filled in
 *      the same step is read before it is overwritten. */
int lsg_batch_fetch(void* d_buf, const uint32_t* d_ids, const uint32_t* d_slots, uint64_t n,
                    uint64_t sample_bytes, uint64_t fill_seed, void* d_out, void* stream);

/* Same for every node of [node_begin, node_end) of one step in two launches:
 * d_items/d_slots point at the step's first item (lsg_plan_out.items +
 * step base), d_node_off at the step's [N+1] offsets, d_bufs/d_outs are
 * DEVICE arrays of (node_end - node_begin) buffer / batch pointers. rows_hint
 * (the number of rows in the range, or 0) only sizes the grid. */
int lsg_fetch_step(void* const* d_bufs, void* const* d_outs, const uint32_t* d_items,
                   const uint32_t* d_slots, const uint32_t* d_node_off, uint32_t node_begin,
                   uint32_t node_end, uint64_t rows_hint, uint64_t sample_bytes, uint64_t fill_seed,
                   void* stream);

/* The loading phase of steps [step_begin, step_end) of a plan, in step order
 * (lsg_fetch_job without a host tier: misses synthesised on device; the
 * job's miss list is built on the device, then two launches per step from C
 * without host round trips):
 * d_items/d_slots/d_node_off are the WHOLE plan's arrays (lsg_plan_out
 * layout, [T][N+1] offsets), h_node_off a host copy of the offsets (step
 * bases and grid sizes). When the call returns the batch tensors hold the
 * LAST step's rows (rows past its list are unspecified): the fused kernel
 * alternates steps between the tensors and an internal scratch set, so one
 * step's batch-row stores need not wait for the previous step's. */
int lsg_fetch_steps(void* const* d_bufs, void* const* d_outs, const uint32_t* d_items, const uint32_t* d_slots,
                    const uint32_t* d_node_off, const uint32_t* h_node_off, uint64_t step_begin,
                    uint64_t step_end, uint32_t N, uint32_t node_begin, uint32_t node_end,
                    uint64_t sample_bytes, uint64_t fill_seed, void* stream);

/* ---- The loading phase of a whole job with a real miss source ----
 * The HOST TIER: the Store payload rows of the whole dataset (store.cpp:70-80;
 * row i at byte i * sample_bytes, i.e. the Store file without its 22-byte
 * header) in a file on a tmpfs, mapped and pinned (cudaHostRegister, mapped),
 * so all processes of a box share one copy and the GPU reads it over PCIe.
 * create != 0 writes the file (host threads); else it is opened and must be
 * count x sample_bytes long. Errors: Storage (6). */
typedef struct lsg_host_rows lsg_host_rows;
int lsg_host_rows_open(const char* path, uint64_t count, uint64_t sample_bytes, uint64_t fill_seed, int32_t create,
                       lsg_host_rows** out);
int lsg_host_rows_info(const lsg_host_rows* h, uint64_t* count, uint64_t* sample_bytes, void** host_base);
void lsg_host_rows_close(lsg_host_rows* h);

/* A job's fetch (replaces Store::read_one/read_chunk, store.hpp:42-44, for the
 * batches of steps [step_begin, step_end) of ranks [node_begin, node_end)):
 * hits are gathered from the HBM sample buffers (TMA bulk copies), misses come
 * from `host` (NULL: the Store payload synthesised on device) into their batch
 * row and, unless the replay bypassed them, their new buffer slot.
 * lsg_fetch_job_create builds the job's miss list on `stream` and, with a
 * host tier, starts the miss prefetcher there (a persistent kernel reading
 * the host rows over PCIe into a device ring of about ring_bytes, 0 = 2 GiB)
 * and returns once it is resident; `stream` then stays busy until the job's
 * misses are consumed, so give each job in flight its own. lsg_fetch_job_run
 * enqueues the steps on the fetch stream (it waits for the miss list only);
 * afterwards the batch tensors hold the job's last step (rows past its list
 * unspecified; earlier steps alternate with an internal scratch set).
 * lsg_fetch_job_stats (synchronous) reads {misses, kept misses, host bytes,
 * hits}; lsg_fetch_job_destroy frees stream-ordered after the job. */
typedef struct lsg_fetch_job lsg_fetch_job;
/* A miss ring shared by consecutive jobs of one fetch stream (same ranks and
 * buffers, jobs fetched in creation order): a job's prefetcher runs on into
 * the ring while the previous job still fetches, so a job's all-miss first
 * epoch is largely staged in HBM before its fetch starts. The ring must hold
 * a step's rows; destroy it (a device synchronisation) only when no job that
 * uses it is in flight. */
typedef struct lsg_miss_stream lsg_miss_stream;
int lsg_miss_stream_create(uint64_t sample_bytes, uint64_t ring_bytes, lsg_miss_stream** out);
void lsg_miss_stream_destroy(lsg_miss_stream* ms);
typedef struct {
    void* const* d_bufs;        /* device array of (node_end - node_begin) HBM buffer pointers */
    void* const* d_outs;        /* device array of batch tensor pointers */
    const uint32_t* d_items;    /* the whole plan's items (lsg_plan_out layout) */
    const uint32_t* d_slots;    /* lsg_simulate d_slot of the same plan */
    const uint32_t* d_node_off; /* [T][N+1] */
    const uint32_t* h_node_off; /* host copy of the offsets */
    uint64_t step_begin, step_end;
    uint32_t N, node_begin, node_end;
    uint64_t sample_bytes, fill_seed;
    const lsg_host_rows* host;  /* NULL: synthesised misses */
    uint64_t ring_bytes;        /* the job's own ring (0 = 2 GiB) when misses is NULL */
    lsg_miss_stream* misses;    /* shared ring, or NULL */
} lsg_fetch_job_desc;
int lsg_fetch_job_create(const lsg_fetch_job_desc* desc, lsg_fetch_job** out, void* stream);
int lsg_fetch_job_run(lsg_fetch_job* job, void* stream);
int lsg_fetch_job_stats(lsg_fetch_job* job, uint64_t* h_stats4, void* stream);
void lsg_fetch_job_destroy(lsg_fetch_job* job, void* stream);

/* ---- Run report totals over a device plan (lsg_plan_out layout):
 * total_barrier_cost and total_io_cost (pipeline.cpp:133-151) with
 * barrier_time (balance.cpp:41-47) and read_cost (cost_model.cpp:9-18),
 * bit-identical doubles (reference summation order, no FMA). A list's fetch
 * count is its untagged items (d_items), or d_fetches[T][N] when given.
 * d_read_* may be NULL (then *h_io_total = 0). */
int lsg_plan_costs(const uint32_t* d_items, const uint32_t* d_fetches, const uint32_t* d_node_off,
                   const uint32_t* d_read_start,
                   const uint32_t* d_read_end, const uint32_t* d_read_count, uint64_t T, uint32_t N,
                   double seek_cost, double stream_cost, double* h_barrier_total, double* h_io_total, void* stream);

/* ---- The sample Store (store.hpp:13-81, store.cpp:37-148): SLRD files
 *      (22-byte header + one continuous splitmix64 payload stream).
 *      Errors: Storage (6) for I/O, format and budget failures, Validation
 *      (3) for bad ranges, as the reference throws them. */
typedef struct lsg_store lsg_store;

/* create_store(path, count, size, fill_seed, max_bytes) (store.cpp:37-82);
 * the payload is computed on the GPU and written out. Byte-identical to the
 * reference file. */
int lsg_store_create(const char* path, uint64_t sample_count, uint64_t sample_size, uint64_t fill_seed,
                     uint64_t max_bytes, void* stream);

/* Store::Store (store.cpp:84-117): validates magic, version, file length. */
int lsg_store_open(const char* path, lsg_store** out);
int lsg_store_info(const lsg_store* h, uint64_t* sample_count, uint64_t* sample_size);
void lsg_store_close(lsg_store* h);

/* Store::read_chunk (store.cpp:141-148) into host memory; read_one is
 * count == 1 (store.cpp:134-139). */
int lsg_store_read(const lsg_store* h, uint64_t start, uint64_t count, void* h_dst);

/* Samples h_ids[0..n) into device rows (pitch = sample size): the ids are
 * cut into chunk reads of span <= threshold (plan_chunks, chunking.cpp:9-33)
 * read in parallel into pinned staging, moved to HBM in one async copy and
 * scattered to their rows. Stream-ordered. */
int lsg_store_read_rows(lsg_store* h, const uint32_t* h_ids, uint64_t n, uint64_t threshold, void* d_rows,
                        void* stream);

/* lsg_fetch_step with the misses read from the Store instead of
 * synthesised: hits gathered from the HBM buffers, misses read from the file
 * (chunk reads of span <= threshold) into their batch rows and, unless the
 * replay bypassed them, their new buffer slots. h_bufs / h_outs: HOST arrays
 * holding the same device pointers as d_bufs / d_outs. */
int lsg_fetch_step_store(lsg_store* h, void* const* d_bufs, void* const* d_outs, void* const* h_bufs,
                         void* const* h_outs, const uint32_t* d_items, const uint32_t* d_slots,
                         const uint32_t* d_node_off, uint32_t node_begin, uint32_t node_end, uint64_t rows_hint,
                         uint64_t threshold, void* stream);

/* ---- Per-call pieces of the reference API around the path ----
 * first_buffer_window / last_buffer_window (reuse_graph.cpp:43-75): window
 * bitsets of every epoch, [E][W][ceil(D/32)] words, W = 1 (Global) or N. */
int lsg_buffer_windows(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D, uint32_t N, uint64_t b,
                       int32_t drop_last, uint64_t buffer_size, int32_t mode, uint32_t* d_first, uint32_t* d_last,
                       void* stream);
/* brute_force_order (epoch_order.cpp:32-52): exact minimum over all E! open
 * paths, ties to the lexicographically smallest order; E <= 10. */
int lsg_brute_force_order(const uint64_t* d_w, uint32_t E, uint32_t* d_order, uint64_t* d_cost, void* stream);
/* remap_step / slice_step (locality.cpp:7-73, slice != 0) of one batch
 * against explicit residency sets (node k holds h_res_ids[h_res_off[k] ..
 * h_res_off[k+1])): node lists into h_items (len, id | LSG_HIT_BIT) at
 * h_node_off[N+1]. Runs the cluster step loop for one step, no advance. */
int lsg_remap_step(const uint64_t* h_res_off, const uint32_t* h_res_ids, uint32_t N, const uint32_t* h_batch,
                   uint64_t len, uint64_t local_batch, int32_t slice, uint32_t* h_items, uint32_t* h_node_off,
                   void* stream);
/* balance_step (balance.cpp:10-39) of one step's lists, in place; *h_moves
 * receives the number of moves. */
int lsg_balance_step(uint32_t* h_items, uint32_t* h_node_off, uint32_t N, uint64_t* h_moves, void* stream);
/* ---- Buffer (buffer.hpp:21-79): one node's buffer as a device-resident
 *      slot array; make_buffer == lsg_buffer_create. Accesses are applied in
 *      order by one CTA (silent != 0: insert_silent). Host arrays. */
typedef struct lsg_buffer lsg_buffer;
int lsg_buffer_create(int32_t policy, uint64_t capacity, lsg_buffer** out);
void lsg_buffer_destroy(lsg_buffer* b);
int lsg_buffer_access(lsg_buffer* b, const uint64_t* h_ids, const uint64_t* h_next_use, uint64_t n, int32_t silent,
                      uint8_t* h_hits, void* stream);
int lsg_buffer_clear(lsg_buffer* b);
int lsg_buffer_resident(lsg_buffer* b, uint64_t* h_ids, uint64_t cap, uint64_t* h_n);
/* simulate_sequence (buffer.cpp:116-125): misses of one access sequence
 * through one buffer, via the K7 replay (one node, one access per step). */
int lsg_simulate_sequence(const uint32_t* h_seq, uint64_t len, uint64_t capacity, int32_t policy,
                          uint64_t* h_misses, void* stream);
/* optimal_miss_oracle (buffer.cpp:132-182): exhaustive optimum, length <= 16,
 * capacity in [1, 4]; a backward DP over (position, resident mask). */
int lsg_optimal_miss_oracle(const uint64_t* h_seq, uint64_t len, uint64_t capacity, uint64_t* h_misses,
                            void* stream);
/* plan_chunks (chunking.cpp:9-33) of one host fetch list: reads into h_start /
 * h_end (capacity n; start == end: Single), h_meta = {reads, needed, redundant}. */
int lsg_plan_chunks(const uint32_t* h_ids, uint64_t n, uint64_t threshold, uint32_t* h_start, uint32_t* h_end,
                    uint64_t* h_meta, void* stream);

/* ---- Text artifacts (trace.cpp:72-162, reuse_graph.cpp:103-140,
 *      plan.cpp:44-214). Writers format on the GPU into h_out when
 *      cap >= *nbytes (call with h_out = NULL for the size); the bytes are
 *      identical to the reference's ostream output. Readers accept exactly
 *      what the reference accepts, with its error classes and messages. */
int lsg_format_trace(const uint32_t* d_trace, uint64_t dataset_size, uint32_t num_epochs, uint32_t num_nodes,
                     uint64_t local_batch, uint64_t seed, int32_t drop_last, uint64_t keep, char* h_out,
                     uint64_t cap, uint64_t* nbytes, void* stream);
/* Plan rows: N balance rows, the assign rows and the read rows of every
 * step (T = E * S steps, execution order); reads as lsg_plan_out (NULL:
 * no read rows); a read with start == end is written as "single". */
int lsg_format_plan(const uint32_t* d_items, const uint32_t* d_node_off, const uint32_t* d_fetch_before,
                    const uint32_t* d_fetch_after, const uint32_t* d_read_start, const uint32_t* d_read_end,
                    const uint32_t* d_read_count, const uint32_t* d_order, uint64_t cost, uint32_t E, uint64_t T,
                    uint32_t N, uint64_t S, uint64_t dataset_size, uint64_t local_batch, uint64_t chunk_threshold,
                    char* h_out, uint64_t cap, uint64_t* nbytes, void* stream);
int lsg_format_graph(const uint64_t* d_w, uint32_t E, char* h_out, uint64_t cap, uint64_t* nbytes, void* stream);

typedef struct lsg_trace_text {
    uint64_t dataset_size;
    uint32_t num_epochs, num_nodes;
    uint64_t local_batch, seed;
    int32_t drop_last;
    uint64_t keep; /* ids per epoch */
} lsg_trace_text;
/* read_trace (trace.cpp:103-147): header into *hdr; ids ([E][keep]) into
 * h_ids when cap >= E * keep. */
int lsg_parse_trace(const char* text, uint64_t len, lsg_trace_text* hdr, uint32_t* h_ids, uint64_t cap);
/* read_graph (reuse_graph.cpp:114-128): *E, weights into h_w when cap >= E*E. */
int lsg_parse_graph(const char* text, uint64_t len, uint32_t* E, uint64_t* h_w, uint64_t cap);

/* read_plan (plan.cpp:85-214) in the flat layout: steps in the file's epoch
 * order (epoch_steps[i] steps for its i-th epoch), node lists in file order,
 * reads as CSR per (step, node). Arrays are owned by the handle. */
typedef struct lsg_parsed_plan lsg_parsed_plan;
typedef struct lsg_plan_view {
    uint64_t dataset_size, local_batch, chunk_threshold, cost;
    uint32_t num_nodes, num_epochs;
    uint64_t num_steps, num_items, num_reads;
    const uint32_t* order;        /* [num_epochs] (the order line) */
    const uint32_t* epoch_ids;    /* [num_epochs] */
    const uint64_t* epoch_steps;  /* [num_epochs] */
    const uint32_t* items;        /* [num_items] id | LSG_HIT_BIT */
    const uint32_t* node_off;     /* [num_steps][N+1] */
    const uint64_t* fetch_before; /* [num_steps][N] */
    const uint64_t* fetch_after;  /* [num_steps][N] */
    const uint64_t* read_off;     /* [num_steps*N+1] */
    const uint64_t* read_start;   /* [num_reads] */
    const uint64_t* read_end;     /* [num_reads] */
    const uint8_t* read_chunk;    /* [num_reads] 1 = chunk, 0 = single */
    const uint64_t* needed;       /* [num_steps][N] ChunkPlan.needed */
    const uint64_t* redundant;    /* [num_steps][N] ChunkPlan.redundant */
} lsg_plan_view;
int lsg_parse_plan(const char* text, uint64_t len, lsg_parsed_plan** out, lsg_plan_view* view);
void lsg_free_plan(lsg_parsed_plan* p);

/* Number of kernel launches issued by this library since load (for the
 * bench's gpu_launches claim). */
uint64_t lsg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif

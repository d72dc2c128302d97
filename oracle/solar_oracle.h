/* oracle/solar_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement ("port") of the reference SOLAR loading-planner path
 * (/root/reference/proj, namespace loadsched). Used by tests/ as the parity
 * checker, by __graft_entry__.smoke() and by bench.py's cpu_baseline leg.
 * The product (paper_2211_00224_b200) never links or calls this.
 *
 * Every function cites the reference file:line it restates. Return values are
 * the reference ErrorClass codes (errors.hpp:11-18): 0 ok, 2 Config,
 * 3 Validation, 4 Capability, 7 Internal.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * reference's golden vectors (tests/test_prng.cpp, test_trace.cpp,
 * test_reuse_graph.cpp, test_balance.cpp, test_locality.cpp, README demo)
 * and, when oracle/_ref/ref_dump is built, against the compiled reference
 * on seeded configs (bit-exact on every output array).
 */
#ifndef SOLAR_ORACLE_H
#define SOLAR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_NEVER UINT64_C(0xFFFFFFFFFFFFFFFF)
#define OR_HIT_BIT 0x80000000u

/* Same field meaning as the reference PipelineConfig (config.hpp:17-36). */
typedef struct {
    uint64_t dataset_size;   /* D */
    uint32_t num_epochs;     /* E */
    uint32_t num_nodes;      /* N */
    uint64_t local_batch;    /* b */
    uint64_t seed;
    int32_t drop_last;
    int32_t policy;          /* 0 clairvoyant, 1 lru */
    uint64_t buffer_capacity;/* C, per node */
    int32_t graph_mode;      /* 0 global, 1 pernode */
    int32_t insert_redundant;
    uint64_t chunk_threshold;
    int32_t optim_order, optim_remap, optim_balance, optim_chunk;
    uint32_t pso_swarm, pso_iters, pso_stagnation, pso_restart;
    double pso_p_personal, pso_p_global, pso_inertia, pso_kick;
} or_config;

uint64_t or_splitmix_next(uint64_t* state);
uint64_t or_steps_per_epoch(uint64_t D, uint32_t N, uint64_t b, int drop_last);

/* trace.cpp:26-43 */
int or_generate_trace(uint64_t D, uint32_t E, uint32_t N, uint64_t b, uint64_t seed,
                      int drop_last, uint32_t* out /* E*keep */);

/* reuse_graph.cpp:77-101 over a general (possibly repeating) trace. */
int or_build_reuse_graph(const uint32_t* ids, uint32_t E, uint64_t len, uint64_t D, uint32_t N,
                         uint64_t b, int drop_last, uint64_t buffer_size, int mode,
                         uint64_t* w /* E*E */);

/* epoch_order.cpp:121-221 */
int or_pso_order(const uint64_t* w, uint32_t E, uint32_t swarm, uint32_t iters, double p_personal,
                 double p_global, double inertia, double kick, uint32_t stagnation,
                 uint32_t restart, uint64_t seed, uint32_t* order, uint64_t* cost,
                 uint64_t* hist /* iters */, uint32_t* n_iters);

/* epoch_order.cpp:32-52 */
int or_brute_force_order(const uint64_t* w, uint32_t E, uint32_t* order, uint64_t* cost);

/* locality.cpp:7-42 / :57-73 on holder masks (bit k = resident on node k,
 * N <= 64): out_ids/out_tags in node order, node_off[N+1]. */
int or_remap_step(const uint64_t* holders, const uint32_t* batch, uint64_t len, uint32_t N,
                  uint64_t b, int slice, uint32_t* out_items, uint32_t* node_off);

/* balance.cpp:10-39 on a CSR step (items carry OR_HIT_BIT for hits). */
int or_balance_step(uint32_t* items, uint32_t* node_off, uint32_t N, uint64_t* moves);

/* pipeline.cpp:32-120. Outputs (caller-sized):
 *   trace[E*keep], graph[E*E], order[E], cost, hist[pso_iters], n_iters,
 *   items[E*keep] (id | OR_HIT_BIT when tagged hit), node_off[T*(N+1)],
 *   fb[T*N], fa[T*N]; residency[T*N*3] (count,sum,xor digest) may be NULL. */
int or_plan(const or_config* cfg, uint32_t* trace, uint64_t* graph, uint32_t* order,
            uint64_t* cost, uint64_t* hist, uint32_t* n_iters, uint32_t* items,
            uint32_t* node_off, uint32_t* fb, uint32_t* fa, uint64_t* residency);

/* buffer.cpp:183-247 (insert_redundant = false). Steps in execution order;
 * hits/misses[T*N]. */
int or_simulate_ex(const uint32_t* items, const uint32_t* node_off, uint64_t T, uint32_t N,
                   uint64_t D, uint64_t C, int policy, const uint32_t* rstart, const uint32_t* rend,
                   const uint32_t* rcount, uint32_t* hits, uint32_t* misses);
int or_simulate(const uint32_t* items, const uint32_t* node_off, uint64_t T, uint32_t N,
                uint64_t D, uint64_t C, int policy, uint32_t* hits, uint32_t* misses);

/* buffer.cpp:114-123: misses of one sequence through one buffer. */
int or_simulate_sequence(const uint32_t* seq, uint64_t n, uint64_t D, uint64_t C, int policy,
                         uint64_t* misses);

/* chunking.cpp:9-33 / pipeline.cpp:21-28 on a finished plan: reads of list
 * (g, k) at its item offsets (start == end: Single), per-list counts. */
int or_plan_reads(const uint32_t* items, const uint32_t* node_off, uint64_t T, uint32_t N,
                  int chunked, uint64_t thr, uint32_t* rstart, uint32_t* rend, uint32_t* rcount,
                  uint32_t* needed, uint32_t* redundant);

/* store.cpp:70-80: payload bytes [offset, offset+n) of a store with fill_seed. */
void or_store_payload(uint64_t fill_seed, uint64_t offset, uint64_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif

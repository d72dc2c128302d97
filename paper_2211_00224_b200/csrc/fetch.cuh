// fetch.cuh — the step fetch's launch descriptor, shared by the single-step
// path (gather.cu) and the whole-job path with a real miss source
// (fetch_job.cu).
#pragma once
#include "common.cuh"

namespace lsg {

// One step of the loading phase for the contiguous node range [k0, k1): their
// lists are contiguous in the step's item array (rows node_off[k0] ..
// node_off[k1]), so one launch covers every local rank of the step. Row r of
// node k goes to outs[k - k0] row r - node_off[k] and, for hits, comes from
// bufs[k - k0].
struct StepFetch {
    const uint32_t* items;     // step's items (ids | hit tag)
    const uint32_t* slots;     // step's replay slots (bit 31 = resident at step start)
    const uint32_t* node_off;  // [N+1] of the step
    uint4* const* bufs;        // [k1-k0] HBM sample buffers
    uint4* const* outs;        // [k1-k0] batch tensors
    uint32_t k0, k1;
    uint64_t vec_per_row, tiles_per_row, seed;
    uint32_t* claim;           // the TMA kernel's tile-chunk counter for this step (zeroed) or null
    uint32_t* mlist;           // miss rows of the step (listed by the TMA hit kernel) or null
    uint32_t* mctl;            // [1] listed miss count (may exceed mcap: then scan every row)
    uint32_t mcap;             // capacity of mlist
    int l2hint;                // TMA copies tagged L2::evict_first (streaming)
};

__device__ __forceinline__ uint32_t node_of_row(const StepFetch& f, uint32_t r) {
    uint32_t k = f.k0;
    while (k + 1 < f.k1 && __ldg(&f.node_off[k + 1]) <= r) ++k;
    return k;
}

// Hit rows of one step (TMA bulk copies when rows are whole 8 KiB tiles,
// else 128-bit loads/stores). *tma reports which kernel ran.
int launch_fetch_hits(StepFetch f, uint64_t rows, uint64_t sample_bytes, cudaStream_t st, bool* tma);

// launch with programmatic stream serialization (PDL); which: 0 = hit
// kernels, 1 = miss kernels (LSG_PDL bit mask, default 1)
bool pdl_on(int which);

}  // namespace lsg

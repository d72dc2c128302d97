// report.cu — the run report's totals over a flat device plan:
// total_barrier_cost and total_io_cost (pipeline.cpp:133-151), with the
// per-step barrier (balance.cpp:41-47: the slowest node's fetch count x
// (seek + stream)) and read-plan cost (cost_model.cpp:9-18: per read, seek +
// span x stream, summed in read order; the step costs its slowest node).
//
// Doubles are summed in the reference's order, so the totals are
// bit-identical: one thread per (step, node) list sums its reads in order;
// per-step maxima are order-free; the T step values are then added in step
// order by one thread (T <= ~1e5, far below the planner's cost).
#include "common.cuh"

namespace lsg {

namespace {

struct CostArgs {
    const uint32_t* items;        // ids | hit tag (lsg_plan_out layout), or null
    const uint32_t* fetches;      // [T][N] fetch counts, or null: counted from items' tags
    const uint32_t* node_off;     // [T][N+1]
    const uint64_t* base;         // [T] item offset of each step
    const uint32_t* rstart;       // reads at their list's item offsets (may be null)
    const uint32_t* rend;
    const uint32_t* rcount;       // [T][N]
    uint32_t T, N;
    double seek, stream;
    double* step_barrier;         // [T]
    double* step_io;              // [T]
    double* totals;               // [2]
};

__global__ void __launch_bounds__(256) k_step_costs(CostArgs a) {
    const uint32_t g = blockIdx.x;
    const double per_fetch = __dadd_rn(a.seek, a.stream);
    double bar = 0.0, io = 0.0;
    for (uint32_t k = threadIdx.x; k < a.N; k += blockDim.x) {
        uint32_t nf;
        if (a.fetches) {
            nf = a.fetches[size_t(g) * a.N + k];
        } else {  // StepAssignment::fetch_counts (plan.cpp:11-16): untagged items
            const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
            nf = 0;
            for (uint32_t i = off[k]; i < off[k + 1]; ++i) nf += !(a.items[a.base[g] + i] & kHit);
        }
        bar = fmax(bar, __dmul_rn(double(nf), per_fetch));
        if (a.rcount) {
            const uint64_t lo = a.base[g] + a.node_off[size_t(g) * (a.N + 1) + k];
            const uint32_t n = a.rcount[size_t(g) * a.N + k];
            double c = 0.0;
            // no FMA contraction: the reference's g++ -std=c++20 build rounds the
            // product and the two sums separately
            for (uint32_t r = 0; r < n; ++r)
                c = __dadd_rn(c, __dadd_rn(a.seek, __dmul_rn(double(a.rend[lo + r] - a.rstart[lo + r] + 1), a.stream)));
            io = fmax(io, c);
        }
    }
    __shared__ double sb[256], si[256];
    sb[threadIdx.x] = bar;
    si[threadIdx.x] = io;
    __syncthreads();
    for (uint32_t s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) {
            sb[threadIdx.x] = fmax(sb[threadIdx.x], sb[threadIdx.x + s]);
            si[threadIdx.x] = fmax(si[threadIdx.x], si[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.step_barrier[g] = sb[0];
        a.step_io[g] = si[0];
    }
}

__global__ void k_sum_in_order(CostArgs a) {
    double b = 0.0, io = 0.0;
    for (uint32_t g = 0; g < a.T; ++g) {
        b = __dadd_rn(b, a.step_barrier[g]);
        io = __dadd_rn(io, a.step_io[g]);
    }
    a.totals[0] = b;
    a.totals[1] = io;
}

__global__ void k_bases(const uint32_t* __restrict__ node_off, uint32_t T, uint32_t N, uint64_t* __restrict__ base) {
    uint64_t s = 0;
    for (uint32_t g = 0; g < T; ++g) {
        base[g] = s;
        s += node_off[size_t(g) * (N + 1) + N];
    }
}

}  // namespace

}  // namespace lsg

using namespace lsg;

extern "C" int lsg_plan_costs(const uint32_t* d_items, const uint32_t* d_fetches, const uint32_t* d_node_off,
                              const uint32_t* d_read_start,
                              const uint32_t* d_read_end, const uint32_t* d_read_count, uint64_t T, uint32_t N,
                              double seek_cost, double stream_cost, double* h_barrier_total, double* h_io_total,
                              void* stream) {
    if (T && (!d_node_off || (!d_items && !d_fetches)))
        return set_error(kValidation, "plan_costs: offsets and items or fetch counts required");
    if (d_read_count && (!d_read_start || !d_read_end)) return set_error(kValidation, "plan_costs: incomplete reads");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (T == 0) {
        if (h_barrier_total) *h_barrier_total = 0.0;
        if (h_io_total) *h_io_total = 0.0;
        return kOk;
    }
    Scratch sc(st);
    CostArgs a{d_items, d_fetches, d_node_off, sc.get<uint64_t>(T), d_read_start, d_read_end, d_read_count,
               uint32_t(T), N, seek_cost, stream_cost, sc.get<double>(T), sc.get<double>(T), sc.get<double>(2)};
    if (!a.base || !a.step_barrier || !a.step_io || !a.totals)
        return set_error(kInternal, "plan_costs: scratch allocation failed");
    k_bases<<<1, 1, 0, st>>>(d_node_off, uint32_t(T), N, const_cast<uint64_t*>(a.base));
    LSG_LAUNCH_CHECK("k_bases");
    k_step_costs<<<unsigned(T), 256, 0, st>>>(a);
    LSG_LAUNCH_CHECK("k_step_costs");
    k_sum_in_order<<<1, 1, 0, st>>>(a);
    LSG_LAUNCH_CHECK("k_sum_in_order");
    double h[2] = {0, 0};
    if (int rc = d2h_small(h, a.totals, sizeof h, st)) return rc;
    if (h_barrier_total) *h_barrier_total = h[0];
    if (h_io_total) *h_io_total = h[1];
    return kOk;
}

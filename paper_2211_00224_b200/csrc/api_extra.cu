// api_extra.cu — the per-call pieces of the reference API around the hot
// path, on the device:
//  * first_buffer_window / last_buffer_window (reuse_graph.cpp:43-75): the K2
//    window bitsets of one epoch;
//  * brute_force_order (epoch_order.cpp:32-52): all E! open paths for E <= 10,
//    one CTA enumerating them in lexicographic chunks (Lehmer-coded starts,
//    next_permutation inside a chunk), min (cost, index) so ties keep the
//    lexicographically smallest order like the reference's strict-improvement
//    scan;
//  * plan_chunks (chunking.cpp:9-33) of one fetch list through the K-reads
//    kernel of the plan path.
#include <vector>

#include "common.cuh"

namespace lsg {

int window_bits_device(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D, uint32_t N, uint64_t b,
                       bool drop_last, uint64_t buffer_size, int mode, bool rows_distinct_known, uint32_t* Fb,
                       uint32_t* Lb, cudaStream_t st);
int plan_reads_device(const uint32_t* d_items, const uint32_t* d_node_off, uint32_t T, uint32_t N, uint32_t S,
                      uint32_t B, uint32_t keep, int chunked, uint64_t thr, uint32_t* rstart, uint32_t* rend,
                      uint32_t* rcount, uint32_t* needed, uint32_t* redundant, cudaStream_t st);

namespace {

constexpr int kBfT = 1024;

__device__ __forceinline__ void decode_perm(uint64_t idx, uint32_t E, uint32_t* p) {
    // factorial number system, lexicographic rank idx -> permutation
    uint32_t avail = (1u << E) - 1u;
    uint64_t f = 1;
    for (uint32_t i = 2; i < E; ++i) f *= i;  // (E-1)!
    for (uint32_t i = 0; i < E; ++i) {
        const uint64_t d = E - 1 - i > 0 ? idx / f : 0;
        if (E - 1 - i > 0) idx -= d * f;
        // d-th remaining element
        uint32_t m = avail;
        for (uint64_t q = 0; q < d; ++q) m &= m - 1;
        const uint32_t x = __ffs(m) - 1;
        p[i] = x;
        avail &= ~(1u << x);
        if (E - 1 - i > 1) f /= (E - 1 - i);
    }
}

__device__ __forceinline__ bool next_perm(uint32_t* a, uint32_t n) {
    if (n < 2) return false;
    int i = int(n) - 2;
    while (i >= 0 && a[i] >= a[i + 1]) --i;
    if (i < 0) return false;
    int j = int(n) - 1;
    while (a[j] <= a[i]) --j;
    uint32_t t = a[i];
    a[i] = a[j];
    a[j] = t;
    for (int l = i + 1, r = int(n) - 1; l < r; ++l, --r) {
        t = a[l];
        a[l] = a[r];
        a[r] = t;
    }
    return true;
}

__global__ void __launch_bounds__(kBfT) k_brute_force(const uint64_t* __restrict__ w, uint32_t E, uint64_t total,
                                                      uint32_t* order, uint64_t* cost) {
    __shared__ uint64_t sw[100];
    __shared__ unsigned long long bc[kBfT];
    __shared__ unsigned long long bi[kBfT];
    for (uint32_t i = threadIdx.x; i < E * E; i += kBfT) sw[i] = w[i];
    __syncthreads();
    const uint64_t per = (total + kBfT - 1) / kBfT;
    const uint64_t i0 = uint64_t(threadIdx.x) * per, i1 = min(total, i0 + per);
    unsigned long long best = ~0ull, bidx = ~0ull;
    if (i0 < i1) {
        uint32_t p[10];
        decode_perm(i0, E, p);
        for (uint64_t idx = i0; idx < i1; ++idx) {
            unsigned long long c = 0;
            for (uint32_t i = 0; i + 1 < E; ++i) c += sw[p[i] * E + p[i + 1]];
            if (c < best) {
                best = c;
                bidx = idx;
            }
            next_perm(p, E);
        }
    }
    bc[threadIdx.x] = best;
    bi[threadIdx.x] = bidx;
    __syncthreads();
    for (int s = kBfT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < uint32_t(s)) {
            const unsigned long long c2 = bc[threadIdx.x + s], i2 = bi[threadIdx.x + s];
            if (c2 < bc[threadIdx.x] || (c2 == bc[threadIdx.x] && i2 < bi[threadIdx.x])) {
                bc[threadIdx.x] = c2;
                bi[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        uint32_t p[10];
        decode_perm(bi[0], E, p);
        for (uint32_t i = 0; i < E; ++i) order[i] = p[i];
        *cost = bc[0];
    }
}

}  // namespace
}  // namespace lsg

using namespace lsg;

extern "C" {

int lsg_buffer_windows(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D, uint32_t N, uint64_t b,
                       int32_t drop_last, uint64_t buffer_size, int32_t mode, uint32_t* d_first, uint32_t* d_last,
                       void* stream) {
    if (buffer_size == 0) return set_error(kValidation, "buffer window: buffer_size must be >= 1");
    if (E == 0) return kOk;
    return window_bits_device(d_trace, E, len, D, N, b, drop_last != 0, buffer_size, mode, false, d_first, d_last,
                              static_cast<cudaStream_t>(stream));
}

int lsg_brute_force_order(const uint64_t* d_w, uint32_t E, uint32_t* d_order, uint64_t* d_cost, void* stream) {
    if (E == 0) return set_error(kValidation, "brute_force_order: empty graph");
    if (E > 10) return set_error(kCapability, "brute_force_order: guarded to num_epochs <= 10");
    uint64_t total = 1;
    for (uint32_t i = 2; i <= E; ++i) total *= i;
    k_brute_force<<<1, kBfT, 0, static_cast<cudaStream_t>(stream)>>>(d_w, E, total, d_order, d_cost);
    LSG_LAUNCH_CHECK("k_brute_force");
    return kOk;
}

// plan_chunks(fetch_ids, threshold) for one list (host ids, any order,
// repeats allowed): reads into h_start/h_end (capacity n), count / needed /
// redundant into *h_meta[3].
int lsg_plan_chunks(const uint32_t* h_ids, uint64_t n, uint64_t threshold, uint32_t* h_start, uint32_t* h_end,
                    uint64_t* h_meta, void* stream) {
    if (threshold == 0) return set_error(kValidation, "plan_chunks: threshold must be >= 1");
    if (n >= (1ull << 31)) return set_error(kCapability, "plan_chunks: list too long for the device");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    h_meta[0] = h_meta[1] = h_meta[2] = 0;
    if (n == 0) return kOk;
    Scratch sc(st);
    uint32_t* d = sc.get<uint32_t>(3 * n + 8);
    if (!d) return set_error(kInternal, "plan_chunks: scratch allocation failed");
    uint32_t *items = d, *rs = d + n, *re = d + 2 * n, *off = d + 3 * n, *meta = d + 3 * n + 2;
    for (uint64_t i = 0; i < n; ++i)
        if (h_ids[i] & kHit) return set_error(kCapability, "plan_chunks: sample ids must be < 2^31 on the device");
    const uint32_t hoff[2] = {0, uint32_t(n)};
    LSG_CUDA(cudaMemcpyAsync(items, h_ids, n * 4, cudaMemcpyHostToDevice, st));
    LSG_CUDA(cudaMemcpyAsync(off, hoff, 8, cudaMemcpyHostToDevice, st));
    if (int rc = plan_reads_device(items, off, 1, 1, 1, uint32_t(n), uint32_t(n), 1, threshold, rs, re, meta,
                                   meta + 1, meta + 2, st))
        return rc;
    uint32_t m[3];
    LSG_CUDA(cudaMemcpyAsync(m, meta, 12, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    LSG_CUDA(cudaMemcpyAsync(h_start, rs, size_t(m[0]) * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaMemcpyAsync(h_end, re, size_t(m[0]) * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    h_meta[0] = m[0];
    h_meta[1] = m[1];
    h_meta[2] = m[2];
    return kOk;
}

}  // extern "C"

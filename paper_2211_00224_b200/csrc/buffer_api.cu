// buffer_api.cu — the reference's per-node Buffer object (buffer.hpp:21-79)
// as a device-resident state, plus the two single-sequence entry points.
//
//  * lsg_buffer_*: make_buffer / Buffer::access / insert_silent / clear /
//    resident. The state lives in HBM as a slot array {id, key} of capacity
//    C+1 (the +1 holds the incoming sample, which may itself be the victim:
//    buffer.cpp:36-44). One CTA applies a batch of accesses in order; every
//    access is a block-wide membership scan plus, on overflow, a block-wide
//    argmax: the max (next_use, id) for the clairvoyant policy (the lazy
//    heap's valid top, buffer.cpp:19-35) or the oldest touch for LRU (the
//    recency list's tail, buffer.cpp:61-77). The planner's step loop and the
//    replay keep their own structures; this object serves per-call users.
//  * lsg_simulate_sequence (buffer.cpp:116-125): one node's replay through
//    the K7 kernels, one access per step.
//  * lsg_optimal_miss_oracle (buffer.cpp:132-182): the exhaustive optimum as a
//    backward dynamic programme over (position, resident mask), one CTA, two
//    mask rows in shared memory.
#include <vector>

#include "common.cuh"

namespace lsg {

int simulate_device(const uint32_t* d_items, const uint32_t* d_node_off, uint64_t T, uint32_t N, uint64_t D,
                    uint64_t C, int policy, uint32_t k0, uint32_t k1, uint32_t* d_hits, uint32_t* d_misses,
                    uint32_t* d_slot, const uint32_t* rstart, const uint32_t* rend, const uint32_t* rcount,
                    int insred, uint32_t* status, cudaStream_t st);

namespace {

constexpr int kBT = 512;

struct BufState {
    unsigned long long* id;   // [C+1]
    unsigned long long* key;  // [C+1] clairvoyant: next_use; LRU: touch time
    unsigned long long* ctl;  // [0] size, [1] clock
};

// (a_hi, a_lo) > (b_hi, b_lo)
__device__ __forceinline__ bool gt2(unsigned long long ah, unsigned long long al, unsigned long long bh,
                                    unsigned long long bl) {
    return ah > bh || (ah == bh && al > bl);
}

__global__ void __launch_bounds__(kBT) k_buffer_ops(BufState s, uint64_t C, int lru, int silent,
                                                    const unsigned long long* __restrict__ ids,
                                                    const unsigned long long* __restrict__ nus, uint64_t n,
                                                    uint8_t* __restrict__ hit) {
    __shared__ unsigned long long w_hi[kBT / 32], w_lo[kBT / 32], w_slot[kBT / 32];
    __shared__ unsigned long long found;
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint64_t size = s.ctl[0];
    unsigned long long clock = s.ctl[1];
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned long long x = ids[i];
        const unsigned long long key = lru ? clock++ : nus[i];
        if (tid == 0) found = ~0ull;
        __syncthreads();
        for (uint64_t j = tid; j < size; j += kBT)
            if (s.id[j] == x) found = j;  // ids are unique among residents
        __syncthreads();
        const unsigned long long f = found;
        if (f != ~0ull) {
            // hit: re-key (clairvoyant access, any LRU touch); a silent
            // clairvoyant insert of a resident id changes nothing
            if (tid == 0) {
                if (lru || !silent) s.key[f] = key;
                if (!silent) hit[i] = 1;
            }
            __syncthreads();
            continue;
        }
        if (tid == 0) {
            s.id[size] = x;
            s.key[size] = key;
            if (!silent) hit[i] = 0;
        }
        ++size;
        __syncthreads();
        if (size <= C) continue;
        // overflow: victim over all size = C+1 slots (the incoming included).
        // Clairvoyant: max (next_use, id). LRU: min touch time = max of ~time.
        unsigned long long bh = 0, bl = 0, bs = ~0ull;
        for (uint64_t j = tid; j < size; j += kBT) {
            const unsigned long long hi = lru ? ~s.key[j] : s.key[j], lo = lru ? 0ull : s.id[j];
            if (bs == ~0ull || gt2(hi, lo, bh, bl)) {
                bh = hi;
                bl = lo;
                bs = j;
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const unsigned long long oh = __shfl_xor_sync(0xFFFFFFFFu, bh, d);
            const unsigned long long ol = __shfl_xor_sync(0xFFFFFFFFu, bl, d);
            const unsigned long long os = __shfl_xor_sync(0xFFFFFFFFu, bs, d);
            if (os != ~0ull && (bs == ~0ull || gt2(oh, ol, bh, bl))) {
                bh = oh;
                bl = ol;
                bs = os;
            }
        }
        if (lane == 0) {
            w_hi[w] = bh;
            w_lo[w] = bl;
            w_slot[w] = bs;
        }
        __syncthreads();
        if (tid == 0) {
            for (int q = 1; q < kBT / 32; ++q)
                if (w_slot[q] != ~0ull && (bs == ~0ull || gt2(w_hi[q], w_lo[q], bh, bl))) {
                    bh = w_hi[q];
                    bl = w_lo[q];
                    bs = w_slot[q];
                }
            // drop slot bs: the last slot moves into it
            s.id[bs] = s.id[size - 1];
            s.key[bs] = s.key[size - 1];
        }
        --size;
        __syncthreads();
    }
    if (tid == 0) {
        s.ctl[0] = size;
        s.ctl[1] = clock;
    }
}

// f[pos][mask] backwards; cur/nxt rows of 2^k int8 in shared memory
__global__ void __launch_bounds__(1024) k_opt_oracle(const unsigned long long* __restrict__ seq, uint32_t n,
                                                     uint32_t C, uint32_t* out) {
    extern __shared__ int8_t rows[];
    __shared__ uint8_t lab[16];
    __shared__ uint32_t nk;
    if (threadIdx.x == 0) {
        uint32_t k = 0;
        for (uint32_t i = 0; i < n; ++i) {
            uint32_t l = k;
            for (uint32_t q = 0; q < i; ++q)
                if (seq[q] == seq[i]) {
                    l = lab[q];
                    break;
                }
            lab[i] = uint8_t(l);
            if (l == k) ++k;
        }
        nk = k;
    }
    __syncthreads();
    const uint32_t masks = 1u << nk;
    int8_t* nxt = rows;
    int8_t* cur = rows + masks;
    for (uint32_t m = threadIdx.x; m < masks; m += blockDim.x) nxt[m] = 0;
    __syncthreads();
    for (int pos = int(n) - 1; pos >= 0; --pos) {
        const uint32_t bit = 1u << lab[pos];
        for (uint32_t m = threadIdx.x; m < masks; m += blockDim.x) {
            if (uint32_t(__popc(m)) > C) continue;
            int8_t best;
            if (m & bit) {
                best = nxt[m];
            } else {
                const uint32_t g = m | bit;
                if (uint32_t(__popc(g)) <= C) {
                    best = int8_t(1 + nxt[g]);
                } else {
                    best = int8_t(n + 1);
                    for (uint32_t v = g; v; v &= v - 1) {
                        const uint32_t low = v & (~v + 1);
                        best = min(best, int8_t(1 + nxt[g & ~low]));
                    }
                }
            }
            cur[m] = best;
        }
        __syncthreads();
        int8_t* t = nxt;
        nxt = cur;
        cur = t;
    }
    if (threadIdx.x == 0) *out = uint32_t(nxt[0]);
}

__global__ void k_seq_offsets(uint32_t* off, uint64_t len) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < len; g += uint64_t(gridDim.x) * blockDim.x) {
        off[2 * g] = 0;
        off[2 * g + 1] = 1;
    }
}

__global__ void k_sum_u32(const uint32_t* __restrict__ v, uint64_t n, unsigned long long* out) {
    unsigned long long s = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        s += v[i];
    const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, uint32_t(s));
    if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(ws));
}

}  // namespace
}  // namespace lsg

using namespace lsg;

struct lsg_buffer {
    int policy;
    uint64_t capacity;
    BufState s;
    void* mem;
};

extern "C" {

int lsg_buffer_create(int32_t policy, uint64_t capacity, lsg_buffer** out) {
    *out = nullptr;
    if (capacity == 0) return set_error(kValidation, "buffer capacity must be >= 1");
    if (policy != 0 && policy != 1) return set_error(kConfig, "buffer: policy must be clairvoyant (0) or lru (1)");
    if (capacity > (1ull << 32)) return set_error(kCapability, "buffer: capacity <= 2^32 on the device");
    auto* b = new lsg_buffer{policy, capacity, {}, nullptr};
    const size_t slots = capacity + 1;
    if (cudaMalloc(&b->mem, (2 * slots + 2) * sizeof(unsigned long long)) != cudaSuccess) {
        delete b;
        cudaGetLastError();
        return set_error(kInternal, "buffer: device allocation failed");
    }
    auto* p = static_cast<unsigned long long*>(b->mem);
    b->s = BufState{p, p + slots, p + 2 * slots};
    LSG_CUDA(cudaMemset(b->s.ctl, 0, 2 * sizeof(unsigned long long)));
    *out = b;
    return kOk;
}

void lsg_buffer_destroy(lsg_buffer* b) {
    if (!b) return;
    cudaFree(b->mem);
    delete b;
}

// n accesses (silent = 0: Buffer::access, hits[i] = 1 on a hit) or silent
// inserts (Buffer::insert_silent, hits unused), applied in order. Host arrays.
int lsg_buffer_access(lsg_buffer* b, const uint64_t* h_ids, const uint64_t* h_next_use, uint64_t n, int32_t silent,
                      uint8_t* h_hits, void* stream) {
    if (!b) return set_error(kValidation, "buffer: null handle");
    if (n == 0) return kOk;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    auto* d = sc.get<unsigned long long>(2 * n);
    auto* hit = sc.get<uint8_t>(n);
    if (!d || !hit) return set_error(kInternal, "buffer: scratch allocation failed");
    LSG_CUDA(cudaMemcpyAsync(d, h_ids, n * 8, cudaMemcpyHostToDevice, st));
    if (h_next_use) LSG_CUDA(cudaMemcpyAsync(d + n, h_next_use, n * 8, cudaMemcpyHostToDevice, st));
    else LSG_CUDA(cudaMemsetAsync(d + n, 0, n * 8, st));
    k_buffer_ops<<<1, kBT, 0, st>>>(b->s, b->capacity, b->policy, silent != 0, d, d + n, n, hit);
    LSG_LAUNCH_CHECK("k_buffer_ops");
    if (!silent && h_hits) LSG_CUDA(cudaMemcpyAsync(h_hits, hit, n, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    return kOk;
}

int lsg_buffer_clear(lsg_buffer* b) {
    if (!b) return set_error(kValidation, "buffer: null handle");
    LSG_CUDA(cudaMemset(b->s.ctl, 0, 2 * sizeof(unsigned long long)));
    return kOk;
}

// resident ids (any order) into h_ids (capacity cap); *h_n = count
int lsg_buffer_resident(lsg_buffer* b, uint64_t* h_ids, uint64_t cap, uint64_t* h_n) {
    if (!b) return set_error(kValidation, "buffer: null handle");
    unsigned long long size = 0;
    LSG_CUDA(cudaMemcpy(&size, b->s.ctl, 8, cudaMemcpyDeviceToHost));
    *h_n = size;
    if (h_ids && size) LSG_CUDA(cudaMemcpy(h_ids, b->s.id, std::min<uint64_t>(size, cap) * 8, cudaMemcpyDeviceToHost));
    return kOk;
}

// simulate_sequence(seq, capacity, policy) -> misses (buffer.cpp:116-125):
// node 0 of a one-node plan with one access per step, through the K7 replay.
int lsg_simulate_sequence(const uint32_t* h_seq, uint64_t len, uint64_t capacity, int32_t policy,
                          uint64_t* h_misses, void* stream) {
    if (capacity == 0) return set_error(kValidation, "buffer capacity must be >= 1");
    if (policy != 0 && policy != 1) return set_error(kConfig, "simulate: policy must be clairvoyant (0) or lru (1)");
    *h_misses = 0;
    if (len == 0) return kOk;
    uint64_t D = 1;
    for (uint64_t i = 0; i < len; ++i) {
        if (h_seq[i] >= kHit) return set_error(kCapability, "simulate_sequence: sample ids must be < 2^31 on device");
        D = std::max<uint64_t>(D, uint64_t(h_seq[i]) + 1);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    uint32_t* items = sc.get<uint32_t>(len);
    uint32_t* off = sc.get<uint32_t>(2 * len);
    uint32_t* hits = sc.get<uint32_t>(len);
    uint32_t* miss = sc.get<uint32_t>(len);
    uint32_t* status = sc.get<uint32_t>(1);
    auto* tot = sc.get<unsigned long long>(1);
    if (!items || !off || !hits || !miss || !status || !tot)
        return set_error(kInternal, "simulate_sequence: scratch allocation failed");
    LSG_CUDA(cudaMemcpyAsync(items, h_seq, len * 4, cudaMemcpyHostToDevice, st));
    LSG_CUDA(cudaMemsetAsync(status, 0, 4, st));
    LSG_CUDA(cudaMemsetAsync(tot, 0, 8, st));
    k_seq_offsets<<<grid_for(len, 256, 1184), 256, 0, st>>>(off, len);
    LSG_LAUNCH_CHECK("k_seq_offsets");
    if (int rc = simulate_device(items, off, len, 1, D, capacity, policy, 0, 1, hits, miss, nullptr, nullptr,
                                 nullptr, nullptr, 0, status, st))
        return rc;
    k_sum_u32<<<grid_for(len, 256, 1184), 256, 0, st>>>(miss, len, tot);
    LSG_LAUNCH_CHECK("k_sum_u32");
    uint32_t h = 0;
    unsigned long long m = 0;
    if (int _rc = d2h_small(&h, status, 4, st)) return _rc;
    if (int _rc = d2h_small(&m, tot, 8, st)) return _rc;
    LSG_CUDA(cudaStreamSynchronize(st));
    if (h) return set_error(kInternal, "simulate_sequence: device invariant violated");
    *h_misses = m;
    return kOk;
}

// optimal_miss_oracle(seq, capacity) (buffer.cpp:132-182), same guards.
int lsg_optimal_miss_oracle(const uint64_t* h_seq, uint64_t len, uint64_t capacity, uint64_t* h_misses,
                            void* stream) {
    if (len > 16) return set_error(kCapability, "optimal_miss_oracle: guarded to length <= 16");
    if (capacity == 0 || capacity > 4)
        return set_error(kCapability, "optimal_miss_oracle: guarded to capacity in [1, 4]");
    *h_misses = 0;
    if (len == 0) return kOk;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    auto* seq = sc.get<unsigned long long>(len);
    uint32_t* out = sc.get<uint32_t>(1);
    if (!seq || !out) return set_error(kInternal, "optimal_miss_oracle: scratch allocation failed");
    LSG_CUDA(cudaMemcpyAsync(seq, h_seq, len * 8, cudaMemcpyHostToDevice, st));
    const int smem = 2 << 16;  // two rows of up to 2^16 masks
    LSG_CUDA(cudaFuncSetAttribute(k_opt_oracle, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_opt_oracle<<<1, 1024, smem, st>>>(seq, uint32_t(len), uint32_t(capacity), out);
    LSG_LAUNCH_CHECK("k_opt_oracle");
    uint32_t m = 0;
    if (int _rc = d2h_small(&m, out, 4, st)) return _rc;
    LSG_CUDA(cudaStreamSynchronize(st));
    *h_misses = m;
    return kOk;
}

}  // extern "C"

// trace.cu — K1: per-epoch shuffled index lists, bit-exact with
// generate_trace (trace.cpp:26-43) / fisher_yates_shuffle (prng.hpp:45-53).
//
// The reference runs a sequential Fisher–Yates per epoch: for t = D-1 … 1,
// swap(A[t], A[H[t]]) with H[t] = next() % (t+1). splitmix64 is
// counter-based, so H[t] = mix(s_e + (D-t)*gamma) % (t+1) for every t at
// once. The swap sequence is then resolved without any sequential loop:
//
//   position t is final after step t (later steps only touch indices < t),
//   so F[t] = value sitting at H[t] just before step t. Group the steps by
//   their target p = H[t]; inside a group, steps run in descending t. With
//     succ(t) = smallest t' > t with H[t'] = H[t]    (previous writer of H[t])
//     m(p)    = smallest t  > p with H[t]  = p        (last writer of p before step p)
//     V[p]    = value at p just before step p = V[m(p)] if m(p) exists else p
//   we get F[t] = V[succ(t)] if succ(t) exists else H[t]   (t >= 1),
//          F[0] = V[m(0)]    if m(0)    exists else 0.
//
// Groups are collected with an atomicExch linked list (no sort, no scan):
// group sizes are ~ln(D/p), so one thread per group resolves succ() in
// registers. Four passes over HBM-resident per-epoch arrays; every epoch of a
// batch runs in the same launches (blockIdx.y = epoch).
#include "common.cuh"

namespace lsg {

namespace {

constexpr int kTB = 256;

// Pass 1: draws + linked-list group insertion.
__global__ void __launch_bounds__(kTB) k_shuffle_draws(uint64_t seed, uint32_t D, uint32_t e0,
                                                       uint32_t* __restrict__ H,
                                                       uint32_t* __restrict__ nxt,
                                                       uint32_t* __restrict__ head) {
    const uint32_t eb = blockIdx.y;
    const uint64_t s = seed ^ (kGamma * (uint64_t(e0 + eb) + 1));
    const size_t base = size_t(eb) * D;
    for (uint32_t t = blockIdx.x * kTB + threadIdx.x; t < D; t += gridDim.x * kTB) {
        if (t == 0) continue;
        const uint64_t r = draw(s, uint64_t(D - t));
        const uint32_t h = uint32_t(r % (uint64_t(t) + 1));
        H[base + t] = h;
        nxt[base + t] = atomicExch(&head[base + h], t);
    }
}

// Pass 2: per target p, walk its group; succ(t) for members, m(p).
__global__ void __launch_bounds__(kTB) k_shuffle_groups(uint32_t D, const uint32_t* __restrict__ nxt,
                                                        const uint32_t* __restrict__ head,
                                                        uint32_t* __restrict__ succ,
                                                        uint32_t* __restrict__ mfirst) {
    const size_t base = size_t(blockIdx.y) * D;
    constexpr int kLocal = 24;
    for (uint32_t p = blockIdx.x * kTB + threadIdx.x; p < D; p += gridDim.x * kTB) {
        uint32_t mem[kLocal];
        int n = 0;
        uint32_t mp = kNone;
        bool spill = false;
        for (uint32_t t = head[base + p]; t != kNone; t = nxt[base + t]) {
            if (n < kLocal) mem[n] = t;
            else spill = true;
            ++n;
            if (t > p && t < mp) mp = t;
        }
        mfirst[base + p] = mp;
        if (!spill) {
            for (int a = 0; a < n; ++a) {
                uint32_t best = kNone;
                for (int c = 0; c < n; ++c)
                    if (mem[c] > mem[a] && mem[c] < best) best = mem[c];
                succ[base + mem[a]] = best;
            }
        } else {  // rare long group: quadratic walk over the list itself
            for (uint32_t a = head[base + p]; a != kNone; a = nxt[base + a]) {
                uint32_t best = kNone;
                for (uint32_t c = head[base + p]; c != kNone; c = nxt[base + c])
                    if (c > a && c < best) best = c;
                succ[base + a] = best;
            }
        }
    }
}

// Pass 3: V[p] = root of the m() chain starting at p (chains strictly rise).
__global__ void __launch_bounds__(kTB) k_shuffle_chain(uint32_t D, const uint32_t* __restrict__ mfirst,
                                                       uint32_t* __restrict__ V) {
    const size_t base = size_t(blockIdx.y) * D;
    for (uint32_t p = blockIdx.x * kTB + threadIdx.x; p < D; p += gridDim.x * kTB) {
        uint32_t q = p;
        for (uint32_t m = mfirst[base + q]; m != kNone; m = mfirst[base + q]) q = m;
        V[base + p] = q;
    }
}

// Pass 4: final value at every kept position (+ optional inverse map).
__global__ void __launch_bounds__(kTB) k_shuffle_final(uint32_t D, uint32_t keep, uint32_t e0,
                                                       const uint32_t* __restrict__ H,
                                                       const uint32_t* __restrict__ succ,
                                                       const uint32_t* __restrict__ mfirst,
                                                       const uint32_t* __restrict__ V,
                                                       uint32_t* __restrict__ out,
                                                       uint32_t* __restrict__ inv) {
    const uint32_t eb = blockIdx.y;
    const size_t base = size_t(eb) * D;
    const size_t obase = size_t(e0 + eb) * keep;
    for (uint32_t t = blockIdx.x * kTB + threadIdx.x; t < keep; t += gridDim.x * kTB) {
        uint32_t f;
        if (t == 0) {
            const uint32_t m = mfirst[base];
            f = m == kNone ? 0u : V[base + m];
        } else {
            const uint32_t s = succ[base + t];
            f = s == kNone ? H[base + t] : V[base + s];
        }
        out[obase + t] = f;
        if (inv) inv[size_t(e0 + eb) * D + f] = t;
    }
}

}  // namespace

// Generates trace[E][keep]; when d_inv != nullptr also writes inv[E][D]
// (position of id x in epoch e, kNone when dropped by drop_last).
int generate_trace_device(uint64_t D, uint32_t E, uint64_t keep, uint64_t seed, uint32_t* d_trace,
                          uint32_t* d_inv, cudaStream_t st) {
    if (D == 0 || E == 0) return kOk;
    if (d_inv) LSG_CUDA(cudaMemsetAsync(d_inv, 0xFF, size_t(E) * D * sizeof(uint32_t), st));
    // epochs per batch: keep scratch (5 arrays) around 5 x 64 MB.
    uint32_t EB = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(E, (1ull << 24) / D)));
    EB = std::min<uint32_t>(EB, 65535u);
    Scratch sc(st);
    const size_t n = size_t(EB) * D;
    uint32_t* H = sc.get<uint32_t>(n);
    uint32_t* nxt = sc.get<uint32_t>(n);
    uint32_t* head = sc.get<uint32_t>(n);
    uint32_t* succ = sc.get<uint32_t>(n);
    uint32_t* mf = sc.get<uint32_t>(n);
    if (!H || !nxt || !head || !succ || !mf) return set_error(kInternal, "trace: scratch allocation failed");
    uint32_t* V = nxt;  // nxt is dead after pass 2
    for (uint32_t e0 = 0; e0 < E; e0 += EB) {
        const uint32_t eb = std::min<uint32_t>(EB, E - e0);
        LSG_CUDA(cudaMemsetAsync(head, 0xFF, size_t(eb) * D * sizeof(uint32_t), st));
        dim3 grid(grid_for(D, kTB, 4096), eb);
        k_shuffle_draws<<<grid, kTB, 0, st>>>(seed, uint32_t(D), e0, H, nxt, head);
        LSG_LAUNCH_CHECK("k_shuffle_draws");
        k_shuffle_groups<<<grid, kTB, 0, st>>>(uint32_t(D), nxt, head, succ, mf);
        LSG_LAUNCH_CHECK("k_shuffle_groups");
        k_shuffle_chain<<<grid, kTB, 0, st>>>(uint32_t(D), mf, V);
        LSG_LAUNCH_CHECK("k_shuffle_chain");
        dim3 gridk(grid_for(keep, kTB, 4096), eb);
        k_shuffle_final<<<gridk, kTB, 0, st>>>(uint32_t(D), uint32_t(keep), e0, H, succ, mf, V,
                                               d_trace, d_inv);
        LSG_LAUNCH_CHECK("k_shuffle_final");
    }
    return kOk;
}

}  // namespace lsg

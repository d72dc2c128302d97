// ubench_gather.cu — variants of the K8 row gather (cfg2 shape: 4096 rows of
// 256 KiB from a 12.8 GiB buffer into a 1 GiB batch), CUDA-event timed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench_gather.cu -o tools/ubench_gather
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

template <int kThreads, int kUnroll>
__global__ void __launch_bounds__(kThreads) k_lsu(const uint4* __restrict__ buf, const uint32_t* __restrict__ slots,
                                                  uint64_t n, uint64_t vpr, uint4* __restrict__ out) {
    constexpr uint32_t kTile = kThreads * kUnroll;
    const uint64_t tpr = (vpr + kTile - 1) / kTile, nt = n * tpr;
    for (uint64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        const uint64_t row = t / tpr, c0 = (t - row * tpr) * kTile;
        const uint4* src = buf + uint64_t(slots[row]) * vpr;
        uint4* dst = out + row * vpr;
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kThreads + threadIdx.x;
            if (c < vpr) v[u] = __ldcs(&src[c]);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kThreads + threadIdx.x;
            if (c < vpr) __stcs(&dst[c], v[u]);
        }
    }
}

// TMA bulk copies: one elected thread per block streams tiles global -> smem
// (mbarrier complete_tx) -> global, kStages tiles in flight
template <int kTileBytes, int kStages>
__global__ void __launch_bounds__(32) k_tma(const char* __restrict__ buf, const uint32_t* __restrict__ slots,
                                            uint64_t n, uint64_t row_bytes, char* __restrict__ out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[kStages];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kStages; ++s) {
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    const uint64_t tpr = row_bytes / kTileBytes, nt = n * tpr;
    uint32_t phase[kStages];
    for (int s = 0; s < kStages; ++s) phase[s] = 0;
    uint64_t issued = 0;
    auto issue = [&](uint64_t t, int s) {
        const uint64_t row = t / tpr, c = (t - row * tpr) * kTileBytes;
        const char* src = buf + uint64_t(slots[row]) * row_bytes + c;
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sm + s * kTileBytes));
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTileBytes));
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                     "l"(src), "r"(kTileBytes), "r"(b)
                     : "memory");
    };
    uint64_t t0 = blockIdx.x;
    int s = 0;
    for (uint64_t t = t0; t < nt && issued < kStages; t += gridDim.x, ++issued) issue(t, int(issued));
    for (uint64_t t = t0, k = 0; t < nt; t += gridDim.x, ++k) {
        s = int(k % kStages);
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done)
                         : "r"(b), "r"(phase[s]));
        phase[s] ^= 1;
        const uint64_t row = t / tpr, c = (t - row * tpr) * kTileBytes;
        const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(sm + s * kTileBytes));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + row * row_bytes + c),
                     "r"(sp), "r"(kTileBytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        // the smem tile is free once its store has read it
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        const uint64_t tn = t + uint64_t(kStages) * gridDim.x;
        if (tn < nt) issue(tn, s);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// lagged variant: slot of tile k is refilled only after the store of tile k
// has read it, checked L stores later (wait_group.read L), so up to L+1
// stores and S-L-1 loads are in flight per CTA
template <int kTileBytes, int kStages, int kLag>
__global__ void __launch_bounds__(32) k_tma2(const char* __restrict__ buf, const uint32_t* __restrict__ slots,
                                             uint64_t n, uint64_t row_bytes, char* __restrict__ out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[kStages];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kStages; ++s) {
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    const uint64_t tpr = row_bytes / kTileBytes, nt = n * tpr;
    const uint64_t mine = nt > blockIdx.x ? (nt - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;  // my tiles
    auto tile = [&](uint64_t k) { return blockIdx.x + k * gridDim.x; };
    auto issue = [&](uint64_t k) {
        const uint64_t t = tile(k), row = t / tpr, c = (t - row * tpr) * kTileBytes;
        const int s = int(k % kStages);
        const char* src = buf + uint64_t(slots[row]) * row_bytes + c;
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sm + s * kTileBytes));
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTileBytes));
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                     "l"(src), "r"(kTileBytes), "r"(b)
                     : "memory");
    };
    const uint64_t pre = mine < uint64_t(kStages - kLag) ? mine : uint64_t(kStages - kLag);
    for (uint64_t k = 0; k < pre; ++k) issue(k);
    for (uint64_t k = 0; k < mine; ++k) {
        const int s = int(k % kStages);
        const uint32_t par = uint32_t((k / kStages) & 1);
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
        uint32_t done = 0, spins = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done)
                         : "r"(b), "r"(par));
            if (++spins > (1u << 24)) __trap();  // never hang the box
        }
        const uint64_t t = tile(k), row = t / tpr, c = (t - row * tpr) * kTileBytes;
        const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(sm + s * kTileBytes));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + row * row_bytes + c),
                     "r"(sp), "r"(kTileBytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        // tile k+S-L goes into slot (k-L)%S: fresh while k < L, else free once
        // tile k-L's store has read it (at most L newer stores pending)
        const uint64_t kn = k + uint64_t(kStages) - kLag;
        if (k >= uint64_t(kLag)) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kLag) : "memory");
        if (kn < mine) issue(kn);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const uint64_t C = 52428, RB = 262144, n = 4096;
    char *buf, *out;
    uint32_t* slots;
    cudaMalloc(&buf, C * RB);
    cudaMalloc(&out, n * RB * 2);
    cudaMalloc(&slots, n * 4);
    cudaMemset(buf, 1, C * RB);
    std::vector<uint32_t> h(n);
    std::mt19937 r(1);
    for (auto& x : h) x = r() % C;
    cudaMemcpy(slots, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    char* flush;
    cudaMalloc(&flush, 256 << 20);
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        float best = 1e9, tot = 0;
        const int reps = 20;
        for (int i = 0; i < reps; ++i) {
            cudaMemsetAsync(flush, i, 256 << 20);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
            tot += ms;
        }
        const double bytes = 2.0 * n * RB;
        std::printf("%-28s best %.1f us (%.0f GB/s)  mean %.1f us (%.0f GB/s)  %s\n", name, best * 1e3,
                    bytes / (best * 1e-3) / 1e9, tot / reps * 1e3, bytes / (tot / reps * 1e-3) / 1e9,
                    cudaGetErrorString(cudaGetLastError()));
    };
    const uint64_t vpr = RB / 16;
    const uint4* b4 = reinterpret_cast<const uint4*>(buf);
    uint4* o4 = reinterpret_cast<uint4*>(out);
    run("lsu 256x4 g1184", [&] { k_lsu<256, 4><<<1184, 256>>>(b4, slots, n, vpr, o4); });
#define TMA(T, S, G)                                                                              \
    {                                                                                             \
        auto k = k_tma<T, S>;                                                                     \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T * S);              \
        char nm[64];                                                                              \
        std::snprintf(nm, sizeof nm, "tma %dK x%d g%d", T / 1024, S, G);                        \
        run(nm, [&] { k<<<G, 32, T * S>>>(buf, slots, n, RB, out); });                           \
    }
#define TMA2(T, S, L, G)                                                                          \
    {                                                                                             \
        auto k = k_tma2<T, S, L>;                                                                 \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T * S);              \
        char nm[64];                                                                              \
        std::snprintf(nm, sizeof nm, "tma2 %dK x%d lag%d g%d", T / 1024, S, L, G);              \
        run(nm, [&] { k<<<G, 32, T * S>>>(buf, slots, n, RB, out); });                           \
    }
    TMA(16384, 6, 592) TMA(16384, 4, 1184)
    TMA2(16384, 6, 0, 296) TMA2(16384, 6, 1, 296) TMA2(16384, 6, 2, 296) TMA2(16384, 12, 2, 148)
    TMA2(16384, 12, 4, 148) TMA2(16384, 8, 2, 296) TMA2(16384, 4, 1, 444) TMA2(32768, 6, 2, 148)
    TMA2(32768, 3, 1, 296) TMA2(8192, 12, 3, 296) TMA2(8192, 8, 2, 444) TMA2(16384, 4, 1, 592)
    run("cudaMemcpy D2D 1 GiB", [&] { cudaMemcpyAsync(out, buf, n * RB, cudaMemcpyDeviceToDevice); });
    return 0;
}

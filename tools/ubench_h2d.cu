// ubench_h2d.cu — miss-path probe: 256 KiB rows scattered in a pinned host
// dataset -> contiguous device staging. Copy-engine variants (per-row
// cudaMemcpyAsync on 1 / 4 streams) vs SM-driven reads
// of mapped host memory (LSU uint4, TMA bulk copies). CUDA-event timed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench_h2d.cu -o tools/ubench_h2d
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e = (x);                                                     \
        if (e != cudaSuccess) {                                                  \
            std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            return 1;                                                            \
        }                                                                        \
    } while (0)

__global__ void __launch_bounds__(512) k_lsu(const uint4* __restrict__ host, const uint32_t* __restrict__ ids,
                                             uint32_t n, uint64_t vpr, uint4* __restrict__ out) {
    // one CTA per row at a time, 8 x 16 B per thread in flight
    for (uint32_t r = blockIdx.x; r < n; r += gridDim.x) {
        const uint4* src = host + uint64_t(ids[r]) * vpr;
        uint4* dst = out + uint64_t(r) * vpr;
        for (uint64_t c0 = 0; c0 < vpr; c0 += 512 * 8) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = src[c0 + u * 512 + threadIdx.x];
#pragma unroll
            for (int u = 0; u < 8; ++u) dst[c0 + u * 512 + threadIdx.x] = v[u];
        }
    }
}

template <int kTile, int kStages>
__global__ void __launch_bounds__(32) k_tma(const char* __restrict__ host, const uint32_t* __restrict__ ids,
                                            uint32_t n, uint64_t row, char* __restrict__ out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[kStages];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kStages; ++s) {
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    const uint64_t tpr = row / kTile, nt = uint64_t(n) * tpr;
    uint32_t phase[kStages] = {};
    uint64_t t0 = blockIdx.x;
    // simple: load kStages tiles, wait each, store, loop
    for (uint64_t base = t0; base < nt; base += uint64_t(gridDim.x) * kStages) {
        int cnt = 0;
        for (int s = 0; s < kStages; ++s) {
            const uint64_t t = base + uint64_t(s) * gridDim.x;
            if (t >= nt) break;
            const uint64_t r = t / tpr, c = (t % tpr) * kTile;
            const char* src = host + uint64_t(ids[r]) * row + c;
            const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sm + s * kTile));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTile));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                         "l"(src), "r"(kTile), "r"(b)
                         : "memory");
            ++cnt;
        }
        for (int s = 0; s < cnt; ++s) {
            const uint64_t t = base + uint64_t(s) * gridDim.x;
            const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[s]));
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(b), "r"(phase[s]) : "memory");
            phase[s] ^= 1;
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(sm + s * kTile));
            char* dst = out + t / tpr * row + (t % tpr) * kTile;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(d), "r"(kTile) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const uint64_t SB = 262144, HOST = 16ull << 30, NROWS = HOST / SB;
    const uint32_t n = argc > 1 ? atoi(argv[1]) : 4096;
    char* h = nullptr;
    CK(cudaHostAlloc(&h, HOST, cudaHostAllocMapped | cudaHostAllocPortable));
    for (uint64_t i = 0; i < HOST; i += 4096) h[i] = char(i >> 12);
    char *d = nullptr, *dh = nullptr;
    CK(cudaMalloc(&d, uint64_t(n) * SB));
    CK(cudaHostGetDevicePointer((void**)&dh, h, 0));
    std::vector<uint32_t> ids(n);
    std::mt19937_64 rng(1);
    for (auto& v : ids) v = uint32_t(rng() % NROWS);
    uint32_t* dids;
    CK(cudaMalloc(&dids, n * 4));
    CK(cudaMemcpy(dids, ids.data(), n * 4, cudaMemcpyHostToDevice));
    cudaStream_t s[4];
    for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto report = [&](const char* name) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("%-34s %8.3f ms  %7.2f GB/s\n", name, ms, double(n) * SB / (ms * 1e-3) / 1e9);
    };
    for (int rep = 0; rep < 2; ++rep) {
        // 1: per-row copies, one stream
        CK(cudaEventRecord(e0, s[0]));
        for (uint32_t r = 0; r < n; ++r)
            CK(cudaMemcpyAsync(d + uint64_t(r) * SB, h + uint64_t(ids[r]) * SB, SB, cudaMemcpyHostToDevice, s[0]));
        CK(cudaEventRecord(e1, s[0]));
        CK(cudaDeviceSynchronize());
        report("memcpyAsync per row, 1 stream");
        // 2: four streams
        CK(cudaEventRecord(e0, s[0]));
        for (int j = 1; j < 4; ++j) CK(cudaStreamWaitEvent(s[j], e0));
        for (uint32_t r = 0; r < n; ++r)
            CK(cudaMemcpyAsync(d + uint64_t(r) * SB, h + uint64_t(ids[r]) * SB, SB, cudaMemcpyHostToDevice, s[r & 3]));
        cudaEvent_t ej[4];
        for (int j = 1; j < 4; ++j) {
            CK(cudaEventCreateWithFlags(&ej[j], cudaEventDisableTiming));
            CK(cudaEventRecord(ej[j], s[j]));
            CK(cudaStreamWaitEvent(s[0], ej[j]));
        }
        CK(cudaEventRecord(e1, s[0]));
        CK(cudaDeviceSynchronize());
        report("memcpyAsync per row, 4 streams");
        // 4: LSU zero-copy
        for (int g : {16, 32, 64, 148}) {
            CK(cudaEventRecord(e0, s[0]));
            k_lsu<<<g, 512, 0, s[0]>>>((const uint4*)dh, dids, n, SB / 16, (uint4*)d);
            CK(cudaEventRecord(e1, s[0]));
            CK(cudaDeviceSynchronize());
            char nm[64];
            std::snprintf(nm, sizeof nm, "LSU zero-copy grid %d", g);
            report(nm);
        }
        // 5: TMA from host memory
        CK(cudaFuncSetAttribute(k_tma<16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8));
        for (int g : {16, 32, 64, 148}) {
            CK(cudaMemset(d, 0, uint64_t(n) * SB));
            CK(cudaEventRecord(e0, s[0]));
            k_tma<16384, 8><<<g, 32, 16384 * 8, s[0]>>>(dh, dids, n, SB, d);
            CK(cudaEventRecord(e1, s[0]));
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                std::printf("TMA from host: %s\n", cudaGetErrorString(e));
                return 0;
            }
            char nm[64];
            std::snprintf(nm, sizeof nm, "TMA zero-copy grid %d", g);
            report(nm);
        }
        // verify the last TMA result
        std::vector<char> chk(SB);
        bool ok = true;
        for (uint32_t r = 0; r < n; r += 97) {
            CK(cudaMemcpy(chk.data(), d + uint64_t(r) * SB, SB, cudaMemcpyDeviceToHost));
            if (std::memcmp(chk.data(), h + uint64_t(ids[r]) * SB, SB)) ok = false;
        }
        std::printf("TMA bytes %s\n", ok ? "match" : "MISMATCH");
    }
    return 0;
}

// common.cuh — shared device helpers for the lsg kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/lsg.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "lsg kernels target sm_100a (B200) only"
#endif

namespace lsg {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;  // prng.hpp:42
constexpr uint32_t kNone = 0xFFFFFFFFu;             // "not resident" / "no value"
constexpr uint32_t kNever = LSG_NEVER;              // kNeverUsed (buffer.hpp:19)
constexpr uint32_t kHit = LSG_HIT_BIT;

// splitmix64 finaliser (prng.hpp:18-23). Draw k (1-based) of a stream seeded
// s is mix(s + k*gamma): the generator is counter-based, which is what lets
// every kernel below compute its draws independently.
// fire-and-forget global OR / AND (RED: no return value, so no scoreboard
// entry; atomicOr with an unused result compiles to a returning ATOMG)
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_and(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t k) {
    return mix64(seed + k * kGamma);
}
// next_double (prng.hpp:31-33)
__host__ __device__ __forceinline__ double to_unit(uint64_t r) {
    return static_cast<double>(r >> 11) * (1.0 / 9007199254740992.0);
}

// Errors -------------------------------------------------------------------
enum Err : int { kOk = 0, kConfig = 2, kValidation = 3, kCapability = 4, kStorage = 6, kInternal = 7 };
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* where);
void count_launch();
void keep_pool();  // stream-ordered pool keeps its memory between calls
bool profiling();  // LSG_PROFILE=1: per-phase cycle counters to stderr

#define LSG_CUDA(call)                                          \
    do {                                                        \
        cudaError_t _e = (call);                                \
        if (_e != cudaSuccess) return ::lsg::cuda_error(_e, #call); \
    } while (0)

#define LSG_LAUNCH_CHECK(where)                                  \
    do {                                                         \
        ::lsg::count_launch();                                   \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return ::lsg::cuda_error(_e, where); \
    } while (0)

// Stream-ordered scratch (cudaMallocAsync pool). Freed on the same stream.
struct Scratch {
    cudaStream_t s;
    void* ptrs[64];
    int n = 0;
    explicit Scratch(cudaStream_t st) : s(st) { keep_pool(); }
    template <typename T>
    T* get(size_t count) {
        void* p = nullptr;
        if (count == 0) count = 1;
        if (cudaMallocAsync(&p, count * sizeof(T), s) != cudaSuccess) return nullptr;
        ptrs[n++] = p;
        return static_cast<T*>(p);
    }
    ~Scratch() {
        for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], s);
    }
};

// L2 set-aside for a latency-bound kernel's random-access state (LSG_L2PIN=1,
// default off: measured slower): kernels launched on `st` until l2_unpin see [p, p + bytes) as
// a persisting access-policy window, so a fetch streaming through L2 beside
// them does not evict their lines. Returns false (and does nothing) when the
// device has no persisting L2 or the feature is off.
bool l2_pin(cudaStream_t st, const void* p, size_t bytes);
void l2_unpin(cudaStream_t st);

// Dynamic shared memory for the latency-bound single-CTA-per-unit kernels
// (the planner's persistent step loop, the per-rank replay): rounded up so the
// CTA holds its SM alone (LSG_EXCLUSIVE_SM=0: the bare need). Beside the
// fetch's TMA CTAs or each other they otherwise share an SM's issue slots and
// load/store pipes, and one shared SM stretches the whole stage.
size_t exclusive_smem(size_t need);

// Small device->host readback (status words, counts; <= 64 bytes) through a
// per-thread PINNED staging buffer, then a sync of `st` only. A copy into
// pageable host memory is staged by the driver and waited for beside other
// streams' kernels: a replay's status read sat behind a concurrent planner's
// persistent kernel (the whole plan) on another stream.
int d2h_small(void* h, const void* d, size_t bytes, cudaStream_t st);

struct PlanDims {
    uint64_t D, B, S, keep, T;
    uint32_t N, E, b;
};

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
    uint64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

}  // namespace lsg

// fetch_job.cu — the loading phase of a whole job (a step range of a plan)
// with a real miss source.
//
// The reference reads every sample of a batch from its Store (store.cpp:123-148,
// pread at 22 + i*size). Here hits come from the rank's HBM sample buffer
// (K8, TMA bulk copies, gather.cu) and misses from the HOST TIER: the Store
// payload rows of the whole dataset in host memory (a tmpfs file, mapped and
// pinned, so every process of a box shares one copy), read over PCIe.
//
//   lsg_host_rows      the host tier: payload byte j of the file = byte j%8 of
//                      mix(fill_seed + (j/8+1)*gamma) (store.cpp:70-80), row i
//                      at i*sample_bytes — the Store file without its 22-byte
//                      header, so rows stay 16-byte aligned for TMA.
//   miss list          per job: the rows of every step whose replay slot is
//                      not a hit, in step order (k_miss_list count pass,
//                      scan, list pass), built on the device.
//   K10 prefetcher     a persistent kernel (32 single-thread CTAs) walks the
//                      miss list ahead of the fetch: TMA bulk copies from the
//                      MAPPED host rows (cp.async.bulk global->shared reads
//                      host memory over PCIe: 51 GB/s measured,
//                      tools/ubench_h2d.cu) into a device ring, publishing
//                      each row with a release flag. It waits for ring space
//                      on a consumed counter. It is launched when the job is
//                      created, so it runs ahead while earlier work (the
//                      previous job's fetch) still holds the fetch stream.
//   misses kernel      after step g's hit kernel: every miss row of g copied
//                      ring -> batch row and, unless the replay bypassed the
//                      sample, -> its new HBM slot; the last block of the step
//                      releases the step's ring rows. Without a host tier the
//                      payload is synthesised on device instead (K9).
//
// Slot order: a miss may refill a slot whose previous sample was hit earlier
// in the same step, so misses run after the step's hit kernel (as the
// single-step path does); the next step's hit kernel runs after them.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fetch.cuh"

struct lsg_host_rows {
    std::string path;
    int fd = -1;
    unsigned char* base = nullptr;
    unsigned char* dev = nullptr;  // device alias of base (mapped, pinned)
    uint64_t count = 0, sample_bytes = 0, bytes = 0;
    bool registered = false;
};

namespace lsg {

namespace {

constexpr int kPfTile = 8192, kPfStages = 3, kPfCtas = 32;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acquire64(const uint32_t* p) {  // (8-byte aligned)
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// per-step row counts of the node range and the job's step item bases
struct ListArgs {
    const uint32_t* items;
    const uint32_t* slots;
    const uint32_t* node_off;  // job's first step's [N+1] offsets
    const uint32_t* base;      // [nsteps] item offset of each step (job-relative)
    uint32_t N, k0, k1, nsteps;
    uint32_t* cnt;             // [nsteps] misses per step
    uint32_t* moff;            // [nsteps+1] exclusive scan of cnt
    uint32_t* mrow;            // [M] step-relative row of each miss
    uint32_t* mid;             // [M] its sample id
    unsigned long long* stats; // [4] misses, kept, host bytes, hits
    uint64_t host_row_bytes;   // 0 without a host tier
};

// one block per step: count (pass 0) or list (pass 1) the step's miss rows
// in row order
__global__ void __launch_bounds__(256) k_miss_list(ListArgs a, int pass) {
    __shared__ uint32_t wsum[8];
    __shared__ uint32_t carry;
    const uint32_t g = blockIdx.x;
    const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
    const uint32_t r0 = off[a.k0], r1 = off[a.k1];
    const uint64_t b = a.base[g];  // job-relative item offset of the step
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = pass ? a.moff[g] : 0u;
    __syncthreads();
    uint32_t kept = 0;
    for (uint32_t c = r0; c < r1; c += 256) {
        const uint32_t r = c + threadIdx.x;
        bool miss = false;
        uint32_t sl = kNever;
        if (r < r1) {
            sl = __ldg(&a.slots[b + r]);
            miss = sl == kNever || !(sl & kHit);
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, miss);
        if (lane == 0) wsum[w] = __popc(bal);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (int q = 0; q < 8; ++q) {
            before += q < int(w) ? wsum[q] : 0u;
            total += wsum[q];
        }
        if (miss) {
            kept += sl != kNever;
            if (pass) {
                const uint32_t at = carry + before + __popc(bal & ((1u << lane) - 1));
                a.mrow[at] = r;
                a.mid[at] = __ldg(&a.items[b + r]) & ~kHit;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (pass == 0) {
        kept = __reduce_add_sync(0xFFFFFFFFu, kept);
        if (lane == 0 && kept) atomicAdd(&a.stats[1], (unsigned long long)kept);
        if (threadIdx.x == 0) {
            a.cnt[g] = carry;
            atomicAdd(&a.stats[0], (unsigned long long)carry);
            atomicAdd(&a.stats[2], (unsigned long long)carry * a.host_row_bytes);
            atomicAdd(&a.stats[3], (unsigned long long)(r1 - r0 - carry));
        }
    }
}

// single-block exclusive scan of u32 values in[i * stride] (n up to a few
// 1e5) -> out[n+1]
__global__ void __launch_bounds__(1024) k_scan_u32(const uint32_t* __restrict__ in, uint32_t n, uint32_t stride,
                                                   uint32_t* __restrict__ out) {
    __shared__ uint32_t part[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint32_t c = 0; c < n; c += 1024) {
        const uint32_t i = c + threadIdx.x;
        const uint32_t v = i < n ? in[size_t(i) * stride] : 0u;
        uint32_t inc = v;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= uint32_t(d)) inc += o;
        }
        if (lane == 31) part[w] = inc;
        __syncthreads();
        if (w == 0) {
            const uint32_t p = part[lane];
            uint32_t pi = p;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, pi, d);
                if (lane >= uint32_t(d)) pi += o;
            }
            part[lane] = pi - p;
        }
        __syncthreads();
        if (i < n) out[i] = carry + part[w] + inc - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += part[w] + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[n] = carry;
}

struct PrefetchArgs {
    const unsigned char* host;  // device alias of the mapped host rows
    const uint32_t* mid;        // sample id of each miss, job order
    const uint32_t* total;      // &moff[nsteps]
    uint64_t row_bytes;
    unsigned char* ring;
    uint32_t R;                 // ring rows
    uint32_t* ready;            // [R] row m is in ring slot m % R once ready[m % R] == m + 1
    const uint32_t* consumed;   // sequence numbers released by the consumers (a prefix)
    unsigned int* resident;     // host-mapped: CTAs that started
    const uint32_t* seq0;       // sequence number of the job's first miss (0 with a private ring)
    uint32_t* pf_done;          // sequence numbers fully prefetched (jobs prefetch one after another)
    uint32_t* ctas_done;        // this job's finished prefetch CTAs
};

// Jobs sharing a ring prefetch strictly in sequence order: a prefetcher
// starts once the previous job's prefetcher has published every row, so it
// never takes PCIe bandwidth from an earlier job whose fetch waits on it; the
// last CTA to finish passes the baton.
__device__ __forceinline__ void pf_wait_turn(const PrefetchArgs& a, uint32_t s0) {
    while (ld_acquire(a.pf_done) < s0) __nanosleep(512);
}
__device__ __forceinline__ void pf_pass_turn(const PrefetchArgs& a, uint32_t s0, uint32_t M) {
    __threadfence();
    if (atomicAdd(a.ctas_done, 1u) == gridDim.x - 1) atomicMax(a.pf_done, s0 + M);
}

// K10: TMA bulk copies host -> shared -> ring, kPfStages tiles in flight per
// CTA, rows round-robin over the CTAs
__global__ void __launch_bounds__(32) k_miss_prefetch_tma(PrefetchArgs a) {
    extern __shared__ __align__(128) unsigned char psm[];
    __shared__ __align__(8) unsigned long long bar[kPfStages];
    if (threadIdx.x != 0) return;
    atomicAdd_system(a.resident, 1u);
    for (int q = 0; q < kPfStages; ++q) {
        const unsigned bq = static_cast<unsigned>(__cvta_generic_to_shared(&bar[q]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bq));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    const uint32_t M = *a.total, s0 = *a.seq0;
    const uint64_t tpr = a.row_bytes / kPfTile;
    uint32_t phase[kPfStages] = {};
    pf_wait_turn(a, s0);
    for (uint32_t m = blockIdx.x; m < M; m += gridDim.x) {
        const uint32_t q = s0 + m;  // sequence number: ring slot q % R
        if (q >= a.R)
            while (ld_acquire(a.consumed) < q - a.R + 1) __nanosleep(256);
        const unsigned char* src = a.host + uint64_t(__ldg(&a.mid[m])) * a.row_bytes;
        unsigned char* dst = a.ring + uint64_t(q % a.R) * a.row_bytes;
        auto load = [&](uint64_t t) {
            const int q = int(t % kPfStages);
            const unsigned bq = static_cast<unsigned>(__cvta_generic_to_shared(&bar[q]));
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(psm + q * kPfTile));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bq), "r"(kPfTile));
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(d), "l"(src + t * kPfTile), "r"(kPfTile), "r"(bq) : "memory");
        };
        for (uint64_t t = 0; t < tpr && t < uint64_t(kPfStages); ++t) load(t);
        for (uint64_t t = 0; t < tpr; ++t) {
            const int q = int(t % kPfStages);
            const unsigned bq = static_cast<unsigned>(__cvta_generic_to_shared(&bar[q]));
            uint32_t done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(done) : "r"(bq), "r"(phase[q]) : "memory");
            phase[q] ^= 1u;
            const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(psm + q * kPfTile));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * kPfTile),
                         "r"(sp), "r"(kPfTile) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            if (t + kPfStages < tpr) {  // stage q is reloaded once its store has read it
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                load(t + kPfStages);
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the row is in the ring
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        st_release(&a.ready[q % a.R], q + 1);
    }
    pf_pass_turn(a, s0, M);
}

// K10 for rows that are not whole TMA tiles: 128-bit loads of mapped host memory
__global__ void __launch_bounds__(256) k_miss_prefetch_lsu(PrefetchArgs a) {
    if (threadIdx.x == 0) atomicAdd_system(a.resident, 1u);
    const uint32_t M = *a.total, s0 = *a.seq0;
    const uint64_t vpr = a.row_bytes / 16;
    if (threadIdx.x == 0) pf_wait_turn(a, s0);
    __syncthreads();
    for (uint32_t m = blockIdx.x; m < M; m += gridDim.x) {
        const uint32_t q = s0 + m;
        if (threadIdx.x == 0 && q >= a.R)
            while (ld_acquire(a.consumed) < q - a.R + 1) __nanosleep(256);
        __syncthreads();
        const uint4* src = reinterpret_cast<const uint4*>(a.host + uint64_t(__ldg(&a.mid[m])) * a.row_bytes);
        uint4* dst = reinterpret_cast<uint4*>(a.ring + uint64_t(q % a.R) * a.row_bytes);
        uint64_t p = threadIdx.x;
        for (; p + 3 * blockDim.x < vpr; p += 4 * blockDim.x) {  // 4 loads in flight per thread
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = src[p + u * blockDim.x];
#pragma unroll
            for (int u = 0; u < 4; ++u) __stcg(&dst[p + u * blockDim.x], v[u]);
        }
        for (; p < vpr; p += blockDim.x) __stcg(&dst[p], src[p]);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(&a.ready[q % a.R], q + 1);
        }
    }
    if (threadIdx.x == 0) pf_pass_turn(a, s0, M);
}

struct MissArgs {
    StepFetch f;               // step g (items/slots/node_off at the step)
    const uint32_t* moff;      // [nsteps+1]
    uint32_t gi;               // step index in the job
    const uint32_t* mrow;
    const unsigned char* ring; // null: synthesise the Store payload
    uint32_t R;
    const uint32_t* ready;
    uint32_t* consumed;
    uint32_t* done;            // [nsteps] finished blocks per step
    const uint32_t* seq0;      // sequence number of the job's first miss
};

// the misses of one step: batch row and (kept) new slot from the ring or the
// synthesised payload; the step's last block releases its ring rows
__global__ void __launch_bounds__(256) k_job_misses(MissArgs a) {
    asm volatile("griddepcontrol.launch_dependents;");  // the next step's early loads avoid this step's slots
    const StepFetch& f = a.f;
    const uint32_t m0 = __ldg(&a.moff[a.gi]), m1 = __ldg(&a.moff[a.gi + 1]);
    const uint32_t s0 = a.ring ? __ldg(a.seq0) : 0u;
    const uint64_t vpr = f.vec_per_row;
    const uint64_t row_bytes = vpr * 16;
    for (uint32_t m = m0 + blockIdx.y; m < m1; m += gridDim.y) {
        const uint32_t r = __ldg(&a.mrow[m]);
        const uint32_t sl = __ldg(&f.slots[r]);
        const uint32_t k = node_of_row(f, r);
        uint4* out = f.outs[k - f.k0] + uint64_t(r - __ldg(&f.node_off[k])) * vpr;
        uint4* buf = sl != kNever ? f.bufs[k - f.k0] + uint64_t(sl) * vpr : nullptr;
        if (a.ring) {
            const uint32_t q = s0 + m;
            if (threadIdx.x == 0)
                while (ld_acquire(&a.ready[q % a.R]) != q + 1) __nanosleep(128);
            __syncthreads();
            const uint4* src = reinterpret_cast<const uint4*>(a.ring + uint64_t(q % a.R) * row_bytes);
            for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < vpr;
                 p += uint64_t(gridDim.x) * blockDim.x) {
                const uint4 v = __ldcg(&src[p]);
                __stcs(&out[p], v);
                if (buf) __stcs(&buf[p], v);
            }
        } else {
            const uint64_t word0 = uint64_t(__ldg(&f.items[r]) & ~kHit) * (2 * vpr);
            ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out);
            ulonglong2* b2 = reinterpret_cast<ulonglong2*>(buf);
            for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < vpr;
                 p += uint64_t(gridDim.x) * blockDim.x) {
                ulonglong2 v;
                v.x = mix64(f.seed + (word0 + 2 * p + 1) * kGamma);
                v.y = mix64(f.seed + (word0 + 2 * p + 2) * kGamma);
                __stcs(&o2[p], v);
                if (b2) __stcs(&b2[p], v);
            }
        }
    }
    if (a.ring) {  // every block has read its ring rows: the last one releases the step's
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const uint32_t t = atomicAdd(&a.done[a.gi], 1u);
            if (t == gridDim.x * gridDim.y - 1) atomicMax(a.consumed, s0 + m1);
        }
    }
}

// ---- the fused step kernel (rows of whole 8 KiB tiles) ----------------------
// Per row of a step a flag word (k_row_flags), miss index in the upper bits:
//   kRowEarly    a hit whose slot content was NOT written in the previous
//                step: its loads may start before the previous step's kernel
//                has finished (programmatic dependent launch);
//   kRowInplace  a kept miss whose slot was not read by a hit of the same
//                step: its slot is written by this kernel, beside the batch
//                row; other kept misses are written to their slot in the
//                step's deferred-fill phase, after the step's hits.
//   kRowSlotOld  an in-place miss whose slot no row of the previous step read
//                or wrote: its slot write waits only for the step two back.
constexpr uint32_t kRowEarly = 1u, kRowInplace = 2u, kRowSlotOld = 4u, kRowShift = 3;

struct FlagArgs {
    const uint32_t* slots;
    const uint32_t* node_off;  // job's first step
    const uint32_t* base;      // [ns] job-relative step bases
    const uint32_t* moff;      // [ns+1] job miss offsets
    uint32_t N, k0, k1, P2;
    uint32_t* flags;           // [job items] per row: (miss index << 2) | bits
    uint32_t* ndefer;          // [ns] deferred slot writes per step
};

__device__ __forceinline__ bool sl_hit(uint32_t sl) { return sl != kNever && (sl & kHit); }

// one block per step, nodes [k0, k1) in turn: sort the node's hit slots of
// this step and its kept-miss and hit slots of the previous step, then flag
// every row
__global__ void __launch_bounds__(256) k_row_flags(FlagArgs a) {
    extern __shared__ uint32_t fsm[];
    uint32_t* hs = fsm;              // [P2] hit slots of (g, k), sorted
    uint32_t* ps = fsm + a.P2;       // [P2] kept-miss slots of (g-1, k), sorted
    uint32_t* hp = fsm + 2 * a.P2;   // [P2] hit slots of (g-1, k), sorted
    __shared__ uint32_t cnt[3], carry, ndef;
    __shared__ uint32_t wc[8];
    const uint32_t gi = blockIdx.x;
    const uint32_t* off = a.node_off + size_t(gi) * (a.N + 1);
    const uint64_t b = a.base[gi];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        carry = a.moff[gi];  // miss index of the step's next miss
        ndef = 0;
    }
    auto has = [](const uint32_t* v, uint32_t n, uint32_t x) {
        uint32_t l0 = 0, l1 = n;
        while (l0 < l1) {
            const uint32_t mid = (l0 + l1) >> 1;
            if (v[mid] < x) l0 = mid + 1; else l1 = mid;
        }
        return l0 < n && v[l0] == x;
    };
    for (uint32_t k = a.k0; k < a.k1; ++k) {
        const uint32_t lo = off[k], hi = off[k + 1];
        if (threadIdx.x == 0) cnt[0] = cnt[1] = cnt[2] = 0;
        for (uint32_t i = threadIdx.x; i < a.P2; i += blockDim.x) hs[i] = ps[i] = hp[i] = 0xFFFFFFFFu;
        __syncthreads();
        for (uint32_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
            const uint32_t sl = a.slots[b + r];
            if (sl_hit(sl)) hs[atomicAdd(&cnt[0], 1u)] = sl & ~kHit;
        }
        if (gi > 0) {  // the first step of a job never loads early
            const uint32_t* off0 = off - (a.N + 1);
            const uint64_t b0 = a.base[gi - 1];
            for (uint32_t r = off0[k] + threadIdx.x; r < off0[k + 1]; r += blockDim.x) {
                const uint32_t sl = a.slots[b0 + r];
                if (!sl_hit(sl) && sl != kNever) ps[atomicAdd(&cnt[1], 1u)] = sl;
                else if (sl_hit(sl)) hp[atomicAdd(&cnt[2], 1u)] = sl & ~kHit;
            }
        }
        __syncthreads();
        for (uint32_t size = 2; size <= a.P2; size <<= 1)  // the three arrays at once, bitonic
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t t = threadIdx.x; t < 3 * (a.P2 / 2); t += blockDim.x) {
                    const uint32_t q = t & (a.P2 / 2 - 1);
                    uint32_t* v = fsm + (t / (a.P2 / 2)) * a.P2;
                    const uint32_t x0 = 2 * stride * (q / stride) + (q % stride), x1 = x0 + stride;
                    const bool up = (x0 & size) == 0;
                    const uint32_t p = v[x0], r2 = v[x1];
                    if ((p > r2) == up) { v[x0] = r2; v[x1] = p; }
                }
                __syncthreads();
            }
        // rows in order: a miss's index is the step's misses before it
        for (uint32_t c = lo; c < hi; c += blockDim.x) {
            const uint32_t r = c + threadIdx.x;
            const uint32_t sl = r < hi ? a.slots[b + r] : kHit;
            const bool miss = r < hi && !sl_hit(sl);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, miss);
            if (lane == 0) wc[w] = __popc(bal);
            __syncthreads();
            uint32_t pre = carry;
            for (uint32_t q = 0; q < w; ++q) pre += wc[q];
            if (r < hi) {
                uint32_t f;
                if (!miss) {
                    f = (gi > 0 && !has(ps, cnt[1], sl & ~kHit)) ? kRowEarly : 0u;
                } else {
                    const uint32_t m = pre + __popc(bal & ((1u << lane) - 1));
                    const bool inplace = sl == kNever || !has(hs, cnt[0], sl);
                    if (!inplace) atomicAdd(&ndef, 1u);
                    const bool old = inplace && sl != kNever && gi > 0 && !has(ps, cnt[1], sl) && !has(hp, cnt[2], sl);
                    f = (m << kRowShift) | (inplace ? kRowInplace : 0u) | (old ? kRowSlotOld : 0u);
                }
                a.flags[b + r] = f;
            }
            __syncthreads();
            if (threadIdx.x == 0)
                for (uint32_t q = 0; q < blockDim.x / 32; ++q) carry += wc[q];
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) a.ndefer[gi] = ndef;
}

// the deferred slot writes of every step as a list (rows in order, step gi's
// at doff[gi]): kept misses whose slot a hit of the same step reads
__global__ void __launch_bounds__(256) k_defer_list(FlagArgs a, const uint32_t* __restrict__ doff,
                                                    uint32_t* __restrict__ drow) {
    __shared__ uint32_t wc[8], carry;
    const uint32_t gi = blockIdx.x;
    const uint32_t* off = a.node_off + size_t(gi) * (a.N + 1);
    const uint64_t b = a.base[gi];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = doff[gi];
    __syncthreads();
    for (uint32_t c = off[a.k0]; c < off[a.k1]; c += blockDim.x) {
        const uint32_t r = c + threadIdx.x;
        bool d = false;
        if (r < off[a.k1]) {
            const uint32_t sl = a.slots[b + r];
            d = !sl_hit(sl) && sl != kNever && !(a.flags[b + r] & kRowInplace);
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, d);
        if (lane == 0) wc[w] = __popc(bal);
        __syncthreads();
        uint32_t pre = carry;
        for (uint32_t q = 0; q < w; ++q) pre += wc[q];
        if (d) drow[pre + __popc(bal & ((1u << lane) - 1))] = r;
        __syncthreads();
        if (threadIdx.x == 0)
            for (uint32_t q = 0; q < blockDim.x / 32; ++q) carry += wc[q];
        __syncthreads();
    }
}

constexpr int kFTile = 8192, kFStages = 6, kFLag = 2, kFChunk = 16, kFTail = 4;
constexpr unsigned kFCtasPerSm = 4;

struct FusedStep {
    const uint32_t* items;     // job's items (job-relative: step s at base[s])
    const uint32_t* slots;     // job's replay slots
    const uint32_t* flags;     // job's row flags
    const uint32_t* node_off;  // job's [ns][N+1]
    const uint32_t* base;      // [ns] job-relative step bases
    uint32_t N;
    unsigned char* const* bufs;
    unsigned char* const* outs;
    uint32_t k0, k1;
    uint64_t row_bytes, seed;
    uint32_t* claim;            // [2ns] tile claims per phase
    uint32_t* stored;           // [2ns] tiles NOT yet stored per phase (done at 0; 8-byte aligned pairs)
    const uint32_t* ptiles;     // [2ns] tiles per phase
    const uint32_t* ndefer;     // [ns] deferred slot writes per step
    const uint32_t* doff;       // [ns+1] their list offsets
    const uint32_t* drow;       // their rows (step-relative)
    const unsigned char* ring;  // host-tier misses (null: synthesised payload)
    uint32_t R;
    const uint32_t* ready;
    const uint32_t* seq0;
    const uint32_t* moff;       // [ns+1] job miss offsets
    uint32_t* consumed;         // ring sequence numbers released
    uint32_t gA, gB;            // the kernel's steps [gA, gB) of the job (phases [2gA, 2gB))
    uint32_t ns;                // the job's steps: the last one lands in outs, and steps
    unsigned char* scratch;     //   alternate back from it between outs and scratch
    uint32_t srows;             //   ([local rank][srows] rows of row_bytes); null scratch:
                                //   every step in outs, behind a step-wide barrier
    int skip_misses;            // misses left to k_job_misses (large synthesised rows)
};

__device__ __forceinline__ uint32_t fnode_of_row(const uint32_t* off, uint32_t k0, uint32_t k1, uint32_t r) {
    uint32_t k = k0;
    while (k + 1 < k1 && __ldg(&off[k + 1]) <= r) ++k;
    return k;
}

// Steps [gA, gB) of ranks [k0, k1) in ONE persistent launch: every row's
// 8 KiB tiles through an S-stage TMA pipeline per CTA, split between two
// warps so neither's instruction stream bounds the copy rate: warp 0 (the
// producer) claims tiles and loads them — hit tiles HBM slot -> shared, miss
// tiles from the ring (host tier, after the row's ready flag) or as the Store
// payload computed by the warp; warp 1 (the consumer) stores each landed
// tile. Stages hand over through full (TMA transaction) and empty (store has
// read the stage) mbarriers.
//
// Work is a sequence of PHASES: phase 2s is step s's batch rows; phase 2s+1
// fills the slots of the step's kept misses (their payload again, into the
// slot only). CTAs claim tile chunks phase after phase, so a CTA that runs
// out of work in one phase starts loading the next while others finish.
// Batch rows alternate between the caller's tensors and a scratch set, the
// job's last step landing in the caller's. Ordering, with rdy = the number of
// leading phases whose tiles are all stored (per-phase counters), for a tile
// of phase P:
//   a hit loads once rdy >= P (the fills of step s-1 are done), or
//     rdy >= P-2 for an early row (its slot was not filled in step s-1); a
//     miss or a fill (reads no slot) loads once rdy >= P-2;
//   a fill stores once rdy >= P (every hit of its step has loaded the slot);
//   a batch row stores once rdy >= P-2 (step s-2 wrote the same buffer):
//     no step-wide barrier between consecutive steps' batch rows.
// Tiles, not CTAs, are counted, so a CTA that never became resident holds
// nothing anyone waits for; a consumer with nothing to store publishes what
// it holds before waiting. Before griddepcontrol.wait, rdy = 2gA - 2: the
// previous kernel runs at most its last step (both phases) behind.
// PP = phases per step: 2, or 1 when the job has no kept misses (no fills;
// per-phase arrays are indexed 2s (+1) either way).
template <int S, int L, int PP>
__global__ void __launch_bounds__(64) k_fetch_fused(FusedStep f) {
    extern __shared__ __align__(128) unsigned char fsm2[];
    __shared__ __align__(8) unsigned long long full[S], empty[S];
    __shared__ unsigned char* sdst[S];
    __shared__ unsigned char* sdst2[S];
    __shared__ int sstep[S];
    __shared__ uint8_t sslot_old[S];  // the stage's slot write needs only the step two back
    __shared__ uint32_t s_total;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[q])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[q])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        s_total = 0xFFFFFFFFu;
    }
    __syncthreads();
    const uint32_t tpr = uint32_t(f.row_bytes / kFTile);
    const uint32_t s0 = f.ring ? __ldg(f.seq0) : 0u;
    const int PA = PP * int(f.gA), PB = PP * int(f.gB);  // (phases before PA: never polled)
    auto ix = [](int P) -> int { return PP == 2 ? P : 2 * P; };  // a phase's slot in the per-phase arrays
    int rdy = PA - PP;
    // advance rdy over completed phases (all lanes: the warp stays converged); one
    // acquire load covers a step's two phases, so an empty deferred-fill phase is free
    auto poll = [&]() -> bool {
        const int r0 = rdy;
        while (rdy >= PA && rdy < PB) {
            const uint64_t v = ld_acquire64(&f.stored[ix(rdy) & ~1]);
            if (PP == 1 || !(rdy & 1)) {
                if (uint32_t(v)) break;
                if (++rdy >= PB || PP == 1) continue;
            }
            if (uint32_t(v >> 32)) break;
            ++rdy;
        }
        if (rdy != r0) asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads see those stores
        return rdy != r0;
    };
    if (warp == 0) {
        // ---------------- producer ----------------
        const uint32_t guide = gridDim.x * 2 * kFChunk;
        int sc = PA;  // the claim cursor's phase
        const uint32_t* off_s = f.node_off + size_t(sc / PP) * (f.N + 1);
        uint32_t r0 = __ldg(&off_s[f.k0]), bs = __ldg(&f.base[sc / PP]), db = 0;
        // a step's two phase sizes in one load (ptiles is 8-byte aligned)
        uint2 pt = __ldg(reinterpret_cast<const uint2*>(f.ptiles + ix(sc)));
        uint32_t nt = pt.x, te = 0, tn = 0, cur = 0xFFFFFFFFu;
        // the next phase with tiles; an odd phase shares its step's offsets, and
        // an empty one (no deferred fills: the common case) costs one load
        auto advance = [&]() -> bool {
            for (;;) {
                if (++sc >= PB) return false;
                te = tn = 0;
                if (PP == 2 && (sc & 1)) {
                    nt = pt.y;
                    if (nt == 0) continue;
                    db = __ldg(&f.doff[sc >> 1]);
                    return true;
                }
                pt = __ldg(reinterpret_cast<const uint2*>(f.ptiles + ix(sc)));
                off_s = f.node_off + size_t(sc / PP) * (f.N + 1);
                r0 = __ldg(&off_s[f.k0]);
                bs = __ldg(&f.base[sc / PP]);
                nt = pt.x;
                if (nt) return true;
            }
        };
        int cur_step = -1;
        const unsigned char* src_row = nullptr;
        unsigned char* dst_row = nullptr;
        unsigned char* dst2_row = nullptr;
        uint32_t row_flags = 0, row_id = 0;
        bool row_hit = false, row_ready = false;
        // the next tile's row state; 1 = ready, 0 = not yet (inputs not final), -1 = no more tiles
        auto next = [&]() -> int {
            for (;;) {
                if (tn >= te) {  // a new chunk: this phase's, else the next phase's
                    if (sc >= PB) return -1;
                    if (nt == 0) {  // an empty phase: no claim
                        if (!advance()) return -1;
                        continue;
                    }
                    uint32_t v = 0;
                    const uint32_t sz = (nt > te ? nt - te : 0u) > guide ? kFChunk : kFTail;
                    if (lane == 0) v = atomicAdd(&f.claim[ix(sc)], sz);
                    const uint32_t tb = __shfl_sync(0xFFFFFFFFu, v, 0);
                    if (tb >= nt) {
                        if (!advance()) return -1;
                        continue;
                    }
                    te = min(nt, tb + sz);
                    tn = tb;
                }
                const uint32_t rr = tn / tpr;
                if (rr != cur || sc != cur_step) {
                    const bool fill = PP == 2 && (sc & 1);  // a deferred slot write of step sc/2
                    const uint32_t r = fill ? __ldg(&f.drow[db + rr]) : r0 + rr;
                    const uint32_t sl = __ldg(&f.slots[bs + r]);
                    const uint32_t fl = __ldg(&f.flags[bs + r]);
                    const bool hit = !fill && sl_hit(sl);
                    if (!hit && f.skip_misses) {  // k_job_misses writes this row: skip its tiles
                        tn = (rr + 1) * tpr;
                        continue;
                    }
                    const int need = (!hit || (fl & kRowEarly)) ? sc - PP : sc;
                    if (rdy < need && (!poll() || rdy < need)) return 0;
                    cur = rr;
                    cur_step = sc;
                    const uint32_t kk = fnode_of_row(off_s, f.k0, f.k1, r);
                    row_hit = hit;
                    row_flags = fl;
                    row_id = __ldg(&f.items[bs + r]) & ~kHit;
                    row_ready = false;
                    src_row = hit ? f.bufs[kk - f.k0] + uint64_t(sl & ~kHit) * f.row_bytes : nullptr;
                    dst2_row = nullptr;
                    if (fill) {  // the slot only
                        dst_row = f.bufs[kk - f.k0] + uint64_t(sl) * f.row_bytes;
                    } else {  // the batch row, and the slot of an in-place miss
                        const uint32_t ri = r - __ldg(&off_s[kk]);
                        dst_row = (f.scratch && ((f.ns - 1 - uint32_t(sc / PP)) & 1))
                                      ? f.scratch + (uint64_t(kk - f.k0) * f.srows + ri) * f.row_bytes
                                      : f.outs[kk - f.k0] + uint64_t(ri) * f.row_bytes;
                        if (!hit && sl != kNever && (fl & kRowInplace))
                            dst2_row = f.bufs[kk - f.k0] + uint64_t(sl) * f.row_bytes;
                    }
                }
                if (!row_hit && f.ring && !row_ready) {  // host-tier miss: wait for the prefetcher's row
                    uint32_t ok = 0;
                    if (lane == 0) ok = ld_acquire(&f.ready[(s0 + (row_flags >> kRowShift)) % f.R]) == s0 + (row_flags >> kRowShift) + 1;
                    if (!__shfl_sync(0xFFFFFFFFu, ok, 0)) return 0;
                    row_ready = true;
                }
                return 1;
            }
        };
        uint32_t k = 0;
        bool waited = false, trig = false;
        for (;;) {
            const int n = next();
            if (n < 0) break;
            if (n == 0) {  // blocked on earlier phases or a ring row
                if (!waited) {
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    waited = true;
                    rdy = max(rdy, PA);
                } else if (!poll()) {
                    __nanosleep(100);
                }
                continue;
            }
            const int q = int(k % S);
            if (k >= uint32_t(S)) {  // the stage's previous store has read it
                const unsigned eb = smem_u32(&empty[q]);
                const uint32_t par = ((k / S) - 1) & 1;
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(ok) : "r"(eb), "r"(par) : "memory");
            }
            const uint64_t c = uint64_t(tn - cur * tpr) * kFTile;
            const unsigned fb = smem_u32(&full[q]);
            unsigned char* st = fsm2 + q * kFTile;
            if (lane == 0) {
                sdst[q] = dst_row + c;
                sdst2[q] = dst2_row ? dst2_row + c : nullptr;
                sstep[q] = cur_step;
                sslot_old[q] = (row_flags & kRowSlotOld) ? 1 : 0;
            }
            if (row_hit || f.ring) {
                if (lane == 0) {
                    const unsigned char* src =
                        row_hit ? src_row : f.ring + uint64_t((s0 + (row_flags >> kRowShift)) % f.R) * f.row_bytes;
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(kFTile)
                                 : "memory");
                    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(smem_u32(st)), "l"(src + c), "r"(kFTile), "r"(fb) : "memory");
                }
            } else {  // synthesised Store payload (store.cpp:70-80): words of this tile
                const uint64_t w0 = (uint64_t(row_id) * f.row_bytes + c) / 8;
                ulonglong2* sw = reinterpret_cast<ulonglong2*>(st);
                // two consecutive words per lane per 16-byte store; word counter x gamma stepped by adds
                uint64_t x = f.seed + (w0 + 2 * lane + 1) * kGamma;
#pragma unroll 8
                for (uint32_t i = lane; i < kFTile / 16; i += 32, x += 64 * kGamma)
                    sw[i] = make_ulonglong2(mix64(x), mix64(x + kGamma));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
            }
            ++tn;
            ++k;
            if (!waited && k == uint32_t(S)) {  // every stage was free: the rest waits for the previous kernel
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
                rdy = max(rdy, PA);
            }
            if (!trig && rdy >= PB - PP) {  // the next kernel assumes at most step gB-1 still runs
                asm volatile("griddepcontrol.launch_dependents;");
                trig = true;
            }
        }
        if (!waited) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            rdy = max(rdy, PA);
        }
        if (!trig) {
            while (rdy < PB - PP)
                if (!poll()) __nanosleep(128);
            asm volatile("griddepcontrol.launch_dependents;");
        }
        if (lane == 0) {
            asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(smem_u32(&s_total)), "r"(k) : "memory");
        }
    } else {
        // ---------------- consumer ----------------
        asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous kernel on the stream is done
        rdy = max(rdy, PA);
        int pend = -1;
        uint32_t pend_cnt = 0, freed = 0, k = 0;
        auto release = [&](uint32_t upto) {  // stages [freed, upto) have been read by their stores
            if (upto <= freed) return;
            if (lane == 0)
                for (uint32_t i = freed; i < upto; ++i)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[i % S])) : "memory");
            freed = upto;
        };
        auto publish = [&]() {  // this warp's stores of phase pend have landed: count them
            if (pend_cnt) {
                if (lane == 0) {
                    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    __threadfence();
                    const uint32_t left = atomicSub(&f.stored[ix(pend)], pend_cnt) - pend_cnt;
                    // every ring row of step pend/2 has landed (in its deferred fills too, if any)
                    if (f.ring && left == 0 && (PP == 1 || (pend & 1) || !__ldg(&f.ptiles[pend + 1])))
                        atomicMax(f.consumed, s0 + __ldg(&f.moff[pend / PP + 1]));
                }
                __syncwarp();
                release(k);
            }
            pend_cnt = 0;
        };
        for (;; ++k) {
            const int q = int(k % S);
            const unsigned fb = smem_u32(&full[q]);
            const uint32_t par = (k / S) & 1;
            uint32_t ok = 0, spins = 0;
            bool end = false;
            for (;;) {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok) : "r"(fb), "r"(par) : "memory");
                if (ok) break;
                uint32_t tot;
                asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(tot) : "r"(smem_u32(&s_total)) : "memory");
                if (tot <= k) {
                    end = true;
                    break;
                }
                if (++spins == 16) publish();  // idle: others may wait for what this CTA holds
            }
            if (end) break;
            const int sk = sstep[q];
            if (sk != pend) {
                publish();
                pend = sk;
            }
            // a slot write (a fill, an in-place miss) waits for every phase before it; a
            // batch row alone only for the step two back, which wrote the same buffer
            // (steps alternate outs / scratch)
            const int gate = (!f.scratch || (PP == 2 && (sk & 1)) || (sdst2[q] && !sslot_old[q])) ? sk : sk - PP;
            while (rdy < gate)
                if (!poll()) __nanosleep(64);
            if (lane == 0) {
                const unsigned sp = smem_u32(fsm2 + q * kFTile);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sdst[q]), "r"(sp),
                             "r"(kFTile) : "memory");
                if (sdst2[q])
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sdst2[q]),
                                 "r"(sp), "r"(kFTile) : "memory");
                asm volatile("cp.async.bulk.commit_group;");
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(L) : "memory");
            }
            __syncwarp();
            ++pend_cnt;
            if (k + 1 > uint32_t(L)) release(k + 1 - L);
        }
        publish();
    }
}

// a job's place in a shared miss stream: its misses take the next M sequence
// numbers (jobs reserve in the order their fetches run)
__global__ void k_reserve(const uint32_t* __restrict__ total, uint32_t* __restrict__ next_seq,
                          uint32_t* __restrict__ seq0) {
    const uint32_t s = *next_seq;
    *seq0 = s;
    *next_seq = s + *total;
}

}  // namespace

}  // namespace lsg

// A ring shared by consecutive jobs of one fetch stream (same ranks, same
// buffers): job j+1's miss prefetcher fills the ring while job j is still
// fetching, so the all-miss first epoch of job j+1 is largely in HBM when its
// fetch starts. Sequence numbers run on across jobs.
struct lsg_miss_stream {
    unsigned char* ring = nullptr;
    uint32_t* words = nullptr;  // ready [R] | next_seq | consumed | pf_done
    uint32_t R = 0;
    uint64_t sample_bytes = 0;
    cudaEvent_t reserved = nullptr;  // the last job's reservation
    bool any = false;
};

struct lsg_fetch_job {
    lsg_fetch_job_desc d;
    std::vector<uint64_t> base;  // [nsteps+1] item offset of each step (absolute)
    std::vector<uint32_t> rows;  // [nsteps] rows of the node range per step
    uint64_t nsteps = 0;
    // device state (stream-ordered pool)
    uint32_t* d_base = nullptr;  // [nsteps+1] job-relative step bases
    uint32_t* d_ctl = nullptr;   // claims [2ns] | done [2ns] | cnt [ns] | moff [ns+1] | consumed | seq0 | pf_done | ctas
    uint32_t* mrow = nullptr;
    uint32_t* mid = nullptr;
    unsigned char* ring = nullptr;  // the job's own ring, or the shared stream's
    uint32_t* ready = nullptr;
    uint32_t* consumed = nullptr;
    uint32_t* seq0 = nullptr;
    uint32_t* pf_done = nullptr;
    bool own_ring = false;
    // fused step kernel (rows of whole 8 KiB tiles)
    bool fused = false;
    uint32_t* flags = nullptr;       // [job items] row flags
    uint32_t* ndefer_d = nullptr;    // [ns]
    uint32_t* doff = nullptr;        // [ns+1] deferred rows before each step
    uint32_t* ptiles = nullptr;      // [2ns] tiles per phase (step s: 2s rows, 2s+1 deferred fills)
    uint64_t ndefer_rows = 0;        // slot fills (kept misses) in the job
    unsigned char* scratch = nullptr;  // the alternate batch rows [local rank][srows][sample_bytes]
    uint32_t srows = 0;
    uint32_t* drow = nullptr;        // the deferred rows, step by step (step-relative)
    std::vector<uint32_t> ndefer;    // deferred slot writes per step (host)
    bool skip_misses = false;        // fused kernel does hits only; k_job_misses after it
    unsigned long long* stats = nullptr;
    uint32_t R = 0;
    unsigned int* resident = nullptr;  // mapped pinned counter (recycled, never freed)
    int resident_idx = -1;
    cudaEvent_t listed = nullptr;      // the miss list is built (run waits for it)
    cudaEvent_t prefetched = nullptr;  // the prefetcher finished (destroy waits for it)
    bool prefetching = false;
    cudaStream_t prep = nullptr;       // the stream the prefetcher holds
};

namespace lsg {

namespace {

// Residency counters of the miss prefetchers: mapped pinned words from one
// page allocated once per process. cudaFreeHost may synchronise the whole
// device, which would wait for a LATER job's prefetcher that in turn waits for
// kernels the calling thread has not enqueued yet, so counters are recycled
// instead of freed.
std::mutex g_res_mu;
unsigned int* g_res = nullptr;
std::vector<int> g_res_free;
constexpr int kResSlots = 1024;

unsigned int* resident_acquire(int* idx) {
    std::lock_guard<std::mutex> lk(g_res_mu);
    if (!g_res) {
        if (cudaHostAlloc(&g_res, kResSlots * sizeof(unsigned int), cudaHostAllocMapped | cudaHostAllocPortable) !=
            cudaSuccess) {
            g_res = nullptr;
            return nullptr;
        }
        for (int i = kResSlots - 1; i >= 0; --i) g_res_free.push_back(i);
    }
    if (g_res_free.empty()) return nullptr;
    *idx = g_res_free.back();
    g_res_free.pop_back();
    g_res[*idx] = 0;
    return g_res + *idx;
}

void resident_release(int idx) {
    std::lock_guard<std::mutex> lk(g_res_mu);
    g_res_free.push_back(idx);
}

// a per-thread pinned bounce buffer for small device->host reads, grown by
// replacing (never freed: cudaFreeHost may synchronise the device)
void* pinned_bounce(size_t bytes) {
    static thread_local void* buf = nullptr;
    static thread_local size_t cap = 0;
    if (cap < bytes) {
        void* p = nullptr;
        if (cudaMallocHost(&p, std::max<size_t>(bytes, size_t(4) << 20)) != cudaSuccess) return nullptr;
        buf = p;
        cap = std::max<size_t>(bytes, size_t(4) << 20);
    }
    return buf;
}

void fill_payload(unsigned char* base, uint64_t bytes, uint64_t seed) {
    const uint64_t words = bytes / 8;
    const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([=] {
            const uint64_t w0 = words * t / nt, w1 = words * (t + 1) / nt;
            uint64_t* p = reinterpret_cast<uint64_t*>(base);
            for (uint64_t w = w0; w < w1; ++w) p[w] = mix64(seed + (w + 1) * kGamma);  // little-endian bytes
        });
    for (auto& x : th) x.join();
    for (uint64_t j = words * 8; j < bytes; ++j)  // tail bytes
        base[j] = uint8_t(mix64(seed + (j / 8 + 1) * kGamma) >> (8 * (j % 8)));
}

}  // namespace

}  // namespace lsg

using namespace lsg;

extern "C" {

int lsg_host_rows_open(const char* path, uint64_t count, uint64_t sample_bytes, uint64_t fill_seed, int32_t create,
                       lsg_host_rows** out) {
    if (!path || !out) return set_error(kValidation, "host_rows: path and out are required");
    if (count == 0 || sample_bytes == 0 || sample_bytes % 16)
        return set_error(kValidation, "host_rows: count >= 1 and sample_bytes a positive multiple of 16 required");
    auto* h = new lsg_host_rows();
    h->path = path;
    h->count = count;
    h->sample_bytes = sample_bytes;
    h->bytes = count * sample_bytes;
    h->fd = ::open(path, create ? (O_RDWR | O_CREAT | O_TRUNC) : O_RDWR, 0644);
    auto fail = [&](const std::string& msg) {
        if (h->base) munmap(h->base, h->bytes);
        if (h->fd >= 0) ::close(h->fd);
        delete h;
        return set_error(kStorage, msg);
    };
    if (h->fd < 0) return fail("host_rows: cannot open " + h->path);
    if (create) {
        if (ftruncate(h->fd, off_t(h->bytes)) != 0) return fail("host_rows: cannot size " + h->path);
    } else {
        struct stat st{};
        if (fstat(h->fd, &st) != 0 || uint64_t(st.st_size) != h->bytes)
            return fail("host_rows: " + h->path + " is not count x sample_bytes long");
    }
    void* p = mmap(nullptr, h->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, h->fd, 0);
    if (p == MAP_FAILED) return fail("host_rows: mmap failed for " + h->path);
    h->base = static_cast<unsigned char*>(p);
    if (create) fill_payload(h->base, h->bytes, fill_seed);
    if (cudaHostRegister(h->base, h->bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
        cudaGetLastError();
        return fail("host_rows: cudaHostRegister failed for " + h->path);
    }
    h->registered = true;
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, h->base, 0) != cudaSuccess) {
        cudaGetLastError();
        cudaHostUnregister(h->base);
        return fail("host_rows: no device alias for " + h->path);
    }
    h->dev = static_cast<unsigned char*>(dp);
    *out = h;
    return kOk;
}

int lsg_host_rows_info(const lsg_host_rows* h, uint64_t* count, uint64_t* sample_bytes, void** host_base) {
    if (!h) return set_error(kValidation, "host_rows: null handle");
    if (count) *count = h->count;
    if (sample_bytes) *sample_bytes = h->sample_bytes;
    if (host_base) *host_base = h->base;
    return kOk;
}

void lsg_host_rows_close(lsg_host_rows* h) {
    if (!h) return;
    if (h->registered) cudaHostUnregister(h->base);
    if (h->base) munmap(h->base, h->bytes);
    if (h->fd >= 0) ::close(h->fd);
    delete h;
}

int lsg_fetch_job_create(const lsg_fetch_job_desc* desc, lsg_fetch_job** out, void* stream) {
    if (!desc || !out) return set_error(kValidation, "fetch_job: desc and out are required");
    const lsg_fetch_job_desc& d = *desc;
    if (d.node_begin > d.node_end || d.node_end > d.N) return set_error(kValidation, "fetch_job: bad node range");
    if (d.step_begin > d.step_end) return set_error(kValidation, "fetch_job: bad step range");
    if (!d.h_node_off) return set_error(kValidation, "fetch_job: host node offsets required");
    if (d.sample_bytes == 0 || d.sample_bytes % 16)
        return set_error(kValidation, "fetch_job: sample_bytes must be a positive multiple of 16");
    if (d.host && d.host->sample_bytes != d.sample_bytes)
        return set_error(kValidation, "fetch_job: host rows differ in sample size");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    keep_pool();
    auto* j = new lsg_fetch_job();
    j->d = d;
    const uint32_t N = d.N;
    j->nsteps = d.step_end - d.step_begin;
    uint64_t b = 0;
    for (uint64_t g = 0; g < d.step_begin; ++g) b += d.h_node_off[g * (N + 1) + N];
    uint64_t total_rows = 0, max_rows = 0, max_list = 1;
    for (uint64_t g = d.step_begin; g < d.step_end; ++g) {
        const uint32_t* o = d.h_node_off + g * (N + 1);
        for (uint32_t k = d.node_begin; k < d.node_end; ++k)
            max_list = std::max<uint64_t>(max_list, o[k + 1] > o[k] ? o[k + 1] - o[k] : 0);
        if (o[d.node_end] < o[d.node_begin]) {
            delete j;
            return set_error(kValidation, "fetch_job: node offsets not ascending");
        }
        j->base.push_back(b);
        j->rows.push_back(o[d.node_end] - o[d.node_begin]);
        total_rows += j->rows.back();
        max_rows = std::max<uint64_t>(max_rows, j->rows.back());
        b += o[N];
    }
    j->base.push_back(b);
    if (total_rows >= 0xFFFFFFF0ull || b - j->base[0] >= 0xFFFFFFF0ull) {
        delete j;
        return set_error(kCapability, "fetch_job: more than 2^32 items in one job");
    }
    auto fail = [&](int rc) {
        lsg_fetch_job_destroy(j, stream);
        return rc;
    };
    const uint64_t ns = j->nsteps;
    auto alloc = [&](void** p, size_t bytes) { return cudaMallocAsync(p, std::max<size_t>(bytes, 16), st) == cudaSuccess; };
    if (!alloc(reinterpret_cast<void**>(&j->d_base), (ns + 1) * 4) ||
        !alloc(reinterpret_cast<void**>(&j->d_ctl), (6 * ns + 5) * 4) ||
        !alloc(reinterpret_cast<void**>(&j->stats), 32) ||
        !alloc(reinterpret_cast<void**>(&j->mrow), total_rows * 4) ||
        !alloc(reinterpret_cast<void**>(&j->mid), total_rows * 4))
        return fail(set_error(kInternal, "fetch_job: device allocation failed"));
    if (cudaMemsetAsync(j->d_ctl, 0, (6 * ns + 5) * 4, st) != cudaSuccess ||
        cudaMemsetAsync(j->stats, 0, 32, st) != cudaSuccess)
        return fail(cuda_error(cudaGetLastError(), "fetch_job setup"));
    uint32_t* cnt = j->d_ctl + 4 * ns;
    uint32_t* moff = j->d_ctl + 5 * ns;
    if (ns) {
        const uint32_t* noff = d.d_node_off + d.step_begin * (N + 1);
        k_scan_u32<<<1, 1024, 0, st>>>(noff + N, uint32_t(ns), N + 1, j->d_base);  // step bases
        count_launch();
        ListArgs la{d.d_items + j->base[0], d.d_slots + j->base[0], noff, j->d_base, N, d.node_begin, d.node_end,
                    uint32_t(ns), cnt, moff, j->mrow, j->mid, j->stats, d.host ? d.sample_bytes : 0};
        k_miss_list<<<unsigned(ns), 256, 0, st>>>(la, 0);
        count_launch();
        k_scan_u32<<<1, 1024, 0, st>>>(cnt, uint32_t(ns), 1, moff);
        count_launch();
        k_miss_list<<<unsigned(ns), 256, 0, st>>>(la, 1);
        count_launch();
    }
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return fail(cuda_error(e, "fetch_job: miss list"));
    static const bool two_kernels = [] {  // LSG_FETCH_FUSED=0: the hit + misses kernel pair per step
        const char* e = std::getenv("LSG_FETCH_FUSED");
        return e && e[0] == '0';
    }();
    uint32_t P2 = 2;
    while (P2 < max_list) P2 <<= 1;
    j->fused = ns && d.sample_bytes % kFTile == 0 && !two_kernels && P2 <= 16384;
    // LSG_FETCH_SKIP=1: synthesised misses written by the wide k_job_misses after each
    // step's hits. The one-warp-per-CTA step kernel stalled its copies computing 16 MiB
    // payload rows (cfg3), so that was the default above 1 MiB; with a producer warp per
    // CTA the fused kernel is faster for them too (cfg3 3.92-4.01 s vs 4.39 s per job)
    static const int skip_env = [] {
        const char* e = std::getenv("LSG_FETCH_SKIP");
        return e ? std::atoi(e) : 0;
    }();
    j->skip_misses = j->fused && !d.host && skip_env == 1;
    if (j->fused) {
        if (!alloc(reinterpret_cast<void**>(&j->flags), (j->base[ns] - j->base[0]) * 4) ||
            !alloc(reinterpret_cast<void**>(&j->ndefer_d), ns * 4))
            return fail(set_error(kInternal, "fetch_job: device allocation failed"));
        const size_t smem = size_t(3) * P2 * 4;
        static std::atomic<uint64_t> attr_done{0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_done.load() & (1ull << (dev & 63)))) {
            cudaFuncSetAttribute(k_row_flags, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 16384 * 4);
            cudaFuncSetAttribute(k_fetch_fused<kFStages, kFLag, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kFTile * kFStages);
            cudaFuncSetAttribute(k_fetch_fused<kFStages, kFLag, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kFTile * kFStages);
            attr_done.fetch_or(1ull << (dev & 63));
        }
        FlagArgs fa{d.d_slots + j->base[0], d.d_node_off + d.step_begin * (N + 1), j->d_base, moff, N,
                    d.node_begin, d.node_end, P2, j->flags, j->ndefer_d};
        k_row_flags<<<unsigned(ns), 256, smem, st>>>(fa);
        count_launch();
        if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return fail(cuda_error(e, "k_row_flags"));
        // the host needs the steps with deferred slot writes (one read per job)
        void* hb = pinned_bounce(ns * 4);
        if (!hb) return fail(set_error(kInternal, "fetch_job: pinned bounce buffer"));
        if (cudaMemcpyAsync(hb, j->ndefer_d, ns * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(cuda_error(cudaGetLastError(), "fetch_job: deferred counts"));
        j->ndefer.assign(static_cast<uint32_t*>(hb), static_cast<uint32_t*>(hb) + ns);
        {  // their list, for the fused kernel's deferred-fill phases
            // ptiles [2ns] | doff [ns+1], uploaded together; ptiles also seeds the
            // per-phase remaining-tile counters (d_ctl's done region)
            const uint64_t tpr = d.sample_bytes / kFTile;
            std::vector<uint32_t> up(3 * ns + 1, 0);
            for (uint64_t g = 0; g < ns; ++g) {
                up[2 * g] = uint32_t(j->rows[g] * tpr);
                up[2 * g + 1] = j->skip_misses ? 0u : uint32_t(j->ndefer[g] * tpr);
                up[2 * ns + g + 1] = up[2 * ns + g] + j->ndefer[g];
            }
            if (!alloc(reinterpret_cast<void**>(&j->ptiles), up.size() * 4) ||
                !alloc(reinterpret_cast<void**>(&j->drow), size_t(up[3 * ns]) * 4))
                return fail(set_error(kInternal, "fetch_job: device allocation failed"));
            j->doff = j->ptiles + 2 * ns;
            void* hd = pinned_bounce(up.size() * 4);  // (a pageable copy can wait for other streams' kernels)
            if (!hd) return fail(set_error(kInternal, "fetch_job: pinned bounce buffer"));
            std::memcpy(hd, up.data(), up.size() * 4);
            if (cudaMemcpyAsync(j->ptiles, hd, up.size() * 4, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                cudaMemcpyAsync(j->d_ctl + 2 * ns, j->ptiles, 2 * ns * 4, cudaMemcpyDeviceToDevice, st) !=
                    cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess)
                return fail(cuda_error(cudaGetLastError(), "fetch_job: deferred offsets"));
            j->ndefer_rows = up[3 * ns];
            // steps alternate between the caller's batch tensors and these (one more batch
            // per local rank: 128 MiB at cfg2, 256 MiB at cfg3), where a step is short
            // enough for its boundary to matter (<= 512 MiB of rows; fetch alone at one
            // rank, cfg2 44.6 -> 42.2 us per step, cfg3 47.7 -> 46.4; at 8 ranks per GPU
            // (1 GiB per step) no gain, and a GiB per job in flight is HBM the e2e miss
            // ring needs). LSG_FETCH_PINGPONG=0/1 forces it.
            static const int pp_env = [] {
                const char* e = std::getenv("LSG_FETCH_PINGPONG");
                return e ? std::atoi(e) : -1;
            }();
            const bool pp = pp_env >= 0 ? pp_env == 1 : max_rows * d.sample_bytes <= (uint64_t(512) << 20);
            if (ns >= 2 && pp) {
                j->srows = uint32_t((max_list + 63) / 64 * 64);  // (a stable size class across jobs for the pool)
                if (!alloc(reinterpret_cast<void**>(&j->scratch),
                           size_t(d.node_end - d.node_begin) * j->srows * d.sample_bytes))
                    return fail(set_error(kInternal, "fetch_job: device allocation failed (scratch batch rows)"));
            }
            if (up[3 * ns]) {
                k_defer_list<<<unsigned(ns), 256, 0, st>>>(fa, j->doff, j->drow);
                count_launch();
                if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return fail(cuda_error(e, "k_defer_list"));
            }
        }
        if (std::getenv("LSG_FETCH_VERBOSE")) {
            uint64_t steps = 0, rows = 0;
            for (uint32_t v : j->ndefer) steps += v != 0, rows += v;
            fprintf(stderr, "fetch_job: %llu steps, %llu with deferred slot writes (%llu rows)\n",
                    (unsigned long long)ns, (unsigned long long)steps, (unsigned long long)rows);
        }
    }
    cudaEventCreateWithFlags(&j->listed, cudaEventDisableTiming);
    cudaEventRecord(j->listed, st);
    if (d.host && ns && total_rows) {
        j->seq0 = j->d_ctl + 6 * ns + 2;
        if (lsg_miss_stream* ms = d.misses) {  // the shared ring: reserve the job's sequence numbers
            if (ms->sample_bytes != d.sample_bytes)
                return fail(set_error(kValidation, "fetch_job: miss stream differs in sample size"));
            if (max_rows > ms->R)
                return fail(set_error(kCapability, "fetch_job: a step has more rows than the miss stream's ring"));
            j->R = ms->R;
            j->ring = ms->ring;
            j->ready = ms->words;
            j->consumed = ms->words + ms->R + 1;
            j->pf_done = ms->words + ms->R + 2;
            if (ms->any) LSG_CUDA(cudaStreamWaitEvent(st, ms->reserved, 0));  // jobs reserve in creation order
            k_reserve<<<1, 1, 0, st>>>(moff + ns, ms->words + ms->R, j->seq0);
            count_launch();
            if (!ms->reserved) cudaEventCreateWithFlags(&ms->reserved, cudaEventDisableTiming);
            cudaEventRecord(ms->reserved, st);
            ms->any = true;
        } else {
            // own ring: at least the largest step (a step's misses are
            // consumed together), at most ring_bytes beyond that
            const uint64_t want = d.ring_bytes ? d.ring_bytes : (uint64_t(2) << 30);
            const uint64_t R = std::min<uint64_t>(total_rows, std::max<uint64_t>(max_rows, want / d.sample_bytes));
            j->R = uint32_t(R);
            j->own_ring = true;
            if (!alloc(reinterpret_cast<void**>(&j->ring), R * d.sample_bytes) ||
                !alloc(reinterpret_cast<void**>(&j->ready), R * 4))
                return fail(set_error(kInternal, "fetch_job: ring allocation failed"));
            if (cudaMemsetAsync(j->ready, 0, R * 4, st) != cudaSuccess)
                return fail(cuda_error(cudaGetLastError(), "fetch_job ring"));
            j->consumed = j->d_ctl + 6 * ns + 1;
            j->pf_done = j->d_ctl + 6 * ns + 3;
        }
        j->resident = resident_acquire(&j->resident_idx);
        if (!j->resident) return fail(set_error(kInternal, "fetch_job: no residency counter"));
        unsigned int* dres = nullptr;
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&dres), j->resident, 0);
        PrefetchArgs pa{d.host->dev, j->mid, moff + ns, d.sample_bytes, j->ring, j->R, j->ready,
                        j->consumed, dres, j->seq0, j->pf_done, j->d_ctl + 6 * ns + 4};
        static const bool lsu = [] {  // LSG_PF_LSU=1: 128-bit loads instead of TMA
            const char* e = std::getenv("LSG_PF_LSU");
            return e && e[0] == '1';
        }();
        const bool tma = d.sample_bytes % kPfTile == 0 && !lsu;
        if (tma) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_miss_prefetch_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kPfTile * kPfStages);
                attr = true;
            }
            k_miss_prefetch_tma<<<kPfCtas, 32, kPfTile * kPfStages, st>>>(pa);
        } else {
            k_miss_prefetch_lsu<<<kPfCtas, 256, 0, st>>>(pa);
        }
        count_launch();
        if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return fail(cuda_error(e, "k_miss_prefetch"));
        cudaEventCreateWithFlags(&j->prefetched, cudaEventDisableTiming);
        cudaEventRecord(j->prefetched, st);
        j->prefetching = true;
        j->prep = st;
        // the consumers spin on ring rows: return only once every prefetch
        // CTA is resident (it then runs to completion beside anything)
        const auto t0 = std::chrono::steady_clock::now();
        while (__atomic_load_n(j->resident, __ATOMIC_ACQUIRE) < unsigned(kPfCtas)) {
            if (cudaStreamQuery(st) == cudaSuccess) break;  // finished already (tiny job)
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
                return fail(set_error(kInternal, "fetch_job: the miss prefetcher never became resident"));
            std::this_thread::yield();
        }
    }
    *out = j;
    return kOk;
}

int lsg_fetch_job_run(lsg_fetch_job* j, void* stream) {
    if (!j) return set_error(kValidation, "fetch_job: null job");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (j->prefetching && st == j->prep)
        return set_error(kValidation, "fetch_job: run on the stream the miss prefetcher holds (it would wait for itself)");
    const lsg_fetch_job_desc& d = j->d;
    const uint32_t N = d.N, ns = uint32_t(j->nsteps);
    if (j->listed) LSG_CUDA(cudaStreamWaitEvent(st, j->listed, 0));  // NOT the prefetcher: it needs these kernels
    uint32_t* claims = j->d_ctl;      // [2ns]: per step, or per phase (fused)
    uint32_t* done = j->d_ctl + 2 * ns;
    uint32_t* moff = j->d_ctl + 5 * ns;
    if (j->fused) {
        // one persistent launch per run of steps (and, with LSG_FETCH_SKIP=1,
        // one per step followed by k_job_misses)
        FusedStep fs{d.d_items + j->base[0], d.d_slots + j->base[0], j->flags,
                     d.d_node_off + d.step_begin * (N + 1), j->d_base, N,
                     reinterpret_cast<unsigned char* const*>(d.d_bufs),
                     reinterpret_cast<unsigned char* const*>(d.d_outs), d.node_begin, d.node_end, d.sample_bytes,
                     d.fill_seed, claims, done, j->ptiles, j->ndefer_d, j->doff, j->drow, j->ring, j->R, j->ready,
                     j->seq0, moff, j->consumed, 0, 0, ns, j->scratch, j->srows, j->skip_misses ? 1 : 0};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        const int npdl = pdl_on(0) ? 1 : 0;
        // a launch holds every SM it runs on, so launches are cut every ~1 GiB of tiles
        // (~0.3 ms): the plan loop and replay kernels on their high-priority streams get
        // SMs at the next cut (LSG_FETCH_SEG_TILES overrides)
        static const uint64_t seg_tiles = [] {
            const char* e = std::getenv("LSG_FETCH_SEG_TILES");
            return e ? std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) : (uint64_t(1) << 17);
        }();
        // stages per CTA x CTAs per SM (LSG_FETCH_S / LSG_FETCH_CPS: 5x5, 6x4, 12x2). At one rank
        // per GPU more, shallower pipelines won (43.3 us per step at 6x4 vs 44.9 at 12x2):
        // a step's stores wait for the whole previous step, so the slowest CTA's queue of
        // loaded tiles sets the step boundary
        static const int nst = [] {
            const char* e = std::getenv("LSG_FETCH_S");
            const int v = e ? std::atoi(e) : kFStages;
            return v == 5 || v == 12 ? v : kFStages;
        }();
        static const unsigned cps = [] {
            const char* e = std::getenv("LSG_FETCH_CPS");
            return e ? unsigned(std::max(1, std::atoi(e))) : kFCtasPerSm;
        }();
        // the grid leaves 8 SMs' worth of CTA slots to the planner and replay streams: their
        // many short launches (the next-use pass: 100 per job) otherwise wait for the fetch's
        // launch cuts. At one rank per GPU beside a fetch: replay 195 -> 157 ms, job period
        // 334 -> 295 ms; the fetch itself unchanged (HBM-bound at 140 SMs). LSG_FETCH_RESERVE_SMS
        static const unsigned fetch_sms = [] {
            const char* e = std::getenv("LSG_FETCH_RESERVE_SMS");
            const int r = e ? std::atoi(e) : 8;
            return unsigned(std::max(1, 148 - std::max(0, r)));
        }();
        const bool fills = j->ndefer_rows > 0;  // deferred-fill phases needed
        auto kern = nst == 5    ? (fills ? k_fetch_fused<5, 2, 2> : k_fetch_fused<5, 2, 1>)
                    : nst == 12 ? (fills ? k_fetch_fused<12, 3, 2> : k_fetch_fused<12, 3, 1>)
                                : (fills ? k_fetch_fused<kFStages, kFLag, 2> : k_fetch_fused<kFStages, kFLag, 1>);
        static std::atomic<uint32_t> vattr{0};
        if (!(vattr.fetch_or(1u) & 1u)) {
            for (auto kf : {k_fetch_fused<5, 2, 1>, k_fetch_fused<5, 2, 2>})
                cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, kFTile * 5);
            for (auto kf : {k_fetch_fused<12, 3, 1>, k_fetch_fused<12, 3, 2>})
                cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, kFTile * 12);
        }
        for (uint32_t ga = 0; ga < ns;) {
            uint32_t gb = ga + 1;
            const uint64_t tpr = d.sample_bytes / kFTile;
            uint64_t tiles = j->rows[ga] * tpr;
            while (gb < ns && !j->skip_misses && tiles + j->rows[gb] * tpr <= seg_tiles)
                tiles += j->rows[gb++] * tpr;
            fs.gA = ga;
            fs.gB = gb;
            if (tiles && d.node_begin != d.node_end) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(unsigned(std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(fetch_sms) * cps))));
                cfg.blockDim = dim3(64);
                cfg.dynamicSmemBytes = size_t(kFTile) * nst;
                cfg.stream = st;
                cfg.attrs = attr;
                cfg.numAttrs = npdl;
                LSG_CUDA(cudaLaunchKernelEx(&cfg, kern, fs));
                LSG_LAUNCH_CHECK("k_fetch_fused");
            }
            const uint32_t gl = gb - 1;  // the segment's last step
            const uint64_t g = d.step_begin + gl;
            if (j->skip_misses && j->rows[gl]) {  // large synthesised rows: a wide kernel writes the misses
                StepFetch f{};
                f.items = d.d_items + j->base[gl];
                f.slots = d.d_slots + j->base[gl];
                f.node_off = d.d_node_off + g * (N + 1);
                f.bufs = reinterpret_cast<uint4* const*>(d.d_bufs);
                f.outs = reinterpret_cast<uint4* const*>(d.d_outs);
                f.k0 = d.node_begin;
                f.k1 = d.node_end;
                f.vec_per_row = d.sample_bytes / 16;
                f.tiles_per_row = (f.vec_per_row + 1023) / 1024;
                f.seed = d.fill_seed;
                MissArgs ma{f, moff, gl, j->mrow, nullptr, 0, nullptr, nullptr, done, nullptr};
                const dim3 grid(unsigned(std::min<uint64_t>(std::max<uint64_t>(f.vec_per_row / 4096, 1), 64)),
                                unsigned(std::min<uint64_t>(j->rows[gl], 148)));
                k_job_misses<<<grid, 256, 0, st>>>(ma);
                LSG_LAUNCH_CHECK("k_job_misses");
            }
            ga = gb;
        }
        return kOk;
    }
    for (uint32_t gi = 0; gi < ns; ++gi) {
        const uint64_t g = d.step_begin + gi;
        const uint64_t b = j->base[gi];
        StepFetch f{};
        f.items = d.d_items + b;
        f.slots = d.d_slots + b;
        f.node_off = d.d_node_off + g * (N + 1);
        f.bufs = reinterpret_cast<uint4* const*>(d.d_bufs);
        f.outs = reinterpret_cast<uint4* const*>(d.d_outs);
        f.k0 = d.node_begin;
        f.k1 = d.node_end;
        f.vec_per_row = d.sample_bytes / 16;
        f.tiles_per_row = (f.vec_per_row + 1023) / 1024;
        f.seed = d.fill_seed;
        f.claim = claims + gi;
        const uint64_t rows = j->rows[gi];
        if (rows == 0 || d.node_begin == d.node_end) continue;
        if (int rc = launch_fetch_hits(f, rows, d.sample_bytes, st, nullptr)) return rc;
        MissArgs ma{f, moff, gi, j->mrow, j->ring, j->R, j->ready, j->consumed, done, j->seq0};
        const dim3 grid(unsigned(std::min<uint64_t>(std::max<uint64_t>(f.vec_per_row / 4096, 1), 64)),
                        unsigned(std::min<uint64_t>(rows, 148)));
        k_job_misses<<<grid, 256, 0, st>>>(ma);
        LSG_LAUNCH_CHECK("k_job_misses");
    }
    return kOk;
}

int lsg_fetch_job_stats(lsg_fetch_job* j, uint64_t* h_stats, void* stream) {
    if (!j || !h_stats) return set_error(kValidation, "fetch_job: null argument");
    unsigned long long s[4] = {};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    LSG_CUDA(cudaMemcpyAsync(s, j->stats, 32, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < 4; ++i) h_stats[i] = s[i];
    return kOk;
}

void lsg_fetch_job_destroy(lsg_fetch_job* j, void* stream) {
    if (!j) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (j->prefetching) cudaStreamWaitEvent(st, j->prefetched, 0);
    for (void* p : {static_cast<void*>(j->d_base), static_cast<void*>(j->d_ctl), static_cast<void*>(j->mrow),
                    static_cast<void*>(j->mid), static_cast<void*>(j->stats)})
        if (p) cudaFreeAsync(p, st);
    if (j->flags) cudaFreeAsync(j->flags, st);
    if (j->ndefer_d) cudaFreeAsync(j->ndefer_d, st);
    if (j->ptiles) cudaFreeAsync(j->ptiles, st);
    if (j->scratch) cudaFreeAsync(j->scratch, st);
    if (j->drow) cudaFreeAsync(j->drow, st);
    if (j->own_ring) {
        if (j->ring) cudaFreeAsync(j->ring, st);
        if (j->ready) cudaFreeAsync(j->ready, st);
    }
    if (j->prefetched) cudaEventDestroy(j->prefetched);
    if (j->listed) cudaEventDestroy(j->listed);
    // the counter is written only when the prefetcher starts, which create
    // waited for: it can be recycled now
    if (j->resident_idx >= 0) resident_release(j->resident_idx);
    delete j;
}

int lsg_miss_stream_create(uint64_t sample_bytes, uint64_t ring_bytes, lsg_miss_stream** out) {
    if (!out || sample_bytes == 0 || sample_bytes % 16)
        return set_error(kValidation, "miss_stream: sample_bytes must be a positive multiple of 16");
    const uint64_t R = ring_bytes / sample_bytes;
    if (R == 0 || R >= 0x7FFFFFFFull) return set_error(kValidation, "miss_stream: ring_bytes out of range");
    auto* ms = new lsg_miss_stream();
    ms->R = uint32_t(R);
    ms->sample_bytes = sample_bytes;
    if (cudaMalloc(&ms->ring, R * sample_bytes) != cudaSuccess ||
        cudaMalloc(&ms->words, (R + 3) * 4) != cudaSuccess || cudaMemset(ms->words, 0, (R + 3) * 4) != cudaSuccess) {
        cudaGetLastError();
        lsg_miss_stream_destroy(ms);
        return set_error(kInternal, "miss_stream: ring allocation failed");
    }
    *out = ms;
    return kOk;
}

void lsg_miss_stream_destroy(lsg_miss_stream* ms) {
    if (!ms) return;
    if (ms->ring) cudaFree(ms->ring);
    if (ms->words) cudaFree(ms->words);
    if (ms->reserved) cudaEventDestroy(ms->reserved);
    delete ms;
}

}  // extern "C"

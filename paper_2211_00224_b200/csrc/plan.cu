// plan.cu — K5 (step-granular next use), sorted step batches, and K6: the
// persistent planner step loop of plan_schedule (pipeline.cpp:32-120):
// per step, locality remap (locality.cpp:7-42) or slicing (:57-73), fetch
// balancing (balance.cpp:10-39) and the clairvoyant buffer advance
// (buffer.cpp:37-46) for every node, bit-exact.
//
// The step recurrence (6,400 dependent steps at config 2) runs inside ONE
// persistent CTA: no per-step launches, no host round trips; all state stays
// in HBM/L2 (keys, holder masks, bucket bitmaps) and shared memory (the
// current batch). Per step:
//
//  A  load batch ids, next-use keys and N-bit holder masks; classify items
//     as no-holder / single-holder / multi-holder; per-warp ranks of singles
//     with __match_any_sync (order-preserving, no atomics).
//  B  per-node exclusive scan of the per-warp counts (warp k scans node k).
//  C  exact S_k(j) (singles of node k before j) for every multi item.
//  D  ONE warp resolves the multi-holder items serially, lanes = nodes:
//     c_k = min(b, S_k(j) + M_k); argmin over holders with c_k < b,
//     ties -> lowest k (__reduce_min_sync on (c<<5)|k).  This is the only
//     serial part of the remap; singles then need no serial pass:
//     single j (holder k) is a hit iff S_k(j) + M_k(<j) < b.
//  E/F fetches fill nodes in ascending order up to b (prefix over free slots).
//  G  balance is simulated on the N fetch counts only (thread 0); donors and
//     recipients are disjoint, donor d's i-th move gives its i-th largest
//     fetch id, recipients append in move order.
//  H  final node lists -> plan output (ids | hit tag), offsets, fetch counts.
//  I  buffer advance, nodes in parallel. Within a (node, step) an item is a
//     hit iff it was resident at step start (every miss inserts a key beyond
//     the current step, so current-step residents are never the eviction
//     maximum). Runs of hits re-key; runs of misses insert then drop the
//     (size - C)+ largest (key, id): streaming "keep the C smallest".
//     Eviction walks a per-node "maybe non-empty" bucket bitmap over future
//     steps (key = next-use step) and, inside bucket g', the step-g' batch in
//     descending id order testing key == g' (the reference's tie rule: equal
//     keys evict the larger id first). kNeverUsed keys live in an exact
//     per-node id bitmap scanned from the top.
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"

namespace lsg {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kMaxN = 32;
constexpr uint32_t kOvN = 8;  // the overlapped loop's node limit
constexpr uint32_t kOvW = 4096 / 32;  // words of a step bitmap at the overlapped loop's largest B
constexpr uint32_t kDWarps = 4;  // its team D: one warp per scheduler of CTA 2, one per step mod 4
constexpr uint32_t kMaxSmemB = 8192;   // per-item arrays in shared memory up to here
constexpr uint32_t kMaxB = 16384;      // then in L2-resident global scratch
constexpr uint32_t kFetch = 0xFFFFFFFFu;
constexpr uint32_t kDmv = 32;       // G: moves per donor kept in shared memory
constexpr uint32_t kNotMoved = 0xFFFFFFFFu;
constexpr uint32_t kWinWords = 40;  // I1 bucket-bit window (covers 2S <= 1216 steps)
constexpr uint32_t kPk16B = 2048;   // D8 with 16-bit packed keys below this local batch

// ----------------------------------------------------------------- K5 ----
// nu for the access of x at execution epoch i, position pos: the first
// later execution epoch j whose kept prefix contains x gives
// j*S + floor(inv/B) (the global step of its next use), else kNever.
__global__ void k_nextuse(const uint32_t* __restrict__ trace, const uint32_t* __restrict__ order,
                          const uint32_t* __restrict__ inv, uint32_t E, uint32_t keep, uint32_t D,
                          uint32_t S, uint32_t B, uint32_t* __restrict__ nu) {
    const uint32_t i = blockIdx.y;
    const uint32_t e = order[i];
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < keep; pos += gridDim.x * blockDim.x) {
        const uint32_t x = trace[size_t(e) * keep + pos];
        uint32_t r = kNever;
        for (uint32_t j = i + 1; j < E; ++j) {
            const uint32_t p2 = inv[size_t(order[j]) * D + x];
            if (p2 != kNone) {
                r = j * S + p2 / B;
                break;
            }
        }
        nu[size_t(i) * keep + pos] = r;
    }
}

// Each step's batch sorted by descending id (bucket enumeration order).
__global__ void __launch_bounds__(1024) k_sort_batches(const uint32_t* __restrict__ trace,
                                                       const uint32_t* __restrict__ order,
                                                       uint32_t keep, uint32_t S, uint32_t B,
                                                       uint32_t P2, uint32_t* __restrict__ sb) {
    extern __shared__ uint32_t sk[];
    const uint32_t g = blockIdx.x, i = g / S, t = g % S;
    const uint32_t lo = t * B, len = min(B, keep - lo);
    const uint32_t* row = trace + size_t(order[i]) * keep + lo;
    for (uint32_t r = threadIdx.x; r < P2; r += blockDim.x) sk[r] = r < len ? row[r] : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t size = 2; size <= P2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t r = threadIdx.x; r < P2 / 2; r += blockDim.x) {
                const uint32_t a = 2 * stride * (r / stride) + (r % stride), c = a + stride;
                const bool up = (a & size) == 0;
                const uint32_t x = sk[a], y = sk[c];
                if ((x > y) == up) { sk[a] = y; sk[c] = x; }
            }
            __syncthreads();
        }
    }
    uint32_t* out = sb + size_t(i) * keep + lo;
    for (uint32_t r = threadIdx.x; r < len; r += blockDim.x) out[r] = sk[len - 1 - r];
}

// Rank of x inside the descending-sorted batch of its next-use step (binary
// search of the step's sorted row); kNone for kNeverUsed. The eviction buckets
// index residents by this rank, so rank order == the reference's tie order.
__global__ void k_nextrank(const uint32_t* __restrict__ trace, const uint32_t* __restrict__ order,
                           const uint32_t* __restrict__ nu, const uint32_t* __restrict__ sb,
                           uint32_t E, uint32_t keep, uint32_t S, uint32_t B,
                           uint32_t* __restrict__ nr) {
    const uint32_t i = blockIdx.y;
    const uint32_t* row = trace + size_t(order[i]) * keep;
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < keep; pos += gridDim.x * blockDim.x) {
        const uint32_t v = nu[size_t(i) * keep + pos];
        uint32_t r = kNever;
        if (v != kNever) {
            const uint32_t x = row[pos];
            const uint32_t gi = v / S, gt = v % S, lo = gt * B, blen = min(B, keep - lo);
            const uint32_t* cand = sb + size_t(gi) * keep + lo;
            uint32_t a0 = 0, a1 = blen;  // first index with cand[idx] <= x (descending)
            while (a0 < a1) {
                const uint32_t mid = (a0 + a1) >> 1;
                if (cand[mid] > x) a0 = mid + 1; else a1 = mid;
            }
            r = v * B + a0;  // packed resident key: next-use step, rank
        }
        nr[size_t(i) * keep + pos] = r;
    }
}

// ----------------------------------------------------------------- K6 ----
struct LoopArgs {
    uint32_t D, N, b, B, S, E, keep, T, C;
    int remap, balance;
    uint32_t nzw;                    // words per node in the bucket bitmap
    uint32_t infw;                   // words per node in the never-used bitmap
    const uint32_t* trace;           // [E][keep]
    const uint32_t* order;           // [E]
    const uint32_t* nu;              // [E*keep] execution order
    const uint32_t* sb;              // [E*keep] execution order, desc per step
    const uint32_t* nr;              // [E*keep] packed next-use key: step * B + rank in sb, or kNever
    unsigned long long bdiv;         // ceil(2^64 / B) (B >= 2): step = umul64hi(key, bdiv)
    uint32_t* bm;                    // [N][T][BW] bucket membership bitmaps over ranks
    uint32_t BW;                     // words per bucket bitmap (ceil(B/32))
    uint32_t* key;                   // [N][D] next-use step * B + rank, kNever, or kNone
    uint32_t* hm;                    // [D] holder masks
    uint32_t* nz;                    // [N][nzw]
    uint32_t* infbm;                 // [N][infw]
    uint32_t* smul;                  // [B][N] scratch: warp-local S_k(j)
    uint32_t* sx;                    // [B][N] scratch: exact S_k(j) by multi index
    uint32_t* dmoves;                // [N][B] donor's i-th move (r | q<<8) beyond kDmv
    uint32_t* items;                 // [E*keep] output
    uint32_t* node_off;              // [T][N+1] output
    uint32_t* fb;                    // [T][N] output (may be null)
    uint32_t* fa;                    // [T][N] output (may be null)
    uint32_t* status;
    uint32_t* gitems;                // [6][B] per-item arrays when they do not fit smem
    unsigned long long* prof;        // [8] per-phase cycles (LSG_PROFILE) or null
    int dbg_skip;                    // timing experiments only (LSG_DEBUG_SKIP)
    uint32_t* nb;                    // [3][D] overlapped loop: per batch mod 3, the latest batch each id was
                                     // classified in, or null
};

struct Shared {
    uint32_t* sx;     // [B] ids
    uint32_t* snu;    // [B] packed next-use keys (step * B + rank, kNever)
    uint32_t* smask;  // [B] holder masks at step start
    uint32_t* sinfo;  // [B] per-item scratch
    uint32_t* pre;    // [B] pre-balance lists, node k at k*b (j | hit tag)
    uint32_t* fin;    // [B] final lists (j | k<<16 | hit tag)
};

struct Small {
    uint32_t wcnt[kWarps][kMaxN];   // per-warp single counts -> bases
    uint32_t cm[kWarps][kMaxN];     // per-chunk single lanes per holder
    uint32_t wmul[kWarps];          // per-warp multi counts -> bases
    uint32_t wfet[kWarps];          // per-warp fetch counts -> bases
    uint32_t tot[kMaxN];            // singles per node
    uint32_t mtot[kMaxN];           // multi assigned per node
    uint32_t size[kMaxN];           // hits per node (list prefix)
    uint32_t free_pre[kMaxN + 1];   // prefix of free capacity
    uint32_t lenk[kMaxN];           // pre-balance list length
    uint32_t fcnt[kMaxN];           // fetches before balance
    uint32_t outk[kMaxN], ink[kMaxN];
    uint32_t noff[kMaxN + 1];       // final offsets
    uint32_t bsize[kMaxN];          // buffer occupancy
    uint32_t top[kMaxN];            // bucket upper bound
    uint32_t inftop[kMaxN];         // never-used bitmap upper word bound
    uint32_t infcnt[kMaxN];         // never-used residents
    uint32_t nmulti, nfetch, nmoves;
    alignas(16) uint32_t stg[2][32][kMaxN];  // D: staged S_k(j) of 32 multi items
    uint32_t dmv[kMaxN][kDmv];      // G: donor's i-th move (r | q<<8), i < kDmv
    uint32_t rq[kMaxN];             // G: recipient of each rank in a round
    uint32_t win_base;              // I1: first bucket word of the window
    uint32_t win[kMaxN][kWinWords]; // I1: bucket bits aggregated per step
    uint32_t stamp, conflict, conflict2, conflict3;  // (overlapped loop only; unused here)
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// buffer.cpp:37-41 (re-key) / :42-46 (insert) without the eviction: key
// update plus the bucket / never-used summaries.
__device__ __forceinline__ uint32_t key_step(const LoopArgs& a, uint32_t pk) {
    return a.B == 1 ? pk : uint32_t(__umul64hi(pk, a.bdiv));
}

template <class SM>
__device__ __forceinline__ void set_key(const LoopArgs& a, SM& sm, uint32_t k, uint32_t x, uint32_t pk) {
    // one word per resident: (next-use step, rank in that step's sorted batch)
    a.key[size_t(k) * a.D + x] = pk;
    const uint32_t nu = pk == kNever ? kNever : key_step(a, pk), rank = pk - nu * a.B;
    if (nu != kNever)
        red_or(&a.bm[(size_t(k) * a.T + nu) * a.BW + (rank >> 5)], 1u << (rank & 31));
    if (nu == kNever) {
        red_or(&a.infbm[size_t(k) * a.infw + (x >> 5)], 1u << (x & 31));
        atomicAdd(&sm.infcnt[k], 1u);
        atomicMax(&sm.inftop[k], x >> 5);
    } else {
        red_or(&a.nz[size_t(k) * a.nzw + (nu >> 5)], 1u << (nu & 31));
        atomicMax(&sm.top[k], nu);
    }
}

// with the overlapped loop (a.nb), a holder mask that changes for an id of
// one of the next three, already classified batches (sm.stamp = g+1, g+2, g+3)
// invalidates that classification. The classifier stamps, fences, then reads
// masks; the advance changes a mask, fences, then reads the stamps: one of
// the two sees the other.
template <class SM>
__device__ __forceinline__ void nb_check(const LoopArgs& a, SM& sm, uint32_t x) {
    __threadfence();
    const uint32_t s1 = sm.stamp, s2 = s1 + 1, s3 = s1 + 2;
    if (__ldcg(&a.nb[size_t(s1 % 3) * a.D + x]) == s1) sm.conflict = 1;
    if (__ldcg(&a.nb[size_t(s2 % 3) * a.D + x]) == s2) sm.conflict2 = 1;
    if (__ldcg(&a.nb[size_t(s3 % 3) * a.D + x]) == s3) sm.conflict3 = 1;
}
template <class SM>
__device__ __forceinline__ void drop(const LoopArgs& a, SM& sm, uint32_t k, uint32_t x) {
    a.key[size_t(k) * a.D + x] = kNone;
    red_and(&a.hm[x], ~(1u << k));
    if (a.nb) nb_check(a, sm, x);
}

// Remove the `need` largest (key, id) residents of node k. Whole warp.
template <class SM>
__device__ void evict_walk(const LoopArgs& a, SM& sm, uint32_t k, uint32_t need, uint32_t lane,
                           uint32_t g) {
    const uint32_t lt = lanemask_lt();
    while (need > 0) {
        if (sm.infcnt[k] > 0) {  // kNeverUsed bucket: ids descending
            uint32_t* bm = a.infbm + size_t(k) * a.infw;
            int32_t wi = int32_t(sm.inftop[k]);
            bool found = false;
            while (wi >= 0 && !found) {
                const int32_t myw = wi - int32_t(lane);
                const uint32_t v = myw >= 0 ? __ldcg(&bm[myw]) : 0u;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v != 0);
                if (bal) {
                    const uint32_t src = __ffs(bal) - 1;
                    const int32_t hw = wi - int32_t(src);
                    uint32_t word = __shfl_sync(0xFFFFFFFFu, v, src);
                    // take bits from the top of this word
                    while (word && need > 0) {
                        const uint32_t bit = 31 - __clz(word);
                        word &= ~(1u << bit);
                        const uint32_t x = uint32_t(hw) * 32 + bit;
                        if (lane == 0) {
                            drop(a, sm, k, x);
                            atomicAnd(&bm[hw], ~(1u << bit));
                        }
                        --need;
                        if (lane == 0) { sm.infcnt[k] -= 1; sm.bsize[k] -= 1; }
                    }
                    if (lane == 0) sm.inftop[k] = uint32_t(hw);
                    found = true;
                } else {
                    wi -= 32;
                }
                __syncwarp();
            }
            if (!found) {  // bookkeeping says never-used residents exist
                if (lane == 0) { atomicOr(a.status, 2u); sm.infcnt[k] = 0; }
                __syncwarp();
            }
            continue;
        }
        // highest possibly non-empty finite bucket
        uint32_t* nzk = a.nz + size_t(k) * a.nzw;
        int32_t wi = int32_t(sm.top[k] >> 5);
        int32_t beta = -1;
        while (wi >= 0) {
            const int32_t myw = wi - int32_t(lane);
            const uint32_t v = myw >= 0 ? __ldcg(&nzk[myw]) : 0u;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v != 0);
            if (bal) {
                const uint32_t src = __ffs(bal) - 1;
                const uint32_t word = __shfl_sync(0xFFFFFFFFu, v, src);
                beta = (wi - int32_t(src)) * 32 + (31 - __clz(word));
                break;
            }
            wi -= 32;
        }
        if (beta < 0) {
            if (lane == 0) atomicOr(a.status, 4u);
            return;
        }
        // take members of bucket beta in rank order (rank 0 = largest id):
        // future buckets are exact (an entry goes stale only once its step is
        // reached, and evictions clear their own bits); a past bucket (only
        // reached when nothing has a future use) is validated against key/rank.
        const uint32_t gi = uint32_t(beta) / a.S, gt = uint32_t(beta) % a.S;
        const uint32_t lo = gt * a.B, blen = min(a.B, a.keep - lo);
        const uint32_t* cand = a.sb + size_t(gi) * a.keep + lo;
        uint32_t* bw = a.bm + (size_t(k) * a.T + uint32_t(beta)) * a.BW;
        const bool past = uint32_t(beta) <= g;
        const uint32_t nwords = (blen + 31) >> 5;
        bool left = false;  // members remain in the scanned words
        uint32_t w0 = 0;
        for (; w0 < nwords && need > 0; w0 += 32) {
            const uint32_t wi2 = w0 + lane;
            uint32_t word = wi2 < nwords ? __ldcg(&bw[wi2]) : 0u;
            if (past && word) {  // drop stale bits
                uint32_t m = word;
                while (m) {
                    const uint32_t bit = __ffs(m) - 1;
                    m &= m - 1;
                    const uint32_t x = cand[wi2 * 32 + bit];
                    if (__ldcg(&a.key[size_t(k) * a.D + x]) != uint32_t(beta) * a.B + wi2 * 32 + bit)
                        word &= ~(1u << bit);
                }
            }
            const uint32_t cnt = __popc(word);
            uint32_t inc = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (lane >= uint32_t(d)) inc += o;
            }
            const uint32_t before = inc - cnt, total = __shfl_sync(0xFFFFFFFFu, inc, 31);
            const uint32_t take = before < need ? min(cnt, need - before) : 0u;
            uint32_t rest = word;
            for (uint32_t t2 = 0; t2 < take; ++t2) {
                const uint32_t bit = __ffs(rest) - 1;
                rest &= rest - 1;
                drop(a, sm, k, cand[wi2 * 32 + bit]);
            }
            if (wi2 < nwords && (rest != word || past)) bw[wi2] = rest;
            left = left || (__ballot_sync(0xFFFFFFFFu, rest != 0) != 0);
            const uint32_t took = min(total, need);
            need -= took;
            if (lane == 0) sm.bsize[k] -= took;
        }
        __syncwarp();
        // every word scanned and nothing left: the bucket is empty now
        if (w0 >= nwords && !left && lane == 0) atomicAnd(&nzk[beta >> 5], ~(1u << (beta & 31)));
        if (lane == 0) sm.top[k] = uint32_t(beta);
        __syncwarp();
    }
}

// kD8: N <= 8 (register-only multi-holder pass); the other path is not
// instantiated, which keeps the step's instruction footprint small.
template <bool kSmemItems, bool kD8>
__global__ void __launch_bounds__(kThreads, 1) k_plan_loop(LoopArgs a) {
    extern __shared__ __align__(16) uint32_t dyn[];
    __shared__ Small sm;
    Shared s;
    uint32_t* const items_base = kSmemItems ? dyn : a.gitems;
    s.sx = items_base;
    s.snu = items_base + a.B;
    s.smask = items_base + 2 * a.B;
    s.sinfo = items_base + 3 * a.B;
    s.pre = items_base + 4 * a.B;
    s.fin = items_base + 5 * a.B;
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t N = a.N, b = a.b;
    const uint32_t lt = lanemask_lt();
    if (tid < kMaxN) {
        sm.bsize[tid] = 0;
        sm.top[tid] = 0;
        sm.inftop[tid] = 0;
        sm.infcnt[tid] = 0;
    }
    __syncthreads();
    size_t gbase = 0;
    unsigned long long pacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tprev = clock64();
#define LSG_PHASE(n)                                              \
    if (a.prof && tid == 0) {                                     \
        const unsigned long long tnow = clock64();                \
        pacc[n] += tnow - tprev;                                  \
        tprev = tnow;                                             \
    }
    for (uint32_t g = 0; g < a.T; ++g) {
        const uint32_t i = g / a.S, t = g % a.S;
        const uint32_t lo = t * a.B, len = min(a.B, a.keep - lo);
        const uint32_t* row = a.trace + size_t(a.order[i]) * a.keep + lo;
        const uint32_t* pkrow = a.nr + size_t(i) * a.keep + lo;
        const uint32_t R = ((len + kThreads - 1) / kThreads) * 32;  // items per warp
        const uint32_t j0 = w * R, j1 = min(j0 + R, len);

        // ---------------- A: load + classify + per-warp single ranks
        if (lane < kMaxN) sm.wcnt[w][lane] = 0;
        uint32_t wm = 0;
        // all of the warp's global loads first (coalesced ids/keys, then the
        // independent random holder-mask loads), so they overlap in flight
#pragma unroll 4
        for (uint32_t j = j0 + lane; j < j1; j += 32) {
            s.sx[j] = row[j];
            s.snu[j] = pkrow[j];
        }
        __syncwarp();
#pragma unroll 4
        for (uint32_t j = j0 + lane; j < j1; j += 32) s.smask[j] = __ldcg(&a.hm[s.sx[j]]);
        __syncwarp();
        for (uint32_t c = j0; c < j0 + R && a.remap; c += 32) {
            const uint32_t j = c + lane;
            const bool valid = j < j1;
            const uint32_t m = valid ? s.smask[j] : 0u;
            const uint32_t hc = __popc(m);
            const bool single = valid && hc == 1, multi = valid && hc >= 2;
            const uint32_t h = single ? __ffs(m) - 1 : 0;
            if (lane < kMaxN) sm.cm[w][lane] = 0;
            __syncwarp();
            const uint32_t grp = __match_any_sync(0xFFFFFFFFu, single ? h : 0x100u + lane);
            if (single && lane == uint32_t(__ffs(grp) - 1)) sm.cm[w][h] = grp;
            __syncwarp();
            if (single) s.sinfo[j] = sm.wcnt[w][h] + __popc(grp & lt);
            const uint32_t mb = __ballot_sync(0xFFFFFFFFu, multi);
            if (multi) {
                s.sinfo[j] = wm + __popc(mb & lt);
                uint32_t mm = m;
                while (mm) {
                    const uint32_t k = __ffs(mm) - 1;
                    mm &= mm - 1;
                    a.smul[size_t(j) * N + k] = sm.wcnt[w][k] + __popc(sm.cm[w][k] & lt);
                }
            }
            __syncwarp();
            if (single && lane == uint32_t(__ffs(grp) - 1)) sm.wcnt[w][h] += __popc(grp);
            wm += __popc(mb);
            __syncwarp();
        }
        if (lane == 0) sm.wmul[w] = wm;
        __syncthreads();
        LSG_PHASE(0)

        if (a.remap) {
            // ------------ B: scans over warps (warp k: node k; warp 31: multi)
            for (uint32_t k = w; k < N; k += kWarps) {
                const uint32_t v = lane < uint32_t(kWarps) ? sm.wcnt[lane][k] : 0u;
                uint32_t inc = v;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                    if (lane >= uint32_t(d)) inc += o;
                }
                if (lane < uint32_t(kWarps)) sm.wcnt[lane][k] = inc - v;
                if (lane == 31) sm.tot[k] = inc;
            }
            if (w == kWarps - 1) {
                const uint32_t v = lane < uint32_t(kWarps) ? sm.wmul[lane] : 0u;
                uint32_t inc = v;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                    if (lane >= uint32_t(d)) inc += o;
                }
                if (lane < uint32_t(kWarps)) sm.wmul[lane] = inc - v;
                if (lane == 31) sm.nmulti = inc;
            }
            __syncthreads();
            // ------------ C: global ranks; exact S_k(j) for multi items
            for (uint32_t j = j0 + lane; j < j1; j += 32) {
                const uint32_t m = s.smask[j];
                const uint32_t hc = __popc(m);
                if (hc == 1) {
                    s.sinfo[j] += sm.wcnt[w][__ffs(m) - 1];
                } else if (hc >= 2) {
                    const uint32_t mi = sm.wmul[w] + s.sinfo[j];
                    s.sinfo[j] = mi;
                    s.pre[mi] = j;  // multi list (pre is free until F)
                }
            }
            __syncwarp();
            // exact S_k(j) rows of the warp's multi items (warp-local part from
            // A + warp base; b for non-holders), compact by multi index for
            // D's staging. Lane per item: the row's loads are all in flight.
            {
                const uint32_t mb0 = sm.wmul[w];
                const uint32_t mcnt = (w + 1 < uint32_t(kWarps) ? sm.wmul[w + 1] : sm.nmulti) - mb0;
                for (uint32_t q = lane; q < mcnt; q += 32) {
                    const uint32_t mi = mb0 + q, j = s.pre[mi], m = s.smask[j];
                    const uint32_t* sm_row = a.smul + size_t(j) * N;
                    if (kD8) {
                        // D8 keys: T_k = (S_k << 4) | k in rows of 8 words
                        uint32_t t[8];
#pragma unroll
                        for (uint32_t k = 0; k < 8; ++k)
                            t[k] = (k < N && ((m >> k) & 1u)) ? __ldcg(&sm_row[k]) : 0u;
#pragma unroll
                        for (uint32_t k = 0; k < 8; ++k)
                            t[k] = ((k < N && ((m >> k) & 1u)) ? min(b, t[k] + sm.wcnt[w][k]) : b) << 4 | k;
                        if (b < kPk16B) {  // 16-bit keys, two nodes per word
                            reinterpret_cast<uint4*>(a.sx)[mi] = make_uint4(
                                t[0] | t[1] << 16, t[2] | t[3] << 16, t[4] | t[5] << 16, t[6] | t[7] << 16);
                        } else {
                            uint4* dst = reinterpret_cast<uint4*>(a.sx + size_t(mi) * 8);
                            dst[0] = make_uint4(t[0], t[1], t[2], t[3]);
                            dst[1] = make_uint4(t[4], t[5], t[6], t[7]);
                        }
                    } else {
                        for (uint32_t k = 0; k < N; ++k)
                            a.sx[size_t(mi) * N + k] =
                                ((m >> k) & 1u) ? min(b, __ldcg(&sm_row[k]) + sm.wcnt[w][k]) : b;
                    }
                }
            }
            __syncthreads();
            LSG_PHASE(1)
            // ------------ D: serial multi-holder pass
            // the other warps idle through D: pull the next step's id and key
            // rows into L2 for phase A
            if (w != 0 && g + 1 < a.T) {
                const uint32_t i2 = (g + 1) / a.S, t2 = (g + 1) % a.S;
                const uint32_t lo2 = t2 * a.B, len2 = min(a.B, a.keep - lo2);
                const char* r0 = reinterpret_cast<const char*>(a.trace + size_t(a.order[i2]) * a.keep + lo2);
                const char* r1 = reinterpret_cast<const char*>(a.nr + size_t(i2) * a.keep + lo2);
                for (uint32_t off = (tid - 32) * 128; off < len2 * 4; off += (kThreads - 32) * 128) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(r0 + off));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(r1 + off));
                }
            }
            if (w == 0 && (a.dbg_skip & 1)) {  // timing experiment: every multi item fetches
                for (uint32_t mi = lane; mi < sm.nmulti; mi += 32) s.sinfo[s.pre[mi]] = 0xFFFFFFFFu;
                if (lane < N) sm.mtot[lane] = 0;
            }
            for (int drep = 0; drep < ((a.dbg_skip & 2) ? 2 : 1); ++drep)  // timing: D is idempotent
            if (kD8 && w == 0 && !(a.dbg_skip & 1) && b < kPk16B) {
                // N <= 8 and b < 2048: the register decision below with the
                // 8 keys packed two per word (16 bits: (S + M) << 4 | k stays
                // below 2^16), so a key row is ONE broadcast 16-byte load, the
                // minimum is two VIMNMX3.U16x2 plus one 32-bit min, and the
                // winner's count moves by a per-pair increment: ~23
                // instructions per item instead of ~38 on the serial chain.
                uint32_t M01 = 0, M23 = 0, M45 = 0, M67 = 0;  // (M_k << 4) per 16-bit half
                unsigned long long dchain = 0;
                const uint32_t nm = sm.nmulti;
                const uint32_t kSent = (b << 4) - 1u;
                const uint32_t kSent2 = kSent | kSent << 16;
                auto stage = [&](uint32_t base, uint32_t buf) {
                    const uint32_t cnt = min(32u, nm - base);
                    const uint4* src = reinterpret_cast<const uint4*>(a.sx) + base;
                    uint4* dst4 = reinterpret_cast<uint4*>(&sm.stg[buf][0][0]);
                    if (lane < cnt) {
                        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst4 + lane));
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + lane));
                    } else {  // padding rows: no candidate
                        const uint32_t p = b << 4;
                        dst4[lane] = make_uint4(p | (p | 1) << 16, (p | 2) | (p | 3) << 16, (p | 4) | (p | 5) << 16,
                                                (p | 6) | (p | 7) << 16);
                    }
                    asm volatile("cp.async.commit_group;\n" ::);
                };
                if (nm) stage(0, 0);
                for (uint32_t base = 0, buf = 0; base < nm; base += 32, buf ^= 1) {
                    if (base + 32 < nm) {
                        stage(base + 32, buf ^ 1);
                        asm volatile("cp.async.wait_group 1;\n" ::);
                    } else {
                        asm volatile("cp.async.wait_group 0;\n" ::);
                    }
                    __syncwarp();
                    const uint32_t cnt = min(32u, nm - base);
                    const uint32_t myj = lane < cnt ? s.pre[base + lane] : 0u;
                    const uint4* rows = reinterpret_cast<const uint4*>(&sm.stg[buf][0][0]);
                    uint32_t myres = kSent;
                    const unsigned long long tc0 = a.prof ? clock64() : 0ull;
                    // v (per 16-bit half) = 0 for the previous item's winner,
                    // else 1; its count moves by 16 - 16 v. The next keys are
                    // (r + M + 16) - 16 v: the sum is off the chain, so the
                    // chain is IMAD -> 2 VIMNMX3 -> half swap + VIMNMX -> IADD
                    // (K - min, >= 0 per half) -> VIMNMX (v)
                    uint32_t v01 = 0x10001u, v23 = 0x10001u, v45 = 0x10001u, v67 = 0x10001u;
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        const uint4 r = rows[u];
                        const uint32_t K01 = (r.x + M01 + 0x100010u) - (v01 << 4);
                        const uint32_t K23 = (r.y + M23 + 0x100010u) - (v23 << 4);
                        const uint32_t K45 = (r.z + M45 + 0x100010u) - (v45 << 4);
                        const uint32_t K67 = (r.w + M67 + 0x100010u) - (v67 << 4);
                        M01 += 0x100010u - (v01 << 4);
                        M23 += 0x100010u - (v23 << 4);
                        M45 += 0x100010u - (v45 << 4);
                        M67 += 0x100010u - (v67 << 4);
                        const uint32_t m2 = __vimin3_u16x2(__vimin3_u16x2(K01, K23, K45), K67, kSent2);
                        const uint32_t mm = __vminu2(m2, __byte_perm(m2, 0, 0x1032));  // min in both halves
                        v01 = __vminu2(K01 - mm, 0x10001u);
                        v23 = __vminu2(K23 - mm, 0x10001u);
                        v45 = __vminu2(K45 - mm, 0x10001u);
                        v67 = __vminu2(K67 - mm, 0x10001u);
                        myres = lane == uint32_t(u) ? (mm & 0xFFFFu) : myres;
                    }
                    M01 += 0x100010u - (v01 << 4);  // the chunk's last decision
                    M23 += 0x100010u - (v23 << 4);
                    M45 += 0x100010u - (v45 << 4);
                    M67 += 0x100010u - (v67 << 4);
                    if (a.prof) {
                        const uint32_t dep = myres & 1u;  // keep the timer after the chain
                        const unsigned long long tc1 = clock64() + dep;
                        if (lane == 0) dchain += tc1 - tc0;
                    }
                    if (lane < cnt) {
                        if (myres != kSent) {
                            const uint32_t kk = myres & 15u, c = myres >> 4;
                            const uint32_t Sk =
                                reinterpret_cast<const uint16_t*>(&sm.stg[buf][0][0])[lane * 8 + kk] >> 4;
                            s.fin[kk * b + (c - Sk)] = myj;
                            s.sinfo[myj] = (c << 5) | kk;  // consumed by E
                        } else {
                            s.sinfo[myj] = 0xFFFFFFFFu;
                        }
                    }
                    __syncwarp();
                }
                if (a.prof && lane == 0) {
                    atomicAdd(&a.prof[12], (unsigned long long)nm);
                    atomicAdd(&a.prof[13], dchain);
                }
                const uint32_t Mp[4] = {M01, M23, M45, M67};
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (lane == uint32_t(k) && uint32_t(k) < N) sm.mtot[k] = ((Mp[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) >> 4;
            } else
            if (kD8 && w == 0 && !(a.dbg_skip & 1)) {
                // N <= 8: no warp reduction at all. Every lane runs the same
                // serial decision on registers: node k's running count is
                // Mk[k] = M_k << 4, item keys are T_k + Mk[k] with
                // T_k = (S_k << 4) | k (phase C), and the winner is the
                // minimum key below b << 4 (lowest k on ties, locality.cpp:
                // 24-31). Clamping the minimum at kSent = (b << 4) - 1, whose
                // low nibble no key has, makes "no candidate" update nothing.
                // The rows of a chunk are staged in shared memory and read
                // with broadcast 16-byte loads, off the dependency chain.
                uint32_t Mk[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) Mk[k] = 0;
                unsigned long long dchain = 0;
                const uint32_t nm = sm.nmulti;
                const uint32_t kSent = (b << 4) - 1u;
                auto stage = [&](uint32_t base, uint32_t buf) {
                    const uint32_t cnt = min(32u, nm - base);
                    const uint32_t* src = a.sx + size_t(base) * 8;
                    uint4* dst4 = reinterpret_cast<uint4*>(&sm.stg[buf][0][0]);
                    for (uint32_t q = lane; q < 64; q += 32) {
                        if (q < 2 * cnt) {
                            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst4 + q));
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 4 * q));
                        } else {
                            const uint32_t k0 = (q & 1) * 4;  // padding rows: no candidate
                            dst4[q] = make_uint4(b << 4 | k0, b << 4 | (k0 + 1), b << 4 | (k0 + 2), b << 4 | (k0 + 3));
                        }
                    }
                    asm volatile("cp.async.commit_group;\n" ::);
                };
                if (nm) stage(0, 0);
                for (uint32_t base = 0, buf = 0; base < nm; base += 32, buf ^= 1) {
                    if (base + 32 < nm) {
                        stage(base + 32, buf ^ 1);
                        asm volatile("cp.async.wait_group 1;\n" ::);
                    } else {
                        asm volatile("cp.async.wait_group 0;\n" ::);
                    }
                    __syncwarp();
                    const uint32_t cnt = min(32u, nm - base);
                    const uint32_t myj = lane < cnt ? s.pre[base + lane] : 0u;
                    const uint4* rows = reinterpret_cast<const uint4*>(&sm.stg[buf][0][0]);
                    uint32_t myres = kSent;
                    const unsigned long long tc0 = a.prof ? clock64() : 0ull;
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        const uint4 r0 = rows[2 * u], r1 = rows[2 * u + 1];
                        const uint32_t K0 = r0.x + Mk[0], K1 = r0.y + Mk[1], K2 = r0.z + Mk[2], K3 = r0.w + Mk[3];
                        const uint32_t K4 = r1.x + Mk[4], K5 = r1.y + Mk[5], K6 = r1.z + Mk[6], K7 = r1.w + Mk[7];
                        const uint32_t cl = __vimin3_u32(__vimin3_u32(K0, K1, K2), __vimin3_u32(K3, K4, K5),
                                                         __vimin3_u32(K6, K7, kSent));
                        Mk[0] += cl == K0 ? 16u : 0u; Mk[1] += cl == K1 ? 16u : 0u;
                        Mk[2] += cl == K2 ? 16u : 0u; Mk[3] += cl == K3 ? 16u : 0u;
                        Mk[4] += cl == K4 ? 16u : 0u; Mk[5] += cl == K5 ? 16u : 0u;
                        Mk[6] += cl == K6 ? 16u : 0u; Mk[7] += cl == K7 ? 16u : 0u;
                        myres = lane == uint32_t(u) ? cl : myres;
                    }
                    if (a.prof) {
                        const uint32_t dep = myres & 1u;  // keep the timer after the chain
                        const unsigned long long tc1 = clock64() + dep;
                        if (lane == 0) dchain += tc1 - tc0;
                    }
                    // lane u: item u's decision -> node list position + E's input
                    if (lane < cnt) {
                        if (myres != kSent) {
                            const uint32_t kk = myres & 15u, c = myres >> 4;
                            const uint32_t Sk = (&sm.stg[buf][0][0])[lane * 8 + kk] >> 4;  // row-major 8 words/item
                            s.fin[kk * b + (c - Sk)] = myj;
                            s.sinfo[myj] = (c << 5) | kk;  // consumed by E
                        } else {
                            s.sinfo[myj] = 0xFFFFFFFFu;
                        }
                    }
                    __syncwarp();
                }
                if (a.prof && lane == 0) {
                    atomicAdd(&a.prof[12], (unsigned long long)nm);
                    atomicAdd(&a.prof[13], dchain);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (lane == uint32_t(k) && uint32_t(k) < N) sm.mtot[k] = Mk[k] >> 4;
            } else
            if (!kD8 && w == 0 && !(a.dbg_skip & 1)) {
                // The warp-local part of S_k(j) for 32 multi items at a time is
                // staged global->smem with cp.async one chunk ahead. A
                // lane-parallel pass then packs the exact S_k(j) of the chunk
                // (plus the phase-B warp base; S = b when k is no holder) into
                // 16 registers per lane, so the fully unrolled serial loop
                // touches no memory at all (shared stores inside it serialize
                // with REDUX in the MIO pipe):
                //   key = ((S + M) << 5) | k, candidate iff M < b - S,
                // lane k holding Msh = M_k << 5. Results stay in registers
                // (lane u keeps item u's decision); list positions are rebuilt
                // after the chunk with __match_any_sync (a node's items of one
                // chunk take consecutive positions in item order).
                uint32_t Msh = 0;
                const uint32_t nm = sm.nmulti;
                // stage the chunk's exact S rows (contiguous 32*N words) with
                // 16-byte cp.async, one chunk ahead
                auto stage = [&](uint32_t base, uint32_t buf) {
                    const uint32_t cnt = min(32u, nm - base);
                    const uint32_t words = cnt * N;  // N <= 32, rows of N words
                    const uint32_t* src = a.sx + size_t(base) * N;
                    uint32_t* dstw = &sm.stg[buf][0][0];
                    for (uint32_t q = lane * 4; q < words; q += 128) {
                        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(dstw + q));
                        if (q + 4 <= words && ((reinterpret_cast<uintptr_t>(src + q) & 15) == 0)) {
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + q));
                        } else {
                            for (uint32_t r = q; r < min(q + 4, words); ++r) {
                                const unsigned d1 = static_cast<unsigned>(__cvta_generic_to_shared(dstw + r));
                                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d1), "l"(src + r));
                            }
                        }
                    }
                    asm volatile("cp.async.commit_group;\n" ::);
                };
                if (nm) stage(0, 0);
                for (uint32_t base = 0, buf = 0; base < nm; base += 32, buf ^= 1) {
                    if (base + 32 < nm) {
                        stage(base + 32, buf ^ 1);
                        asm volatile("cp.async.wait_group 1;\n" ::);
                    } else {
                        asm volatile("cp.async.wait_group 0;\n" ::);
                    }
                    __syncwarp();
                    const uint32_t cnt = min(32u, nm - base);
                    const uint32_t myj = lane < cnt ? s.pre[base + lane] : 0u;
                    const uint32_t* stw = &sm.stg[buf][0][0];  // row u at stw[u * N]
                    uint32_t P[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const uint32_t u0 = 2 * q, u1 = 2 * q + 1;
                        const uint32_t s0 = (u0 < cnt && lane < N) ? stw[u0 * N + lane] : b;
                        const uint32_t s1 = (u1 < cnt && lane < N) ? stw[u1 * N + lane] : b;
                        P[q] = s0 | (s1 << 16);
                    }
                    const uint32_t Mstart = Msh >> 5;
                    uint32_t myres = 0xFFFFFFFFu;
                    for (int lrep = 0; lrep < ((a.dbg_skip & 4) ? 2 : 1); ++lrep) {  // timing only
                    if (lrep) Msh = Mstart << 5;
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        if (uint32_t(u) < cnt) {
                            const uint32_t S = (P[u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
                            const uint32_t thr = (b - S) << 5, kb = (S << 5) | lane;
                            const uint32_t keyv = Msh < thr ? kb + Msh : 0xFFFFFFFFu;
                            const uint32_t best = __reduce_min_sync(0xFFFFFFFFu, keyv);
                            Msh += (keyv == best && best != 0xFFFFFFFFu) ? 32u : 0u;
                            myres = lane == uint32_t(u) ? best : myres;
                        }
                    }
                    }
                    // lane u: item u's decision -> node list position + E's input
                    const bool chose = lane < cnt && myres != 0xFFFFFFFFu;
                    const uint32_t kk = myres & 31;
                    const uint32_t grp = __match_any_sync(0xFFFFFFFFu, chose ? kk : 0x100u + lane);
                    const uint32_t m0 = __shfl_sync(0xFFFFFFFFu, Mstart, kk);
                    if (chose) s.fin[kk * b + m0 + __popc(grp & lt)] = myj;
                    if (lane < cnt) s.sinfo[myj] = myres;  // consumed by E
                    __syncwarp();
                }
                if (a.prof && lane == 0) atomicAdd(&a.prof[12], (unsigned long long)nm);
                if (lane < N) sm.mtot[lane] = Msh >> 5;
            }
            __syncthreads();
            LSG_PHASE(2)
            // ------------ E: hits/positions for singles; fetch ranks
            uint32_t wf = 0;
            for (uint32_t c = j0; c < j0 + R; c += 32) {
                const uint32_t j = c + lane;
                const bool valid = j < j1;
                bool fetch = false;
                if (valid) {
                    const uint32_t m = s.smask[j];
                    const uint32_t hc = __popc(m);
                    if (hc == 1) {
                        const uint32_t h = __ffs(m) - 1;
                        const uint32_t S = s.sinfo[j];
                        // M_h(<j): multi items before j assigned to h
                        const uint32_t* mp = s.fin + h * b;
                        uint32_t lo2 = 0, hi2 = sm.mtot[h];
                        while (lo2 < hi2) {
                            const uint32_t mid = (lo2 + hi2) >> 1;
                            if (mp[mid] < j) lo2 = mid + 1; else hi2 = mid;
                        }
                        const uint32_t pos = S + lo2;
                        if (pos < b) s.sinfo[j] = (h << 24) | pos;
                        else fetch = true;
                    } else if (hc >= 2) {
                        const uint32_t r = s.sinfo[j];
                        if (r != 0xFFFFFFFFu) s.sinfo[j] = ((r & 31) << 24) | (r >> 5);
                        else fetch = true;
                    } else {
                        fetch = true;
                    }
                }
                const uint32_t fbal = __ballot_sync(0xFFFFFFFFu, fetch);
                if (fetch) s.sinfo[j] = kFetch - (wf + __popc(fbal & lt)) ;  // encoded below
                wf += __popc(fbal);
            }
            if (lane == 0) sm.wfet[w] = wf;
            if (tid < N) sm.size[tid] = min(b, sm.tot[tid] + sm.mtot[tid]);
            __syncthreads();
            if (w == 0) {
                const uint32_t v = lane < uint32_t(kWarps) ? sm.wfet[lane] : 0u;
                uint32_t inc = v;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                    if (lane >= uint32_t(d)) inc += o;
                }
                if (lane < uint32_t(kWarps)) sm.wfet[lane] = inc - v;
                const uint32_t F = __shfl_sync(0xFFFFFFFFu, inc, 31);
                // free-capacity prefix over nodes (ascending fill, locality.cpp:33-39)
                const uint32_t fr = lane < N ? b - sm.size[lane] : 0;
                uint32_t pinc = fr;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, pinc, d);
                    if (lane >= uint32_t(d)) pinc += o;
                }
                const uint32_t pex = pinc - fr;
                if (lane < N) {
                    sm.free_pre[lane] = pex;
                    const uint32_t got = F > pex ? min(fr, F - pex) : 0u;
                    sm.fcnt[lane] = got;
                    sm.lenk[lane] = sm.size[lane] + got;
                }
                if (lane == N - 1) sm.free_pre[N] = pinc;
                if (lane == 0) sm.nfetch = F;
                const uint32_t totfree = __shfl_sync(0xFFFFFFFFu, pinc, N - 1);
                if (lane == 0 && F > totfree) atomicOr(a.status, 8u);  // ran out of capacity
            }
            __syncthreads();
            LSG_PHASE(3)
            // ------------ F: pre-balance lists [hits in batch order][fetches]
            for (uint32_t j = j0 + lane; j < j1; j += 32) {
                const uint32_t v = s.sinfo[j];
                if (v >= kFetch - 65536u) {
                    const uint32_t f = sm.wfet[w] + (kFetch - v);
                    // node with free_pre[k] <= f < free_pre[k+1]
                    uint32_t k = 0;
                    while (k + 1 < N && sm.free_pre[k + 1] <= f) ++k;
                    const uint32_t pos = sm.size[k] + (f - sm.free_pre[k]);
                    s.pre[k * b + pos] = j;
                } else {
                    s.pre[(v >> 24) * b + (v & 0xFFFFFF)] = j | kHit;
                }
            }
        } else {
            // slice_step (locality.cpp:57-73): node k = positions [k*b, (k+1)*b)
            for (uint32_t j = tid; j < len; j += kThreads) {
                const uint32_t k = j / b;
                const bool hit = (s.smask[j] >> k) & 1u;
                s.pre[j] = j | (hit ? kHit : 0u);
            }
            if (tid < N) {
                const uint32_t l0 = min(tid * b, len), l1 = min(l0 + b, len);
                sm.lenk[tid] = l1 - l0;
                sm.size[tid] = 0;
            }
            __syncthreads();
            if (tid < N) {
                uint32_t f = 0;
                for (uint32_t p = 0; p < sm.lenk[tid]; ++p) f += (s.pre[tid * b + p] & kHit) ? 0u : 1u;
                sm.fcnt[tid] = f;
            }
        }
        __syncthreads();

        LSG_PHASE(4)
        // ---------------- G: balance on counts (balance.cpp:10-39)
        // warp 0, lanes = nodes. One move takes from the first argmax and gives
        // to the first argmin, so donors at the top level M give one each in
        // node order while recipients at the bottom level m receive one each
        // in node order (donors and recipients stay disjoint): a round pairs
        // the first n = min(#top, #bottom) of each, all while M - m >= 2.
        // The donor's i-th move goes to recipient r as its q-th appended fetch.
        if (w == 0) {
            uint32_t c = lane < N ? sm.fcnt[lane] : 0u;
            if (a.fb && lane < N) a.fb[size_t(g) * N + lane] = c;
            uint32_t outc = 0, inn = 0, nmv = 0;
            const bool in = lane < N;
            bool rounds = a.balance;
            if (a.balance) {
                // closed form (as wide_balance_cf, plan_wide.cu): with L = F / N
                // the loop consumes donor units (k gives one at count l) in
                // (l desc, k asc) order and recipient units in (l asc, k asc)
                // order and pairs the t-th of each; mandatory units are the
                // donor levels >= L+2 and recipient levels <= L-1, the shorter
                // side padded at level L+1 (donors) / L (recipients) in node
                // order. Recipient units are tabled in the (free) D staging.
                const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, in ? c : 0u);
                const uint32_t mn = __reduce_min_sync(0xFFFFFFFFu, in ? c : 0xFFFFFFFFu);
                const uint32_t F = __reduce_add_sync(0xFFFFFFFFu, in ? c : 0u);
                const uint32_t L = F / N;
                const uint32_t dm = __reduce_add_sync(0xFFFFFFFFu, in && c > L + 1 ? c - L - 1 : 0u);
                const uint32_t rm = __reduce_add_sync(0xFFFFFFFFu, in && c < L ? L - c : 0u);
                const uint32_t mv = max(dm, rm), od = mv - dm, orr = mv - rm;
                uint32_t* urq = &sm.stg[0][0][0];
                if (mx - mn <= 1) {
                    rounds = false;
                } else if (mv <= 2u * 32u * kMaxN) {
                    rounds = false;
                    uint32_t t = 0;
                    for (uint32_t l = mn; l <= L; ++l) {
                        const uint32_t br = __ballot_sync(0xFFFFFFFFu, in && c <= l);
                        const uint32_t lim = l < L ? 32u : orr;
                        const uint32_t rk = __popc(br & lt);
                        if (in && c <= l && rk < lim) {
                            urq[t + rk] = lane | ((l - c) << 8);
                            ++inn;
                        }
                        t += min(uint32_t(__popc(br)), lim);
                    }
                    __syncwarp();
                    t = 0;
                    for (uint32_t l = mx; l >= L + 1; --l) {
                        const uint32_t bd = __ballot_sync(0xFFFFFFFFu, in && c >= l);
                        const uint32_t lim = l > L + 1 ? 32u : od;
                        const uint32_t rk = __popc(bd & lt);
                        if (in && c >= l && rk < lim) {
                            const uint32_t rq = urq[t + rk];
                            if (outc < kDmv) sm.dmv[lane][outc] = rq;
                            else a.dmoves[size_t(lane) * a.B + outc] = rq;
                            ++outc;
                        }
                        t += min(uint32_t(__popc(bd)), lim);
                    }
                    nmv = mv;
                    c = c - outc + inn;
                }
            }
            while (rounds) {  // very wide count spread: the round simulation
                const uint32_t M = __reduce_max_sync(0xFFFFFFFFu, lane < N ? c : 0u);
                const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, lane < N ? c : 0xFFFFFFFFu);
                if (M - m <= 1) break;
                const uint32_t dm = __ballot_sync(0xFFFFFFFFu, lane < N && c == M);
                const uint32_t rm = __ballot_sync(0xFFFFFFFFu, lane < N && c == m);
                const uint32_t n = min(__popc(dm), __popc(rm));
                const bool isd = (dm >> lane) & 1u, isr = (rm >> lane) & 1u;
                const uint32_t rk = __popc((isd ? dm : rm) & lt);  // rank in its set
                // the recipient of rank rk publishes (r, q) for the donor of rank rk
                if (isr && rk < n) {
                    sm.rq[rk] = lane | (inn << 8);
                    ++c;
                    ++inn;
                }
                __syncwarp();
                if (isd && rk < n) {
                    const uint32_t rq = sm.rq[rk];
                    if (outc < kDmv) sm.dmv[lane][outc] = rq;
                    else a.dmoves[size_t(lane) * a.B + outc] = rq;
                    --c;
                    ++outc;
                }
                __syncwarp();
                nmv += n;
            }
            if (lane < N) {
                sm.outk[lane] = outc;
                sm.ink[lane] = inn;
            }
            if (lane == 0) sm.nmoves = nmv;
        }
        __syncthreads();
        LSG_PHASE(5)
        // donors (warp per donor): the i-th largest fetch id takes move i
        // (balance.cpp:27-33 erases the largest remaining fetch id each move)
        if (a.balance && sm.nmoves) {
            for (uint32_t k = w; k < N; k += kWarps) {
                const uint32_t out = sm.outk[k];
                if (!out) continue;
                // remap lists are [hits][fetches]: fetches start at size[k]
                // (slice lists are mixed; size[k] = 0 there)
                const uint32_t L = sm.lenk[k], f0 = sm.size[k];
                for (uint32_t c = f0; c < L; c += 32) {
                    const uint32_t p = c + lane;
                    const uint32_t e = p < L ? s.pre[k * b + p] : kHit;
                    const bool isf = !(e & kHit);
                    const uint32_t x = isf ? s.sx[e & 0xFFFF] : 0u;
                    uint32_t rank = 0;
                    for (uint32_t c2 = f0; c2 < L; c2 += 32) {
                        const uint32_t p2 = c2 + lane;
                        const uint32_t e2 = p2 < L ? s.pre[k * b + p2] : kHit;
                        const uint32_t y = !(e2 & kHit) ? s.sx[e2 & 0xFFFF] : 0u;  // 0 is never > x
#pragma unroll
                        for (int q = 0; q < 32; ++q) rank += __shfl_sync(0xFFFFFFFFu, y, q) > x ? 1u : 0u;
                    }
                    if (isf)
                        s.sinfo[e & 0xFFFF] = rank >= out ? kNotMoved
                                              : rank < kDmv ? sm.dmv[k][rank] : a.dmoves[size_t(k) * a.B + rank];
                }
            }
            __syncthreads();
        }
        LSG_PHASE(6)
        // ---------------- H: final lists + outputs
        if (w == 0) {
            const uint32_t L = lane < N ? sm.lenk[lane] - sm.outk[lane] + sm.ink[lane] : 0;
            uint32_t inc = L;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (lane >= uint32_t(d)) inc += o;
            }
            if (lane < N) {
                sm.noff[lane] = inc - L;
                a.node_off[size_t(g) * (N + 1) + lane] = inc - L;
                if (a.fa) a.fa[size_t(g) * N + lane] = sm.fcnt[lane] - sm.outk[lane] + sm.ink[lane];
            }
            if (lane == N - 1) {
                sm.noff[N] = inc;
                a.node_off[size_t(g) * (N + 1) + N] = inc;
                if (inc != len) atomicOr(a.status, 16u);  // multiset size check
            }
        }
        __syncthreads();
        // warp k places node k's pre-balance list (k < N)
        for (uint32_t k = w; k < N; k += kWarps) {
            const uint32_t L = sm.lenk[k], out = sm.outk[k];
            uint32_t shift = 0;
            for (uint32_t c = 0; c < L; c += 32) {
                const uint32_t p = c + lane;
                uint32_t e = 0;
                bool moved = false;
                if (p < L) {
                    e = s.pre[k * b + p];
                    moved = out && !(e & kHit) && s.sinfo[e & 0xFFFF] != kNotMoved;
                }
                const uint32_t mbal = __ballot_sync(0xFFFFFFFFu, moved);
                if (p < L) {
                    uint32_t dst;
                    if (moved) {
                        const uint32_t mvv = s.sinfo[e & 0xFFFF];  // (r, q) from G
                        const uint32_t r = mvv & 0xFF, q = mvv >> 8;
                        dst = sm.noff[r] + (sm.lenk[r]) + q;
                        s.fin[dst] = (e & 0xFFFF) | (r << 16);
                    } else {
                        dst = sm.noff[k] + p - (shift + __popc(mbal & lt));
                        s.fin[dst] = (e & 0xFFFF) | (k << 16) | (e & kHit);
                    }
                    a.items[gbase + dst] = s.sx[e & 0xFFFF] | (e & kHit);
                }
                shift += __popc(mbal);
            }
        }
        __syncthreads();

        LSG_PHASE(7)
        // ---------------- I: buffer advance, nodes in parallel
        if (a.remap) {  // tagged hits form each list's prefix: one re-key run
            // their new keys fall in (g, g+2S): aggregate the bucket bits in a
            // shared window, then flush one atomic per non-empty word
            const uint32_t wbase = (g + 1) >> 5;
            for (uint32_t q = tid; q < N * kWinWords; q += kThreads) sm.win[q / kWinWords][q % kWinWords] = 0;
            __syncthreads();
            for (uint32_t p = tid; p < len; p += kThreads) {
                const uint32_t e = s.fin[p];
                if (!(e & kHit)) continue;
                const uint32_t j = e & 0xFFFF, k = (e >> 16) & 0xFF;
                const uint32_t x = s.sx[j], pk = s.snu[j];
                const uint32_t nu = pk == kNever ? kNever : key_step(a, pk), rank = pk - nu * a.B;
                const uint32_t wd = nu >> 5;
                if (nu != kNever && wd >= wbase && wd - wbase < kWinWords) {
                    a.key[size_t(k) * a.D + x] = pk;
                    red_or(&a.bm[(size_t(k) * a.T + nu) * a.BW + (rank >> 5)], 1u << (rank & 31));
                    atomicOr(&sm.win[k][wd - wbase], 1u << (nu & 31));
                } else {
                    set_key(a, sm, k, x, pk);
                }
            }
            __syncthreads();
            for (uint32_t q = tid; q < N * kWinWords; q += kThreads) {
                const uint32_t k = q / kWinWords, wd = q % kWinWords;
                const uint32_t v = sm.win[k][wd];
                if (v) {
                    red_or(&a.nz[size_t(k) * a.nzw + wbase + wd], v);
                    atomicMax(&sm.top[k], (wbase + wd) * 32 + 31 - __clz(v));
                }
            }
            __syncthreads();
        }
        LSG_PHASE(8)
        for (uint32_t k = w; k < N; k += kWarps) {
            const uint32_t begin = sm.noff[k] + (a.remap ? sm.size[k] : 0u), end = sm.noff[k + 1];
            // a miss run may span chunks: insert as we go, evict once when the
            // run ends (before the next hit run, or at the end of the list)
            bool pending = false;
            auto flush = [&]() {
                uint32_t need = 0;
                if (lane == 0) need = sm.bsize[k] > a.C ? sm.bsize[k] - a.C : 0u;
                need = __shfl_sync(0xFFFFFFFFu, need, 0);
                __syncwarp();
                if (need) evict_walk(a, sm, k, need, lane, g);
                __syncwarp();
                pending = false;
            };
            for (uint32_t c = begin; c < end; c += 32) {
                const uint32_t p = c + lane;
                const bool valid = p < end;
                uint32_t j = 0;
                bool res = false;
                if (valid) {
                    j = s.fin[p] & 0xFFFF;
                    res = (s.smask[j] >> k) & 1u;  // residency at step start
                }
                const uint32_t vbal = __ballot_sync(0xFFFFFFFFu, valid);
                const uint32_t rbal = __ballot_sync(0xFFFFFFFFu, res);
                // walk the chunk's runs in order
                uint32_t done = 0;
                while (done != vbal) {
                    const uint32_t first = __ffs(vbal & ~done) - 1;
                    const bool hitrun = (rbal >> first) & 1u;
                    // run = maximal lanes from `first` with the same residency
                    const uint32_t same = hitrun ? rbal : (vbal & ~rbal);
                    const uint32_t after = (~same) & vbal & ~((1u << first) - 1u) & ~(1u << first);
                    const uint32_t stop = after ? __ffs(after) - 1 : 32u;
                    const uint32_t run = (stop == 32 ? 0xFFFFFFFFu : ((1u << stop) - 1u)) & ~((1u << first) - 1u) & vbal;
                    const bool mine = (run >> lane) & 1u;
                    if (hitrun && pending) flush();  // the miss run before it ends here
                    if (mine) {
                        const uint32_t x = s.sx[j];
                        set_key(a, sm, k, x, s.snu[j]);
                        if (!hitrun) red_or(&a.hm[x], 1u << k);
                    }
                    __syncwarp();
                    if (!hitrun) {
                        if (lane == 0) sm.bsize[k] += __popc(run);
                        pending = true;
                    }
                    __syncwarp();
                    done |= run;
                }
            }
            if (pending) flush();
        }
        __syncthreads();
        LSG_PHASE(9)
        gbase += len;
    }
#undef LSG_PHASE
    if (a.prof && tid == 0)
        for (int q = 0; q < 10; ++q) a.prof[q] = pacc[q];
}

// ---------------------------------------------------------------------------
// K6o: the step loop with its phases PIPELINED over three teams (N <= 8,
// b < 2048, B <= 4096, remap on; clairvoyant): team C classifies step h
// (A..C), team D runs the serial multi-holder chain D of step h, team P
// applies D and runs the buffer-side phases E..I of step h. Step h is
// classified once I(h-4) has advanced the buffers, i.e. against holder masks
// three advances old, so the loop P(h-4) -> C(h) -> D(h) -> P(h) spans four
// steps. Only ids of batch h whose mask I(h-3)..I(h-1) changes can alter its
// classification: an insert or a drop of such an id (an id in nearby batches
// at an epoch boundary, or an eviction reaching next-step keys) is detected
// through per-id stamps (one array per batch mod 3, so an id in several
// pending batches keeps every stamp), and then step h is classified and
// resolved again after I(h-1) (around epoch boundaries, in practice). Team
// P's step arrays are double-buffered by step parity (team C classifies into
// its own shared memory, two sets, and copies a step over once P is done
// with the step two back); team D's inputs and results are in global memory
// by step mod 4. The teams hand off through shared-memory step counters with
// cluster-scope release/acquire.
struct OvPar {  // per step parity
    uint32_t tot[kMaxN];   // singles per node
    uint32_t mtot[kMaxN];  // multi assigned per node (D)
    uint32_t nmulti;
    uint32_t cf;           // I(g-1) found this batch's masks changed
};

struct SmallOv {
    uint32_t wcnt[kWarps][kMaxN];
    uint32_t cm[kWarps][kMaxN];
    uint32_t wmul[kWarps];
    uint32_t wfet[kWarps];
    uint32_t size[kMaxN];
    uint32_t free_pre[kMaxN + 1];
    uint32_t lenk[kMaxN];
    uint32_t fcnt[kMaxN];
    uint32_t outk[kMaxN], ink[kMaxN];
    uint32_t noff[kMaxN + 1];
    uint32_t bsize[kMaxN];
    uint32_t top[kMaxN];
    uint32_t inftop[kMaxN];
    uint32_t infcnt[kMaxN];
    uint32_t nfetch, nmoves;
    alignas(16) uint32_t stg[kDWarps][2][32][kOvN];  // team D: staging per D warp (32 packed rows of 16 B)
    uint32_t dmv[kMaxN][kDmv];
    uint32_t rq[kMaxN];
    uint32_t win[kMaxN][kWinWords];
    uint32_t stamp, conflict, conflict2, conflict3;  // I(g): stamps g+1..g+3, their batches' verdicts
    OvPar par[2];
    uint32_t cfv[8];   // verdict per batch (mod 8): a mask it was classified with changed
    uint32_t mbm[kOvN][kOvW];   // team P: the multi items team D assigned to node k, by batch position
    uint32_t mpre[kOvN][kOvW];  //   and their count before each word
    uint32_t cnm[4];   // (team C's copy) multi items per step (mod 4), for team D
    // team hand-off counters (monotone): steps classified, resolved (D
    // final), buffer-advanced, speculative-D-finished-on-conflict,
    // re-classified, copied into team P's arrays, resolved (first pass)
    volatile uint32_t ac_cnt, d_cnt, i_cnt, spec_cnt, redo_cnt, copy_cnt, ds_cnt[kDWarps];
};

// The teams run on the three SMs of a thread-block cluster: team C (all 16
// warps of CTA 0), team P (all 16 warps of CTA 1), whose per-step arrays and
// hand-off counters live in CTA 1's shared memory, and team D (four warps of
// CTA 2, one per scheduler). Teams C and D reach team P's state through
// distributed shared memory.
constexpr uint32_t kPWarps = kWarps, kPThreads = kPWarps * 32;
constexpr uint32_t kOvDepth = 4;  // steps in flight: step h is classified once I(h-4) is done
// team C (classification): CTA 0's 12 warps that do not share warp 0's
// scheduler (warp w issues on SMSP w % 4)
constexpr uint32_t kCWarps = 16, kCThreads = kCWarps * 32;

__device__ __forceinline__ void bar_p() { asm volatile("bar.sync 1, %0;" ::"n"(kPThreads) : "memory"); }
__device__ __forceinline__ void bar_c() { asm volatile("bar.sync 2, %0;" ::"n"(kCThreads) : "memory"); }
// hand-offs between the cluster's CTAs: release/acquire at cluster scope
// (the counters live in shared memory; partner writes are DSMEM and global)
__device__ __forceinline__ void wait_ge(volatile uint32_t* c, uint32_t v) {
    while (*c < v) {
    }
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
}
__device__ __forceinline__ void publish(volatile uint32_t* c, uint32_t v) {
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
    *c = v;
}

struct OvBufs {
    uint32_t *sx, *snu, *smask, *sinfo, *pre, *fin;
};

// A..C of step g by team C (CTA 0, 12 warps): load + classify + ranks, exact
// S_k(j) rows of the multi items for D (global, buffer g % 3)
__device__ void ov_classify(const LoopArgs& a, SmallOv& sm, const OvBufs& s, OvPar& pp, uint32_t* smul,
                            uint32_t* dsx, uint32_t* dpre, uint32_t g, uint32_t pw, uint32_t lane, bool stamp) {
    // sm, s, pp: team C's own scratch, step arrays and totals (local shared
    // memory; ov_copy moves them to team P)
    const uint32_t N = a.N, b = a.b;
    const uint32_t lt = lanemask_lt();
    const uint32_t i = g / a.S, t = g % a.S;
    const uint32_t lo = t * a.B, len = min(a.B, a.keep - lo);
    const uint32_t* row = a.trace + size_t(a.order[i]) * a.keep + lo;
    const uint32_t R = ((len + kCThreads - 1) / kCThreads) * 32;
    const uint32_t j0 = pw * R, j1 = min(j0 + R, len);
    if (lane < kMaxN) sm.wcnt[pw][lane] = 0;
    uint32_t wm = 0;
    // every lane's (at most 8: B <= 4096 over 16 warps) ids, then their masks,
    // each as one batch of independent loads
    constexpr int kCU = 8;
    uint32_t xs[kCU];
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
        const uint32_t j = j0 + lane + 32u * u;
        xs[u] = j < j1 ? __ldg(&row[j]) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
        const uint32_t j = j0 + lane + 32u * u;
        if (j < j1) {
            s.sx[j] = xs[u];
            if (stamp) a.nb[size_t(g % 3) * a.D + xs[u]] = g;  // this batch's classification is checked by I(g-3)..I(g-1)
        }
    }
    __threadfence();  // stamps before the masks are read (nb_check)
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
        const uint32_t j = j0 + lane + 32u * u;
        xs[u] = j < j1 ? __ldcg(&a.hm[xs[u]]) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
        const uint32_t j = j0 + lane + 32u * u;
        if (j < j1) s.smask[j] = xs[u];
    }
    __syncwarp();
    for (uint32_t c = j0; c < j0 + R; c += 32) {
        const uint32_t j = c + lane;
        const bool valid = j < j1;
        const uint32_t m = valid ? s.smask[j] : 0u;
        const uint32_t hc = __popc(m);
        const bool single = valid && hc == 1, multi = valid && hc >= 2;
        const uint32_t h = single ? __ffs(m) - 1 : 0;
        if (lane < kMaxN) sm.cm[pw][lane] = 0;
        __syncwarp();
        const uint32_t grp = __match_any_sync(0xFFFFFFFFu, single ? h : 0x100u + lane);
        if (single && lane == uint32_t(__ffs(grp) - 1)) sm.cm[pw][h] = grp;
        __syncwarp();
        if (single) s.sinfo[j] = sm.wcnt[pw][h] + __popc(grp & lt);
        const uint32_t mb = __ballot_sync(0xFFFFFFFFu, multi);
        if (multi) {
            s.sinfo[j] = wm + __popc(mb & lt);
            uint32_t mm = m;
            while (mm) {
                const uint32_t k = __ffs(mm) - 1;
                mm &= mm - 1;
                smul[size_t(j) * N + k] = sm.wcnt[pw][k] + __popc(sm.cm[pw][k] & lt);
            }
        }
        __syncwarp();
        if (single && lane == uint32_t(__ffs(grp) - 1)) sm.wcnt[pw][h] += __popc(grp);
        wm += __popc(mb);
        __syncwarp();
    }
    if (lane == 0) sm.wmul[pw] = wm;
    bar_c();
    // B: scans over the P warps (warp k: node k; the last warp: multi)
    for (uint32_t k = pw; k < N; k += kCWarps) {
        const uint32_t v = lane < kCWarps ? sm.wcnt[lane][k] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= uint32_t(d)) inc += o;
        }
        if (lane < kCWarps) sm.wcnt[lane][k] = inc - v;
        if (lane == 31) pp.tot[k] = inc;
    }
    if (pw == kCWarps - 1) {
        const uint32_t v = lane < kCWarps ? sm.wmul[lane] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= uint32_t(d)) inc += o;
        }
        if (lane < kCWarps) sm.wmul[lane] = inc - v;
        if (lane == 31) pp.nmulti = inc;
    }
    bar_c();
    // C: global ranks; exact S_k(j) rows of the multi items (16-bit packed)
    for (uint32_t j = j0 + lane; j < j1; j += 32) {
        const uint32_t m = s.smask[j];
        const uint32_t hc = __popc(m);
        if (hc == 1) {
            s.sinfo[j] += sm.wcnt[pw][__ffs(m) - 1];
        } else if (hc >= 2) {
            const uint32_t mi = sm.wmul[pw] + s.sinfo[j];
            s.sinfo[j] = mi;
            s.pre[mi] = j;
        }
    }
    __syncwarp();
    {
        const uint32_t mb0 = sm.wmul[pw];
        const uint32_t mcnt = (pw + 1 < kCWarps ? sm.wmul[pw + 1] : pp.nmulti) - mb0;
        for (uint32_t q = lane; q < mcnt; q += 32) {
            const uint32_t mi = mb0 + q, j = s.pre[mi], m = s.smask[j];
            const uint32_t* sm_row = smul + size_t(j) * N;
            uint32_t tk[8];
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) tk[k] = (k < N && ((m >> k) & 1u)) ? __ldcg(&sm_row[k]) : 0u;
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k)
                tk[k] = ((k < N && ((m >> k) & 1u)) ? min(b, tk[k] + sm.wcnt[pw][k]) : b) << 4 | k;
            reinterpret_cast<uint4*>(dsx)[mi] =
                make_uint4(tk[0] | tk[1] << 16, tk[2] | tk[3] << 16, tk[4] | tk[5] << 16, tk[6] | tk[7] << 16);
            dpre[mi] = j;  // the multi list for team D, in global memory (no DSMEM on its chain)
        }
    }
    if (pw == 0 && lane == 0) sm.cnm[g % kOvDepth] = pp.nmulti;
    __threadfence_block();
    bar_c();
}

// the classified step g (team C's arrays + totals; the packed next-use keys
// straight from their global row) into team P's parity buffers (16-byte
// DSMEM stores), once team P is done with step g-2
__device__ void ov_copy(const LoopArgs& a, const OvBufs& s, const OvPar& pc, const OvBufs& sr, OvPar& pp, uint32_t g,
                        uint32_t pw, uint32_t lane) {
    const uint32_t lo = (g % a.S) * a.B, len = min(a.B, a.keep - lo);
    const uint32_t* pkrow = a.nr + size_t(g / a.S) * a.keep + lo;  // (any alignment: read by words)
    const uint32_t ctid = pw * 32 + lane, nm = pc.nmulti;
    const uint32_t len4 = (len + 3) / 4, nm4 = (nm + 3) / 4;
    for (uint32_t q = ctid; q < 4 * len4 + nm4; q += kCThreads) {
        const uint32_t arr = q < 4 * len4 ? q / len4 : 4, e = (q < 4 * len4 ? q - arr * len4 : q - 4 * len4) * 4;
        uint32_t* dst = arr == 0 ? sr.sx : arr == 1 ? sr.snu : arr == 2 ? sr.smask : arr == 3 ? sr.sinfo : sr.pre;
        uint4 v;
        if (arr == 1) {
            v.x = __ldcg(&pkrow[e]);
            v.y = e + 1 < len ? __ldcg(&pkrow[e + 1]) : 0u;
            v.z = e + 2 < len ? __ldcg(&pkrow[e + 2]) : 0u;
            v.w = e + 3 < len ? __ldcg(&pkrow[e + 3]) : 0u;
        } else {
            const uint32_t* src = arr == 0 ? s.sx : arr == 2 ? s.smask : arr == 3 ? s.sinfo : s.pre;
            v = *reinterpret_cast<const uint4*>(src + e);
        }
        *reinterpret_cast<uint4*>(dst + e) = v;
    }
    if (ctid < a.N) pp.tot[ctid] = pc.tot[ctid];
    if (ctid == 0) pp.nmulti = nm;
    __threadfence_block();
    bar_c();
}

// D of one step by warp 0: the packed register chain of k_plan_loop. Inputs
// from global memory (the multi list and the packed rows), outputs into team
// D's own shared memory (res[mi] = the chain's minimum key, or kSent; mtot);
// team P applies them to its lists (ov_apply).
__device__ void ov_resolve(const LoopArgs& a, uint32_t (*stg)[32][kOvN], const uint32_t* dsx, const uint32_t* dpre,
                           uint32_t nm, uint32_t* res, uint32_t* mtot, uint32_t lane) {
    const uint32_t N = a.N, b = a.b;
    uint32_t M01 = 0, M23 = 0, M45 = 0, M67 = 0;
    const uint32_t kSent = (b << 4) - 1u;
    const uint32_t kSent2 = kSent | kSent << 16;
    (void)dpre;
    auto stage = [&](uint32_t base, uint32_t buf) {
        const uint32_t cnt = min(32u, nm - base);
        const uint4* src = reinterpret_cast<const uint4*>(dsx) + base;
        uint4* dst4 = reinterpret_cast<uint4*>(&stg[buf][0][0]);
        if (lane < cnt) {
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst4 + lane));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + lane));
        } else {
            const uint32_t p = b << 4;
            dst4[lane] = make_uint4(p | (p | 1) << 16, (p | 2) | (p | 3) << 16, (p | 4) | (p | 5) << 16,
                                    (p | 6) | (p | 7) << 16);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (nm) stage(0, 0);
    for (uint32_t base = 0, buf = 0; base < nm; base += 32, buf ^= 1) {
        if (base + 32 < nm) {
            stage(base + 32, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncwarp();
        const uint32_t cnt = min(32u, nm - base);
        const uint4* rows = reinterpret_cast<const uint4*>(&stg[buf][0][0]);
        uint32_t myres = kSent;
        uint32_t v01 = 0x10001u, v23 = 0x10001u, v45 = 0x10001u, v67 = 0x10001u;
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const uint4 r = rows[u];
            const uint32_t K01 = (r.x + M01 + 0x100010u) - (v01 << 4);
            const uint32_t K23 = (r.y + M23 + 0x100010u) - (v23 << 4);
            const uint32_t K45 = (r.z + M45 + 0x100010u) - (v45 << 4);
            const uint32_t K67 = (r.w + M67 + 0x100010u) - (v67 << 4);
            M01 += 0x100010u - (v01 << 4);
            M23 += 0x100010u - (v23 << 4);
            M45 += 0x100010u - (v45 << 4);
            M67 += 0x100010u - (v67 << 4);
            const uint32_t m2 = __vimin3_u16x2(__vimin3_u16x2(K01, K23, K45), K67, kSent2);
            const uint32_t mm = __vminu2(m2, __byte_perm(m2, 0, 0x1032));
            v01 = __vminu2(K01 - mm, 0x10001u);
            v23 = __vminu2(K23 - mm, 0x10001u);
            v45 = __vminu2(K45 - mm, 0x10001u);
            v67 = __vminu2(K67 - mm, 0x10001u);
            myres = lane == uint32_t(u) ? (mm & 0xFFFFu) : myres;
        }
        M01 += 0x100010u - (v01 << 4);
        M23 += 0x100010u - (v23 << 4);
        M45 += 0x100010u - (v45 << 4);
        M67 += 0x100010u - (v67 << 4);
        if (lane < cnt) res[base + lane] = myres;
        __syncwarp();
    }
    const uint32_t Mp[4] = {M01, M23, M45, M67};
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (lane == uint32_t(k) && uint32_t(k) < N) mtot[k] = ((Mp[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) >> 4;
    __syncwarp();
}

// team P: team D's decisions for the multi items of step g into the lists
// (node positions in fin, E's input in sinfo) — what k_plan_loop's D writes
// (a bit per multi item in its node's batch-position bitmap: E counts the
// multi items of node h before a single at j with a prefix and a popc, where
// the single-CTA loop binary-searches a sorted list)
__device__ void ov_apply(const LoopArgs& a, const OvBufs& s, OvPar& pp, SmallOv& sm, const uint32_t* res_d,
                         const uint32_t* mtot_d, uint32_t ptid) {
    const uint32_t b = a.b, nm = pp.nmulti;
    const uint32_t kSent = (b << 4) - 1u;
    for (uint32_t mi = ptid; mi < nm; mi += kPThreads) {
        const uint32_t r = __ldcg(&res_d[mi]), j = s.pre[mi];
        if (r != kSent) {
            const uint32_t kk = r & 15u, c = r >> 4;
            atomicOr(&sm.mbm[kk][j >> 5], 1u << (j & 31));
            s.sinfo[j] = (c << 5) | kk;
        } else {
            s.sinfo[j] = 0xFFFFFFFFu;
        }
    }
    if (ptid < a.N) pp.mtot[ptid] = __ldcg(&mtot_d[ptid]);
}

__global__ void __launch_bounds__(kThreads, 1) k_plan_loop_ov(LoopArgs a) {
    extern __shared__ __align__(16) uint32_t dyn[];
    __shared__ SmallOv sm_local;
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t crank = cl.block_rank();
    // team P's state (CTA 1), as seen from either CTA
    SmallOv& sm = *cl.map_shared_rank(&sm_local, 1);
    uint32_t* pdyn = cl.map_shared_rank(dyn, 1);
    OvBufs S2[2];
    for (int p = 0; p < 2; ++p) {
        uint32_t* b0 = pdyn + size_t(p) * 6 * a.B;
        S2[p] = OvBufs{b0, b0 + a.B, b0 + 2 * a.B, b0 + 3 * a.B, b0 + 4 * a.B, b0 + 5 * a.B};
    }
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t N = a.N, b = a.b;
    const uint32_t lt = lanemask_lt();
    if (crank == 1) {
        if (tid < kMaxN) {
            sm_local.bsize[tid] = 0;
            sm_local.top[tid] = 0;
            sm_local.inftop[tid] = 0;
            sm_local.infcnt[tid] = 0;
        }
        if (tid == 0) {
            sm_local.ac_cnt = sm_local.d_cnt = sm_local.i_cnt = sm_local.spec_cnt = sm_local.redo_cnt = 0;
            sm_local.copy_cnt = 0;
            for (uint32_t q = 0; q < kDWarps; ++q) sm_local.ds_cnt[q] = 0;
            for (int q = 0; q < 8; ++q) sm_local.cfv[q] = 0;
            sm_local.conflict = sm_local.conflict2 = sm_local.conflict3 = 0;
        }
    }
    cl.sync();
    // global scratch: smul [B][N] (team C only), the D rows [3][B] x 16 B and multi lists [3][B]
    // global scratch (a.sx): the D rows [4][B] x 16 B, multi lists [4][B], team D's
    // results res [4][B] and mtot [4][kMaxN], by step mod 4; smul [2][B][N] (team C only)
    auto smul_of = [&](uint32_t g) { return a.smul + size_t(g & 1) * a.B * N; };
    auto dsx_of = [&](uint32_t g) { return a.sx + size_t(g % kOvDepth) * a.B * 4; };
    auto dpre_of = [&](uint32_t g) { return a.sx + size_t(kOvDepth) * a.B * 4 + size_t(g % kOvDepth) * a.B; };
    auto res_of = [&](uint32_t g) { return a.sx + size_t(kOvDepth) * a.B * 5 + size_t(g % kOvDepth) * a.B; };
    auto mtot_of = [&](uint32_t g) { return a.sx + size_t(kOvDepth) * a.B * 6 + size_t(g % kOvDepth) * kMaxN; };
    unsigned long long pf[12] = {}, t0 = clock64();
    auto tick = [&](int q) {
        if (a.prof) {
            const unsigned long long t1 = clock64();
            pf[q] += t1 - t0;
            t0 = t1;
        }
    };
    // LSG_PROFILE_OV: global-timer stamps of each team's events for steps 2000..2015
    auto ev = [&](uint32_t g, int e) {
        const uint32_t g0 = uint32_t(a.dbg_skip) >> 8;
        if (a.prof && g >= g0 && g < g0 + 16) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.prof[32 + (g - g0) * 8 + e] = t;
        }
    };
    if (crank == 0) {
        // -------------------------------------------- team C (CTA 0, all warps)
        const uint32_t cw = w;
        // team C's step arrays, two sets (it classifies step h before copying
        // step h-1): sx, smask, sinfo, pre (the next-use keys are copied from
        // their global row)
        auto sc_of = [&](uint32_t h) {
            uint32_t* c0 = dyn + size_t(h & 1) * 4 * a.B;
            return OvBufs{c0, nullptr, c0 + a.B, c0 + 2 * a.B, c0 + 3 * a.B, nullptr};
        };
        auto pc_of = [&](uint32_t h) -> OvPar& { return sm_local.par[h & 1]; };  // its totals, per set
        for (uint32_t h = 0; h < a.T + kOvDepth - 1; ++h) {
            // classify step h once I(h-4) is done; first the final verdict (I(h-6)..I(h-4))
            // on step h-3, whose re-classification uses set h (not yet written this round)
            if (h >= kOvDepth - 1) {
                if (cw == 0) wait_ge(&sm.i_cnt, h - (kOvDepth - 1));
                bar_c();
            }
            if (h >= kOvDepth && h - (kOvDepth - 1) < a.T && sm.cfv[(h - (kOvDepth - 1)) & 7]) {
                const uint32_t q = h - (kOvDepth - 1);
                if (cw == 0) wait_ge(&sm.ds_cnt[q % kDWarps], q + 1);  // team D is done with the speculative D(q)
                bar_c();
                ov_classify(a, sm_local, sc_of(h), pc_of(h), smul_of(q), dsx_of(q), dpre_of(q), q, cw, lane, false);
                // team P has not started step q (it waits for D(q)): its buffers take the new classification
                ov_copy(a, sc_of(h), pc_of(h), S2[q & 1], sm.par[q & 1], q, cw, lane);
                if (cw == 0 && lane == 0) publish(&sm.redo_cnt, q + 1);
            }
            if (h < a.T) {
                tick(0);
                if (cw == 0 && lane == 0) ev(h, 0);
                ov_classify(a, sm_local, sc_of(h), pc_of(h), smul_of(h), dsx_of(h), dpre_of(h), h, cw, lane, true);
                if (cw == 0 && lane == 0) publish(&sm.ac_cnt, h + 1);
                if (cw == 0 && lane == 0) ev(h, 1);
                tick(1);
            }
            if (h >= 1 && h - 1 < a.T) {  // copy step h-1 once team P is done with step h-3
                const uint32_t q = h - 1;
                if (q >= 2) {
                    if (cw == 0) wait_ge(&sm.i_cnt, q - 1);
                    bar_c();
                }
                tick(2);
                if (cw == 0 && lane == 0) ev(q, 2);
                ov_copy(a, sc_of(q), pc_of(q), S2[q & 1], sm.par[q & 1], q, cw, lane);
                if (cw == 0 && lane == 0) publish(&sm.copy_cnt, q + 1);
                if (cw == 0 && lane == 0) ev(q, 3);
                tick(3);
            }
        }
        if (cw == 0 && lane == 0) publish(&sm.ac_cnt, a.T + 1);  // team D: no more re-classifications
        if (a.prof && cw == 0 && lane == 0)
            for (int q = 0; q < 4; ++q) a.prof[20 + q] = pf[q];
        cl.sync();  // team P's shared memory stays alive until every team is done with it
        return;
    }
    if (crank == 2) {
        if (w < kDWarps) {
            // -------------------------------------------- team D (CTA 2)
            // One warp per scheduler, one per step mod 4: D(g) of one step does
            // not depend on D(g-1), and one warp's serial chain leaves most of
            // its scheduler idle. Speculative D(g) as soon as step g is
            // classified; a re-classified step (team C, after I(g-3)..I(g-1)
            // changed one of its masks) is resolved again when it arrives, and
            // team P waits for that only then.
            const uint32_t dp = w;  // this warp's steps: g % 4 == dp
            const SmallOv& smc = *cl.map_shared_rank(&sm_local, 0);  // team C's (cnm)
            uint32_t (*stg)[32][kOvN] = sm_local.stg[dp];
            uint32_t redone = 0;  // re-classifications resolved (redo_cnt values)
            auto pending = [&]() {
                const uint32_t r = sm.redo_cnt;
                return r > redone && ((r - 1) % kDWarps) == dp;
            };
            auto redo = [&]() {
                if (!pending()) return;
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
                const uint32_t r = sm.redo_cnt, q = r - 1;
                ov_resolve(a, stg, dsx_of(q), dpre_of(q), smc.cnm[q % kOvDepth], res_of(q), mtot_of(q), lane);
                __syncwarp();
                if (lane == 0) publish(&sm.d_cnt, r);
                redone = r;
            };
            for (uint32_t g = dp; g < a.T;) {
                // every lane spins: a one-lane spin left the warp diverged through the chain
                while (sm.ac_cnt < g + 1 && !pending()) {
                }
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
                tick(0);
                redo();  // (at most one pending: the next needs P to finish the step this one blocks)
                if (sm.ac_cnt < g + 1) continue;
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
                if (lane == 0) ev(g, 4);
                ov_resolve(a, stg, dsx_of(g), dpre_of(g), smc.cnm[g % kOvDepth], res_of(g), mtot_of(g), lane);
                __syncwarp();
                if (lane == 0) publish(&sm.ds_cnt[dp], g + 1);  // team P knows the verdict itself (it ran I(g-1))
                if (lane == 0) ev(g, 5);
                tick(1);
                g += kDWarps;
            }
            while (sm.ac_cnt <= a.T) redo();  // team C's last re-classifications (it ends with ac_cnt = T+1)
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            redo();
            if (a.prof && w == 0 && lane == 0)
                for (int q = 0; q < 4; ++q) a.prof[q] = pf[q];
        }
        cl.sync();  // team P's shared memory stays alive until team D is done with it
        return;
    }
    // ---------------------------------------------------- team P (CTA 1)
    {
    SmallOv& sm = sm_local;  // its own shared memory, addressed directly
    const uint32_t pw = w, ptid = tid;
    size_t gbase = 0;
    for (uint32_t g = 0; g < a.T; ++g) {
        // the step's arrays straight from the shared-memory symbol (not from the
        // S2 table, which lives on the stack and would make every access generic)
        uint32_t* b0 = dyn + size_t(g & 1) * 6 * a.B;
        const OvBufs s{b0, b0 + a.B, b0 + 2 * a.B, b0 + 3 * a.B, b0 + 4 * a.B, b0 + 5 * a.B};
        OvPar& pp = sm.par[g & 1];
        const uint32_t len = min(a.B, a.keep - (g % a.S) * a.B);
        const uint32_t R = ((len + kPThreads - 1) / kPThreads) * 32;
        const uint32_t j0 = pw * R, j1 = min(j0 + R, len);
        tick(3);
        if (ptid == 0) {  // D(g) resolved, step g copied in; one waiter, the barrier orders the rest
            wait_ge(&sm.ds_cnt[g % kDWarps], g + 1);
            wait_ge(&sm.copy_cnt, g + 1);
            // I(g-2) or I(g-1) changed a mask of this batch: wait for its second classification
            if (g > 0 && sm.cfv[g & 7]) {
                wait_ge(&sm.d_cnt, g + 1);
                if (a.prof) a.prof[24] += 1;
            }
        }
        bar_p();
        if (ptid == 0) ev(g, 6);
        if (a.prof && ptid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.prof[32 + 128 + 2 * g] = t;
        }
        tick(9);
        const uint32_t lenw = (min(a.B, a.keep - (g % a.S) * a.B) + 31) / 32;
        for (uint32_t q = ptid; q < N * kOvW; q += kPThreads) sm.mbm[q / kOvW][q % kOvW] = 0;
        bar_p();
        ov_apply(a, s, pp, sm, res_of(g), mtot_of(g), ptid);
        bar_p();
        for (uint32_t k = pw; k < N; k += kPWarps) {  // per node: multi items before each word
            uint32_t v[4], t = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t wd = lane * 4 + u;
                v[u] = wd < lenw ? __popc(sm.mbm[k][wd]) : 0u;
                t += v[u];
            }
            uint32_t inc = t;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (lane >= uint32_t(d)) inc += o;
            }
            uint32_t run = inc - t;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                sm.mpre[k][lane * 4 + u] = run;
                run += v[u];
            }
        }
        bar_p();
        tick(0);
        if (g + kOvDepth < a.T && !(a.dbg_skip & 8)) {  // batch g+4's rows into L2 for its classification after I(g)
            const uint32_t g2 = g + kOvDepth, i2 = g2 / a.S, t2 = g2 % a.S;
            const uint32_t lo2 = t2 * a.B, len2 = min(a.B, a.keep - lo2);
            const char* r0 = reinterpret_cast<const char*>(a.trace + size_t(a.order[i2]) * a.keep + lo2);
            const char* r1 = reinterpret_cast<const char*>(a.nr + size_t(i2) * a.keep + lo2);
            for (uint32_t off = ptid * 128; off < len2 * 4; off += kPThreads * 128) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(r0 + off));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(r1 + off));
            }
        }
        // ------------ E: hits/positions for singles; fetch ranks
        uint32_t wf = 0;
        for (uint32_t c = j0; c < j0 + R; c += 32) {
            const uint32_t j = c + lane;
            const bool valid = j < j1;
            bool fetch = false;
            if (valid) {
                const uint32_t m = s.smask[j];
                const uint32_t hc = __popc(m);
                if (hc == 1) {
                    const uint32_t h = __ffs(m) - 1;
                    const uint32_t S = s.sinfo[j];
                    // M_h(<j): multi items before j assigned to h
                    const uint32_t pos = S + sm.mpre[h][j >> 5] + __popc(sm.mbm[h][j >> 5] & lanemask_lt());
                    if (pos < b) s.sinfo[j] = (h << 24) | pos;
                    else fetch = true;
                } else if (hc >= 2) {
                    const uint32_t r = s.sinfo[j];
                    if (r != 0xFFFFFFFFu) s.sinfo[j] = ((r & 31) << 24) | (r >> 5);
                    else fetch = true;
                } else {
                    fetch = true;
                }
            }
            const uint32_t fbal = __ballot_sync(0xFFFFFFFFu, fetch);
            if (fetch) s.sinfo[j] = kFetch - (wf + __popc(fbal & lt));
            wf += __popc(fbal);
        }
        if (lane == 0) sm.wfet[pw] = wf;
        if (ptid < N) sm.size[ptid] = min(b, pp.tot[ptid] + pp.mtot[ptid]);
        bar_p();
        if (pw == 0) {
            const uint32_t v = lane < kPWarps ? sm.wfet[lane] : 0u;
            uint32_t inc = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (lane >= uint32_t(d)) inc += o;
            }
            if (lane < kPWarps) sm.wfet[lane] = inc - v;
            const uint32_t F = __shfl_sync(0xFFFFFFFFu, inc, 31);
            const uint32_t fr = lane < N ? b - sm.size[lane] : 0;
            uint32_t pinc = fr;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, pinc, d);
                if (lane >= uint32_t(d)) pinc += o;
            }
            const uint32_t pex = pinc - fr;
            if (lane < N) {
                sm.free_pre[lane] = pex;
                const uint32_t got = F > pex ? min(fr, F - pex) : 0u;
                sm.fcnt[lane] = got;
                sm.lenk[lane] = sm.size[lane] + got;
            }
            if (lane == N - 1) sm.free_pre[N] = pinc;
            if (lane == 0) sm.nfetch = F;
            const uint32_t totfree = __shfl_sync(0xFFFFFFFFu, pinc, N - 1);
            if (lane == 0 && F > totfree) atomicOr(a.status, 8u);
        }
        bar_p();
        tick(4);
        // ------------ F: pre-balance lists [hits in batch order][fetches]
        for (uint32_t j = j0 + lane; j < j1; j += 32) {
            const uint32_t v = s.sinfo[j];
            if (v >= kFetch - 65536u) {
                const uint32_t f = sm.wfet[pw] + (kFetch - v);
                uint32_t k = 0;
                while (k + 1 < N && sm.free_pre[k + 1] <= f) ++k;
                const uint32_t pos = sm.size[k] + (f - sm.free_pre[k]);
                s.pre[k * b + pos] = j;
            } else {
                s.pre[(v >> 24) * b + (v & 0xFFFFFF)] = j | kHit;
            }
        }
        bar_p();
        tick(5);
        // ------------ G: balance on counts (closed form, as k_plan_loop)
        if (pw == 0) {
            uint32_t c = lane < N ? sm.fcnt[lane] : 0u;
            if (a.fb && lane < N) a.fb[size_t(g) * N + lane] = c;
            uint32_t outc = 0, inn = 0, nmv = 0;
            const bool in = lane < N;
            bool rounds = a.balance;
            if (a.balance) {
                const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, in ? c : 0u);
                const uint32_t mn = __reduce_min_sync(0xFFFFFFFFu, in ? c : 0xFFFFFFFFu);
                const uint32_t F = __reduce_add_sync(0xFFFFFFFFu, in ? c : 0u);
                const uint32_t L = F / N;
                const uint32_t dm = __reduce_add_sync(0xFFFFFFFFu, in && c > L + 1 ? c - L - 1 : 0u);
                const uint32_t rm = __reduce_add_sync(0xFFFFFFFFu, in && c < L ? L - c : 0u);
                const uint32_t mv = max(dm, rm), od = mv - dm, orr = mv - rm;
                uint32_t* urq = a.dmoves + size_t(N) * a.B;  // recipient units (D's staging is busy here)
                if (mx - mn <= 1) {
                    rounds = false;
                } else if (mv <= 2u * 32u * kMaxN) {
                    rounds = false;
                    uint32_t t = 0;
                    for (uint32_t l = mn; l <= L; ++l) {
                        const uint32_t br = __ballot_sync(0xFFFFFFFFu, in && c <= l);
                        const uint32_t lim = l < L ? 32u : orr;
                        const uint32_t rk = __popc(br & lt);
                        if (in && c <= l && rk < lim) {
                            urq[t + rk] = lane | ((l - c) << 8);
                            ++inn;
                        }
                        t += min(uint32_t(__popc(br)), lim);
                    }
                    __syncwarp();
                    t = 0;
                    for (uint32_t l = mx; l >= L + 1; --l) {
                        const uint32_t bd = __ballot_sync(0xFFFFFFFFu, in && c >= l);
                        const uint32_t lim = l > L + 1 ? 32u : od;
                        const uint32_t rk = __popc(bd & lt);
                        if (in && c >= l && rk < lim) {
                            const uint32_t rq = urq[t + rk];
                            if (outc < kDmv) sm.dmv[lane][outc] = rq;
                            else a.dmoves[size_t(lane) * a.B + outc] = rq;
                            ++outc;
                        }
                        t += min(uint32_t(__popc(bd)), lim);
                    }
                    nmv = mv;
                    c = c - outc + inn;
                }
            }
            while (rounds) {
                const uint32_t M = __reduce_max_sync(0xFFFFFFFFu, lane < N ? c : 0u);
                const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, lane < N ? c : 0xFFFFFFFFu);
                if (M - m <= 1) break;
                const uint32_t dmk = __ballot_sync(0xFFFFFFFFu, lane < N && c == M);
                const uint32_t rmk = __ballot_sync(0xFFFFFFFFu, lane < N && c == m);
                const uint32_t n = min(__popc(dmk), __popc(rmk));
                const bool isd = (dmk >> lane) & 1u, isr = (rmk >> lane) & 1u;
                const uint32_t rk = __popc((isd ? dmk : rmk) & lt);
                if (isr && rk < n) {
                    sm.rq[rk] = lane | (inn << 8);
                    ++c;
                    ++inn;
                }
                __syncwarp();
                if (isd && rk < n) {
                    const uint32_t rq = sm.rq[rk];
                    if (outc < kDmv) sm.dmv[lane][outc] = rq;
                    else a.dmoves[size_t(lane) * a.B + outc] = rq;
                    --c;
                    ++outc;
                }
                __syncwarp();
                nmv += n;
            }
            if (lane < N) {
                sm.outk[lane] = outc;
                sm.ink[lane] = inn;
            }
            if (lane == 0) sm.nmoves = nmv;
        }
        bar_p();
        if (a.balance && sm.nmoves) {
            for (uint32_t k = pw; k < N; k += kPWarps) {
                const uint32_t out = sm.outk[k];
                if (!out) continue;
                const uint32_t L = sm.lenk[k], f0 = sm.size[k];
                for (uint32_t c = f0; c < L; c += 32) {
                    const uint32_t p = c + lane;
                    const uint32_t e = p < L ? s.pre[k * b + p] : kHit;
                    const bool isf = !(e & kHit);
                    const uint32_t x = isf ? s.sx[e & 0xFFFF] : 0u;
                    uint32_t rank = 0;
                    for (uint32_t c2 = f0; c2 < L; c2 += 32) {
                        const uint32_t p2 = c2 + lane;
                        const uint32_t e2 = p2 < L ? s.pre[k * b + p2] : kHit;
                        const uint32_t y = !(e2 & kHit) ? s.sx[e2 & 0xFFFF] : 0u;
#pragma unroll
                        for (int q = 0; q < 32; ++q) rank += __shfl_sync(0xFFFFFFFFu, y, q) > x ? 1u : 0u;
                    }
                    if (isf)
                        s.sinfo[e & 0xFFFF] = rank >= out ? kNotMoved
                                              : rank < kDmv ? sm.dmv[k][rank] : a.dmoves[size_t(k) * a.B + rank];
                }
            }
            bar_p();
        }
        tick(6);
        // ------------ H: final lists + outputs
        if (pw == 0) {
            const uint32_t L = lane < N ? sm.lenk[lane] - sm.outk[lane] + sm.ink[lane] : 0;
            uint32_t inc = L;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (lane >= uint32_t(d)) inc += o;
            }
            if (lane < N) {
                sm.noff[lane] = inc - L;
                a.node_off[size_t(g) * (N + 1) + lane] = inc - L;
                if (a.fa) a.fa[size_t(g) * N + lane] = sm.fcnt[lane] - sm.outk[lane] + sm.ink[lane];
            }
            if (lane == N - 1) {
                sm.noff[N] = inc;
                a.node_off[size_t(g) * (N + 1) + N] = inc;
                if (inc != len) atomicOr(a.status, 16u);
            }
        }
        bar_p();
        for (uint32_t k = pw; k < N; k += kPWarps) {
            const uint32_t L = sm.lenk[k], out = sm.outk[k];
            uint32_t shift = 0;
            for (uint32_t c = 0; c < L; c += 32) {
                const uint32_t p = c + lane;
                uint32_t e = 0;
                bool moved = false;
                if (p < L) {
                    e = s.pre[k * b + p];
                    moved = out && !(e & kHit) && s.sinfo[e & 0xFFFF] != kNotMoved;
                }
                const uint32_t mbal = __ballot_sync(0xFFFFFFFFu, moved);
                if (p < L) {
                    uint32_t dst;
                    if (moved) {
                        const uint32_t mvv = s.sinfo[e & 0xFFFF];
                        const uint32_t r = mvv & 0xFF, q = mvv >> 8;
                        dst = sm.noff[r] + (sm.lenk[r]) + q;
                        s.fin[dst] = (e & 0xFFFF) | (r << 16);
                    } else {
                        dst = sm.noff[k] + p - (shift + __popc(mbal & lt));
                        s.fin[dst] = (e & 0xFFFF) | (k << 16) | (e & kHit);
                    }
                    a.items[gbase + dst] = s.sx[e & 0xFFFF] | (e & kHit);
                }
                shift += __popc(mbal);
            }
        }
        bar_p();
        tick(7);
        // ------------ I: buffer advance; changes to the masks of batches g+1
        // and g+2 (already classified) are caught by the stamp checks
        if (ptid == 0) {
            sm.stamp = g + 1;
            sm.conflict = sm.conflict2 = sm.conflict3 = 0;
        }
        bar_p();
        {
            const uint32_t wbase = (g + 1) >> 5;
            for (uint32_t q = ptid; q < N * kWinWords; q += kPThreads) sm.win[q / kWinWords][q % kWinWords] = 0;
            bar_p();
            for (uint32_t p = ptid; p < len; p += kPThreads) {
                const uint32_t e = s.fin[p];
                if (!(e & kHit)) continue;
                const uint32_t j = e & 0xFFFF, k = (e >> 16) & 0xFF;
                const uint32_t x = s.sx[j], pk = s.snu[j];
                const uint32_t nu = pk == kNever ? kNever : key_step(a, pk), rank = pk - nu * a.B;
                const uint32_t wd = nu >> 5;
                if (nu != kNever && wd >= wbase && wd - wbase < kWinWords) {
                    a.key[size_t(k) * a.D + x] = pk;
                    red_or(&a.bm[(size_t(k) * a.T + nu) * a.BW + (rank >> 5)], 1u << (rank & 31));
                    atomicOr(&sm.win[k][wd - wbase], 1u << (nu & 31));
                } else {
                    set_key(a, sm, k, x, pk);
                }
            }
            bar_p();
            for (uint32_t q = ptid; q < N * kWinWords; q += kPThreads) {
                const uint32_t k = q / kWinWords, wd = q % kWinWords;
                const uint32_t v = sm.win[k][wd];
                if (v) {
                    red_or(&a.nz[size_t(k) * a.nzw + wbase + wd], v);
                    atomicMax(&sm.top[k], (wbase + wd) * 32 + 31 - __clz(v));
                }
            }
            bar_p();
        }
        tick(8);
        for (uint32_t k = pw; k < N; k += kPWarps) {
            const uint32_t begin = sm.noff[k] + sm.size[k], end = sm.noff[k + 1];
            bool pending = false;
            auto flush = [&]() {
                uint32_t need = 0;
                if (lane == 0) need = sm.bsize[k] > a.C ? sm.bsize[k] - a.C : 0u;
                need = __shfl_sync(0xFFFFFFFFu, need, 0);
                __syncwarp();
                if (need) evict_walk(a, sm, k, need, lane, g);
                __syncwarp();
                pending = false;
            };
            for (uint32_t c = begin; c < end; c += 32) {
                const uint32_t p = c + lane;
                const bool valid = p < end;
                uint32_t j = 0;
                bool res = false;
                if (valid) {
                    j = s.fin[p] & 0xFFFF;
                    res = (s.smask[j] >> k) & 1u;
                }
                const uint32_t vbal = __ballot_sync(0xFFFFFFFFu, valid);
                const uint32_t rbal = __ballot_sync(0xFFFFFFFFu, res);
                uint32_t done = 0;
                while (done != vbal) {
                    const uint32_t first = __ffs(vbal & ~done) - 1;
                    const bool hitrun = (rbal >> first) & 1u;
                    const uint32_t same = hitrun ? rbal : (vbal & ~rbal);
                    const uint32_t after = (~same) & vbal & ~((1u << first) - 1u) & ~(1u << first);
                    const uint32_t stop = after ? __ffs(after) - 1 : 32u;
                    const uint32_t run = (stop == 32 ? 0xFFFFFFFFu : ((1u << stop) - 1u)) & ~((1u << first) - 1u) & vbal;
                    const bool mine = (run >> lane) & 1u;
                    if (hitrun && pending) flush();
                    if (mine) {
                        const uint32_t x = s.sx[j];
                        set_key(a, sm, k, x, s.snu[j]);
                        if (!hitrun) {
                            red_or(&a.hm[x], 1u << k);
                            nb_check(a, sm, x);
                        }
                    }
                    __syncwarp();
                    if (!hitrun) {
                        if (lane == 0) sm.bsize[k] += __popc(run);
                        pending = true;
                    }
                    __syncwarp();
                    done |= run;
                }
            }
            if (pending) flush();
        }
        bar_p();
        tick(1);
        gbase += len;
        // the verdicts on steps g+1 (final) and g+2 (first half); team C re-classifies on a conflict
        if (ptid == 0) {
            sm.cfv[(g + 1) & 7] |= sm.conflict;
            sm.cfv[(g + 2) & 7] |= sm.conflict2;
            sm.cfv[(g + 3) & 7] = sm.conflict3;
            publish(&sm.i_cnt, g + 1);
            ev(g, 7);
            if (a.prof) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                a.prof[32 + 128 + 2 * g + 1] = t;
            }
        }
        tick(2);
    }
    if (a.prof && ptid == 0)
        for (int q = 0; q < 12; ++q) a.prof[4 + q] = pf[q];
    }
    cl.sync();
}

}  // namespace


int plan_wide_device(const PlanDims& dm, uint64_t C, int lru, int remap, int balance, int insred, uint64_t thr,
                     const uint32_t* d_trace, const uint32_t* d_order, const uint32_t* d_inv, const uint32_t* d_nu,
                     uint32_t* d_items, uint32_t* d_node_off, uint32_t* d_fb, uint32_t* d_fa, uint32_t* d_status,
                     cudaStream_t st, const uint32_t* d_hm_init = nullptr, int advance = 1);

int plan_loop_device(const PlanDims& dm, uint64_t C, int policy, int remap, int balance, int insred, uint64_t thr,
                     const uint32_t* d_trace,
                     const uint32_t* d_order, const uint32_t* d_inv, uint32_t* d_items,
                     uint32_t* d_node_off, uint32_t* d_fb, uint32_t* d_fa, uint32_t* d_status,
                     cudaStream_t st) {
    // wide worlds (N > 32, a global batch beyond shared memory, or packed
    // keys beyond 32 bits) run the cluster step loop of plan_wide.cu, which
    // is faster there (cfg5 N=32: 292 vs 528 us/step); LSG_PLAN_WIDE=1 / 0
    // forces / forbids it (parity tests of both kernels on the same configs)
    const char* fw = std::getenv("LSG_PLAN_WIDE");
    bool wide = dm.N > kMaxN || dm.B > kMaxSmemB || dm.T * dm.B >= 0xFFFFFFF0ull || policy == 1 || insred;
    if (fw && fw[0] == '1') wide = true;
    if (fw && fw[0] == '0' && dm.N <= kMaxN && dm.B <= kMaxB && dm.T * dm.B < 0xFFFFFFF0ull && policy == 0 &&
        !insred)
        wide = false;
    Scratch sc(st);
    const size_t EK = size_t(dm.E) * dm.keep;
    uint32_t* nu = sc.get<uint32_t>(EK);
    if (wide) {
        if (!nu) return set_error(kInternal, "plan: scratch allocation failed");
        k_nextuse<<<dim3(grid_for(dm.keep, 256, 1024), dm.E), 256, 0, st>>>(
            d_trace, d_order, d_inv, dm.E, uint32_t(dm.keep), uint32_t(dm.D), uint32_t(dm.S), uint32_t(dm.B), nu);
        LSG_LAUNCH_CHECK("k_nextuse");
        return plan_wide_device(dm, C, policy == 1, remap, balance, insred, thr, d_trace, d_order, d_inv, nu, d_items,
                                d_node_off, d_fb, d_fa,
                                d_status, st);
    }
    uint32_t* sb = sc.get<uint32_t>(EK);
    uint32_t* nr = sc.get<uint32_t>(EK);
    LoopArgs a{};
    a.D = uint32_t(dm.D);
    a.N = dm.N;
    a.b = dm.b;
    a.B = uint32_t(dm.B);
    a.S = uint32_t(dm.S);
    a.E = dm.E;
    a.keep = uint32_t(dm.keep);
    a.T = uint32_t(dm.T);
    a.C = uint32_t(std::min<uint64_t>(C, 0xFFFFFFF0ull));
    a.remap = remap;
    a.balance = balance;
    a.nzw = uint32_t((dm.T + 31) / 32 + 1);
    a.infw = uint32_t((dm.D + 31) / 32);
    a.key = sc.get<uint32_t>(size_t(dm.N) * dm.D);
    a.BW = uint32_t((dm.B + 31) / 32);
    a.bm = sc.get<uint32_t>(size_t(dm.N) * dm.T * a.BW);
    a.hm = sc.get<uint32_t>(dm.D);
    a.nz = sc.get<uint32_t>(size_t(dm.N) * a.nzw);
    a.infbm = sc.get<uint32_t>(size_t(dm.N) * a.infw);
    // the overlapped loop (K6o): team D resolves step g+1 while team P
    // advances step g and classifies step g+2 (LSG_PLAN_OV=0: the plain loop)
    const char* ov_env = std::getenv("LSG_PLAN_OV");
    // (below B = 2048 the team hand-offs cost more than the overlap wins: cfg4, B = 512, 7.8 s
    // overlapped vs 5.4 s; cfg1, B = 256, 35 vs 22.5 ms)
    // LSG_PLAN_OV=1 forces it for any B the kernel supports (tests), =0 turns it off
    const bool ov = remap && dm.N <= 8 && dm.b < kPk16B && dm.B <= 4096 && dm.B % 4 == 0 && !profiling() &&
                    !std::getenv("LSG_DEBUG_SKIP") && !(ov_env && ov_env[0] == '0') &&
                    (dm.B >= 2048 || (ov_env && ov_env[0] == '1'));
    a.smul = sc.get<uint32_t>(size_t(dm.B) * dm.N * (ov ? 2 : 1));
    a.sx = sc.get<uint32_t>(ov ? size_t(dm.B) * 4 * 7 + 4 * kMaxN
                               : size_t(dm.B) * std::max<uint32_t>(dm.N, 8u));  // D rows (+ ov: 4 sets, lists, results)
    a.dmoves = sc.get<uint32_t>(size_t(dm.N) * dm.B + 2 * 32 * kMaxN);
    a.nb = ov ? sc.get<uint32_t>(size_t(3) * dm.D) : nullptr;
    if (ov && !a.nb) return set_error(kInternal, "plan: scratch allocation failed");
    if (ov) LSG_CUDA(cudaMemsetAsync(a.nb, 0xFF, size_t(3) * dm.D * 4, st));
    if (!nu || !sb || !nr || !a.bm || !a.key || !a.hm || !a.nz || !a.infbm || !a.smul || !a.sx || !a.dmoves)
        return set_error(kInternal, "plan: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(a.key, 0xFF, size_t(dm.N) * dm.D * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.hm, 0, dm.D * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.nz, 0, size_t(dm.N) * a.nzw * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.bm, 0, size_t(dm.N) * dm.T * a.BW * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.infbm, 0, size_t(dm.N) * a.infw * 4, st));
    // K5
    k_nextuse<<<dim3(grid_for(dm.keep, 256, 1024), dm.E), 256, 0, st>>>(
        d_trace, d_order, d_inv, dm.E, uint32_t(dm.keep), uint32_t(dm.D), uint32_t(dm.S), uint32_t(dm.B), nu);
    LSG_LAUNCH_CHECK("k_nextuse");
    // sorted batches
    uint32_t P2 = 1;
    while (P2 < dm.B) P2 <<= 1;
    LSG_CUDA(cudaFuncSetAttribute(k_sort_batches, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P2 * 4)));
    k_sort_batches<<<uint32_t(dm.T), 1024, P2 * 4, st>>>(d_trace, d_order, uint32_t(dm.keep),
                                                          uint32_t(dm.S), uint32_t(dm.B), P2, sb);
    LSG_LAUNCH_CHECK("k_sort_batches");
    a.trace = d_trace;
    a.order = d_order;
    k_nextrank<<<dim3(grid_for(dm.keep, 256, 1024), dm.E), 256, 0, st>>>(
        d_trace, d_order, nu, sb, dm.E, uint32_t(dm.keep), uint32_t(dm.S), uint32_t(dm.B), nr);
    LSG_LAUNCH_CHECK("k_nextrank");
    a.nu = nu;
    a.sb = sb;
    a.nr = nr;
    a.bdiv = dm.B >= 2 ? ~0ull / dm.B + 1 : 0;
    a.items = d_items;
    a.node_off = d_node_off;
    a.fb = d_fb;
    a.fa = d_fa;
    a.status = d_status;
    const bool smem_items = dm.B <= kMaxSmemB;
    a.gitems = smem_items ? nullptr : sc.get<uint32_t>(size_t(6) * dm.B);
    if (!smem_items && !a.gitems) return set_error(kInternal, "plan: scratch allocation failed");
    a.prof = profiling() ? sc.get<unsigned long long>(16 + 256) : nullptr;
    a.dbg_skip = std::getenv("LSG_DEBUG_SKIP") ? std::atoi(std::getenv("LSG_DEBUG_SKIP")) : 0;
    if (ov && std::getenv("LSG_OV_NOPF")) a.dbg_skip = 8;  // experiments: no L2 prefetch of batch g+3
    if (ov && std::getenv("LSG_OV_EVSTEP")) a.dbg_skip |= std::atoi(std::getenv("LSG_OV_EVSTEP")) << 8;
    if (a.prof) LSG_CUDA(cudaMemsetAsync(a.prof, 0, (16 + 256) * 8, st));
    const bool ov_prof = ov && std::getenv("LSG_PROFILE_OV");
    if (ov_prof) {
        a.prof = sc.get<unsigned long long>(32 + 8 * 16 + 2 * dm.T);
        if (!a.prof) return set_error(kInternal, "plan: scratch allocation failed");
        LSG_CUDA(cudaMemsetAsync(a.prof, 0, (32 + 8 * 16 + 2 * dm.T) * 8, st));
    }
    if (ov) {
        // team P: two parity sets of the six per-step arrays; CTA 0: team C's two sets of four
        const size_t smem = size_t(12) * dm.B * 4;
        LSG_CUDA(cudaFuncSetAttribute(k_plan_loop_ov, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(3);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 3;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        LSG_CUDA(cudaLaunchKernelEx(&cfg, k_plan_loop_ov, a));
    } else if (smem_items) {
        const size_t smem = exclusive_smem(size_t(6) * dm.B * 4);
        auto kern = dm.N <= 8 ? k_plan_loop<true, true> : k_plan_loop<true, false>;
        LSG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<1, kThreads, smem, st>>>(a);
    } else {
        const size_t smem = exclusive_smem(0);
        auto kern = dm.N <= 8 ? k_plan_loop<false, true> : k_plan_loop<false, false>;
        LSG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<1, kThreads, smem, st>>>(a);
    }
    LSG_LAUNCH_CHECK("k_plan_loop");
    if (ov_prof) {
        unsigned long long h[32];
        LSG_CUDA(cudaMemcpyAsync(h, a.prof, sizeof h, cudaMemcpyDeviceToHost, st));
        LSG_CUDA(cudaStreamSynchronize(st));
        const double T = double(dm.T ? dm.T : 1);
        fprintf(stderr, "[lsg ov] team D cyc/step: wait-classified %.0f  resolve %.0f  wait-verdict %.0f  publish %.0f\n",
                h[0] / T, h[1] / T, h[2] / T, h[3] / T);
        fprintf(stderr, "[lsg ov] team C cyc/step: wait-verdict %.0f  classify %.0f  wait-copy %.0f  copy %.0f; "
                "re-classified steps %llu\n", h[20] / T, h[21] / T, h[22] / T, h[23] / T, h[24]);
        fprintf(stderr, "[lsg ov] team P cyc/step: wait D/copy %.0f  apply %.0f  I2 %.0f  verdict %.0f  other %.0f  "
                "E %.0f  F %.0f  G1/G2 %.0f  H %.0f  I1 %.0f\n",
                h[13] / T, h[4] / T, h[5] / T, h[6] / T, h[7] / T, h[8] / T, h[9] / T, h[10] / T, h[11] / T, h[12] / T);
        unsigned long long e[8 * 16];
        LSG_CUDA(cudaMemcpyAsync(e, a.prof + 32, sizeof e, cudaMemcpyDeviceToHost, st));
        LSG_CUDA(cudaStreamSynchronize(st));
        const uint32_t g0 = uint32_t(a.dbg_skip) >> 8;
        if (dm.T >= g0 + 16) {
            const unsigned long long z = e[0];
            fprintf(stderr, "[lsg ov] ns from step %u's classify start: step | C classify | C copy | D resolve | P run\n", g0);
            for (int q = 0; q < 16; ++q)
                fprintf(stderr, "[lsg ov] %4u | %7lld %7lld | %7lld %7lld | %7lld %7lld | %7lld %7lld\n", g0 + q,
                        (long long)(e[q * 8 + 0] - z), (long long)(e[q * 8 + 1] - z), (long long)(e[q * 8 + 2] - z),
                        (long long)(e[q * 8 + 3] - z), (long long)(e[q * 8 + 4] - z), (long long)(e[q * 8 + 5] - z),
                        (long long)(e[q * 8 + 6] - z), (long long)(e[q * 8 + 7] - z));
        }
        std::vector<unsigned long long> pt(2 * dm.T);
        LSG_CUDA(cudaMemcpyAsync(pt.data(), a.prof + 32 + 128, pt.size() * 8, cudaMemcpyDeviceToHost, st));
        LSG_CUDA(cudaStreamSynchronize(st));
        std::vector<std::pair<long long, uint32_t>> waits;
        long long wsum = 0, rsum = 0;
        for (uint32_t g = 1; g < dm.T; ++g) {
            const long long wt = (long long)(pt[2 * g] - pt[2 * g - 1]);
            waits.push_back({wt, g});
            wsum += wt;
            rsum += (long long)(pt[2 * g + 1] - pt[2 * g]);
        }
        std::sort(waits.rbegin(), waits.rend());
        fprintf(stderr, "[lsg ov] team P: run %.2f us/step, wait %.2f us/step; longest waits (us@step):", rsum / 1e3 / dm.T,
                wsum / 1e3 / dm.T);
        for (size_t q = 0; q < std::min<size_t>(24, waits.size()); ++q)
            fprintf(stderr, " %.1f@%u", waits[q].first / 1e3, waits[q].second);
        fprintf(stderr, "\n");
        {  // by step in epoch (S steps)
            std::vector<double> wb(dm.S, 0.0), rb(dm.S, 0.0);
            for (uint32_t g = 1; g < dm.T; ++g) {
                wb[g % dm.S] += (double)(long long)(pt[2 * g] - pt[2 * g - 1]);
                rb[g % dm.S] += (double)(long long)(pt[2 * g + 1] - pt[2 * g]);
            }
            fprintf(stderr, "[lsg ov] team P wait/run us summed over epochs, by step in epoch:");
            for (uint32_t q = 0; q < dm.S; ++q) fprintf(stderr, " %u:%.0f/%.0f", q, wb[q] / 1e3, rb[q] / 1e3);
            fprintf(stderr, "\n");
            const uint32_t E = uint32_t(dm.T / dm.S);
            std::vector<double> we(E + 1, 0.0);
            for (uint32_t g = 1; g < dm.T; ++g) we[g / dm.S] += (double)(long long)(pt[2 * g] - pt[2 * g - 1]);
            fprintf(stderr, "[lsg ov] team P wait us by epoch:");
            for (uint32_t q = 0; q < E; ++q) fprintf(stderr, " %.0f", we[q] / 1e3);
            fprintf(stderr, "\n");
        }
        a.prof = nullptr;
    }
    if (a.prof) {
        unsigned long long h[16 + 256];
        LSG_CUDA(cudaMemcpyAsync(h, a.prof, sizeof h, cudaMemcpyDeviceToHost, st));
        LSG_CUDA(cudaStreamSynchronize(st));
        const char* names[10] = {"A load/classify", "B/C ranks", "D multi pass", "E positions/fetch ranks",
                                 "F pre-balance lists", "G1 balance moves", "G2 donor ranks", "H lists",
                                 "I1 hit rekey", "I2 fetch runs+evict"};
        unsigned long long tot = 0;
        for (int q = 0; q < 10; ++q) tot += h[q];

        fprintf(stderr, "[lsg profile] D: %llu multi-holder items (%.1f cyc/item incl. barrier, %.1f in the chain)\n",
                h[12], double(h[2]) / double(h[12] ? h[12] : 1), double(h[13]) / double(h[12] ? h[12] : 1));
        fprintf(stderr, "[lsg profile] plan loop T=%llu steps, %.1f Mcycles total\n",
                (unsigned long long)dm.T, tot / 1e6);
        for (int q = 0; q < 10; ++q)
            fprintf(stderr, "[lsg profile]   %-22s %10.1f kcyc  %6.2f%%  %8.0f cyc/step\n", names[q],
                    h[q] / 1e3, 100.0 * h[q] / (tot ? tot : 1), double(h[q]) / double(dm.T ? dm.T : 1));
    }
    return kOk;
}

}  // namespace lsg

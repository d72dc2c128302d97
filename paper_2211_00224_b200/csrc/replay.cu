// replay.cu — K7: per-rank clairvoyant replay of a plan (simulate_plan,
// buffer.cpp:183-247, with next_use_chain :103-112), bit-exact hits/misses
// per (step, node), plus the HBM slot each access lands in (for K8).
//
// Each node's buffer is independent: one WARP replays one node (4 nodes per
// CTA; ranks shard across GPUs by node range), so the per-run ordering below
// costs warp syncs only and the node state lives in (warp-uniform) registers.
// Keys are positions in the node's own flattened sequence, encoded g*L + i
// (g = step, i = index in the node's step list, L = longest node list),
// which orders exactly like the flattened position.
//
//  1. step bases (exclusive scan of step lengths), one block;
//  2. backward pass per node: next-use key of every access from a per-node
//     last-seen table, one step at a time, lane-parallel inside the step; a
//     (node, step) that repeats an id is rejected (the batched replay below
//     needs ids unique per (node, step), which every plan plan_schedule
//     emits satisfies);
//  3. forward replay per node: an item is a hit iff resident at step start
//     (misses insert keys beyond the step, so no current-step resident is ever
//     the eviction maximum); runs of hits re-key, runs of misses insert and
//     evict the (size-C)+ largest keys once the run ends. Residents are
//     indexed by (step of next use, list position) bitmaps. Every resident's
//     key is in the future, and an eviction never needs more than the future
//     residents, so the walk only meets exact buckets (a re-keyed hit leaves
//     a stale bit in its current step, which is never reached). kNeverUsed
//     residents sit in an id bitmap scanned from the top (ties by larger id,
//     buffer.cpp:27-28).
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "lru.cuh"

namespace lsg {

namespace {

constexpr int kRWarps = 4;  // nodes per CTA
constexpr uint32_t kRMaxList = 16384;

__device__ __forceinline__ uint32_t lanemask_lt_r() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// exclusive scan of node_off[g][N] over g -> gb[g] (one block, chunked)
__global__ void __launch_bounds__(1024) k_step_bases(const uint32_t* __restrict__ node_off, uint32_t T,
                                                     uint32_t N, uint64_t* __restrict__ gb) {
    __shared__ uint64_t part[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint32_t c = 0; c < T; c += 1024) {
        const uint32_t g = c + threadIdx.x;
        const uint64_t v = g < T ? node_off[size_t(g) * (N + 1) + N] : 0;
        uint64_t inc = v;
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= uint32_t(d)) inc += o;
        }
        if (lane == 31) part[w] = inc;
        __syncthreads();
        if (w == 0) {
            uint64_t p = part[lane], pi = p;
            for (int d = 1; d < 32; d <<= 1) {
                const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, pi, d);
                if (lane >= uint32_t(d)) pi += o;
            }
            part[lane] = pi - p;
        }
        __syncthreads();
        if (g < T) gb[g] = carry + part[w] + inc - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += part[w] + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) gb[T] = carry;
}

// largest sample id of a plan's lists (hit bit stripped): the replay indexes
// per-node tables by id, so ids >= dataset_size are rejected up front
__global__ void __launch_bounds__(256) k_max_id(const uint32_t* __restrict__ items, uint64_t n,
                                                uint32_t* __restrict__ out) {
    uint32_t m = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        m = max(m, __ldg(&items[i]) & ~kHit);
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

struct ReplayArgs {
    uint32_t T, N, D, L, C, k0, k1;
    uint32_t nzw, infw, bw;  // words: per-node step bitmap, id bitmap, per-step list bitmap
    const uint32_t* items;
    const uint32_t* node_off;
    const uint64_t* gb;
    uint32_t* nuk;     // [total items] next-use key per access
    uint32_t* last;    // [N][D]
    uint32_t* key;     // [N][D]  kNone = not resident
    uint32_t* slot;    // [N][D]
    uint32_t* nz;      // [N][nzw] next-use steps that may hold residents
    uint32_t* pbm;     // [N][T][bw] list positions per next-use step
    uint32_t* psum;    // [N][psw] non-empty pbm words
    uint32_t psw;
    uint32_t* psum2;   // [N][ps2w] non-empty psum words
    uint32_t ps2w;
    uint32_t* infbm;   // [N][infw]
    uint32_t* infsum;  // [N][sumw] non-empty infbm words
    uint32_t sumw;
    uint32_t* fstack;  // [N][C] freed slots (null when slots are not wanted)
    uint32_t* hits;    // [T][N]
    uint32_t* misses;  // [T][N]
    uint32_t* slot_out;  // [total items] or null
    uint32_t* status;
};

// backward pass: next-use key (g'*L + i') of every access on this node
__global__ void __launch_bounds__(kRWarps * 32) k_replay_nextuse(ReplayArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t k = a.k0 + blockIdx.x * kRWarps + (threadIdx.x >> 5);
    if (k >= a.k1) return;
    uint32_t* last = a.last + size_t(k) * a.D;
    for (int64_t g = int64_t(a.T) - 1; g >= 0; --g) {
        const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
        const uint32_t o = off[k], len = off[k + 1] - o;
        const uint64_t base = a.gb[g] + o;
        for (uint32_t i = lane; i < len; i += 32) {
            const uint32_t x = a.items[base + i] & ~kHit;
            const uint32_t v = __ldcg(&last[x]);
            a.nuk[base + i] = v == kNone ? kNever : v;
        }
        __syncwarp();
        const uint32_t here = uint32_t(g) * a.L;
        for (uint32_t i = lane; i < len; i += 32) {
            const uint32_t x = a.items[base + i] & ~kHit;
            const uint32_t old = atomicExch(&last[x], here + i);
            if (old != kNone && old / a.L == uint32_t(g)) atomicOr(a.status, 32u);  // repeat in step
        }
        __syncwarp();
    }
}

// Warp-uniform node state (every lane holds the same values).
struct NodeState {
    uint32_t size, top, inftop, infcnt, fresh, nfree, ptop;
};

// Take the `want` largest ids of a node's never-used bitmap (whole warp).
// The bitmap (bm, one bit per id) has a summary level (sm1, one bit per
// non-empty bm word), so the walk visits non-empty words only: new never-used
// residents land at random ids above the harvested region, and a flat walk
// would cross the whole id range on every eviction. Up to 32 non-empty words
// are gathered per round (wbuf, 32 shared words of this warp), lane 0 holding
// the highest; prefix sums of their popcounts tell each lane how many of its
// word's top bits go. Freed slots are pushed in eviction order (descending
// id). Returns the ids taken; `top` stays an upper bound of the highest word.
// bm_take generalises it to any summarised bitmap whose bit (word w, bit) names
// a resident through `idof`: the never-used id bitmap (identity) and the
// per-node key-space bitmap of finite keys (pbm, key = (step, list position),
// see key_take below).
template <class IdOf>
__device__ __forceinline__ uint32_t bm_take(uint32_t* bm, uint32_t* sm1, uint32_t* sm2, uint32_t& top, uint32_t want,
                                            IdOf idof, uint32_t* keyk, uint32_t* slotk, uint32_t* fs, uint32_t& nfree,
                                            uint32_t* wbuf, uint32_t lane) {
    const uint32_t lt = lanemask_lt_r();
    uint32_t taken = 0;
    int32_t cur = int32_t(top);  // highest bm word still to visit
    while (taken < want && cur >= 0) {
        // gather up to 32 non-empty bm words <= cur, descending
        uint32_t ngot = 0;
        int32_t sw = cur >> 5;
        uint32_t firstmask = (cur & 31) == 31 ? 0xFFFFFFFFu : ((2u << (cur & 31)) - 1u);
        bool skip = sm2 != nullptr;  // entering a possibly empty stretch
        while (ngot < 32 && sw >= 0) {
            if (skip) {
                // second summary level (one bit per non-empty sm1 word): jump to
                // the highest non-empty sm1 word <= sw, 1,024 sm1 words per round
                int32_t s2 = sw >> 5, found = -1;
                uint32_t m2 = (sw & 31) == 31 ? 0xFFFFFFFFu : ((2u << (sw & 31)) - 1u);
                while (s2 >= 0) {
                    const int32_t my2 = s2 - int32_t(lane);
                    uint32_t v2 = my2 >= 0 ? __ldcg(&sm2[my2]) : 0u;
                    if (lane == 0) v2 &= m2;
                    const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, v2 != 0);
                    if (b2) {
                        const uint32_t src = __ffs(b2) - 1;
                        const uint32_t word = __shfl_sync(0xFFFFFFFFu, v2, src);
                        found = (s2 - int32_t(src)) * 32 + int32_t(31 - __clz(word));
                        break;
                    }
                    s2 -= 32;
                    m2 = 0xFFFFFFFFu;
                }
                if (found < 0) break;
                if (found < sw) {
                    sw = found;
                    firstmask = 0xFFFFFFFFu;
                }
            }
            const int32_t myws = sw - int32_t(lane);
            uint32_t v = myws >= 0 ? __ldcg(&sm1[myws]) : 0u;
            if (lane == 0) v &= firstmask;
            const uint32_t c = __popc(v);
            uint32_t incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= uint32_t(d)) incl += o;
            }
            uint32_t r = ngot + incl - c;
            while (v && r < 32) {
                const uint32_t bit = 31 - __clz(v);
                v &= ~(1u << bit);
                wbuf[r++] = uint32_t(myws) * 32 + bit;
            }
            const uint32_t found1 = __shfl_sync(0xFFFFFFFFu, incl, 31);
            ngot += found1;
            skip = sm2 != nullptr && found1 == 0;
            sw -= 32;
            firstmask = 0xFFFFFFFFu;
        }
        __syncwarp();
        ngot = min(ngot, 32u);
        if (ngot == 0) break;
        const int32_t myw = lane < ngot ? int32_t(wbuf[lane]) : -1;
        const uint32_t lastw = wbuf[ngot - 1];
        __syncwarp();
        const uint32_t v = myw >= 0 ? __ldcg(&bm[myw]) : 0u;
        const uint32_t cnt = __popc(v);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= uint32_t(d)) incl += o;
        }
        const uint32_t before = incl - cnt, left = want - taken;
        const uint32_t take = before < left ? min(cnt, left - before) : 0u;
        // pass 1: which of my taken ids hold a slot (a miss of the current
        // run has none yet). Ids of the word's top `take` bits, 4 at a time so
        // their loads overlap (the key-space bitmap maps a bit to a list item)
        const uint64_t wb = myw >= 0 ? uint64_t(idof.base(uint32_t(myw))) : 0ull;
        uint32_t rest = v, pushes = 0;
        for (uint32_t t = 0; t < take; t += 4) {
            uint32_t xs[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool on = t + u < take;
                const uint32_t bit = on ? 31 - __clz(rest) : 0u;
                if (on) rest &= ~(1u << bit);
                xs[u] = on ? idof.id(wb, bit) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (t + u < take && fs && __ldcg(&slotk[xs[u]]) != kNone) ++pushes;
        }
        uint32_t pinc = pushes;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, pinc, d);
            if (lane >= uint32_t(d)) pinc += o;
        }
        uint32_t q = nfree + pinc - pushes;
        rest = v;
        for (uint32_t t = 0; t < take; t += 4) {
            uint32_t xs[4], sls[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool on = t + u < take;
                const uint32_t bit = on ? 31 - __clz(rest) : 0u;
                if (on) rest &= ~(1u << bit);
                xs[u] = on ? idof.id(wb, bit) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) sls[u] = t + u < take ? slotk[xs[u]] : kNone;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (t + u >= take) break;
                keyk[xs[u]] = kNone;
                if (sls[u] != kNone) {
                    if (fs) fs[q++] = sls[u];
                    slotk[xs[u]] = kNone;
                }
            }
        }
        if (take) {
            bm[myw] = rest;
            if (rest == 0) {
                const uint32_t old1 = atomicAnd(&sm1[myw >> 5], ~(1u << (myw & 31)));
                if (sm2 && (old1 & ~(1u << (myw & 31))) == 0) atomicAnd(&sm2[myw >> 10], ~(1u << ((myw >> 5) & 31)));
            }
        }
        nfree += __shfl_sync(0xFFFFFFFFu, pinc, 31);
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const uint32_t got = min(tot, left);
        taken += got;
        if (got < tot || taken >= want) {  // stopped inside this round
            const uint32_t tb = __ballot_sync(0xFFFFFFFFu, take > 0);
            cur = tb ? int32_t(__shfl_sync(0xFFFFFFFFu, uint32_t(myw), 31 - __clz(tb))) : cur;
            break;
        }
        cur = int32_t(lastw) - 1;
    }
    top = cur < 0 ? 0u : uint32_t(cur);
    __syncwarp();
    return taken;
}

struct IdIdentity {
    __device__ __forceinline__ uint32_t base(uint32_t w) const { return w * 32; }
    __device__ __forceinline__ uint32_t id(uint64_t b, uint32_t bit) const { return uint32_t(b) + bit; }
};

__device__ __forceinline__ uint32_t never_take(uint32_t* bm, uint32_t* sm1, uint32_t& top, uint32_t want,
                                               uint32_t* keyk, uint32_t* slotk, uint32_t* fs, uint32_t& nfree,
                                               uint32_t* wbuf, uint32_t lane) {
    return bm_take(bm, sm1, nullptr, top, want, IdIdentity{}, keyk, slotk, fs, nfree, wbuf, lane);
}

// Finite keys: node k's (step, list position) bitmap is bw words per step, so
// word w = beta * bw + p / 32 and the resident is the item at position p of
// the node's list at step beta. The summary (one bit per non-empty pbm word)
// lets an eviction take the largest keys 32 words per round, whatever the
// spread of next-use steps (a walk bucket by bucket pays a round trip per
// step holding residents: cfg5, 1,000 epochs).
struct IdOfKey {
    const uint32_t* items;
    const uint32_t* node_off;
    const uint64_t* gb;
    uint32_t N, k, bw;
    // item index of the word's bit 0 (64-bit plans: the item array offset)
    __device__ __forceinline__ uint64_t base(uint32_t w) const {
        const uint32_t beta = w / bw;
        return __ldg(&gb[beta]) + __ldg(&node_off[size_t(beta) * (N + 1) + k]) + (w - beta * bw) * 32;
    }
    __device__ __forceinline__ uint32_t id(uint64_t b, uint32_t bit) const { return __ldg(&items[b + bit]) & ~kHit; }
};

__device__ __forceinline__ void key_mark(uint32_t* pbmk, uint32_t* psumk, uint32_t* psum2k, uint32_t bw, uint32_t L,
                                         uint32_t nu) {
    const uint32_t beta = nu / L, p = nu - beta * L;
    const uint32_t w = beta * bw + (p >> 5);
    red_or(&pbmk[w], 1u << (p & 31));  // (idempotent ORs: no need to read the summary back)
    red_or(&psumk[w >> 5], 1u << (w & 31));
    red_or(&psum2k[w >> 10], 1u << ((w >> 5) & 31));
}

// Evict the `need` largest keys of node k (whole warp).
__device__ void r_evict(const ReplayArgs& a, NodeState& ns, uint32_t k, uint32_t need, uint32_t lane,
                        uint32_t lt, uint32_t* wbuf) {
    uint32_t* keyk = a.key + size_t(k) * a.D;
    uint32_t* slotk = a.slot + size_t(k) * a.D;
    uint32_t* fs = a.fstack ? a.fstack + size_t(k) * a.C : nullptr;
    while (need > 0) {
        if (ns.infcnt > 0) {  // never used again on this node: ids descending
            const uint32_t got = never_take(a.infbm + size_t(k) * a.infw, a.infsum + size_t(k) * a.sumw, ns.inftop,
                                            min(need, ns.infcnt), keyk, slotk, fs, ns.nfree, wbuf, lane);
            if (got == 0) {
                if (lane == 0) atomicOr(a.status, 2u);
                ns.infcnt = 0;
            }
            ns.infcnt -= min(got, ns.infcnt);
            ns.size -= got;
            need -= got;
            continue;
        }
        const IdOfKey idof{a.items, a.node_off, a.gb, a.N, k, a.bw};
        const uint32_t got = bm_take(a.pbm + size_t(k) * a.T * a.bw, a.psum + size_t(k) * a.psw,
                                     a.psum2 + size_t(k) * a.ps2w, ns.ptop, need, idof,
                                     keyk, slotk, fs, ns.nfree, wbuf, lane);
        if (got == 0) {
            if (lane == 0) atomicOr(a.status, 4u);
            return;
        }
        ns.size -= got;
        need -= got;
    }
}

__global__ void __launch_bounds__(kRWarps * 32) k_replay(ReplayArgs a) {
    extern __shared__ __align__(16) uint32_t rdyn[];
    __shared__ uint32_t rwbuf[kRWarps][32];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t k = a.k0 + blockIdx.x * kRWarps + wib;
    if (k >= a.k1) return;
    const uint32_t lt = lanemask_lt_r();
    uint32_t* sx = rdyn + size_t(wib) * a.L;  // this node's list: id | resident-at-start bit
    uint32_t* keyk = a.key + size_t(k) * a.D;
    uint32_t* slotk = a.slot + size_t(k) * a.D;
    uint32_t* fs = a.fstack ? a.fstack + size_t(k) * a.C : nullptr;
    uint32_t* infk = a.infbm + size_t(k) * a.infw;
    NodeState ns{0, 0, 0, 0, 0, 0, 0};
    for (uint32_t g = 0; g < a.T; ++g) {
        const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
        const uint32_t o = off[k], len = off[k + 1] - o;
        const uint64_t base = a.gb[g] + o;
        // load + residency at step start
        uint32_t hitc = 0;
        for (uint32_t i = lane; i < len; i += 32) {
            const uint32_t x = a.items[base + i] & ~kHit;
            const bool res = __ldcg(&keyk[x]) != kNone;
            sx[i] = x | (res ? kHit : 0u);
            if (a.slot_out && res) a.slot_out[base + i] = slotk[x] | kHit;
            hitc += res;
        }
        hitc = __reduce_add_sync(0xFFFFFFFFu, hitc);
        if (lane == 0) {
            a.hits[size_t(g) * a.N + k] = hitc;
            a.misses[size_t(g) * a.N + k] = len - hitc;
        }
        __syncwarp();
        // runs in list order; a miss run may span chunks and is evicted once
        bool pending = false;
        uint32_t run0 = 0;
        auto flush = [&](uint32_t run1) {
            const uint32_t need = ns.size > a.C ? ns.size - a.C : 0u;
            if (need) r_evict(a, ns, k, need, lane, lt, rwbuf[wib]);
            __syncwarp();
            if (fs) {  // survivors of the run take slots, in list order
                for (uint32_t c = run0; c < run1; c += 32) {
                    const uint32_t i = c + lane;
                    bool surv = false;
                    uint32_t x = 0;
                    if (i < run1) {
                        x = sx[i] & ~kHit;
                        surv = __ldcg(&keyk[x]) != kNone;
                    }
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, surv);
                    const uint32_t rank = __popc(bal & lt);
                    if (surv) slotk[x] = rank < ns.nfree ? fs[ns.nfree - 1 - rank] : ns.fresh + (rank - ns.nfree);
                    const uint32_t n = __popc(bal);
                    const uint32_t from_stack = min(n, ns.nfree);
                    ns.nfree -= from_stack;
                    ns.fresh += n - from_stack;
                    __syncwarp();
                }
            }
            pending = false;
        };
        for (uint32_t c = 0; c < len; c += 32) {
            const uint32_t i = c + lane;
            const bool valid = i < len;
            const uint32_t v = valid ? sx[i] : 0u;
            const uint32_t x = v & ~kHit;
            const uint32_t nu = valid ? a.nuk[base + i] : kNever;
            const uint32_t vbal = __ballot_sync(0xFFFFFFFFu, valid);
            const uint32_t rbal = __ballot_sync(0xFFFFFFFFu, valid && (v & kHit));
            uint32_t done = 0;
            while (done != vbal) {
                const uint32_t first = __ffs(vbal & ~done) - 1;
                const bool hitrun = (rbal >> first) & 1u;
                const uint32_t same = hitrun ? rbal : (vbal & ~rbal);
                const uint32_t after = (~same) & vbal & ~((2u << first) - 1u);
                const uint32_t stop = after ? __ffs(after) - 1 : 32u;
                const uint32_t run = (stop == 32 ? 0xFFFFFFFFu : ((1u << stop) - 1u)) & ~((1u << first) - 1u) & vbal;
                if (hitrun && pending) flush(c + first);
                const bool mine = (run >> lane) & 1u;
                const bool nev = mine && nu == kNever;
                if (mine) {  // buffer.cpp:37-46 without the eviction
                    keyk[x] = nu;
                    if (nev) {
                        red_or(&infk[x >> 5], 1u << (x & 31));
                        red_or(&a.infsum[size_t(k) * a.sumw + (x >> 10)], 1u << ((x >> 5) & 31));
                    } else {
                        key_mark(a.pbm + size_t(k) * a.T * a.bw, a.psum + size_t(k) * a.psw,
                                 a.psum2 + size_t(k) * a.ps2w, a.bw, a.L, nu);
                    }
                }
                const uint32_t nevb = __ballot_sync(0xFFFFFFFFu, nev);
                ns.infcnt += __popc(nevb);
                ns.inftop = max(ns.inftop, __reduce_max_sync(0xFFFFFFFFu, nev ? (x >> 5) : 0u));
                ns.ptop = max(ns.ptop, __reduce_max_sync(0xFFFFFFFFu, (mine && !nev) ? (nu / a.L) * a.bw +
                                                                               ((nu - (nu / a.L) * a.L) >> 5) : 0u));
                if (!hitrun) {
                    ns.size += __popc(run);
                    if (!pending) run0 = c + first;
                    pending = true;
                }
                __syncwarp();
                done |= run;
            }
        }
        if (pending) flush(len);
        // misses report the slot they hold at the END of the step (one that a
        // later run of the same step evicted again is a bypass)
        if (a.slot_out)
            for (uint32_t i = lane; i < len; i += 32) {
                const uint32_t v = sx[i];
                if (v & kHit) continue;
                const uint32_t x = v & ~kHit;
                a.slot_out[base + i] = __ldcg(&keyk[x]) != kNone ? slotk[x] : kNever;
            }
        __syncwarp();
    }
}

// ---- long node lists (L > 128): one CTA per node, candidates of a bucket are
// the node's list at that step scanned from its end (the round-1 design).
constexpr int kRT = 256;

struct ReplayArgsCta {
    uint32_t T, N, D, B, C, k0;
    uint32_t nzw, infw;
    const uint32_t* items;
    const uint32_t* node_off;
    const uint64_t* gb;
    uint32_t* nuk;     // [total items] next-use key per access
    uint32_t* last;    // [N][D]
    uint32_t* key;     // [N][D]
    uint32_t* slot;    // [N][D]
    uint32_t* nz;      // [N][nzw]
    uint32_t* pbm;     // [N][T][bw] list positions per next-use step, or null (list scan)
    uint32_t bw;
    uint32_t* psum;    // [N][psw] non-empty pbm words
    uint32_t psw;
    uint32_t* psum2;   // [N][ps2w] non-empty psum words
    uint32_t ps2w;
    uint32_t* infbm;   // [N][infw]
    uint32_t* infsum;  // [N][sumw] non-empty infbm words
    uint32_t sumw;
    uint32_t* fstack;  // [N][C] freed slots
    uint32_t* hits;    // [T][N]
    uint32_t* misses;  // [T][N]
    uint32_t* slot_out;  // [total items] or null
    uint32_t* status;
    // simulate_plan(..., insert_redundant = true) (buffer.cpp:224-238): the
    // redundant ids of list (g, k) are red_ids[red_off[g*N+k] .. +1], their
    // next position on the node red_key (filled by the backward pass)
    const uint64_t* red_off;  // [T*N+1] or null
    const uint32_t* red_ids;
    uint32_t* red_key;
};

// backward pass: next-use key (g'*B + i') of every access on this node
__global__ void __launch_bounds__(kRT) k_replay_nextuse_cta(ReplayArgsCta a) {
    const uint32_t k = a.k0 + blockIdx.x;
    uint32_t* last = a.last + size_t(k) * a.D;
    for (int64_t g = int64_t(a.T) - 1; g >= 0; --g) {
        const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
        const uint32_t o = off[k], L = off[k + 1] - o;
        const uint64_t base = a.gb[g] + o;
        for (uint32_t i = threadIdx.x; i < L; i += kRT) {
            const uint32_t x = a.items[base + i] & ~kHit;
            const uint32_t v = __ldcg(&last[x]);
            a.nuk[base + i] = v == kNone ? kNever : v;
        }
        __syncthreads();
        if (a.red_off) {  // silent inserts after step g: next position after the step
            const uint64_t q0 = a.red_off[size_t(g) * a.N + k], q1 = a.red_off[size_t(g) * a.N + k + 1];
            for (uint64_t q = q0 + threadIdx.x; q < q1; q += kRT) {
                const uint32_t v = __ldcg(&last[a.red_ids[q]]);
                a.red_key[q] = v == kNone ? kNever : v;
            }
            __syncthreads();
        }
        const uint32_t here = uint32_t(g) * a.B;
        for (uint32_t i = threadIdx.x; i < L; i += kRT) {
            const uint32_t x = a.items[base + i] & ~kHit;
            const uint32_t old = atomicExch(&last[x], here + i);
            if (old != kNone && old / a.B == uint32_t(g)) atomicOr(a.status, 32u);  // repeat in step
        }
        __syncthreads();
    }
}

// Next-use keys by SEGMENTS of steps, each fully parallel. A plan that
// plan_schedule emits holds every id at most once per epoch (over all
// nodes), so within an epoch-aligned segment an access's next use on its node
// lies in a LATER segment: walking the segments backward, every access of a
// segment reads its node's last-seen key of the id and replaces it with its
// own, all at once (atomicExch; no (node, id) is touched twice). One block per
// step of the segment. An id seen twice on a node inside the segment (a
// foreign plan) shows as a previous key inside the segment: flagged, and the
// caller redoes the pass serially per node. Streaming traffic is the item read
// and the key write (8 B per access); the [N][D] last-seen table is the
// random part (L2-resident at cfg2: 8 MB).
constexpr uint32_t kNuRows = 1024, kNuThreads = 256;  // rows per block, 4 per thread in flight

__global__ void __launch_bounds__(kNuThreads) k_nextuse_seg(const uint32_t* __restrict__ items,
                                                           const uint32_t* __restrict__ node_off,
                                                           const uint64_t* __restrict__ gb, uint32_t N, uint64_t D,
                                                           uint32_t L, uint32_t g0, uint32_t g1, uint32_t chunks,
                                                           uint32_t* __restrict__ last, uint32_t* __restrict__ nuk,
                                                           uint32_t* __restrict__ conflict) {
    extern __shared__ uint32_t soff[];  // [N+1] offsets of this block's step
    const uint32_t g = g0 + blockIdx.x / chunks, r0 = (blockIdx.x % chunks) * kNuRows;
    for (uint32_t k = threadIdx.x; k <= N; k += blockDim.x) soff[k] = __ldg(&node_off[size_t(g) * (N + 1) + k]);
    __syncthreads();
    const uint64_t base = __ldg(&gb[g]);
    const uint32_t len = soff[N];
    const uint64_t seg_lo = uint64_t(g0) * L, seg_hi = uint64_t(g1) * L;
    bool bad = false;
    uint32_t old[kNuRows / kNuThreads], rr[kNuRows / kNuThreads];
#pragma unroll
    for (uint32_t u = 0; u < kNuRows / kNuThreads; ++u) {  // independent atomics, all in flight
        const uint32_t r = r0 + u * kNuThreads + threadIdx.x;
        rr[u] = r;
        old[u] = kNone;
        if (r >= len) continue;
        uint32_t lo = 0, hi = N;  // node of row r: soff[lo] <= r < soff[lo + 1]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (soff[mid] <= r) lo = mid; else hi = mid;
        }
        const uint32_t x = __ldcs(&items[base + r]) & ~kHit;
        old[u] = atomicExch(&last[size_t(lo) * D + x], g * L + (r - soff[lo]));
    }
#pragma unroll
    for (uint32_t u = 0; u < kNuRows / kNuThreads; ++u) {
        if (rr[u] >= len) continue;
        __stcs(&nuk[base + rr[u]], old[u] == kNone ? kNever : old[u]);
        bad |= old[u] != kNone && uint64_t(old[u]) >= seg_lo && uint64_t(old[u]) < seg_hi;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(conflict, 1u);
}

struct RSharedCta {
    uint32_t size, top, inftop, infcnt, fresh, nfree, ptop;
    uint32_t wbuf[32];  // never_take gather
    uint32_t nruns;
    uint32_t hitcnt;
    uint32_t wsum[kRT / 32];
};

__device__ __forceinline__ void r_set_key_cta(const ReplayArgsCta& a, RSharedCta& sh, uint32_t k, uint32_t x,
                                          uint32_t nu) {
    a.key[size_t(k) * a.D + x] = nu;
    if (nu == kNever) {
        red_or(&a.infbm[size_t(k) * a.infw + (x >> 5)], 1u << (x & 31));
        red_or(&a.infsum[size_t(k) * a.sumw + (x >> 10)], 1u << ((x >> 5) & 31));
        atomicAdd(&sh.infcnt, 1u);
        atomicMax(&sh.inftop, x >> 5);
    } else {
        const uint32_t beta = nu / a.B;
        red_or(&a.nz[size_t(k) * a.nzw + (beta >> 5)], 1u << (beta & 31));
        atomicMax(&sh.top, beta);
        if (a.pbm) {
            key_mark(a.pbm + size_t(k) * a.T * a.bw, a.psum + size_t(k) * a.psw, a.psum2 + size_t(k) * a.ps2w, a.bw,
                     a.B, nu);
            atomicMax(&sh.ptop, beta * a.bw + ((nu - beta * a.B) >> 5));
        }
    }
}

// evict the `need` largest keys of node k (warp 0)
__device__ void r_evict_cta(const ReplayArgsCta& a, RSharedCta& sh, uint32_t k, uint32_t need, uint32_t lane) {
    const uint32_t lt = lanemask_lt_r();
    uint32_t* keyk = a.key + size_t(k) * a.D;
    uint32_t* slotk = a.slot + size_t(k) * a.D;
    uint32_t* fs = a.fstack + size_t(k) * a.C;
    while (need > 0) {
        if (sh.infcnt > 0) {  // never used again on this node: ids descending
            uint32_t top = sh.inftop, nf = sh.nfree;
            __syncwarp();
            const uint32_t got = never_take(a.infbm + size_t(k) * a.infw, a.infsum + size_t(k) * a.sumw, top,
                                            min(need, sh.infcnt), keyk, slotk, a.fstack ? fs : nullptr, nf,
                                            sh.wbuf, lane);
            if (lane == 0) {
                sh.inftop = top;
                sh.nfree = nf;
                if (got == 0) {
                    atomicOr(a.status, 2u);
                    sh.infcnt = 0;
                }
                sh.infcnt -= min(got, sh.infcnt);
                sh.size -= got;
            }
            __syncwarp();
            need -= got;
            continue;
        }
        if (a.pbm) {  // largest finite keys, 32 key-space words per round
            uint32_t top = sh.ptop, nf = sh.nfree;
            __syncwarp();
            const IdOfKey idof{a.items, a.node_off, a.gb, a.N, k, a.bw};
            const uint32_t got = bm_take(a.pbm + size_t(k) * a.T * a.bw, a.psum + size_t(k) * a.psw,
                                         a.psum2 + size_t(k) * a.ps2w, top, need, idof,
                                         keyk, slotk, a.fstack ? fs : nullptr, nf, sh.wbuf, lane);
            if (lane == 0) {
                sh.ptop = top;
                sh.nfree = nf;
                sh.size -= got;
                if (got == 0) atomicOr(a.status, 4u);
            }
            __syncwarp();
            if (got == 0) return;
            need -= got;
            continue;
        }
        uint32_t* nzk = a.nz + size_t(k) * a.nzw;
        int32_t wi = int32_t(sh.top >> 5);
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
        const uint32_t* off = a.node_off + size_t(beta) * (a.N + 1);
        const uint32_t o = off[k], L = off[k + 1] - o;
        const uint64_t base = a.gb[beta] + o;

        const uint32_t kb = uint32_t(beta) * a.B;
        uint32_t c = 0;
        for (; c < L && need > 0; c += 128) {
            uint32_t xs[4];
            bool ms[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // reverse list order: largest position first
                const uint32_t r = c + 32 * u + lane;
                xs[u] = r < L ? (a.items[base + (L - 1 - r)] & ~kHit) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t r = c + 32 * u + lane;
                ms[u] = r < L && __ldcg(&keyk[xs[u]]) == kb + (L - 1 - r);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
            const uint32_t x = xs[u];
            const bool mem = ms[u];
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, mem);
            const uint32_t rank = __popc(bal & lt);
            const uint32_t took = min(uint32_t(__popc(bal)), need);
            const bool ev = mem && rank < need;
            uint32_t s = kNone;
            if (ev) {
                keyk[x] = kNone;
                s = slotk[x];
                slotk[x] = kNone;
            }
            // freed slots pushed in eviction order (deterministic)
            const bool push = ev && s != kNone && a.fstack;
            const uint32_t sbal = __ballot_sync(0xFFFFFFFFu, push);
            const uint32_t nf = sh.nfree;
            if (push) fs[nf + __popc(sbal & lt)] = s;
            __syncwarp();
            need -= took;
            if (lane == 0) {
                sh.size -= took;
                sh.nfree = nf + __popc(sbal);
            }
            __syncwarp();
            }
        }
        if (c >= L && need > 0 && lane == 0) atomicAnd(&nzk[beta >> 5], ~(1u << (beta & 31)));
        if (lane == 0) sh.top = uint32_t(beta);
        __syncwarp();
    }
}

// forward replay, one CTA per node
__global__ void __launch_bounds__(kRT) k_replay_cta(ReplayArgsCta a) {
    __shared__ RSharedCta sh;
    extern __shared__ __align__(16) uint32_t rdyn[];
    uint32_t* sx = rdyn;                                       // [B] ids | resident bit
    uint16_t* rstart = reinterpret_cast<uint16_t*>(rdyn + a.B);  // [B+1] run starts
    const uint32_t k = a.k0 + blockIdx.x;
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) {
        sh.size = 0;
        sh.top = 0;
        sh.ptop = 0;
        sh.inftop = 0;
        sh.infcnt = 0;
        sh.fresh = 0;
        sh.nfree = 0;
    }
    __syncthreads();
    uint32_t* keyk = a.key + size_t(k) * a.D;
    uint32_t* slotk = a.slot + size_t(k) * a.D;
    uint32_t* fs = a.fstack + size_t(k) * a.C;
    for (uint32_t g = 0; g < a.T; ++g) {
        const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
        const uint32_t o = off[k], L = off[k + 1] - o;
        const uint64_t base = a.gb[g] + o;
        if (L > kRMaxList) {
            if (tid == 0) atomicOr(a.status, 64u);
            return;
        }
        // load + residency at step start; run boundaries
        uint32_t hitc = 0;
        for (uint32_t c = 0; c < L; c += kRT) {
            const uint32_t i = c + tid;
            bool res = false, chg = false;
            if (i < L) {
                const uint32_t x = a.items[base + i] & ~kHit;
                res = __ldcg(&keyk[x]) != kNone;
                sx[i] = x | (res ? kHit : 0u);
                if (a.slot_out) a.slot_out[base + i] = res ? (slotk[x] | kHit) : kNever;
                hitc += res;
            }
            __syncthreads();
            if (i < L) chg = i == 0 || ((sx[i] ^ sx[i - 1]) & kHit);
            // block-wide prefix of chg (run ids), chunk-local then carried
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, chg);
            if (lane == 0) sh.wsum[w] = __popc(bal);
            __syncthreads();
            if (tid == 0) {
                uint32_t s = c == 0 ? 0u : sh.nruns;
                for (int q = 0; q < kRT / 32; ++q) { const uint32_t v = sh.wsum[q]; sh.wsum[q] = s; s += v; }
                sh.nruns = s;
            }
            __syncthreads();
            if (i < L) {
                const uint32_t rid = sh.wsum[w] + __popc(bal & lanemask_lt_r()) + (chg ? 1u : 0u) - 1u;
                if (chg) rstart[rid] = uint16_t(i);
            }
            __syncthreads();
        }
        // hit count
        for (int s = 16; s > 0; s >>= 1) hitc += __shfl_xor_sync(0xFFFFFFFFu, hitc, s);
        if (lane == 0) sh.wsum[w] = hitc;
        __syncthreads();
        if (tid == 0) {
            uint32_t h = 0;
            for (int q = 0; q < kRT / 32; ++q) h += sh.wsum[q];
            a.hits[size_t(g) * a.N + k] = h;
            a.misses[size_t(g) * a.N + k] = L - h;
            rstart[sh.nruns] = uint16_t(L);
        }
        __syncthreads();
        const uint32_t nruns = L ? sh.nruns : 0;
        for (uint32_t r = 0; r < nruns; ++r) {
            const uint32_t r0 = rstart[r], r1 = rstart[r + 1];
            const bool hitrun = sx[r0] & kHit;
            for (uint32_t i = r0 + tid; i < r1; i += kRT)
                r_set_key_cta(a, sh, k, sx[i] & ~kHit, a.nuk[base + i]);
            __syncthreads();
            if (!hitrun) {
                if (w == 0) {
                    uint32_t need = 0;
                    if (lane == 0) {
                        sh.size += r1 - r0;
                        need = sh.size > a.C ? sh.size - a.C : 0u;
                    }
                    need = __shfl_sync(0xFFFFFFFFu, need, 0);
                    if (need) r_evict_cta(a, sh, k, need, lane);
                    __syncwarp();
                    // survivors of the run take slots, in list order
                    if (a.slot_out) {
                        for (uint32_t c = r0; c < r1; c += 32) {
                            const uint32_t i = c + lane;
                            bool surv = false;
                            uint32_t x = 0;
                            if (i < r1) {
                                x = sx[i] & ~kHit;
                                surv = __ldcg(&keyk[x]) != kNone;
                            }
                            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, surv);
                            const uint32_t rank = __popc(bal & lanemask_lt_r());
                            const uint32_t nf = sh.nfree, fr = sh.fresh;
                            if (surv) {
                                uint32_t s;
                                if (rank < nf) s = fs[nf - 1 - rank];
                                else s = fr + (rank - nf);
                                slotk[x] = s;  // reported at the end of the step
                            }
                            __syncwarp();
                            if (lane == 0) {
                                const uint32_t n = __popc(bal);
                                const uint32_t from_stack = min(n, nf);
                                sh.nfree = nf - from_stack;
                                sh.fresh = fr + (n - from_stack);
                            }
                            __syncwarp();
                        }
                    }
                }
                __syncthreads();
            }
        }
        // insert_silent of the step's redundant ids (buffer.cpp:48-53): the
        // non-resident ones form one more miss run (keep-C-smallest is
        // associative); slots are not tracked on this path
        if (a.red_off) {
            const uint64_t q0 = a.red_off[size_t(g) * a.N + k], q1 = a.red_off[size_t(g) * a.N + k + 1];
            uint32_t ins = 0;
            for (uint64_t q = q0 + tid; q < q1; q += kRT) {
                const uint32_t y = a.red_ids[q];
                if (__ldcg(&keyk[y]) != kNone) continue;
                r_set_key_cta(a, sh, k, y, a.red_key[q]);
                ++ins;
            }
            for (int d = 16; d > 0; d >>= 1) ins += __shfl_xor_sync(0xFFFFFFFFu, ins, d);
            if (lane == 0) atomicAdd(&sh.size, ins);
            __syncthreads();
            if (w == 0) {
                const uint32_t need = sh.size > a.C ? sh.size - a.C : 0u;
                if (need) r_evict_cta(a, sh, k, need, lane);
            }
            __syncthreads();
        }
        // misses report the slot they hold at the END of the step: one that
        // a later run of the same step evicted again is a bypass (its slot may
        // already belong to another miss of this step)
        if (a.slot_out)
            for (uint32_t i = tid; i < L; i += kRT) {
                const uint32_t v = sx[i];
                if (v & kHit) continue;
                const uint32_t x = v & ~kHit;
                a.slot_out[base + i] = __ldcg(&keyk[x]) != kNone ? slotk[x] : kNever;
            }
        __syncthreads();
    }
}

// ---- the CHAIN replay (clairvoyant, no silent inserts): no id-indexed
// key/slot tables. A resident is keyed by the position of its next access on
// the node, so "the access at position q is a hit" is exactly "the key-space
// bitmap holds bit q" (keys are (step, list position); the bit of an access
// already served is never reached again, see r_evict_cta). Slots travel along
// the same chain: when a resident is (re)keyed to position q, its slot is
// written AHEAD into slot_out[q], so a hit finds its slot at its own index
// and an eviction by key reads it there; residents never used again keep
// theirs in an id-indexed array touched once at insert and once at eviction.
// Per access the streaming traffic is the id, the next-use key and the slot
// word; the random part is the key-space bitmap (a window of a few epochs:
// L2-resident).
template <class Take>
__device__ __forceinline__ uint32_t bm_take_h(uint32_t* bm, uint32_t* sm1, uint32_t* sm2, uint32_t& top, uint32_t want,
                                              Take take, uint32_t* fs, uint32_t& nfree, uint32_t* wbuf, uint32_t lane) {
    // bm_take with a per-taken-bit callback: take(word, bit) retires the
    // resident and returns its slot (kNone: none yet) for the free stack
    const uint32_t lt = lanemask_lt_r();
    uint32_t taken = 0;
    int32_t cur = int32_t(top);
    while (taken < want && cur >= 0) {
        uint32_t ngot = 0;
        int32_t sw = cur >> 5;
        uint32_t firstmask = (cur & 31) == 31 ? 0xFFFFFFFFu : ((2u << (cur & 31)) - 1u);
        bool skip = sm2 != nullptr;
        while (ngot < 32 && sw >= 0) {
            if (skip) {
                int32_t s2 = sw >> 5, found = -1;
                uint32_t m2 = (sw & 31) == 31 ? 0xFFFFFFFFu : ((2u << (sw & 31)) - 1u);
                while (s2 >= 0) {
                    const int32_t my2 = s2 - int32_t(lane);
                    uint32_t v2 = my2 >= 0 ? __ldcg(&sm2[my2]) : 0u;
                    if (lane == 0) v2 &= m2;
                    const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, v2 != 0);
                    if (b2) {
                        const uint32_t src = __ffs(b2) - 1;
                        const uint32_t word = __shfl_sync(0xFFFFFFFFu, v2, src);
                        found = (s2 - int32_t(src)) * 32 + int32_t(31 - __clz(word));
                        break;
                    }
                    s2 -= 32;
                    m2 = 0xFFFFFFFFu;
                }
                if (found < 0) break;
                if (found < sw) {
                    sw = found;
                    firstmask = 0xFFFFFFFFu;
                }
            }
            const int32_t myws = sw - int32_t(lane);
            uint32_t v = myws >= 0 ? __ldcg(&sm1[myws]) : 0u;
            if (lane == 0) v &= firstmask;
            const uint32_t c = __popc(v);
            uint32_t incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= uint32_t(d)) incl += o;
            }
            uint32_t r = ngot + incl - c;
            while (v && r < 32) {
                const uint32_t bit = 31 - __clz(v);
                v &= ~(1u << bit);
                wbuf[r++] = uint32_t(myws) * 32 + bit;
            }
            const uint32_t found1 = __shfl_sync(0xFFFFFFFFu, incl, 31);
            ngot += found1;
            skip = sm2 != nullptr && found1 == 0;
            sw -= 32;
            firstmask = 0xFFFFFFFFu;
        }
        __syncwarp();
        ngot = min(ngot, 32u);
        if (ngot == 0) break;
        const int32_t myw = lane < ngot ? int32_t(wbuf[lane]) : -1;
        const uint32_t lastw = wbuf[ngot - 1];
        __syncwarp();
        const uint32_t v = myw >= 0 ? __ldcg(&bm[myw]) : 0u;
        const uint32_t cnt = __popc(v);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= uint32_t(d)) incl += o;
        }
        const uint32_t before = incl - cnt, left = want - taken;
        const uint32_t take_n = before < left ? min(cnt, left - before) : 0u;
        // freed slots are pushed in eviction order (words descending, bits
        // descending): pass 1 counts them, pass 2 writes; 4 slot loads in flight
        uint32_t rest = v, mine = 0;
        if (fs)
            for (uint32_t t = 0; t < take_n; t += 4) {
                uint32_t sv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool on = t + u < take_n;
                    const uint32_t bit = on ? 31 - __clz(rest) : 0u;
                    if (on) rest &= ~(1u << bit);
                    sv[u] = on ? take(uint32_t(myw), bit) : kNone;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) mine += sv[u] != kNone;
            }
        uint32_t pinc = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, pinc, d);
            if (lane >= uint32_t(d)) pinc += o;
        }
        rest = v;
        uint32_t q = nfree + pinc - mine;
        for (uint32_t t = 0; t < take_n; t += 4) {
            uint32_t sv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool on = t + u < take_n;
                const uint32_t bit = on ? 31 - __clz(rest) : 0u;
                if (on) rest &= ~(1u << bit);
                sv[u] = (on && fs) ? take(uint32_t(myw), bit) : kNone;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (sv[u] != kNone) fs[q++] = sv[u];
        }
        if (take_n) {
            bm[myw] = rest;
            if (rest == 0) {
                const uint32_t old1 = atomicAnd(&sm1[myw >> 5], ~(1u << (myw & 31)));
                if (sm2 && (old1 & ~(1u << (myw & 31))) == 0) atomicAnd(&sm2[myw >> 10], ~(1u << ((myw >> 5) & 31)));
            }
        }
        nfree += __shfl_sync(0xFFFFFFFFu, pinc, 31);
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const uint32_t got = min(tot, left);
        taken += got;
        if (got < tot || taken >= want) {
            const uint32_t tb = __ballot_sync(0xFFFFFFFFu, take_n > 0);
            cur = tb ? int32_t(__shfl_sync(0xFFFFFFFFu, uint32_t(myw), 31 - __clz(tb))) : cur;
            break;
        }
        cur = int32_t(lastw) - 1;
        (void)lt;
    }
    top = cur < 0 ? 0u : uint32_t(cur);
    __syncwarp();
    return taken;
}

struct ChainCtx {
    const ReplayArgsCta* a;
    uint32_t k;
    __device__ __forceinline__ uint64_t pos_index(uint32_t key) const {  // key -> item index
        const uint32_t beta = key / a->B, p = key - beta * a->B;
        return __ldg(&a->gb[beta]) + __ldg(&a->node_off[size_t(beta) * (a->N + 1) + k]) + p;
    }
    __device__ __forceinline__ uint32_t* pbmk() const { return a->pbm + size_t(k) * a->T * a->bw; }
    __device__ __forceinline__ bool bit_set(uint32_t key) const {
        const uint32_t beta = key / a->B, p = key - beta * a->B;
        return (__ldcg(&pbmk()[size_t(beta) * a->bw + (p >> 5)]) >> (p & 31)) & 1u;
    }
    __device__ __forceinline__ bool never_set(uint32_t x) const {
        return (__ldcg(&a->infbm[size_t(k) * a->infw + (x >> 5)]) >> (x & 31)) & 1u;
    }
};

// (re)key a resident: finite keys in the key-space bitmap with the slot
// written ahead at that position, never-used ids in the id bitmap with the
// slot in the never-used slot array
__device__ __forceinline__ void chain_set(const ReplayArgsCta& a, RSharedCta& sh, const ChainCtx& cx, uint32_t x,
                                          uint32_t nu, uint32_t slot) {
    const uint32_t k = cx.k;
    if (nu == kNever) {
        red_or(&a.infbm[size_t(k) * a.infw + (x >> 5)], 1u << (x & 31));
        red_or(&a.infsum[size_t(k) * a.sumw + (x >> 10)], 1u << ((x >> 5) & 31));
        atomicAdd(&sh.infcnt, 1u);
        atomicMax(&sh.inftop, x >> 5);
        if (a.slot_out) a.slot[size_t(k) * a.D + x] = slot;
    } else {
        const uint32_t beta = nu / a.B;
        key_mark(cx.pbmk(), a.psum + size_t(k) * a.psw, a.psum2 + size_t(k) * a.ps2w, a.bw, a.B, nu);
        atomicMax(&sh.ptop, beta * a.bw + ((nu - beta * a.B) >> 5));
        if (a.slot_out) a.slot_out[cx.pos_index(nu)] = slot;
    }
}

// evict the `need` largest keys (warp 0)
__device__ void chain_evict(const ReplayArgsCta& a, RSharedCta& sh, const ChainCtx& cx, uint32_t need, uint32_t lane) {
    const uint32_t k = cx.k;
    uint32_t* fs = a.fstack ? a.fstack + size_t(k) * a.C : nullptr;
    while (need > 0) {
        if (sh.infcnt > 0) {  // never used again on this node: ids descending
            uint32_t top = sh.inftop, nf = sh.nfree;
            __syncwarp();
            uint32_t* nvs = a.slot + size_t(k) * a.D;
            const bool sl = a.slot_out != nullptr;
            auto take = [&](uint32_t w, uint32_t bit) -> uint32_t {
                const uint32_t x = w * 32 + bit;
                return sl ? __ldcg(&nvs[x]) : kNone;
            };
            const uint32_t got = bm_take_h(a.infbm + size_t(k) * a.infw, a.infsum + size_t(k) * a.sumw, nullptr, top,
                                           min(need, sh.infcnt), take, fs, nf, sh.wbuf, lane);
            if (lane == 0) {
                sh.inftop = top;
                sh.nfree = nf;
                if (got == 0) {
                    atomicOr(a.status, 2u);
                    sh.infcnt = 0;
                }
                sh.infcnt -= min(got, sh.infcnt);
                sh.size -= got;
            }
            __syncwarp();
            need -= got;
            continue;
        }
        uint32_t top = sh.ptop, nf = sh.nfree;
        __syncwarp();
        const bool sl = a.slot_out != nullptr;
        auto take = [&](uint32_t w, uint32_t bit) -> uint32_t {  // word w = beta * bw + p / 32
            if (!sl) return kNone;
            const uint32_t beta = w / a.bw;
            const uint64_t idx = __ldg(&a.gb[beta]) + __ldg(&a.node_off[size_t(beta) * (a.N + 1) + k]) +
                                 (w - beta * a.bw) * 32 + bit;
            return __ldcg(&a.slot_out[idx]);
        };
        const uint32_t got = bm_take_h(cx.pbmk(), a.psum + size_t(k) * a.psw, a.psum2 + size_t(k) * a.ps2w, top, need,
                                       take, fs, nf, sh.wbuf, lane);
        if (lane == 0) {
            sh.ptop = top;
            sh.nfree = nf;
            sh.size -= got;
            if (got == 0) atomicOr(a.status, 4u);
        }
        __syncwarp();
        if (got == 0) return;
        need -= got;
    }
}

__global__ void __launch_bounds__(kRT) k_replay_chain(ReplayArgsCta a) {
    __shared__ RSharedCta sh;
    extern __shared__ __align__(16) uint32_t rdyn[];
    uint32_t* sx = rdyn;                                         // [B] ids | resident bit
    uint16_t* rstart = reinterpret_cast<uint16_t*>(rdyn + a.B);  // [B+1] run starts
    const uint32_t k = a.k0 + blockIdx.x;
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const ChainCtx cx{&a, k};
    if (tid == 0) {
        sh.size = 0;
        sh.top = 0;
        sh.ptop = 0;
        sh.inftop = 0;
        sh.infcnt = 0;
        sh.fresh = 0;
        sh.nfree = 0;
    }
    __syncthreads();
    uint32_t* fs = a.fstack ? a.fstack + size_t(k) * a.C : nullptr;
    for (uint32_t g = 0; g < a.T; ++g) {
        const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
        const uint32_t o = off[k], L = off[k + 1] - o;
        const uint64_t base = a.gb[g] + o;
        if (L > kRMaxList) {
            if (tid == 0) atomicOr(a.status, 64u);
            return;
        }
        // residency at step start = the key-space bit of the access itself
        uint32_t hitc = 0;
        const uint32_t* pw = cx.pbmk() + size_t(g) * a.bw;
        for (uint32_t c = 0; c < L; c += kRT) {
            const uint32_t i = c + tid;
            bool chg = false;
            if (i < L) {
                const uint32_t x = a.items[base + i] & ~kHit;
                const bool res = (__ldcg(&pw[i >> 5]) >> (i & 31)) & 1u;
                sx[i] = x | (res ? kHit : 0u);
                if (a.slot_out && res) a.slot_out[base + i] |= kHit;  // its slot was written ahead
                hitc += res;
            }
            __syncthreads();
            if (i < L) chg = i == 0 || ((sx[i] ^ sx[i - 1]) & kHit);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, chg);
            if (lane == 0) sh.wsum[w] = __popc(bal);
            __syncthreads();
            if (tid == 0) {
                uint32_t s2 = c == 0 ? 0u : sh.nruns;
                for (int q = 0; q < kRT / 32; ++q) { const uint32_t v = sh.wsum[q]; sh.wsum[q] = s2; s2 += v; }
                sh.nruns = s2;
            }
            __syncthreads();
            if (i < L) {
                const uint32_t rid = sh.wsum[w] + __popc(bal & lanemask_lt_r()) + (chg ? 1u : 0u) - 1u;
                if (chg) rstart[rid] = uint16_t(i);
            }
            __syncthreads();
        }
        for (int d = 16; d > 0; d >>= 1) hitc += __shfl_xor_sync(0xFFFFFFFFu, hitc, d);
        if (lane == 0) sh.wsum[w] = hitc;
        __syncthreads();
        if (tid == 0) {
            uint32_t h = 0;
            for (int q = 0; q < kRT / 32; ++q) h += sh.wsum[q];
            a.hits[size_t(g) * a.N + k] = h;
            a.misses[size_t(g) * a.N + k] = L - h;
            rstart[sh.nruns] = uint16_t(L);
        }
        __syncthreads();
        const uint32_t nruns = L ? sh.nruns : 0;
        for (uint32_t r = 0; r < nruns; ++r) {
            const uint32_t r0 = rstart[r], r1 = rstart[r + 1];
            const bool hitrun = sx[r0] & kHit;
            for (uint32_t i = r0 + tid; i < r1; i += kRT) {
                const uint32_t x = sx[i] & ~kHit;
                // a hit carries its slot on; a miss has none until the run's evictions are done
                const uint32_t s0 = hitrun && a.slot_out ? (a.slot_out[base + i] & ~kHit) : kNone;
                chain_set(a, sh, cx, x, a.nuk[base + i], s0);
            }
            __syncthreads();
            if (!hitrun) {
                if (w == 0) {
                    uint32_t need = 0;
                    if (lane == 0) {
                        sh.size += r1 - r0;
                        need = sh.size > a.C ? sh.size - a.C : 0u;
                    }
                    need = __shfl_sync(0xFFFFFFFFu, need, 0);
                    if (need) chain_evict(a, sh, cx, need, lane);
                }
                __syncthreads();
                // survivors of the run take slots in list order: every warp
                // checks its items, a block scan ranks them
                if (a.slot_out) {
                    for (uint32_t c = r0; c < r1; c += kRT) {
                        const uint32_t i = c + tid;
                        bool surv = false;
                        uint32_t x = 0, nu = kNever;
                        if (i < r1) {
                            x = sx[i] & ~kHit;
                            nu = a.nuk[base + i];
                            surv = nu == kNever ? cx.never_set(x) : cx.bit_set(nu);
                        }
                        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, surv);
                        if (lane == 0) sh.wsum[w] = __popc(bal);
                        __syncthreads();
                        uint32_t before = 0, n = 0;
                        for (int q = 0; q < kRT / 32; ++q) {
                            before += q < int(w) ? sh.wsum[q] : 0u;
                            n += sh.wsum[q];
                        }
                        const uint32_t rank = before + __popc(bal & lanemask_lt_r());
                        const uint32_t nf = sh.nfree, fr = sh.fresh;
                        if (surv) {
                            const uint32_t s2 = rank < nf ? fs[nf - 1 - rank] : fr + (rank - nf);
                            if (nu == kNever) a.slot[size_t(k) * a.D + x] = s2;
                            else a.slot_out[cx.pos_index(nu)] = s2;
                        }
                        __syncthreads();
                        if (tid == 0) {
                            const uint32_t from_stack = min(n, nf);
                            sh.nfree = nf - from_stack;
                            sh.fresh = fr + (n - from_stack);
                        }
                        __syncthreads();
                    }
                }
            }
        }
        // misses report the slot they hold at the END of the step (evicted
        // again by a later run of the step: bypass)
        if (a.slot_out)
            for (uint32_t i = tid; i < L; i += kRT) {
                const uint32_t v = sx[i];
                if (v & kHit) continue;
                const uint32_t x = v & ~kHit, nu = a.nuk[base + i];
                uint32_t s = kNever;
                if (nu == kNever) {
                    if (cx.never_set(x)) s = a.slot[size_t(k) * a.D + x];
                } else if (cx.bit_set(nu)) {
                    s = __ldcg(&a.slot_out[cx.pos_index(nu)]);
                }
                a.slot_out[base + i] = s;
            }
        __syncthreads();
    }
}

// ---- redundant_ids (chunking.cpp:35-45) of every (step, node) list of a
// plan with reads: the ids inside its chunk reads (start < end) that are not
// among the list's fetch ids, unique and ascending. One warp per list; pass 0
// counts, pass 1 writes at red_off.
struct RedArgs {
    const uint32_t* items;
    const uint32_t* node_off;
    const uint64_t* gb;
    const uint32_t* rstart;
    const uint32_t* rend;
    const uint32_t* rcount;
    uint32_t T, N, P2;
    uint64_t* red_cnt;        // pass 0: [T*N]
    const uint64_t* red_off;  // pass 1: [T*N+1]
    uint32_t* red_ids;        // pass 1
    uint32_t* status;
};

__global__ void k_redundant_ids(RedArgs a, int pass) {
    extern __shared__ uint32_t rbuf[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    uint32_t* buf = rbuf + size_t(wib) * a.P2;
    const uint32_t lt = lanemask_lt_r();
    for (uint64_t list = uint64_t(blockIdx.x) * wpb + wib; list < uint64_t(a.T) * a.N;
         list += uint64_t(gridDim.x) * wpb) {
        const uint32_t g = uint32_t(list / a.N), k = uint32_t(list % a.N);
        const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
        const uint64_t lo = a.gb[g] + off[k];
        const uint32_t L = off[k + 1] - off[k], R = a.rcount[list];
        uint32_t F = 0;
        for (uint32_t c = 0; c < L; c += 32) {
            const uint32_t v = c + lane < L ? a.items[lo + c + lane] : kHit;
            const bool f = !(v & kHit);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
            if (f) buf[F + __popc(bal & lt)] = v;
            F += __popc(bal);
        }
        uint32_t P = 1;
        while (P < F) P <<= 1;
        for (uint32_t i = F + lane; i < P; i += 32) buf[i] = 0xFFFFFFFFu;
        __syncwarp();
        for (uint32_t size = 2; size <= P; size <<= 1)
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t r = lane; r < P / 2; r += 32) {
                    const uint32_t x0 = 2 * stride * (r / stride) + (r % stride), x1 = x0 + stride;
                    const bool up = (x0 & size) == 0;
                    const uint32_t p = buf[x0], q = buf[x1];
                    if ((p > q) == up) { buf[x0] = q; buf[x1] = p; }
                }
                __syncwarp();
            }
        // reads in file order may overlap in a foreign plan: ids are emitted
        // once, from the first read that covers them
        uint64_t n = 0;
        const uint64_t wbase = pass ? a.red_off[list] : 0;
        for (uint32_t r = 0; r < R; ++r) {
            const uint32_t st = a.rstart[lo + r], en = a.rend[lo + r];
            if (st >= en) continue;  // a Single read streams nothing extra
            for (uint64_t y0 = st; y0 <= en; y0 += 32) {
                const uint64_t y = y0 + lane;
                bool red = false;
                if (y <= en) {
                    uint32_t l0 = 0, l1 = F;  // fetch ids: binary search
                    while (l0 < l1) {
                        const uint32_t mid = (l0 + l1) >> 1;
                        if (buf[mid] < y) l0 = mid + 1; else l1 = mid;
                    }
                    red = !(l0 < F && buf[l0] == y);
                    for (uint32_t r2 = 0; r2 < r && red; ++r2) {
                        const uint32_t s2 = a.rstart[lo + r2], e2 = a.rend[lo + r2];
                        if (s2 < e2 && y >= s2 && y <= e2) red = false;
                    }
                }
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, red);
                if (pass && red) a.red_ids[wbase + n + __popc(bal & lt)] = uint32_t(y);
                n += __popc(bal);
            }
        }
        if (!pass && lane == 0) a.red_cnt[list] = n;
        __syncwarp();
    }
}

__global__ void k_scan_u64(const uint64_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
    // single block exclusive scan (n = T*N lists), out[n] = total
    __shared__ uint64_t part[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint64_t c = 0; c < n; c += 1024) {
        const uint64_t i = c + threadIdx.x;
        const uint64_t v = i < n ? in[i] : 0;
        uint64_t inc = v;
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= uint32_t(d)) inc += o;
        }
        if (lane == 31) part[w] = inc;
        __syncthreads();
        if (w == 0) {
            const uint64_t p = part[lane];
            uint64_t pi = p;
            for (int d = 1; d < 32; d <<= 1) {
                const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, pi, d);
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

// ---- LRU replay (simulate_plan with Policy::Lru, buffer.cpp:61-82): one
// warp per node walks the node's accesses through lru_step (lru.cuh). Slots:
// a miss takes its victim's slot, or a fresh one while the buffer fills; hits
// report their slot at the access (bit 31), misses the slot they hold at the
// end of the step (LSG_NEVER if a later miss of the step evicted them again).
struct LruReplayArgs {
    uint32_t T, N, D, C, k0, k1;
    const uint32_t* items;
    const uint32_t* node_off;
    const uint64_t* gb;
    uint32_t* last;      // [N][D]
    uint32_t* slot;      // [N][D] or null
    uint32_t* hits;      // [T][N]
    uint32_t* misses;    // [T][N]
    uint32_t* slot_out;  // [total items] or null
    uint32_t* status;
    const uint64_t* red_off;  // [T*N+1] silent inserts after each list (insert_redundant) or null
    const uint32_t* red_ids;
};

__global__ void __launch_bounds__(kRWarps * 32) k_replay_lru(LruReplayArgs a) {
    __shared__ uint32_t hbm_all[kRWarps][kRMaxList / 32];  // hit flags of the step
    uint32_t* hbm = hbm_all[threadIdx.x >> 5];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t k = a.k0 + blockIdx.x * kRWarps + (threadIdx.x >> 5);
    if (k >= a.k1) return;
    uint32_t* last = a.last + size_t(k) * a.D;
    uint32_t* slotk = a.slot ? a.slot + size_t(k) * a.D : nullptr;
    const LruPlanView v{a.items, a.node_off, a.gb, nullptr, a.N, k, a.red_off ? a.red_off + k : nullptr, a.red_ids,
                        a.N};
    LruNode st{0, 0, 0, 0, 0, 0};
    for (uint32_t g = 0; g < a.T; ++g) {
        const uint32_t L = v.llen(g);
        const uint64_t base = a.gb[g] + a.node_off[size_t(g) * (a.N + 1) + k];
        const uint32_t* lst = a.items + base;
        uint32_t* so = a.slot_out ? a.slot_out + base : nullptr;
        if (so) {
            for (uint32_t wd = lane; wd < (L + 31) / 32; wd += 32) hbm[wd] = 0;
            __syncwarp();
        }
        const uint32_t miss = lru_step(
            v, st, last, lst, L, a.C, lane, a.status,
            [&](uint32_t i, uint32_t x) {
                if (so) {
                    so[i] = slotk[x] | kHit;
                    atomicOr(&hbm[i >> 5], 1u << (i & 31));  // (shared memory)
                }
            },
            [&](uint32_t x, uint32_t y) {
                if (!slotk) return;
                if (y != kNone) {
                    slotk[x] = slotk[y];
                    slotk[y] = kNone;
                } else {
                    slotk[x] = st.fresh++;
                }
            });
        st.fresh = __shfl_sync(0xFFFFFFFFu, st.fresh, 0);
        if (so) {
            __syncwarp();
            for (uint32_t i = lane; i < L; i += 32) {
                if ((hbm[i >> 5] >> (i & 31)) & 1u) continue;  // a hit, reported at its access
                const uint32_t x = __ldcg(&lst[i]) & ~kHit;
                so[i] = __ldcg(&last[x]) != kNone ? slotk[x] : kNever;
            }
        }
        if (lane == 0) {
            a.hits[size_t(g) * a.N + k] = L - miss;
            a.misses[size_t(g) * a.N + k] = miss;
        }
        __syncwarp();
        if (a.red_off) {  // the list's redundant ids, touched silently (they follow the list in node time)
            const uint64_t q0 = a.red_off[size_t(g) * a.N + k], q1 = a.red_off[size_t(g) * a.N + k + 1];
            lru_step(v, st, last, a.red_ids + q0, uint32_t(q1 - q0), a.C, lane, a.status,
                     [](uint32_t, uint32_t) {}, [](uint32_t, uint32_t) {});
            __syncwarp();
        }
    }
}

}  // namespace

// redundant_ids of every (step, node) list of a plan with reads, as CSR:
// roff [T*N+1] (u64 offsets), ids [nred] (ascending per list)
int red_csr(Scratch& sc, const uint32_t* d_items, const uint32_t* d_node_off, const uint64_t* gb,
            const uint32_t* d_rstart, const uint32_t* d_rend, const uint32_t* d_rcount, uint64_t T, uint32_t N,
            uint64_t L, uint32_t* d_status, cudaStream_t st, uint64_t** roff_out, uint32_t** ids_out,
            uint64_t* nred_out) {
    uint64_t* cnt = sc.get<uint64_t>(T * N);
    uint64_t* roff = sc.get<uint64_t>(T * N + 1);
    if (!cnt || !roff) return set_error(kInternal, "simulate: scratch allocation failed");
    RedArgs r{d_items, d_node_off, gb, d_rstart, d_rend, d_rcount, uint32_t(T), N, 1, cnt, roff, nullptr, d_status};
    while (r.P2 < L) r.P2 <<= 1;
    const uint32_t wpb = std::max<uint32_t>(1, std::min<uint32_t>(8, (96u * 1024) / (4 * r.P2)));
    const size_t rs = size_t(wpb) * r.P2 * 4;
    LSG_CUDA(cudaFuncSetAttribute(k_redundant_ids, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rs)));
    const unsigned rg = unsigned(std::min<uint64_t>((T * N + wpb - 1) / wpb, 148ull * 8));
    k_redundant_ids<<<rg, wpb * 32, rs, st>>>(r, 0);
    LSG_LAUNCH_CHECK("k_redundant_ids");
    k_scan_u64<<<1, 1024, 0, st>>>(cnt, T * N, roff);
    LSG_LAUNCH_CHECK("k_scan_u64");
    uint64_t nred = 0;
    if (int rc = d2h_small(&nred, roff + T * N, 8, st)) return rc;
    uint32_t* ids = sc.get<uint32_t>(nred);
    if (!ids) return set_error(kInternal, "simulate: scratch allocation failed");
    r.red_ids = ids;
    k_redundant_ids<<<rg, wpb * 32, rs, st>>>(r, 1);
    LSG_LAUNCH_CHECK("k_redundant_ids");
    *roff_out = roff;
    *ids_out = ids;
    *nred_out = nred;
    return kOk;
}

int simulate_device(const uint32_t* d_items, const uint32_t* d_node_off, uint64_t T, uint32_t N,
                    uint64_t D, uint64_t C, int policy, uint32_t k0, uint32_t k1, uint32_t* d_hits,
                    uint32_t* d_misses, uint32_t* d_slot, const uint32_t* d_rstart, const uint32_t* d_rend,
                    const uint32_t* d_rcount, int insred, uint32_t* d_status, cudaStream_t st) {
    if (k1 <= k0 || T == 0) return kOk;
    if (insred && d_slot)
        return set_error(kCapability, "simulate: HBM slots are not tracked with insert_redundant");
    if (insred && (!d_rstart || !d_rend || !d_rcount))
        return set_error(kValidation, "simulate: insert_redundant needs the plan's reads");
    Scratch sc(st);
    uint64_t* gb = sc.get<uint64_t>(T + 1);
    if (!gb) return set_error(kInternal, "simulate: scratch allocation failed");
    k_step_bases<<<1, 1024, 0, st>>>(d_node_off, uint32_t(T), N, gb);
    LSG_LAUNCH_CHECK("k_step_bases");
    uint64_t total = 0, L = 0;
    if (int _rc = d2h_small(&total, gb + T, 8, st)) return _rc;
    std::vector<uint32_t> hv(size_t(T) * (N + 1));
    {
        // key stride = the longest node list of any step (keys are g*L + i)
        uint32_t* hoff = hv.data();
        const size_t nb = size_t(T) * (N + 1) * 4;
        LSG_CUDA(cudaMemcpyAsync(hoff, d_node_off, nb, cudaMemcpyDeviceToHost, st));
        LSG_CUDA(cudaStreamSynchronize(st));
        for (uint64_t g = 0; g < T; ++g)
            for (uint32_t k = 0; k < N; ++k) {
                const uint32_t* o = hoff + g * (N + 1);
                if (o[k + 1] < o[k]) return set_error(kValidation, "simulate: node offsets not ascending");
                L = std::max<uint64_t>(L, o[k + 1] - o[k]);
            }
    }
    if (L == 0) L = 1;
    if (T * L >= 0xFFFFFFF0ull) return set_error(kCapability, "simulate: plan too large for 32-bit position keys");
    if (total) {  // every id must index the per-node [D] tables
        uint32_t* mx = sc.get<uint32_t>(1);
        if (!mx) return set_error(kInternal, "simulate: scratch allocation failed");
        LSG_CUDA(cudaMemsetAsync(mx, 0, 4, st));
        k_max_id<<<grid_for(total, 256, 148u * 8), 256, 0, st>>>(d_items, total, mx);
        LSG_LAUNCH_CHECK("k_max_id");
        uint32_t hmax = 0;
        if (int rc = d2h_small(&hmax, mx, 4, st)) return rc;
        // the reference's buffers are hash sets, so simulate_plan accepts a
        // plan (read_plan, plan.cpp:85-214) whose ids exceed its dataset_size:
        // widen the id space to cover them, within the device tables' budget
        if (uint64_t(hmax) >= D) D = uint64_t(hmax) + 1;
        if (uint64_t(N) * D > (uint64_t(1) << 33))
            return set_error(kCapability, "simulate: nodes x id space (" + std::to_string(N) + " x " +
                                              std::to_string(D) + ") exceeds the replay's device tables");
    }
    if (L > kRMaxList) return set_error(kCapability, "simulate: node list longer than 16384 samples");
    // segments of whole steps holding at most D accesses (over all nodes):
    // epoch-aligned for plan_schedule's plans
    auto nextuse_segments = [&](uint32_t* last, uint32_t* nuk, uint32_t* conflict) -> int {
        std::vector<uint32_t> cut{uint32_t(T)};
        uint64_t acc = 0;
        for (int64_t g = int64_t(T) - 1; g >= 0; --g) {
            const uint64_t len = hv[size_t(g) * (N + 1) + N];
            if (acc + len > D && acc > 0) {
                cut.push_back(uint32_t(g + 1));
                acc = 0;
            }
            acc += len;
        }
        cut.push_back(0);  // cut: descending step boundaries
        const size_t smem = size_t(N + 1) * 4;
        for (size_t c = 0; c + 1 < cut.size(); ++c) {
            const uint32_t g1 = cut[c], g0 = cut[c + 1];
            if (g1 <= g0) continue;
            uint64_t longest = 1;  // rows of the segment's longest step
            for (uint32_t g = g0; g < g1; ++g) longest = std::max<uint64_t>(longest, hv[size_t(g) * (N + 1) + N]);
            const uint32_t chunks = uint32_t((longest + kNuRows - 1) / kNuRows);
            k_nextuse_seg<<<(g1 - g0) * chunks, kNuThreads, smem, st>>>(d_items, d_node_off, gb, N, D, uint32_t(L),
                                                                        g0, g1, chunks, last, nuk, conflict);
            LSG_LAUNCH_CHECK("k_nextuse_seg");
        }
        return kOk;
    };
    if (policy == 1) {  // LRU
        LruReplayArgs r{};
        r.T = uint32_t(T);
        r.N = N;
        r.D = uint32_t(D);
        r.C = uint32_t(std::min<uint64_t>(C, 0xFFFFFFF0ull));
        r.k0 = k0;
        r.k1 = k1;
        r.items = d_items;
        r.node_off = d_node_off;
        r.gb = gb;
        r.last = sc.get<uint32_t>(size_t(N) * D);
        r.slot = d_slot ? sc.get<uint32_t>(size_t(N) * D) : nullptr;
        if (!r.last || (d_slot && !r.slot)) return set_error(kInternal, "simulate: scratch allocation failed");
        LSG_CUDA(cudaMemsetAsync(r.last, 0xFF, size_t(N) * D * 4, st));
        if (r.slot) LSG_CUDA(cudaMemsetAsync(r.slot, 0xFF, size_t(N) * D * 4, st));
        r.hits = d_hits;
        r.misses = d_misses;
        r.slot_out = d_slot;
        r.status = d_status;
        if (insred) {  // LruBuffer::insert_silent = touch_or_insert (buffer.cpp:88-91)
            uint64_t* roff = nullptr;
            uint32_t* ids = nullptr;
            uint64_t nred = 0;
            if (int rc = red_csr(sc, d_items, d_node_off, gb, d_rstart, d_rend, d_rcount, T, N, L, d_status, st,
                                 &roff, &ids, &nred))
                return rc;
            r.red_off = roff;
            r.red_ids = ids;
        }
        const uint32_t nk = k1 - k0;
        k_replay_lru<<<(nk + kRWarps - 1) / kRWarps, kRWarps * 32, 0, st>>>(r);
        LSG_LAUNCH_CHECK("k_replay_lru");
        return kOk;
    }
    ReplayArgs a{};
    a.T = uint32_t(T);
    a.N = N;
    a.D = uint32_t(D);
    a.L = uint32_t(L);
    a.C = uint32_t(std::min<uint64_t>(C, 0xFFFFFFF0ull));
    a.k0 = k0;
    a.k1 = k1;
    a.nzw = uint32_t((T + 31) / 32 + 1);
    a.infw = uint32_t((D + 31) / 32);
    a.bw = uint32_t((L + 31) / 32);
    a.items = d_items;
    a.node_off = d_node_off;
    a.gb = gb;
    // per-node state is indexed by absolute node id; allocate N rows
    a.nuk = sc.get<uint32_t>(total);
    a.last = sc.get<uint32_t>(size_t(N) * D);
    // the forward replay's random-access state in ONE block (key, slot, the
    // never-used bitmaps, the step bitmap), so an L2 access-policy window can
    // pin it while a fetch streams through L2 beside the replay
    a.sumw = (uint32_t((D + 31) / 32) + 31) / 32;
    const size_t hot_words = size_t(N) * D * 2 + size_t(N) * a.infw + size_t(N) * a.sumw + size_t(N) * a.nzw;
    uint32_t* hot = sc.get<uint32_t>(hot_words);
    a.key = hot;
    a.slot = hot ? hot + size_t(N) * D : nullptr;
    a.infbm = hot ? a.slot + size_t(N) * D : nullptr;
    a.infsum = hot ? a.infbm + size_t(N) * a.infw : nullptr;
    a.nz = hot ? a.infsum + size_t(N) * a.sumw : nullptr;
    // (next-use step, position) bitmaps: always for short lists (warp path);
    // for the CTA path when they fit the budget (else its list-scan eviction)
    const size_t pbm_words = size_t(N) * T * a.bw;
    const bool want_pbm = L <= 128 || (pbm_words * 4 <= (size_t(4) << 30) && !std::getenv("LSG_REPLAY_SCAN"));
    a.pbm = want_pbm ? sc.get<uint32_t>(pbm_words) : nullptr;
    a.psw = uint32_t((uint64_t(T) * a.bw + 31) / 32);
    a.psum = want_pbm ? sc.get<uint32_t>(size_t(N) * a.psw) : nullptr;
    a.ps2w = (a.psw + 31) / 32;
    a.psum2 = want_pbm ? sc.get<uint32_t>(size_t(N) * a.ps2w) : nullptr;
    a.fstack = d_slot ? sc.get<uint32_t>(size_t(N) * std::min<uint64_t>(C, D)) : nullptr;
    if (!a.nuk || !a.last || !a.key || !a.slot || !a.nz || (want_pbm && (!a.pbm || !a.psum || !a.psum2)) || !a.infbm || !a.infsum || (d_slot && !a.fstack))
        return set_error(kInternal, "simulate: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(a.last, 0xFF, size_t(N) * D * 4, st));  // kNone = no later access
    LSG_CUDA(cudaMemsetAsync(a.key, 0xFF, size_t(N) * D * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.slot, 0xFF, size_t(N) * D * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.nz, 0, size_t(N) * a.nzw * 4, st));
    if (a.pbm) LSG_CUDA(cudaMemsetAsync(a.pbm, 0, size_t(N) * T * a.bw * 4, st));
    if (a.psum) LSG_CUDA(cudaMemsetAsync(a.psum, 0, size_t(N) * a.psw * 4, st));
    if (a.psum2) LSG_CUDA(cudaMemsetAsync(a.psum2, 0, size_t(N) * a.ps2w * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.infbm, 0, size_t(N) * a.infw * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.infsum, 0, size_t(N) * a.sumw * 4, st));
    a.hits = d_hits;
    a.misses = d_misses;
    a.slot_out = d_slot;
    a.status = d_status;
    const uint32_t nk = k1 - k0;
    const char* fc = std::getenv("LSG_REPLAY_CTA");  // tests: force the CTA variant
    if (L > 128 || insred || (fc && fc[0] == '1')) {  // long lists (and silent inserts): a CTA per node
        ReplayArgsCta c{};
        if (insred) {  // redundant ids per list (CSR) for the silent inserts
            uint64_t* roff = nullptr;
            uint32_t* ids = nullptr;
            uint64_t nred = 0;
            if (int rc = red_csr(sc, d_items, d_node_off, gb, d_rstart, d_rend, d_rcount, T, N, L, d_status, st,
                                 &roff, &ids, &nred))
                return rc;
            uint32_t* keys = sc.get<uint32_t>(nred);
            if (!keys) return set_error(kInternal, "simulate: scratch allocation failed");
            c.red_off = roff;
            c.red_ids = ids;
            c.red_key = keys;
        }
        c.T = a.T; c.N = N; c.D = a.D; c.B = a.L; c.C = a.C; c.k0 = k0;
        c.nzw = a.nzw; c.infw = a.infw;
        c.items = d_items; c.node_off = d_node_off; c.gb = gb;
        c.nuk = a.nuk; c.last = a.last; c.key = a.key; c.slot = a.slot; c.nz = a.nz;
        c.pbm = a.pbm; c.bw = a.bw; c.psum = a.psum; c.psw = a.psw; c.psum2 = a.psum2; c.ps2w = a.ps2w;
        c.infbm = a.infbm; c.infsum = a.infsum; c.sumw = a.sumw; c.fstack = a.fstack; c.hits = d_hits; c.misses = d_misses;
        c.slot_out = d_slot; c.status = d_status;
        bool serial = insred || std::getenv("LSG_NEXTUSE_SERIAL");
        if (!serial) {  // all nodes' keys (the replay reads only nodes [k0, k1))
            uint32_t* conflict = sc.get<uint32_t>(1);
            if (!conflict) return set_error(kInternal, "simulate: scratch allocation failed");
            LSG_CUDA(cudaMemsetAsync(conflict, 0, 4, st));
            if (int rc = nextuse_segments(a.last, a.nuk, conflict)) return rc;
            uint32_t hc = 0;
            if (int rc = d2h_small(&hc, conflict, 4, st)) return rc;
            if (hc) {  // an id twice on a node inside a segment: redo serially
                serial = true;
                LSG_CUDA(cudaMemsetAsync(a.last, 0xFF, size_t(N) * D * 4, st));
            }
        }
        if (serial) {
            k_replay_nextuse_cta<<<nk, kRT, 0, st>>>(c);
            LSG_LAUNCH_CHECK("k_replay_nextuse_cta");
        }
        // a whole SM per rank only while the ranks fit in one wave with room
        // to spare (256 simulated ranks would otherwise run in two waves)
        const size_t need = size_t(L) * 4 + (L + 2) * 2 + 16;
        const size_t smem = nk <= 32 ? exclusive_smem(need) : need;
        LSG_CUDA(cudaFuncSetAttribute(k_replay_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        // the chain replay (no id-indexed key/slot tables) needs the key-space
        // bitmaps and no silent inserts; LSG_REPLAY_TABLES=1 keeps round 1's
        // table replay
        const bool chain = a.pbm && !insred && !std::getenv("LSG_REPLAY_TABLES");
        if (chain) {
            LSG_CUDA(cudaFuncSetAttribute(k_replay_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            k_replay_chain<<<nk, kRT, smem, st>>>(c);
            LSG_LAUNCH_CHECK("k_replay_chain");
            return kOk;
        }
        const bool pinned = l2_pin(st, hot, hot_words * 4);
        k_replay_cta<<<nk, kRT, smem, st>>>(c);
        LSG_LAUNCH_CHECK("k_replay_cta");
        if (pinned) l2_unpin(st);
        return kOk;
    }
    const unsigned grid = (nk + kRWarps - 1) / kRWarps;
    bool serial = std::getenv("LSG_NEXTUSE_SERIAL") != nullptr;
    if (!serial) {
        uint32_t* conflict = sc.get<uint32_t>(1);
        if (!conflict) return set_error(kInternal, "simulate: scratch allocation failed");
        LSG_CUDA(cudaMemsetAsync(conflict, 0, 4, st));
        if (int rc = nextuse_segments(a.last, a.nuk, conflict)) return rc;
        uint32_t hc = 0;
        if (int rc = d2h_small(&hc, conflict, 4, st)) return rc;
        if (hc) {
            serial = true;
            LSG_CUDA(cudaMemsetAsync(a.last, 0xFF, size_t(N) * D * 4, st));
        }
    }
    if (serial) {
        k_replay_nextuse<<<grid, kRWarps * 32, 0, st>>>(a);
        LSG_LAUNCH_CHECK("k_replay_nextuse");
    }
    const size_t smem = size_t(kRWarps) * L * 4;
    LSG_CUDA(cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_replay<<<grid, kRWarps * 32, smem, st>>>(a);
    LSG_LAUNCH_CHECK("k_replay");
    return kOk;
}

}  // namespace lsg

// plan_wide.cu — K6 for wide jobs: the planner step loop of plan_schedule
// (pipeline.cpp:68-118) when the simulated world has more than 32 nodes or a
// global batch beyond one CTA's shared memory (BASELINE cfg5: 1,048,576 ids,
// 32-256 logical ranks, b=512, so B = N*b reaches 131,072 ids per step).
//
// Same semantics as k_plan_loop (plan.cu), bit-exact with remap_step
// (locality.cpp:7-42) / slice_step (:57-73), balance_step (balance.cpp:10-39)
// and ClairvoyantBuffer::access (buffer.cpp:37-46), but laid out for width:
//
//  * one persistent thread-block CLUSTER (16 CTAs x 512 threads when the
//    device allows it) walks the T dependent steps; the phases of a step are
//    separated by cluster barriers, cross-CTA prefix sums read the other CTAs'
//    shared-memory totals through DSMEM;
//  * holder masks are W = ceil(N/32) words per id;
//  * per-item work (classification, single-holder ranks, positions) is spread
//    over every warp of the cluster; the multi-holder remap is the only serial
//    pass (one warp, lanes = candidate holders, REDUX.MIN on (count, node));
//  * balance is simulated on the N fetch counts in rounds: every round pairs
//    the i-th first-argmax node with the i-th first-argmin node, which is the
//    reference's move sequence (the argmax/argmin only change when a level
//    set is exhausted); donor d's q-th move gives its q-th largest fetch id;
//  * each node's buffer is a dense slot array of (next-use step, id) plus a
//    per-node count of residents per next-use step ("bins"). A miss run
//    inserts its ids, then evicts the (size - C)+ largest (key, id): the
//    threshold bin comes from the counts (walked from the top, 32 bins per
//    ballot), one scan of the slots flags everything above it, a radix select
//    on the ids picks the largest ones inside the threshold bin (equal keys
//    evict the larger id first, buffer.cpp:27-28), and the slot array is
//    compacted by moving survivors from the tail into the holes.
//
// Node-level work (lists, buffer advance) runs one warp per node.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "lru.cuh"

namespace cg = cooperative_groups;

namespace lsg {

namespace {

constexpr int kWT = 512;                // threads per CTA
constexpr int kWW = kWT / 32;           // warps per CTA
constexpr uint32_t kWMaxN = 256;        // simulated nodes
constexpr uint32_t kSortCap = 512;      // donor fetch entries sorted in shared memory
constexpr uint32_t kMS = 1024;          // multi items staged per chunk (B pass)
constexpr uint32_t kMP = kWW * kSortCap * 2 - 3 * kMS;  // staged pair words
constexpr uint32_t kLevCap = 2048;      // balance levels handled in closed form
constexpr uint32_t kHitM = 0x80000000u;
constexpr uint32_t kIdM = 0x7FFFFFFFu;
constexpr uint32_t kClsSingle = 1u << 30;
constexpr uint32_t kClsMulti = 2u << 30;

struct WideArgs {
    uint32_t D, N, W, b, B, S, keep, T, C;
    uint32_t SC;                      // slots per node (C + B)
    uint32_t EBW;                     // eviction-flag words per node
    uint32_t MBW;                     // moved-flag words per node
    int remap, balance, lru;
    int insred;                       // chunk_insert_redundant (pipeline.cpp:103-114)
    int advance;                      // 0: assignment only (remap_step / slice_step per call)
    uint32_t thr;                     // chunk threshold
    uint32_t E;
    const uint32_t* inv;              // [E][D] position of id in epoch e's trace, kNone if not kept
    uint32_t* redbuf;                 // [N][B] sort scratch for lists longer than shared memory
    uint32_t* lred;                   // LRU + insred: [N][lcap] each node's silent-touch ids, step by step
    uint64_t* lroff;                  // LRU + insred: [N][T+1] offsets into the node's lred row
    uint64_t lcap;
    const uint32_t* trace;            // [E][keep]
    const uint32_t* order;            // [E]
    const uint32_t* nu;               // [E*keep] next-use step, execution order
    uint32_t* hm;                     // [D][W] holder masks
    uint32_t* where;                  // [N][D] slot of a resident id (LRU: node time of its last access), kNone otherwise
    uint32_t* sbase;                  // [T] first item of each step (LRU front walk)
    unsigned long long* slot;         // [N][SC] (key << 32 | id), dense in [0, size)
    uint32_t* cnt;                    // [N][T+1] residents per key bin (bin T = never used)
    uint32_t* nst;                    // [N][8] size, top finite key | LRU: size, -, t, front step/index/time
    uint32_t* evb;                    // [N][EBW] eviction flags (zero between uses)
    uint32_t* cand;                   // [N][SC] threshold-bin slots
    uint32_t* candid;                 // [N][SC] their ids
    uint32_t* holes;                  // [N][SC] compaction holes
    uint32_t* movedbm;                // [N][MBW] moved pre-list positions (zero between uses)
    // per-step scratch, batch position j
    uint32_t* jx;                     // [B] id
    uint32_t* jnu;                    // [B] next-use step
    uint32_t* jmask;                  // [B][W] holder masks at step start
    uint32_t* jcls;                   // [B] class | holder
    uint32_t* jS;                     // [B] singles: S_k(j); multi: multi index
    uint32_t* pre;                    // [B] pre-balance lists (j | hit)
    uint32_t* fx;                     // [B] final lists: id | resident-at-start << 31
    uint32_t* fnu;                    // [B] final lists: next-use step
    uint32_t* mj;                     // [B] multi index -> j
    uint32_t* mpo;                    // [B] multi index -> pair offset
    uint32_t* mhc;                    // [B] multi index -> candidate pairs
    uint32_t* pairs;                  // [B*N] (S_k << 10 | k), S_k < b
    uint32_t* massign;                // [B] (position << 10 | node) or kNone
    uint32_t* mpos;                   // [N][b] j of node k's assigned multis, in order
    uint32_t* recv;                   // [N][b] donor's q-th move: (ii << 10 | recipient)
    uint32_t* ur;                     // [B] recipient units in move order
    uint32_t* items;                  // [E*keep] output
    uint32_t* node_off;               // [T][N+1] output
    uint32_t* fb;                     // [T][N] output (may be null)
    uint32_t* fa;                     // [T][N] output (may be null)
    uint32_t* status;
    unsigned long long* prof;         // [16] per-phase cycles + counters (LSG_PROFILE) or null
};

__device__ __forceinline__ uint32_t lanemask_lt_w() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
        if (lane >= uint32_t(d)) v += o;
    }
    return v;
}

__device__ __forceinline__ uint32_t bin_of(uint32_t key, uint32_t T) { return key == kNever ? T : key; }

// drop resident (key, x) of node k: residency, holder bit, bin count
__device__ __forceinline__ void evict_one(const WideArgs& a, uint32_t k, unsigned long long v) {
    const uint32_t x = uint32_t(v);
    a.where[size_t(k) * a.D + x] = kNone;
    atomicAnd(&a.hm[size_t(x) * a.W + (k >> 5)], ~(1u << (k & 31)));
    atomicSub(&a.cnt[size_t(k) * (a.T + 1) + bin_of(uint32_t(v >> 32), a.T)], 1u);
}

// Eviction team: the tpn warps that own node k. The leader warp walks the
// node's list; the whole team runs every eviction (scan, select, apply).
struct Team {
    uint32_t tpn, wr, bar_id;
    uint32_t* ctl;   // [8] shared: cmd, tstar, bsz, newsize, hcount, ccount, r, prefix
    uint32_t* hist;  // [256] shared radix histogram (the leader warp's)
    __device__ __forceinline__ void sync() const {
        if (tpn > 1) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(tpn * 32) : "memory");
    }
};

// The team part of an eviction of node k (every warp of the team, identical
// barriers): (1) scan slots [0, bsz) in 128-slot strides per warp, dropping
// residents above the threshold bin at once, appending holes below the new
// size and threshold-bin candidates (slot + id), writing tail flag words;
// (2) radix select (8-bit digits, team histogram) of the r-th largest
// candidate id; (3) drop the candidates at or above it.
__device__ void evict_team(const WideArgs& a, uint32_t k, const Team& tm, uint32_t lane) {
    const uint32_t lt = lanemask_lt_w();
    const uint32_t tstar = tm.ctl[1], bsz = tm.ctl[2], newsize = tm.ctl[3], r = tm.ctl[6];
    const uint32_t wr = tm.wr, tpn = tm.tpn;
    unsigned long long* sk = a.slot + size_t(k) * a.SC;
    uint32_t* evk = a.evb + size_t(k) * a.EBW;
    uint32_t* cak = a.cand + size_t(k) * a.SC;
    uint32_t* cid = a.candid + size_t(k) * a.SC;
    uint32_t* hk = a.holes + size_t(k) * a.SC;
    uint32_t* hcount = &tm.ctl[4];
    for (uint32_t s0 = wr * 128; s0 < bsz; s0 += tpn * 128) {
        unsigned long long v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t s = s0 + u * 32 + lane;
            v[u] = s < bsz ? __ldcg(&sk[s]) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t sb = s0 + u * 32, s = sb + lane;
            const bool valid = s < bsz;
            const uint32_t bn = bin_of(uint32_t(v[u] >> 32), a.T);
            const bool ev = valid && bn > tstar, cd = valid && bn == tstar;
            if (ev) evict_one(a, k, v[u]);
            const bool hole = ev && s < newsize;
            const uint32_t hb = __ballot_sync(0xFFFFFFFFu, hole);
            if (hb) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(hcount, __popc(hb));
                base = __shfl_sync(0xFFFFFFFFu, base, 0);
                if (hole) hk[base + __popc(hb & lt)] = s;
            }
            const uint32_t tw = __ballot_sync(0xFFFFFFFFu, ev && s >= newsize);
            if (lane == 0 && sb < bsz && sb + 31 >= newsize) evk[sb >> 5] = tw;
            const uint32_t cb = __ballot_sync(0xFFFFFFFFu, cd);
            if (cb) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&tm.ctl[5], __popc(cb));
                base = __shfl_sync(0xFFFFFFFFu, base, 0);
                if (cd) {
                    cak[base + __popc(cb & lt)] = s;
                    cid[base + __popc(cb & lt)] = uint32_t(v[u]);
                }
            }
        }
    }
    tm.sync();
    const uint32_t ncand = tm.ctl[5];
    uint32_t thr = 0;
    if (r < ncand) {
        uint32_t prefix = 0, pmask = 0, rem = r;
        for (int sh = 24; sh >= 0; sh -= 8) {
            for (uint32_t q = wr * 32 + lane; q < 256; q += tpn * 32) tm.hist[q] = 0;
            tm.sync();
            __syncwarp();
            for (uint32_t q = wr * 32 + lane; q < ncand; q += tpn * 32) {
                const uint32_t id = __ldcg(&cid[q]);
                if ((id & pmask) == prefix) atomicAdd(&tm.hist[(id >> sh) & 255u], 1u);
            }
            tm.sync();
            __syncwarp();
            // every warp derives the same digit: lane l owns digits 255-8l .. 248-8l
            uint32_t hv[8], lsum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                hv[q] = tm.hist[255 - 8 * lane - q];
                lsum += hv[q];
            }
            const uint32_t incl = warp_incl_scan(lsum, lane);
            const uint32_t excl = incl - lsum;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, excl < rem && incl >= rem);
            const uint32_t L = __ffs(bal) - 1;
            uint32_t dsel = 0, above = 0;
            if (lane == L) {
                uint32_t run = excl;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (run + hv[q] >= rem) {
                        dsel = 255 - 8 * lane - q;
                        above = run;
                        break;
                    }
                    run += hv[q];
                }
            }
            dsel = __shfl_sync(0xFFFFFFFFu, dsel, L);
            above = __shfl_sync(0xFFFFFFFFu, above, L);
            rem -= above;
            prefix |= dsel << sh;
            pmask |= 255u << sh;
            __syncwarp();
            tm.sync();  // histogram reads done before the next pass clears it
        }
        thr = prefix;  // the r-th largest id of the bin (ids are distinct per node)
    }
    for (uint32_t q0 = wr * 32; q0 < ncand; q0 += tpn * 32) {
        const uint32_t q = q0 + lane;
        bool ev = false;
        uint32_t s = 0;
        if (q < ncand && (r >= ncand || __ldcg(&cid[q]) >= thr)) {
            s = __ldcg(&cak[q]);
            ev = true;
            evict_one(a, k, __ldcg(&sk[s]));
            if (s >= newsize) atomicOr(&evk[s >> 5], 1u << (s & 31));
        }
        const bool hole = ev && s < newsize;
        const uint32_t hb = __ballot_sync(0xFFFFFFFFu, hole);
        if (hb) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(hcount, __popc(hb));
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            if (hole) hk[base + __popc(hb & lt)] = s;
        }
    }
    tm.sync();
}

// Remove the m = size - C largest (key, id) residents of node k (leader warp
// of the team): threshold bin from the per-bin counts (never-used first,
// then finite bins walked down from the top, 32 per ballot), the team part
// above, then tail survivors move into the holes.
__device__ void wide_evict(const WideArgs& a, uint32_t k, uint32_t& bsz, uint32_t& top, uint32_t g,
                           uint32_t lane, const Team& tm) {
    const uint32_t lt = lanemask_lt_w();
    const uint32_t m = bsz - a.C;
    uint32_t* cntk = a.cnt + size_t(k) * (a.T + 1);
    unsigned long long* sk = a.slot + size_t(k) * a.SC;
    uint32_t* evk = a.evb + size_t(k) * a.EBW;
    uint32_t* hk = a.holes + size_t(k) * a.SC;
    uint32_t tstar = 0, r = 0;
    const uint32_t nev = __ldcg(&cntk[a.T]);
    if (nev >= m) {
        tstar = a.T;
        r = m;
    } else {
        uint32_t acc = nev;
        int32_t hi = int32_t(top);
        bool found = false;
        while (!found) {
            if (hi <= int32_t(g)) {  // only current/stale keys left: impossible for a miss run
                if (lane == 0) atomicOr(a.status, 8u);
                return;
            }
            const int32_t bn = hi - int32_t(lane);
            const uint32_t v = bn > int32_t(g) ? __ldcg(&cntk[bn]) : 0u;
            const uint32_t incl = warp_incl_scan(v, lane);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, acc + incl >= m);
            if (bal) {
                const uint32_t L = __ffs(bal) - 1;
                const uint32_t before = __shfl_sync(0xFFFFFFFFu, incl - v, L);
                tstar = uint32_t(hi - int32_t(L));
                r = m - (acc + before);
                found = true;
            } else {
                acc += __shfl_sync(0xFFFFFFFFu, incl, 31);
                hi -= 32;
            }
        }
    }
    const uint32_t newsize = bsz - m;
    if (a.prof && lane == 0) {
        atomicAdd(&a.prof[8], 1ull);
        atomicAdd(&a.prof[9], static_cast<unsigned long long>(bsz));
    }
    if (lane == 0) {
        tm.ctl[0] = 1;
        tm.ctl[1] = tstar;
        tm.ctl[2] = bsz;
        tm.ctl[3] = newsize;
        tm.ctl[4] = 0;
        tm.ctl[5] = 0;
        tm.ctl[6] = r;
    }
    __syncwarp();
    tm.sync();
    evict_team(a, k, tm, lane);
    tm.sync();
    const uint32_t nh = tm.ctl[4];
    // ---- survivors from the tail fill the holes
    uint32_t nmv = 0;
    for (uint32_t s0 = newsize & ~31u; s0 < bsz; s0 += 32) {
        const uint32_t s = s0 + lane;
        const uint32_t word = __ldcg(&evk[s0 >> 5]);
        const bool mv = s >= newsize && s < bsz && !((word >> lane) & 1u);
        const uint32_t mb = __ballot_sync(0xFFFFFFFFu, mv);
        if (mv) {
            const uint32_t d = __ldcg(&hk[nmv + __popc(mb & lt)]);
            const unsigned long long v = __ldcg(&sk[s]);
            sk[d] = v;
            a.where[size_t(k) * a.D + uint32_t(v)] = d;
        }
        nmv += __popc(mb);
    }
    if (nmv != nh && lane == 0) atomicOr(a.status, 16u);
    __syncwarp();
    for (uint32_t wd = (newsize >> 5) + lane; wd < (bsz + 31) / 32; wd += 32) evk[wd] = 0;
    bsz = newsize;
    if (tstar != a.T) top = tstar;
    __syncwarp();
}

// Balance (balance.cpp:10-39) on the fetch counts in rounds (one warp).
// Writes outk/ink and, when recv != null, recv[d*b + q] = (ii << 10 | r):
// donor d's q-th move goes to recipient r as its ii-th appended fetch.
__device__ void wide_balance(uint32_t N, uint32_t b, const uint32_t* fcnt, uint32_t* outk, uint32_t* ink,
                             uint32_t* rl, uint32_t* rl2, uint32_t* recv, uint32_t* status, uint32_t lane) {
    const uint32_t lt = lanemask_lt_w();
    uint32_t cv[8], oq[8], iq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t k = q * 32 + lane;
        cv[q] = k < N ? fcnt[k] : 0u;
        oq[q] = iq[q] = 0;
    }
    const uint32_t NQ = (N + 31) / 32;
    for (;;) {
        uint32_t mx = 0, mn = 0xFFFFFFFFu;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (uint32_t(q) < NQ && q * 32 + lane < N) {
                mx = max(mx, cv[q]);
                mn = min(mn, cv[q]);
            }
        }
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        mn = __reduce_min_sync(0xFFFFFFFFu, mn);
        if (mx - mn <= 1) break;
        uint32_t nd = 0, nr = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (uint32_t(q) >= NQ) break;
            const bool in = q * 32 + lane < N;
            nd += __popc(__ballot_sync(0xFFFFFFFFu, in && cv[q] == mx));
            nr += __popc(__ballot_sync(0xFFFFFFFFu, in && cv[q] == mn));
        }
        const uint32_t pn = min(nd, nr);
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (uint32_t(q) >= NQ) break;
            const uint32_t k = q * 32 + lane;
            const bool isr = k < N && cv[q] == mn;
            const uint32_t br = __ballot_sync(0xFFFFFFFFu, isr);
            if (isr) {
                const uint32_t rk = acc + __popc(br & lt);
                if (rk < pn) {
                    rl[rk] = k;
                    rl2[rk] = iq[q];
                    iq[q] += 1;
                    cv[q] += 1;
                }
            }
            acc += __popc(br);
        }
        __syncwarp();
        acc = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (uint32_t(q) >= NQ) break;
            const uint32_t k = q * 32 + lane;
            const bool isd = k < N && cv[q] == mx;
            const uint32_t bd = __ballot_sync(0xFFFFFFFFu, isd);
            if (isd) {
                const uint32_t rk = acc + __popc(bd & lt);
                if (rk < pn) {
                    if (recv) recv[size_t(k) * b + oq[q]] = (rl2[rk] << 10) | rl[rk];
                    oq[q] += 1;
                    cv[q] -= 1;
                }
            }
            acc += __popc(bd);
        }
        __syncwarp();
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t k = q * 32 + lane;
        if (k < N) {
            outk[k] = oq[q];
            ink[k] = iq[q];
            if (oq[q] && iq[q]) atomicOr(status, 32u);  // a recipient became a donor
        }
    }
}

// Balance (balance.cpp:10-39) in closed form, all threads of the CTA.
// With counts c_k, F = sum, L = F / N: the reference loop ends when every
// count is L or L+1. A "donor unit" (k, l) is node k giving one fetch while
// at count l; a "recipient unit" (k, l) is node k receiving one at count l.
// The loop consumes donor units in (l desc, k asc) order and recipient units
// in (l asc, k asc) order (the first argmax / argmin only change when a level
// set is exhausted), and the t-th move pairs the t-th units of both lists.
// Mandatory units: donors at levels >= L+2, recipients at levels <= L-1
// (Dm, Rm of them); the longer side is padded with level-(L+1) donor or
// level-L recipient units in node order. Donor k's q-th move is its unit at
// level c_k - q and gives its q-th largest fetch id; the recipient appends it
// as its (l - c_k)-th incoming fetch. CTA `writer` also writes recv[].
__device__ void wide_balance_cf(const WideArgs& a, uint32_t N, uint32_t b, const uint32_t* fcnt, uint32_t* outk,
                                uint32_t* ink, uint32_t* lv, uint32_t* bsc, uint32_t* rl, uint32_t* rl2,
                                bool writer, uint32_t tid, uint32_t lane, uint32_t w) {
    const uint32_t lt = lanemask_lt_w();
    const uint32_t NQ = (N + 31) / 32;
    uint32_t cv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t k = q * 32 + lane;
        cv[q] = (uint32_t(q) < NQ && k < N) ? fcnt[k] : 0u;
    }
    if (w == 0) {
        uint32_t mx = 0, mn = 0xFFFFFFFFu, sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (uint32_t(q) < NQ && q * 32 + lane < N) {
                mx = max(mx, cv[q]);
                mn = min(mn, cv[q]);
                sum += cv[q];
            }
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        mn = __reduce_min_sync(0xFFFFFFFFu, mn);
        sum = __reduce_add_sync(0xFFFFFFFFu, sum);
        const uint32_t L = sum / N;
        uint32_t dm = 0, rm = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (uint32_t(q) < NQ && q * 32 + lane < N) {
                dm += cv[q] > L + 1 ? cv[q] - L - 1 : 0u;
                rm += cv[q] < L ? L - cv[q] : 0u;
            }
        dm = __reduce_add_sync(0xFFFFFFFFu, dm);
        rm = __reduce_add_sync(0xFFFFFFFFu, rm);
        if (lane == 0) {
            bsc[0] = L;
            bsc[1] = dm;
            bsc[2] = rm;
            bsc[3] = mn;
            bsc[4] = mx;
        }
    }
    __syncthreads();
    const uint32_t L = bsc[0], dm = bsc[1], rm = bsc[2], mn = bsc[3], mx = bsc[4];
    if (mx - mn <= 1) {
        for (uint32_t k = tid; k < N; k += kWT) outk[k] = ink[k] = 0;
        __syncthreads();
        return;
    }
    if (mx - mn + 1 > kLevCap) {  // very wide count spread: the round simulation
        if (w == 0) wide_balance(N, b, fcnt, outk, ink, rl, rl2, writer ? a.recv : nullptr, a.status, lane);
        __syncthreads();
        return;
    }
    const uint32_t mv = max(dm, rm), od = mv - dm, orr = mv - rm;
    uint32_t* lvge = lv;                // #{c_k >= l}
    uint32_t* lvle = lv + kLevCap;      // #{c_k <= l}
    uint32_t* lvds = lv + 2 * kLevCap;  // first donor unit of level l
    uint32_t* lvrs = lv + 3 * kLevCap;  // first recipient unit of level l
    for (uint32_t l = mn + w; l <= mx; l += kWW) {
        uint32_t ge = 0, le = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (uint32_t(q) >= NQ) break;
            const bool in = q * 32 + lane < N;
            ge += __popc(__ballot_sync(0xFFFFFFFFu, in && cv[q] >= l));
            le += __popc(__ballot_sync(0xFFFFFFFFu, in && cv[q] <= l));
        }
        if (lane == 0) {
            lvge[l - mn] = ge;
            lvle[l - mn] = le;
        }
    }
    __syncthreads();
    if (w == 0) {
        // donor levels mx, mx-1, .., L+2 (suffix sums); recipient levels mn .. L-1
        const uint32_t nd = mx >= L + 2 ? mx - L - 1 : 0u, nr = L > mn ? L - mn : 0u;
        uint32_t run = 0;
        for (uint32_t d0 = 0; d0 < nd; d0 += 32) {
            const uint32_t d = d0 + lane;
            const uint32_t v = d < nd ? lvge[mx - d - mn] : 0u;
            const uint32_t incl = warp_incl_scan(v, lane);
            if (d < nd) lvds[mx - d - mn] = run + incl - v;
            run += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        run = 0;
        for (uint32_t d0 = 0; d0 < nr; d0 += 32) {
            const uint32_t d = d0 + lane;
            const uint32_t v = d < nr ? lvle[d] : 0u;
            const uint32_t incl = warp_incl_scan(v, lane);
            if (d < nr) lvrs[d] = run + incl - v;
            run += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        // moves per node: mandatory units + the optional one
        uint32_t accd = 0, accr = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (uint32_t(q) >= NQ) break;
            const uint32_t k = q * 32 + lane;
            const bool in = k < N;
            const bool isd = in && cv[q] >= L + 1, isr = in && cv[q] <= L;
            const uint32_t bd = __ballot_sync(0xFFFFFFFFu, isd), br = __ballot_sync(0xFFFFFFFFu, isr);
            const uint32_t rd = accd + __popc(bd & lt), rr = accr + __popc(br & lt);
            if (in) {
                outk[k] = (cv[q] > L + 1 ? cv[q] - L - 1 : 0u) + ((isd && rd < od) ? 1u : 0u);
                ink[k] = (cv[q] < L ? L - cv[q] : 0u) + ((isr && rr < orr) ? 1u : 0u);
            }
            accd += __popc(bd);
            accr += __popc(br);
        }
    }
    __syncthreads();
    if (writer) {
        // recipient units -> ur[t] = (ii << 10 | r)
        for (uint32_t l = mn + w; l <= L; l += kWW) {
            const uint32_t base = l < L ? lvrs[l - mn] : rm, lim = l < L ? 0xFFFFFFFFu : orr;
            uint32_t acc = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (uint32_t(q) >= NQ) break;
                const uint32_t k = q * 32 + lane;
                const bool isr = k < N && cv[q] <= l;
                const uint32_t br = __ballot_sync(0xFFFFFFFFu, isr);
                const uint32_t rk = acc + __popc(br & lt);
                if (isr && rk < lim) a.ur[base + rk] = ((l - cv[q]) << 10) | k;
                acc += __popc(br);
            }
        }
        __syncthreads();
        // donor units: donor k's (c_k - l)-th move takes the t-th recipient unit
        for (uint32_t l = L + 1 + w; l <= mx; l += kWW) {
            const uint32_t base = l > L + 1 ? lvds[l - mn] : dm, lim = l > L + 1 ? 0xFFFFFFFFu : od;
            uint32_t acc = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (uint32_t(q) >= NQ) break;
                const uint32_t k = q * 32 + lane;
                const bool isd = k < N && cv[q] >= l;
                const uint32_t bd = __ballot_sync(0xFFFFFFFFu, isd);
                const uint32_t rk = acc + __popc(bd & lt);
                if (isd && rk < lim) a.recv[size_t(k) * b + (cv[q] - l)] = __ldcg(&a.ur[base + rk]);
                acc += __popc(bd);
            }
        }
    }
    __syncthreads();
}

// exclusive prefix of v[0..n) into out[0..n], out[n] = total (one warp)
__device__ __forceinline__ void warp_prefix(const uint32_t* v, uint32_t* out, uint32_t n, uint32_t lane) {
    uint32_t run = 0;
    for (uint32_t k0 = 0; k0 < n; k0 += 32) {
        const uint32_t k = k0 + lane;
        const uint32_t x = k < n ? v[k] : 0u;
        const uint32_t incl = warp_incl_scan(x, lane);
        if (k < n) out[k] = run + incl - x;
        run += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    if (lane == 0) out[n] = run;
}

// Multi-holder remap of staged items [mi0, mi0 + cntm) (one warp), exact
// and speculative: lane l evaluates item q0 + l against the counts M at the
// start of the batch. An item's decision depends only on M_k of its own
// candidate holders, so every item before the first one that has a holder
// chosen by an earlier lane of the batch decided exactly; that prefix
// commits (its lanes chose distinct nodes), the batch restarts after it.
// firstch[k] = earliest lane of the batch that chose node k (32: none).
__device__ __forceinline__ void multi_pass(const uint32_t* pairs, uint32_t* mpos, uint32_t* massign, uint32_t* M,
                                           uint32_t* firstch, uint32_t cntm, uint32_t mi0, uint32_t p0, bool pin,
                                           const uint32_t* st_np, const uint32_t* st_po, const uint32_t* st_j,
                                           const uint32_t* st_pr, uint32_t b, uint32_t lane) {
    auto pair_at = [&](uint32_t po, uint32_t t) {
        return pin ? st_pr[po + t] : __ldcg(&pairs[p0 + po + t]);
    };
    for (uint32_t q0 = 0; q0 < cntm;) {
        const uint32_t q = q0 + lane;
        const bool valid = q < cntm;
        const uint32_t np = valid ? st_np[q] : 0u, po = valid ? st_po[q] : 0u;
        uint32_t best = 0xFFFFFFFFu;
        for (uint32_t t = 0; t < np; ++t) {
            const uint32_t pr = pair_at(po, t), k = pr & 0x3FFu;
            const uint32_t cc = min(b, (pr >> 10) + M[k]);
            if (cc < b) best = min(best, (cc << 10) | k);
        }
        const bool chose = best != 0xFFFFFFFFu;
        if (chose) atomicMin(&firstch[best & 0x3FFu], lane);
        __syncwarp();
        bool aff = false;
        for (uint32_t t = 0; t < np && !aff; ++t) aff = firstch[pair_at(po, t) & 0x3FFu] < lane;
        const uint32_t abal = __ballot_sync(0xFFFFFFFFu, aff);
        const uint32_t nval = min(32u, cntm - q0);
        const uint32_t ncommit = abal ? min(nval, uint32_t(__ffs(abal) - 1)) : nval;
        __syncwarp();
        if (chose) firstch[best & 0x3FFu] = 32u;
        if (lane < ncommit) {
            if (chose) {
                const uint32_t k = best & 0x3FFu, mold = M[k];
                M[k] = mold + 1;
                mpos[size_t(k) * b + mold] = st_j[q];
            }
            massign[mi0 + q] = best;
        }
        __syncwarp();
        q0 += ncommit;
    }
}

// First scheduled step of id y after step g (the reference's occ[y][cursor]
// once step g's accesses are walked), from the inverse permutations.
__device__ __forceinline__ uint32_t next_step_after(const WideArgs& a, uint32_t y, uint32_t g) {
    for (uint32_t j = g / a.S; j < a.E; ++j) {
        const uint32_t p = __ldcg(&a.inv[size_t(a.order[j]) * a.D + y]);
        if (p == kNone) continue;
        const uint32_t st = j * a.S + p / a.B;
        if (st > g) return st;
    }
    return kNever;
}

// pipeline.cpp:103-114 for node k after its step-g advance: the ids a chunk
// read of its fetch list streams without being requested (redundant_ids,
// chunking.cpp:35-45, ascending) are inserted silently (buffer.cpp:48-53:
// resident ids are left alone) with their next scheduled step as key. Keep-C-
// smallest is associative, so the inserts form one miss run; the run is
// flushed early only when the slot array is about to overflow. Leader warp of
// the team (the team joins the evictions).
__device__ void redundant_inserts(const WideArgs& a, uint32_t k, uint32_t& bsz, uint32_t& top, uint32_t g,
                                  uint32_t lane, const Team& tm, const uint32_t* list, uint32_t L,
                                  uint32_t* sbuf /*[2*kSortCap] shared*/) {
    const uint32_t lt = lanemask_lt_w();
    // fetch ids of the list (items without the hit tag)
    uint32_t nf = 0;
    for (uint32_t c = 0; c < L; c += 32) {
        const uint32_t it = c + lane < L ? __ldcg(&list[c + lane]) : kHit;
        const bool f = !(it & kHit);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
        nf += __popc(bal);
    }
    if (nf < 2) return;
    uint32_t P2 = 1;
    while (P2 < nf) P2 <<= 1;
    uint32_t* v = P2 <= 2 * kSortCap ? sbuf : a.redbuf + size_t(k) * a.B;
    nf = 0;
    for (uint32_t c = 0; c < L; c += 32) {
        const uint32_t it = c + lane < L ? __ldcg(&list[c + lane]) : kHit;
        const bool f = !(it & kHit);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
        if (f) v[nf + __popc(bal & lt)] = it;
        nf += __popc(bal);
    }
    for (uint32_t q = nf + lane; q < P2; q += 32) v[q] = 0xFFFFFFFFu;
    __syncwarp();
    for (uint32_t sz = 2; sz <= P2; sz <<= 1)
        for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
            for (uint32_t r = lane; r < P2 / 2; r += 32) {
                const uint32_t x0 = 2 * st * (r / st) + (r % st), x1 = x0 + st;
                const bool up = (x0 & sz) == 0;
                const uint32_t p = v[x0], q = v[x1];
                if ((p > q) == up) {
                    v[x0] = q;
                    v[x1] = p;
                }
            }
            __syncwarp();
        }
    // greedy reads of span <= thr over the unique ids (chunking.cpp:17-30);
    // the gaps inside every chunk read are the redundant ids
    const uint32_t kw = k >> 5, kb = 1u << (k & 31);
    uint32_t* cntk = a.cnt + size_t(k) * (a.T + 1);
    unsigned long long* sk = a.slot + size_t(k) * a.SC;
    uint32_t i = 0;
    while (i < nf) {
        const uint32_t start = v[i];
        uint32_t j = i + 1, prev = start;
        // walk the read; between consecutive unique ids the gap ids go in
        while (j < nf && v[j] - start + 1 <= a.thr) {
            const uint32_t cur = v[j];
            if (cur != prev) {
                for (uint32_t y0 = prev + 1; y0 < cur; y0 += 32) {
                    // room for a full batch (SC >= C + 64)
                    if (bsz + 32 > a.SC && bsz > a.C) wide_evict(a, k, bsz, top, g, lane, tm);
                    const uint32_t y = y0 + lane;
                    bool ins = false;
                    uint32_t key = 0;
                    if (y < cur && __ldcg(&a.where[size_t(k) * a.D + y]) == kNone) {
                        ins = true;
                        key = next_step_after(a, y, g);
                    }
                    const uint32_t ib = __ballot_sync(0xFFFFFFFFu, ins);
                    if (ins) {
                        const uint32_t s2 = bsz + __popc(ib & lt);
                        a.where[size_t(k) * a.D + y] = s2;
                        sk[s2] = (static_cast<unsigned long long>(key) << 32) | y;
                        atomicAdd(&cntk[bin_of(key, a.T)], 1u);
                        atomicOr(&a.hm[size_t(y) * a.W + kw], kb);
                    }
                    top = max(top, __reduce_max_sync(0xFFFFFFFFu, ins && key != kNever ? key : 0u));
                    bsz += __popc(ib);
                    __syncwarp();
                }
                prev = cur;
            }
            ++j;
        }
        i = j;
    }
    if (bsz > a.C) wide_evict(a, k, bsz, top, g, lane, tm);
}

// LRU + chunk_insert_redundant (pipeline.cpp:103-114 with LruBuffer::
// insert_silent = touch_or_insert, buffer.cpp:88-91): the redundant ids of
// node k's step-g list (the gaps inside its chunk reads, ascending, as in
// redundant_inserts) are appended to the node's silent-touch row, where the
// LRU front walk finds them after the list in node time. Returns the row
// range [*r0, *r1). Leader warp of the node's team.
__device__ void lru_redundant_ids(const WideArgs& a, uint32_t k, uint32_t g, uint32_t lane, const uint32_t* list,
                                  uint32_t L, uint32_t* sbuf /*[2*kSortCap] shared*/, uint64_t* r0, uint64_t* r1) {
    const uint32_t lt = lanemask_lt_w();
    uint64_t* ro = a.lroff + size_t(k) * (a.T + 1);
    uint32_t* row = a.lred + size_t(k) * a.lcap;
    const uint64_t c0 = __ldcg(&ro[g]);
    uint64_t cur_out = c0;
    uint32_t nf = 0;
    for (uint32_t c = 0; c < L; c += 32) {
        const uint32_t it = c + lane < L ? __ldcg(&list[c + lane]) : kHit;
        nf += __popc(__ballot_sync(0xFFFFFFFFu, !(it & kHit)));
    }
    if (nf >= 2) {
        uint32_t P2 = 1;
        while (P2 < nf) P2 <<= 1;
        uint32_t* v = P2 <= 2 * kSortCap ? sbuf : a.redbuf + size_t(k) * a.B;
        nf = 0;
        for (uint32_t c = 0; c < L; c += 32) {
            const uint32_t it = c + lane < L ? __ldcg(&list[c + lane]) : kHit;
            const bool f = !(it & kHit);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
            if (f) v[nf + __popc(bal & lt)] = it;
            nf += __popc(bal);
        }
        for (uint32_t q = nf + lane; q < P2; q += 32) v[q] = 0xFFFFFFFFu;
        __syncwarp();
        for (uint32_t sz = 2; sz <= P2; sz <<= 1)
            for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
                for (uint32_t r = lane; r < P2 / 2; r += 32) {
                    const uint32_t x0 = 2 * st * (r / st) + (r % st), x1 = x0 + st;
                    const bool up = (x0 & sz) == 0;
                    const uint32_t p = v[x0], q = v[x1];
                    if ((p > q) == up) {
                        v[x0] = q;
                        v[x1] = p;
                    }
                }
                __syncwarp();
            }
        // greedy reads of span <= thr over the unique ids (chunking.cpp:17-30)
        uint32_t i = 0;
        while (i < nf) {
            const uint32_t start = v[i];
            uint32_t j = i + 1, prev = start;
            while (j < nf && v[j] - start + 1 <= a.thr) {
                const uint32_t cur = v[j];
                if (cur != prev) {
                    for (uint32_t y0 = prev + 1; y0 < cur; y0 += 32) {
                        const uint32_t y = y0 + lane;
                        const bool in = y < cur;
                        const uint32_t ib = __ballot_sync(0xFFFFFFFFu, in);
                        const uint64_t at = cur_out + __popc(ib & lt);
                        if (in && at < a.lcap) row[at] = y;
                        cur_out += __popc(ib);
                    }
                    prev = cur;
                }
                ++j;
            }
            i = j;
        }
        __syncwarp();
    }
    if (cur_out > a.lcap) {  // budget exceeded: the plan fails with a CapabilityError
        if (lane == 0) atomicOr(a.status, 1u << 20);
        cur_out = a.lcap;
    }
    if (lane == 0) ro[g + 1] = cur_out;
    __syncwarp();
    *r0 = c0;
    *r1 = cur_out;
}

__global__ void __launch_bounds__(kWT, 1) k_plan_wide(WideArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t P = cl.num_blocks(), c = cl.block_rank();
    extern __shared__ __align__(16) unsigned char wsm[];
    const uint32_t N = a.N, W = a.W, b = a.b;
    unsigned long long* sortb = reinterpret_cast<unsigned long long*>(wsm);  // [kWW][kSortCap]
    uint32_t* hist = reinterpret_cast<uint32_t*>(sortb + kWW * kSortCap);    // [kWW][256]
    uint32_t* wc = hist + kWW * 256;      // [kWW][N]
    uint32_t* cm = wc + kWW * N;          // [kWW][N]
    uint32_t* ctot = cm + kWW * N;        // [N] CTA totals (read remotely)
    uint32_t* base = ctot + N;            // [N]
    uint32_t* tot = base + N;             // [N]
    uint32_t* mk = tot + N;               // [N]
    uint32_t* size = mk + N;              // [N]
    uint32_t* fcnt = size + N;            // [N]
    uint32_t* lenpre = fcnt + N;          // [N]
    uint32_t* outk = lenpre + N;          // [N]
    uint32_t* ink = outk + N;             // [N]
    uint32_t* M = ink + N;                // [N] serial pass (CTA 0, read remotely)
    uint32_t* rl = M + N;                 // [N]
    uint32_t* rl2 = rl + N;               // [N]
    uint32_t* lenfin = rl2 + N;           // [N]
    uint32_t* freepre = lenfin + N;       // [N+1]
    uint32_t* noffpre = freepre + N + 1;  // [N+1]
    uint32_t* noff = noffpre + N + 1;     // [N+1]
    __shared__ unsigned long long wsc[kWW];
    __shared__ unsigned long long ctsc, msbase, mstot;
    __shared__ uint32_t wsf[kWW];
    __shared__ uint32_t ctf, fbase, ftot;
    __shared__ uint32_t bsc[8];

    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t gw = c * kWW + w, GW = P * kWW;
    const uint32_t lt = lanemask_lt_w();
    unsigned long long* my_sort = sortb + w * kSortCap;
    // eviction teams: tpn warps per node (power of two, within one CTA)
    __shared__ uint32_t team_ctl[kWW][8];
    uint32_t tpn = 1;
    while (tpn * 2 <= uint32_t(kWW) && GW / (tpn * 2) >= N) tpn *= 2;
    const Team tm{tpn, w % tpn, 1 + w / tpn, team_ctl[w / tpn], hist + (w - w % tpn) * 256};
    const uint32_t tg = c * (kWW / tpn) + w / tpn, NT = GW / tpn;
    size_t gbase = 0;
    unsigned long long pacc[7] = {0, 0, 0, 0, 0, 0, 0};
    unsigned long long tprev = clock64();
#define WPHASE(n)                                                  \
    if (a.prof && c == 0 && tid == 0) {                            \
        const unsigned long long tnow = clock64();                 \
        pacc[n] += tnow - tprev;                                   \
        tprev = tnow;                                              \
    }

    for (uint32_t g = 0; g < a.T; ++g) {
        const uint32_t i = g / a.S, t = g % a.S;
        const uint32_t lo = t * a.B, len = min(a.B, a.keep - lo);
        const uint32_t* row = a.trace + size_t(a.order[i]) * a.keep + lo;
        const uint32_t* nurow = a.nu + size_t(i) * a.keep + lo;
        const uint32_t R = ((len + GW * 32 - 1) / (GW * 32)) * 32;
        const uint32_t j0 = min(gw * R, len), j1 = min(j0 + R, len);
        if (a.lru && c == 0 && tid == 0) a.sbase[g] = uint32_t(gbase);

        // ------------------------------------------------ A: load + classify
        for (uint32_t k = lane; k < N; k += 32) {
            wc[w * N + k] = 0;
            cm[w * N + k] = 0;
        }
        unsigned long long msc = 0;
        __syncwarp();
        for (uint32_t cb = j0; cb < j1; cb += 32) {
            const uint32_t j = cb + lane;
            const bool valid = j < j1;
            uint32_t hc = 0, h = 0;
            if (valid) {
                const uint32_t x = row[j], nuj = nurow[j];
                uint32_t mw[8];  // all mask loads in flight before any store
#pragma unroll
                for (int q = 0; q < 8; ++q) mw[q] = uint32_t(q) < W ? __ldcg(&a.hm[size_t(x) * W + q]) : 0u;
                a.jx[j] = x;
                a.jnu[j] = nuj;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (uint32_t(q) < W) a.jmask[size_t(j) * W + q] = mw[q];
                    if (mw[q] && hc == 0) h = q * 32 + __ffs(mw[q]) - 1;
                    hc += __popc(mw[q]);
                }
            }
            if (a.remap) {
                const bool single = valid && hc == 1, multi = valid && hc >= 2;
                const uint32_t grp = __match_any_sync(0xFFFFFFFFu, single ? h : 0x10000u + lane);
                if (single && lane == uint32_t(__ffs(grp) - 1)) wc[w * N + h] += __popc(grp);
                const uint32_t mb = __ballot_sync(0xFFFFFFFFu, multi);
                const uint32_t hs = __reduce_add_sync(0xFFFFFFFFu, multi ? hc : 0u);
                msc += (static_cast<unsigned long long>(__popc(mb)) << 32) | hs;
                if (valid) a.jcls[j] = single ? (kClsSingle | h) : (multi ? kClsMulti : 0u);
            }
            __syncwarp();
        }
        if (lane == 0) wsc[w] = msc;
        __syncthreads();
        if (a.remap) {
            for (uint32_t k = tid; k < N; k += kWT) {
                uint32_t s = 0;
                for (uint32_t w2 = 0; w2 < uint32_t(kWW); ++w2) {
                    const uint32_t v = wc[w2 * N + k];
                    wc[w2 * N + k] = s;
                    s += v;
                }
                ctot[k] = s;
            }
            if (tid == 0) {
                unsigned long long s = 0;
                for (int w2 = 0; w2 < kWW; ++w2) {
                    const unsigned long long v = wsc[w2];
                    wsc[w2] = s;
                    s += v;
                }
                ctsc = s;
            }
        }
        cl.sync();  // (1)
        WPHASE(0)
        if (a.remap) {
            for (uint32_t k = tid; k < N; k += kWT) {
                uint32_t bs = 0, tt = 0;
                for (uint32_t c2 = 0; c2 < P; ++c2) {
                    const uint32_t v = cl.map_shared_rank(ctot, c2)[k];
                    if (c2 < c) bs += v;
                    tt += v;
                }
                base[k] = bs;
                tot[k] = tt;
            }
            if (tid == 0) {
                unsigned long long bs = 0, tt = 0;
                for (uint32_t c2 = 0; c2 < P; ++c2) {
                    const unsigned long long v = *cl.map_shared_rank(&ctsc, c2);
                    if (c2 < c) bs += v;
                    tt += v;
                }
                msbase = bs;
                mstot = tt;
            }
            __syncthreads();
            // ------------------------------- A2: exact single ranks, multi pairs
            for (uint32_t k = lane; k < N; k += 32) wc[w * N + k] += base[k];
            unsigned long long mrun = msbase + wsc[w];
            __syncwarp();
            for (uint32_t cb = j0; cb < j1; cb += 32) {
                const uint32_t j = cb + lane;
                const bool valid = j < j1;
                const uint32_t cls = valid ? a.jcls[j] : 0u;
                const bool single = (cls >> 30) == 1u, multi = (cls >> 30) == 2u;
                const uint32_t h = cls & 0x3FFu;
                const uint32_t grp = __match_any_sync(0xFFFFFFFFu, single ? h : 0x10000u + lane);
                const bool leader = single && lane == uint32_t(__ffs(grp) - 1);
                if (leader) cm[w * N + h] = grp;
                __syncwarp();
                if (single) a.jS[j] = wc[w * N + h] + __popc(grp & lt);
                const uint32_t mb = __ballot_sync(0xFFFFFFFFu, multi);
                uint32_t hcv = 0;
                if (multi)
                    for (uint32_t q = 0; q < W; ++q) hcv += __popc(a.jmask[size_t(j) * W + q]);
                const uint32_t hinc = warp_incl_scan(hcv, lane);
                if (multi) {
                    const uint32_t mi = uint32_t(mrun >> 32) + __popc(mb & lt);
                    const uint32_t po = uint32_t(mrun) + hinc - hcv;
                    uint32_t np = 0;
                    for (uint32_t q = 0; q < W; ++q) {
                        uint32_t m = a.jmask[size_t(j) * W + q];
                        while (m) {
                            const uint32_t k = q * 32 + __ffs(m) - 1;
                            m &= m - 1;
                            const uint32_t sk = wc[w * N + k] + __popc(cm[w * N + k] & lt);
                            if (sk < b) a.pairs[po + np++] = (sk << 10) | k;
                        }
                    }
                    a.mj[mi] = j;
                    a.mpo[mi] = po;
                    a.mhc[mi] = np;
                    a.jS[j] = mi;
                }
                __syncwarp();
                if (leader) {
                    wc[w * N + h] += __popc(grp);
                    cm[w * N + h] = 0;
                }
                mrun += (static_cast<unsigned long long>(__popc(mb)) << 32) |
                        __shfl_sync(0xFFFFFFFFu, hinc, 31);
                __syncwarp();
            }
        }
        cl.sync();  // (2)
        WPHASE(1)

        // ---------------- B: serial multi-holder pass (CTA 0; warp 0 decides)
        // The multi items' metadata and candidate pairs are staged in shared
        // memory by the whole CTA, so the serial chain is shared-memory only:
        // per item, lanes take its candidate (S_k, k) pairs, c_k = min(b,
        // S_k + M_k), the winner is REDUX.MIN of (c_k << 10 | k) over c_k < b
        // (lowest count, ties lowest k: locality.cpp:20-31).
        if (a.remap && c == 0) {
            uint32_t* st_np = reinterpret_cast<uint32_t*>(sortb);
            uint32_t* st_po = st_np + kMS;
            uint32_t* st_j = st_po + kMS;
            uint32_t* st_pr = st_j + kMS;
            for (uint32_t k = tid; k < N; k += kWT) {
                M[k] = 0;
                rl[k] = 32u;  // firstch of the speculative multi pass
            }
            const uint32_t nm = uint32_t(mstot >> 32), npairs = uint32_t(mstot);
            if (a.prof && tid == 0) {
                atomicAdd(&a.prof[10], static_cast<unsigned long long>(nm));
                atomicAdd(&a.prof[11], static_cast<unsigned long long>(npairs));
            }
            for (uint32_t mi0 = 0; mi0 < nm; mi0 += kMS) {
                const uint32_t cntm = min(kMS, nm - mi0);
                const uint32_t p0 = __ldcg(&a.mpo[mi0]);
                const uint32_t p1 = mi0 + cntm < nm ? __ldcg(&a.mpo[mi0 + cntm]) : npairs;
                const bool pin = p1 - p0 <= kMP;
                for (uint32_t q = tid; q < cntm; q += kWT) {
                    st_np[q] = __ldcg(&a.mhc[mi0 + q]);
                    st_po[q] = __ldcg(&a.mpo[mi0 + q]) - p0;
                    st_j[q] = __ldcg(&a.mj[mi0 + q]);
                }
                if (pin)
                    for (uint32_t q = tid; q < p1 - p0; q += kWT) st_pr[q] = __ldcg(&a.pairs[p0 + q]);
                __syncthreads();
                const unsigned long long tb0 = clock64();
                if (w == 0) {
                    multi_pass(a.pairs, a.mpos, a.massign, M, rl, cntm, mi0, p0, pin, st_np, st_po, st_j, st_pr,
                               b, lane);
                    if (a.prof && lane == 0) atomicAdd(&a.prof[12], clock64() - tb0);
                }
                __syncthreads();
            }

        }
        cl.sync();  // (3)
        WPHASE(2)

        // ---------------------------------- C1: hit / fetch, fetch counts
        if (a.remap) {
            for (uint32_t k = tid; k < N; k += kWT) {
                const uint32_t v = cl.map_shared_rank(M, 0)[k];
                mk[k] = v;
                size[k] = v + min(tot[k], b - v);
            }
        }
        for (uint32_t k = lane; k < N; k += 32) wc[w * N + k] = 0;
        __syncthreads();
        uint32_t fw = 0;
        for (uint32_t cb = j0; cb < j1; cb += 32) {
            const uint32_t j = cb + lane;
            const bool valid = j < j1;
            bool hit = false;
            uint32_t node = 0;
            if (valid) {
                if (a.remap) {
                    const uint32_t cls = a.jcls[j];
                    if ((cls >> 30) == 1u) hit = a.jS[j] < b - mk[cls & 0x3FFu];
                    else if ((cls >> 30) == 2u) hit = __ldcg(&a.massign[a.jS[j]]) != 0xFFFFFFFFu;
                } else {
                    node = j / b;
                    hit = (a.jmask[size_t(j) * W + (node >> 5)] >> (node & 31)) & 1u;
                }
            }
            const bool isf = valid && !hit;
            const uint32_t fbal = __ballot_sync(0xFFFFFFFFu, isf);
            if (!a.remap) {
                const uint32_t grp = __match_any_sync(0xFFFFFFFFu, isf ? node : 0x10000u + lane);
                if (isf && lane == uint32_t(__ffs(grp) - 1)) wc[w * N + node] += __popc(grp);
            }
            fw += __popc(fbal);
            __syncwarp();
        }
        if (lane == 0) wsf[w] = fw;
        __syncthreads();
        if (tid == 0) {
            uint32_t s = 0;
            for (int w2 = 0; w2 < kWW; ++w2) {
                const uint32_t v = wsf[w2];
                wsf[w2] = s;
                s += v;
            }
            ctf = s;
        }
        if (!a.remap)
            for (uint32_t k = tid; k < N; k += kWT) {
                uint32_t s = 0;
                for (uint32_t w2 = 0; w2 < uint32_t(kWW); ++w2) s += wc[w2 * N + k];
                ctot[k] = s;
            }
        cl.sync();  // (4)
        WPHASE(3)
        if (tid == 0) {
            uint32_t bs = 0, tt = 0;
            for (uint32_t c2 = 0; c2 < P; ++c2) {
                const uint32_t v = *cl.map_shared_rank(&ctf, c2);
                if (c2 < c) bs += v;
                tt += v;
            }
            fbase = bs;
            ftot = tt;
        }
        if (!a.remap)
            for (uint32_t k = tid; k < N; k += kWT) {
                uint32_t s = 0;
                for (uint32_t c2 = 0; c2 < P; ++c2) s += cl.map_shared_rank(ctot, c2)[k];
                fcnt[k] = s;
            }
        __syncthreads();
        // node tables (warp 0 of every CTA; identical everywhere)
        if (w == 0) {
            if (a.remap) {
                for (uint32_t k = lane; k < N; k += 32) rl[k] = b - size[k];
                __syncwarp();
                warp_prefix(rl, freepre, N, lane);
                __syncwarp();
                const uint32_t F = ftot;
                if (lane == 0 && F > freepre[N]) atomicOr(a.status, 64u);  // ran out of capacity
                for (uint32_t k = lane; k < N; k += 32) {
                    const uint32_t f = F > freepre[k] ? min(b - size[k], F - freepre[k]) : 0u;
                    fcnt[k] = f;
                    lenpre[k] = size[k] + f;
                }
            } else {
                for (uint32_t k = lane; k < N; k += 32) {
                    const uint32_t l = len > k * b ? min(b, len - k * b) : 0u;
                    lenpre[k] = l;
                    size[k] = l - fcnt[k];
                }
            }
            __syncwarp();
            warp_prefix(lenpre, noffpre, N, lane);
            __syncwarp();
        }
        __syncthreads();
        // --------------------------- C2: pre-balance positions, then balance
        {
            uint32_t fr = fbase + wsf[w];
            for (uint32_t cb = j0; cb < j1; cb += 32) {
                const uint32_t j = cb + lane;
                const bool valid = j < j1;
                bool hit = false;
                uint32_t node = 0, pos = 0;
                if (valid) {
                    if (a.remap) {
                        const uint32_t cls = a.jcls[j];
                        if ((cls >> 30) == 1u) {
                            const uint32_t h = cls & 0x3FFu, S = a.jS[j];
                            hit = S < b - mk[h];
                            if (hit) {
                                // multis assigned to h before j
                                const uint32_t* mp = a.mpos + size_t(h) * b;
                                uint32_t l0 = 0, l1 = mk[h];
                                while (l0 < l1) {
                                    const uint32_t mid = (l0 + l1) >> 1;
                                    if (__ldcg(&mp[mid]) < j) l0 = mid + 1; else l1 = mid;
                                }
                                node = h;
                                pos = S + l0;
                            }
                        } else if ((cls >> 30) == 2u) {
                            const uint32_t best = __ldcg(&a.massign[a.jS[j]]);
                            if (best != 0xFFFFFFFFu) {
                                hit = true;
                                node = best & 0x3FFu;
                                pos = best >> 10;
                            }
                        }
                    } else {
                        node = j / b;
                        pos = j - node * b;
                        hit = (a.jmask[size_t(j) * W + (node >> 5)] >> (node & 31)) & 1u;
                    }
                }
                const bool isf = valid && !hit;
                const uint32_t fbal = __ballot_sync(0xFFFFFFFFu, isf);
                if (isf && a.remap) {
                    const uint32_t f = fr + __popc(fbal & lt);
                    uint32_t l0 = 0, l1 = N;  // first k with freepre[k+1] > f
                    while (l0 < l1) {
                        const uint32_t mid = (l0 + l1) >> 1;
                        if (freepre[mid + 1] > f) l1 = mid; else l0 = mid + 1;
                    }
                    node = l0;
                    pos = size[node] + f - freepre[node];
                }
                if (valid) a.pre[noffpre[node] + pos] = j | (hit ? kHitM : 0u);
                fr += __popc(fbal);
            }
        }
        if (a.balance) {
            wide_balance_cf(a, N, b, fcnt, outk, ink, reinterpret_cast<uint32_t*>(sortb), bsc, rl, rl2, c == 0,
                            tid, lane, w);
        } else {
            for (uint32_t k = tid; k < N; k += kWT) outk[k] = ink[k] = 0;
            __syncthreads();
        }
        if (w == 0) {
            for (uint32_t k = lane; k < N; k += 32) lenfin[k] = lenpre[k] - outk[k] + ink[k];
            __syncwarp();
            warp_prefix(lenfin, noff, N, lane);
        }
        cl.sync();  // (5)
        WPHASE(4)

        // --------------------------------- D: final lists (one warp per node)
        for (uint32_t k = gw; k < N; k += GW) {
            const uint32_t lp = lenpre[k], pb = noffpre[k], fbk = noff[k], nout = outk[k];
            uint32_t* items = a.items + gbase;
            // final position dst of node kk: the plan item, and the buffer
            // advance record (id | resident-at-step-start on kk, next use)
            auto emit = [&](uint32_t kk, uint32_t dst, uint32_t it) {
                const uint32_t j = it & kIdM, x = __ldcg(&a.jx[j]);
                items[dst] = x | (it & kHitM);
                const uint32_t res = (__ldcg(&a.jmask[size_t(j) * W + (kk >> 5)]) >> (kk & 31)) & 1u;
                a.fx[dst] = x | (res << 31);
                a.fnu[dst] = __ldcg(&a.jnu[j]);
            };
            if (nout == 0) {
                for (uint32_t p = lane; p < lp; p += 32) {
                    const uint32_t it = __ldcg(&a.pre[pb + p]);
                    emit(k, fbk + p, it);
                }
            } else {
                uint32_t* mvk = a.movedbm + size_t(k) * a.MBW;
                const bool fits = fcnt[k] <= kSortCap;
                uint32_t nf = 0;
                for (uint32_t p0 = 0; p0 < lp; p0 += 32) {
                    const uint32_t p = p0 + lane;
                    const uint32_t it = p < lp ? __ldcg(&a.pre[pb + p]) : kHitM;
                    const bool isf = !(it & kHitM);
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, isf);
                    if (isf && fits)
                        my_sort[nf + __popc(bal & lt)] =
                            (static_cast<unsigned long long>(__ldcg(&a.jx[it])) << 32) | p;
                    nf += __popc(bal);
                }
                if (nf != fcnt[k] && lane == 0) atomicOr(a.status, 128u);
                auto move_one = [&](uint32_t q, uint32_t p) {
                    atomicOr(&mvk[p >> 5], 1u << (p & 31));
                    const uint32_t rec = __ldcg(&a.recv[size_t(k) * b + q]);
                    const uint32_t r = rec & 0x3FFu, ii = rec >> 10;
                    const uint32_t dest = noff[r] + lenpre[r] + ii;
                    emit(r, dest, __ldcg(&a.pre[pb + p]));
                };
                if (fits) {
                    uint32_t P2 = 1;
                    while (P2 < nf) P2 <<= 1;
                    for (uint32_t q = nf + lane; q < P2; q += 32) my_sort[q] = 0ull;
                    __syncwarp();
                    for (uint32_t sz = 2; sz <= P2; sz <<= 1) {
                        for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
                            for (uint32_t r = lane; r < P2 / 2; r += 32) {
                                const uint32_t x0 = 2 * st * (r / st) + (r % st), x1 = x0 + st;
                                const bool desc = (x0 & sz) == 0;
                                const unsigned long long u = my_sort[x0], v = my_sort[x1];
                                if ((u < v) == desc) {
                                    my_sort[x0] = v;
                                    my_sort[x1] = u;
                                }
                            }
                            __syncwarp();
                        }
                    }
                    for (uint32_t q = lane; q < nout; q += 32) move_one(q, uint32_t(my_sort[q]));
                } else {
                    // repeated extraction of the largest unmoved fetch id
                    for (uint32_t q = 0; q < nout; ++q) {
                        unsigned long long best = 0;
                        for (uint32_t p0 = 0; p0 < lp; p0 += 32) {
                            const uint32_t p = p0 + lane;
                            if (p < lp) {
                                const uint32_t it = __ldcg(&a.pre[pb + p]);
                                const bool mv = (__ldcg(&mvk[p >> 5]) >> (p & 31)) & 1u;
                                if (!(it & kHitM) && !mv)
                                    best = max(best, (static_cast<unsigned long long>(__ldcg(&a.jx[it]) + 1ull) << 32) | p);
                            }
                        }
#pragma unroll
                        for (int d = 16; d > 0; d >>= 1) best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, d));
                        if (lane == 0) move_one(q, uint32_t(best));
                        __syncwarp();
                    }
                }
                __syncwarp();
                uint32_t kept = 0;
                for (uint32_t p0 = 0; p0 < lp; p0 += 32) {
                    const uint32_t p = p0 + lane;
                    const bool valid = p < lp;
                    const uint32_t it = valid ? __ldcg(&a.pre[pb + p]) : 0u;
                    const bool keep = valid && !((__ldcg(&mvk[p >> 5]) >> (p & 31)) & 1u);
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
                    if (keep) {
                        const uint32_t dst = fbk + kept + __popc(bal & lt);
                        emit(k, dst, it);
                    }
                    kept += __popc(bal);
                }
                __syncwarp();
                for (uint32_t wd = lane; wd < (lp + 31) / 32; wd += 32) mvk[wd] = 0;
            }
            if (lane == 0) {
                a.node_off[size_t(g) * (N + 1) + k] = fbk;
                if (k == N - 1) a.node_off[size_t(g) * (N + 1) + N] = noff[N];
                if (a.fb) a.fb[size_t(g) * N + k] = fcnt[k];
                if (a.fa) a.fa[size_t(g) * N + k] = fcnt[k] - outk[k] + ink[k];
            }
        }
        cl.sync();  // (6)
        WPHASE(5)

        // ------------------------------- E: buffer advance (one warp per node)
        // List order, runs of equal residency-at-step-start (buffer.cpp:37-46
        // per access == re-key runs, and insert runs followed by one eviction
        // of the (size - C)+ largest). Records are prefetched a chunk ahead;
        // a resident's slot is read once per chunk and re-read only after an
        // eviction in the same chunk (compaction may have moved it).
        for (uint32_t k = tg; k < N && a.advance; k += NT) {
            if (tm.wr != 0) {  // helper warp: join the leader's eviction scans
                for (;;) {
                    tm.sync();
                    const uint32_t cmd = tm.ctl[0];
                    if (cmd == 1) evict_team(a, k, tm, lane);
                    tm.sync();
                    if (cmd != 1) break;
                }
                continue;
            }
            if (a.lru) {  // LruBuffer (buffer.cpp:61-82) through lru.cuh
                uint32_t* ns = a.nst + size_t(k) * 8;
                LruNode st{__ldcg(&ns[0]), __ldcg(&ns[2]), __ldcg(&ns[3]), __ldcg(&ns[4]), __ldcg(&ns[5]), 0};
                const LruPlanView v{a.items, a.node_off, nullptr, a.sbase, N, k,
                                    a.lroff ? a.lroff + size_t(k) * (a.T + 1) : nullptr,
                                    a.lred ? a.lred + size_t(k) * a.lcap : nullptr, 1};
                const uint32_t kw = k >> 5, kb = 1u << (k & 31);
                if (a.insred && lane == 0) {  // no silent entries of step g until they are appended
                    uint64_t* ro = a.lroff + size_t(k) * (a.T + 1);
                    ro[g + 1] = __ldcg(&ro[g]);
                }
                __syncwarp();
                auto on_miss = [&](uint32_t x, uint32_t y) {
                    atomicOr(&a.hm[size_t(x) * W + kw], kb);
                    if (y != kNone) atomicAnd(&a.hm[size_t(y) * W + kw], ~kb);
                };
                lru_step(v, st, a.where + size_t(k) * a.D, a.items + gbase + noff[k], noff[k + 1] - noff[k], a.C, lane,
                         a.status, [](uint32_t, uint32_t) {}, on_miss);
                if (a.insred) {  // silent touches after the list (pipeline.cpp:103-114)
                    uint64_t r0 = 0, r1 = 0;
                    lru_redundant_ids(a, k, g, lane, a.items + gbase + noff[k], noff[k + 1] - noff[k],
                                      reinterpret_cast<uint32_t*>(my_sort), &r0, &r1);
                    lru_step(v, st, a.where + size_t(k) * a.D, a.lred + size_t(k) * a.lcap + r0, uint32_t(r1 - r0),
                             a.C, lane, a.status, [](uint32_t, uint32_t) {}, on_miss);
                }
                if (lane == 0) {
                    ns[0] = st.size;
                    ns[2] = st.t;
                    ns[3] = st.fg;
                    ns[4] = st.fi;
                    ns[5] = st.ft;
                    tm.ctl[0] = 0;  // release the helpers
                }
                __syncwarp();
                tm.sync();
                tm.sync();
                continue;
            }
            uint32_t bsz = __ldcg(&a.nst[k * 8 + 0]), top = __ldcg(&a.nst[k * 8 + 1]);
            const uint32_t lb = noff[k], le = noff[k + 1];
            const uint32_t kw = k >> 5, kb = 1u << (k & 31);
            uint32_t* cntk = a.cnt + size_t(k) * (a.T + 1);
            unsigned long long* sk = a.slot + size_t(k) * a.SC;
            const uint32_t* whk = a.where + size_t(k) * a.D;
            bool pending = false;
            uint32_t nxr = 0, nnu = 0;
            if (lb + lane < le) {
                nxr = __ldcg(&a.fx[lb + lane]);
                nnu = __ldcg(&a.fnu[lb + lane]);
            }
            for (uint32_t p0 = lb; p0 < le; p0 += 32) {
                const bool valid = p0 + lane < le;
                const uint32_t xr = nxr, nuv = nnu;
                if (p0 + 32 + lane < le) {
                    nxr = __ldcg(&a.fx[p0 + 32 + lane]);
                    nnu = __ldcg(&a.fnu[p0 + 32 + lane]);
                }
                const uint32_t x = xr & kIdM;
                const bool res = valid && (xr >> 31);
                uint32_t ws = res ? __ldcg(&whk[x]) : 0u;
                uint32_t old = res ? uint32_t(__ldcg(&sk[ws]) >> 32) : 0u;
                const uint32_t vbal = __ballot_sync(0xFFFFFFFFu, valid);
                const uint32_t rbal = __ballot_sync(0xFFFFFFFFu, res);
                uint32_t done = 0;
                while (done != vbal) {
                    const uint32_t first = __ffs(vbal & ~done) - 1;
                    const bool hitrun = (rbal >> first) & 1u;
                    const uint32_t same = hitrun ? rbal : (vbal & ~rbal);
                    const uint32_t after = (~same) & vbal & ~((2u << first) - 1u);
                    const uint32_t stop = after ? __ffs(after) - 1 : 32u;
                    const uint32_t run = (stop == 32 ? 0xFFFFFFFFu : ((1u << stop) - 1u)) & ~((1u << first) - 1u) & vbal;
                    const bool mine = (run >> lane) & 1u;
                    if (hitrun && pending) {
                        if (bsz > a.C) {
                            wide_evict(a, k, bsz, top, g, lane, tm);
                            if (res && !((done >> lane) & 1u)) {  // slots may have moved
                                ws = __ldcg(&whk[x]);
                                old = uint32_t(__ldcg(&sk[ws]) >> 32);
                            }
                        }
                        pending = false;
                    }
                    if (mine) {
                        if (hitrun) {  // buffer.cpp:37-41 re-key
                            sk[ws] = (static_cast<unsigned long long>(nuv) << 32) | x;
                            if (old != nuv) {
                                atomicSub(&cntk[bin_of(old, a.T)], 1u);
                                atomicAdd(&cntk[bin_of(nuv, a.T)], 1u);
                            }
                        } else {  // buffer.cpp:42-46 insert
                            const uint32_t s2 = bsz + __popc(run & lt);
                            a.where[size_t(k) * a.D + x] = s2;
                            sk[s2] = (static_cast<unsigned long long>(nuv) << 32) | x;
                            atomicAdd(&cntk[bin_of(nuv, a.T)], 1u);
                            atomicOr(&a.hm[size_t(x) * W + kw], kb);
                        }
                    }
                    top = max(top, __reduce_max_sync(0xFFFFFFFFu, mine && nuv != kNever ? nuv : 0u));
                    __syncwarp();
                    if (!hitrun) {
                        bsz += __popc(run);
                        pending = true;
                    }
                    done |= run;
                }
            }
            if (pending && bsz > a.C) wide_evict(a, k, bsz, top, g, lane, tm);
            if (a.insred)
                redundant_inserts(a, k, bsz, top, g, lane, tm, a.items + gbase + lb, le - lb,
                                  reinterpret_cast<uint32_t*>(my_sort));
            if (lane == 0) {
                a.nst[k * 8 + 0] = bsz;
                a.nst[k * 8 + 1] = top;
                tm.ctl[0] = 0;  // release the helpers
            }
            __syncwarp();
            tm.sync();
            tm.sync();
        }
        cl.sync();  // (7)
        WPHASE(6)
        gbase += len;
    }
#undef WPHASE
    if (a.prof && c == 0 && tid == 0)
        for (int q = 0; q < 7; ++q) a.prof[q] = pacc[q];
}

// ---- balance_step (balance.cpp:10-39) on one step's lists, one CTA: the
// closed-form move table of wide_balance_cf, then the donors' q-th largest
// fetch ids (first occurrence on equal ids, balance.cpp:27-30) move to their
// recipients' tails; everything else keeps its order.
struct BalArgs {
    const uint32_t* items;  // [total] id | hit
    const uint32_t* off;    // [N+1]
    uint32_t* out;          // [total]
    uint32_t* out_off;      // [N+1]
    uint32_t* moved;        // [total] scratch flags, zero
    unsigned long long* moves;
    uint32_t N, Lmax;
};

__global__ void __launch_bounds__(kWT, 1) k_balance_lists(BalArgs b, WideArgs a) {
    extern __shared__ __align__(16) unsigned char bsm[];
    unsigned long long* sortb = reinterpret_cast<unsigned long long*>(bsm);  // [kWW][kSortCap]
    uint32_t* lv = reinterpret_cast<uint32_t*>(sortb + kWW * kSortCap);     // [4 * kLevCap]
    uint32_t* fcnt = lv + 4 * kLevCap;
    uint32_t* outk = fcnt + b.N;
    uint32_t* ink = outk + b.N;
    uint32_t* rl = ink + b.N;
    uint32_t* rl2 = rl + b.N;
    uint32_t* lenpre = rl2 + b.N;
    uint32_t* lenfin = lenpre + b.N;
    uint32_t* noff = lenfin + b.N;  // [N+1]
    __shared__ uint32_t bsc[8];
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5, N = b.N;
    const uint32_t lt = lanemask_lt_w();
    for (uint32_t k = w; k < N; k += kWW) {
        const uint32_t lo = b.off[k], hi = b.off[k + 1];
        uint32_t f = 0;
        for (uint32_t p = lo + lane; p < hi; p += 32) f += !(b.items[p] & kHitM);
        f = __reduce_add_sync(0xFFFFFFFFu, f);
        if (lane == 0) {
            fcnt[k] = f;
            lenpre[k] = hi - lo;
        }
    }
    __syncthreads();
    wide_balance_cf(a, N, b.Lmax, fcnt, outk, ink, lv, bsc, rl, rl2, true, tid, lane, w);
    if (w == 0) {
        for (uint32_t k = lane; k < N; k += 32) lenfin[k] = lenpre[k] - outk[k] + ink[k];
        __syncwarp();
        warp_prefix(lenfin, noff, N, lane);
    }
    __syncthreads();
    unsigned long long* my_sort = sortb + w * kSortCap;
    unsigned long long mv = 0;
    for (uint32_t k = w; k < N; k += kWW) {
        const uint32_t lo = b.off[k], lp = lenpre[k], nout = outk[k];
        mv += nout;
        auto move_one = [&](uint32_t q, uint32_t p) {
            b.moved[lo + p] = 1;
            const uint32_t rec = __ldcg(&a.recv[size_t(k) * b.Lmax + q]);
            const uint32_t r = rec & 0x3FFu, ii = rec >> 10;
            b.out[noff[r] + lenpre[r] + ii] = b.items[lo + p];
        };
        if (nout) {
            const bool fits = fcnt[k] <= kSortCap;
            uint32_t nf = 0;
            for (uint32_t p0 = 0; p0 < lp; p0 += 32) {
                const uint32_t p = p0 + lane;
                const uint32_t it = p < lp ? b.items[lo + p] : kHitM;
                const bool isf = !(it & kHitM);
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, isf);
                // (id desc, position asc): the largest id, first occurrence
                if (isf && fits)
                    my_sort[nf + __popc(bal & lt)] = (static_cast<unsigned long long>(it) << 32) | (0xFFFFFFFFu - p);
                nf += __popc(bal);
            }
            if (fits) {
                uint32_t P2 = 1;
                while (P2 < nf) P2 <<= 1;
                for (uint32_t q = nf + lane; q < P2; q += 32) my_sort[q] = 0ull;
                __syncwarp();
                for (uint32_t sz = 2; sz <= P2; sz <<= 1)
                    for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
                        for (uint32_t r = lane; r < P2 / 2; r += 32) {
                            const uint32_t x0 = 2 * st * (r / st) + (r % st), x1 = x0 + st;
                            const bool desc = (x0 & sz) == 0;
                            const unsigned long long u = my_sort[x0], v = my_sort[x1];
                            if ((u < v) == desc) {
                                my_sort[x0] = v;
                                my_sort[x1] = u;
                            }
                        }
                        __syncwarp();
                    }
                for (uint32_t q = lane; q < nout; q += 32) move_one(q, 0xFFFFFFFFu - uint32_t(my_sort[q]));
            } else {
                for (uint32_t q = 0; q < nout; ++q) {
                    unsigned long long best = 0;
                    for (uint32_t p = lane; p < lp; p += 32) {
                        const uint32_t it = b.items[lo + p];
                        if (!(it & kHitM) && !__ldcg(&b.moved[lo + p]))
                            best = max(best, (static_cast<unsigned long long>(it + 1ull) << 32) | (0xFFFFFFFFu - p));
                    }
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, d));
                    if (lane == 0) move_one(q, 0xFFFFFFFFu - uint32_t(best));
                    __syncwarp();
                }
            }
            __syncwarp();
        }
        uint32_t kept = 0;
        for (uint32_t p0 = 0; p0 < lp; p0 += 32) {
            const uint32_t p = p0 + lane;
            const bool keep = p < lp && !(nout && __ldcg(&b.moved[lo + p]));
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
            if (keep) b.out[noff[k] + kept + __popc(bal & lt)] = b.items[lo + p];
            kept += __popc(bal);
        }
    }
    if (lane == 0 && mv) atomicAdd(b.moves, mv);
    for (uint32_t k = tid; k <= N; k += kWT) b.out_off[k] = noff[k];
}

__global__ void k_set_holders(const unsigned long long* __restrict__ roff, const uint32_t* __restrict__ ids,
                              uint32_t N, uint32_t W, uint32_t* __restrict__ hm) {
    const uint64_t total = roff[N];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t l0 = 0, l1 = N;  // node k of entry i: first k with roff[k+1] > i
        while (l0 < l1) {
            const uint32_t mid = (l0 + l1) >> 1;
            if (roff[mid + 1] > i) l1 = mid; else l0 = mid + 1;
        }
        atomicOr(&hm[size_t(ids[i]) * W + (l0 >> 5)], 1u << (l0 & 31));
    }
}

}  // namespace

int plan_wide_device(const PlanDims& dm, uint64_t C, int lru, int remap, int balance, int insred, uint64_t thr,
                     const uint32_t* d_trace, const uint32_t* d_order, const uint32_t* d_inv, const uint32_t* d_nu,
                     uint32_t* d_items, uint32_t* d_node_off, uint32_t* d_fb, uint32_t* d_fa, uint32_t* d_status,
                     cudaStream_t st, const uint32_t* d_hm_init, int advance) {
    if (dm.N > kWMaxN)
        return set_error(kCapability, "plan: device planner supports num_nodes <= 256 in this build");
    if (dm.b >= (1u << 21)) return set_error(kCapability, "plan: local_batch must be < 2^21 on device");
    if (dm.B >= (1ull << 30) || dm.T >= 0xFFFFFFF0ull)
        return set_error(kCapability, "plan: global batch / steps too large for the device planner");
    const uint32_t N = dm.N, W = (N + 31) / 32;
    const uint64_t Ceff = std::min<uint64_t>(C, dm.D);
    const uint64_t SC = Ceff + std::max<uint64_t>(dm.B, 64);  // a miss run, or a batch of silent inserts
    if (SC >= (1ull << 31)) return set_error(kCapability, "plan: buffer capacity too large for the device planner");
    Scratch sc(st);
    WideArgs a{};
    a.D = uint32_t(dm.D);
    a.N = N;
    a.W = W;
    a.b = dm.b;
    a.B = uint32_t(dm.B);
    a.S = uint32_t(dm.S);
    a.keep = uint32_t(dm.keep);
    a.T = uint32_t(dm.T);
    a.C = uint32_t(Ceff);
    a.SC = uint32_t(SC);
    a.EBW = uint32_t((SC + 31) / 32);
    a.MBW = (dm.b + 31) / 32;
    a.remap = remap;
    a.balance = balance;
    a.lru = lru;
    a.insred = insred;
    a.thr = uint32_t(std::min<uint64_t>(thr, 0xFFFFFFFFull));
    a.E = dm.E;
    a.inv = d_inv;
    a.redbuf = insred ? sc.get<uint32_t>(size_t(N) * dm.B) : nullptr;
    if (insred && lru) {
        // each node's redundant ids (<= thr - 1 per fetch id), kept for the
        // LRU front walk; beyond the budget the plan reports a CapabilityError
        const uint64_t per_node = (dm.E * dm.keep + N - 1) / N * 2 + dm.B;
        const uint64_t want = per_node * std::max<uint64_t>(1, std::min<uint64_t>(thr, 64) - 1);
        a.lcap = std::min<uint64_t>(want, (uint64_t(2) << 30) / 4 / N);
        a.lred = sc.get<uint32_t>(size_t(N) * a.lcap);
        a.lroff = sc.get<uint64_t>(size_t(N) * (dm.T + 1));
        if (!a.lred || !a.lroff) return set_error(kInternal, "plan: wide planner scratch allocation failed");
        LSG_CUDA(cudaMemsetAsync(a.lroff, 0, size_t(N) * (dm.T + 1) * 8, st));
    }
    if (insred && !a.redbuf) return set_error(kInternal, "plan: wide planner scratch allocation failed");
    a.trace = d_trace;
    a.order = d_order;
    a.nu = d_nu;
    a.hm = sc.get<uint32_t>(size_t(dm.D) * W);
    a.where = sc.get<uint32_t>(size_t(N) * dm.D);
    a.slot = sc.get<unsigned long long>(size_t(N) * SC);
    a.cnt = sc.get<uint32_t>(size_t(N) * (dm.T + 1));
    a.nst = sc.get<uint32_t>(size_t(N) * 8);
    a.sbase = sc.get<uint32_t>(dm.T + 1);
    a.evb = sc.get<uint32_t>(size_t(N) * a.EBW);
    a.cand = sc.get<uint32_t>(size_t(N) * SC);
    a.candid = sc.get<uint32_t>(size_t(N) * SC);
    a.holes = sc.get<uint32_t>(size_t(N) * SC);
    a.movedbm = sc.get<uint32_t>(size_t(N) * a.MBW);
    a.jx = sc.get<uint32_t>(dm.B);
    a.jnu = sc.get<uint32_t>(dm.B);
    a.jmask = sc.get<uint32_t>(size_t(dm.B) * W);
    a.jcls = sc.get<uint32_t>(dm.B);
    a.jS = sc.get<uint32_t>(dm.B);
    a.pre = sc.get<uint32_t>(dm.B);
    a.fx = sc.get<uint32_t>(dm.B);
    a.fnu = sc.get<uint32_t>(dm.B);
    a.mj = sc.get<uint32_t>(dm.B);
    a.mpo = sc.get<uint32_t>(dm.B);
    a.mhc = sc.get<uint32_t>(dm.B);
    a.pairs = sc.get<uint32_t>(size_t(dm.B) * N);
    a.massign = sc.get<uint32_t>(dm.B);
    a.mpos = sc.get<uint32_t>(size_t(N) * dm.b);
    a.recv = sc.get<uint32_t>(size_t(N) * dm.b);
    a.ur = sc.get<uint32_t>(dm.B);
    if (!a.hm || !a.where || !a.slot || !a.cnt || !a.nst || !a.sbase || !a.evb || !a.cand || !a.candid || !a.holes || !a.movedbm ||
        !a.jx || !a.jnu || !a.jmask || !a.jcls || !a.jS || !a.pre || !a.fx || !a.fnu || !a.mj || !a.mpo || !a.mhc ||
        !a.pairs || !a.massign || !a.mpos || !a.recv || !a.ur)
        return set_error(kInternal, "plan: wide planner scratch allocation failed");
    if (d_hm_init) LSG_CUDA(cudaMemcpyAsync(a.hm, d_hm_init, size_t(dm.D) * W * 4, cudaMemcpyDeviceToDevice, st));
    else LSG_CUDA(cudaMemsetAsync(a.hm, 0, size_t(dm.D) * W * 4, st));
    a.advance = advance;
    LSG_CUDA(cudaMemsetAsync(a.where, 0xFF, size_t(N) * dm.D * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.cnt, 0, size_t(N) * (dm.T + 1) * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.nst, 0, size_t(N) * 32, st));
    LSG_CUDA(cudaMemsetAsync(a.evb, 0, size_t(N) * a.EBW * 4, st));
    LSG_CUDA(cudaMemsetAsync(a.movedbm, 0, size_t(N) * a.MBW * 4, st));
    a.items = d_items;
    a.node_off = d_node_off;
    a.fb = d_fb;
    a.fa = d_fa;
    a.status = d_status;
    a.prof = profiling() ? sc.get<unsigned long long>(16) : nullptr;
    if (a.prof) LSG_CUDA(cudaMemsetAsync(a.prof, 0, 128, st));

    const size_t smem = size_t(kWW) * kSortCap * 8 + size_t(kWW) * 256 * 4 +
                        (size_t(2) * kWW * N + 14 * size_t(N) + 3 * size_t(N + 1)) * 4;
    LSG_CUDA(cudaFuncSetAttribute(k_plan_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    LSG_CUDA(cudaFuncSetAttribute(k_plan_wide, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int want = 16;
    if (const char* e = std::getenv("LSG_WIDE_CLUSTER")) want = std::max(1, std::min(16, std::atoi(e)));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.blockDim = dim3(kWT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    int P = want;
    for (; P >= 1; P >>= 1) {
        cfg.gridDim = dim3(P);
        attr[0].val.clusterDim.x = P;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_plan_wide, &cfg) == cudaSuccess && ncl >= 1) break;
        cudaGetLastError();
    }
    if (P < 1) return set_error(kCapability, "plan: no thread-block cluster fits the wide planner");
    LSG_CUDA(cudaLaunchKernelEx(&cfg, k_plan_wide, a));
    LSG_LAUNCH_CHECK("k_plan_wide");
    if (a.prof) {
        unsigned long long h[16];
        LSG_CUDA(cudaMemcpyAsync(h, a.prof, sizeof h, cudaMemcpyDeviceToHost, st));
        fprintf(stderr, "[lsg profile] wide planner: %llu evictions (%.0f slots scanned each), %llu multi items (%llu pairs)\n",
                h[8], double(h[9]) / double(h[8] ? h[8] : 1), h[10], h[11]);
        fprintf(stderr, "[lsg profile] wide planner: serial multi loop %.1f kcyc total (%.0f cyc/item)\n", h[12] / 1e3,
                double(h[12]) / double(h[10] ? h[10] : 1));
        LSG_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[lsg profile] wide planner: cluster of %d CTAs x %d threads, %zu B smem, N=%u B=%llu T=%llu\n",
                P, kWT, smem, N, (unsigned long long)dm.B, (unsigned long long)dm.T);
        const char* names[7] = {"A load/classify", "A2 ranks/pairs", "B multi pass", "C1 hit/fetch counts",
                                "C2 positions+balance", "D final lists", "E buffer advance"};
        unsigned long long tot = 0;
        for (int q = 0; q < 7; ++q) tot += h[q];
        for (int q = 0; q < 7; ++q)
            fprintf(stderr, "[lsg profile]   %-22s %10.1f kcyc  %6.2f%%  %8.0f cyc/step\n", names[q], h[q] / 1e3,
                    100.0 * h[q] / (tot ? tot : 1), double(h[q]) / double(dm.T ? dm.T : 1));
    }
    return kOk;
}

}  // namespace lsg

using namespace lsg;

extern "C" {

// remap_step / slice_step (locality.cpp:7-73) of one batch against explicit
// residency sets: node k holds h_res_ids[h_res_off[k] .. h_res_off[k+1]).
// The cluster step loop runs one step without a buffer advance.
int lsg_remap_step(const uint64_t* h_res_off, const uint32_t* h_res_ids, uint32_t N, const uint32_t* h_batch,
                   uint64_t len, uint64_t local_batch, int32_t slice, uint32_t* h_items, uint32_t* h_node_off,
                   void* stream) {
    const char* who = slice ? "slice_step" : "remap_step";
    if (N == 0) return set_error(kValidation, std::string(who) + ": no nodes");
    if (local_batch == 0) return set_error(kValidation, std::string(who) + ": local_batch must be >= 1");
    if (len > uint64_t(N) * local_batch)
        return set_error(kValidation, std::string(who) + ": batch larger than N * local_batch");
    if (N > kWMaxN) return set_error(kCapability, std::string(who) + ": num_nodes <= 256 on the device");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint64_t D = 1;
    for (uint64_t i = 0; i < len; ++i) D = std::max<uint64_t>(D, uint64_t(h_batch[i]) + 1);
    const uint64_t nres = h_res_off[N];
    for (uint64_t i = 0; i < nres; ++i) D = std::max<uint64_t>(D, uint64_t(h_res_ids[i]) + 1);
    if (D >= (1ull << 31)) return set_error(kCapability, std::string(who) + ": sample ids must be < 2^31 on device");
    for (uint32_t k = 0; k < N; ++k)
        if (h_res_off[k + 1] < h_res_off[k]) return set_error(kValidation, std::string(who) + ": bad residency offsets");
    h_node_off[0] = 0;
    if (len == 0) {
        for (uint32_t k = 0; k <= N; ++k) h_node_off[k] = 0;
        return kOk;
    }
    const uint32_t W = (N + 31) / 32;
    Scratch sc(st);
    uint32_t* hm = sc.get<uint32_t>(size_t(D) * W);
    unsigned long long* roff = sc.get<unsigned long long>(N + 1);
    uint32_t* rid = sc.get<uint32_t>(nres + 1);
    uint32_t* trace = sc.get<uint32_t>(len);
    uint32_t* order = sc.get<uint32_t>(1);
    uint32_t* nu = sc.get<uint32_t>(len);
    uint32_t* items = sc.get<uint32_t>(len);
    uint32_t* off = sc.get<uint32_t>(N + 1);
    uint32_t* status = sc.get<uint32_t>(1);
    if (!hm || !roff || !rid || !trace || !order || !nu || !items || !off || !status)
        return set_error(kInternal, "remap_step: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(hm, 0, size_t(D) * W * 4, st));
    LSG_CUDA(cudaMemsetAsync(order, 0, 4, st));
    LSG_CUDA(cudaMemsetAsync(nu, 0xFF, len * 4, st));
    LSG_CUDA(cudaMemsetAsync(status, 0, 4, st));
    LSG_CUDA(cudaMemcpyAsync(roff, h_res_off, (N + 1) * 8, cudaMemcpyHostToDevice, st));
    if (nres) LSG_CUDA(cudaMemcpyAsync(rid, h_res_ids, nres * 4, cudaMemcpyHostToDevice, st));
    LSG_CUDA(cudaMemcpyAsync(trace, h_batch, len * 4, cudaMemcpyHostToDevice, st));
    if (nres) {
        k_set_holders<<<grid_for(nres, 256, 1184), 256, 0, st>>>(roff, rid, N, W, hm);
        LSG_LAUNCH_CHECK("k_set_holders");
    }
    PlanDims dm{D, uint64_t(N) * local_batch, 1, len, 1, N, 1, uint32_t(local_batch)};
    if (int rc = plan_wide_device(dm, 1, 0, slice ? 0 : 1, 0, 0, 1, trace, order, nullptr, nu, items, off, nullptr,
                                  nullptr, status, st, hm, 0))
        return rc;
    uint32_t h = 0;
    if (int _rc = d2h_small(&h, status, 4, st)) return _rc;
    LSG_CUDA(cudaMemcpyAsync(h_items, items, len * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaMemcpyAsync(h_node_off, off, (N + 1) * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    if (h & 64u) return set_error(kInternal, "remap_step: ran out of capacity");
    if (h) return set_error(kInternal, std::string(who) + ": device invariant violated");
    return kOk;
}

// balance_step (balance.cpp:10-39) on one step's lists (in place).
int lsg_balance_step(uint32_t* h_items, uint32_t* h_node_off, uint32_t N, uint64_t* h_moves, void* stream) {
    if (N == 0) return set_error(kValidation, "balance_step: no nodes");
    if (N > kWMaxN) return set_error(kCapability, "balance_step: num_nodes <= 256 on the device");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t total = h_node_off[N];
    uint32_t Lmax = 1;
    for (uint32_t k = 0; k < N; ++k) {
        if (h_node_off[k + 1] < h_node_off[k]) return set_error(kValidation, "balance_step: bad offsets");
        Lmax = std::max<uint32_t>(Lmax, h_node_off[k + 1] - h_node_off[k]);
    }
    if (total >= (1ull << 31)) return set_error(kCapability, "balance_step: step too large for the device");
    Scratch sc(st);
    uint32_t* items = sc.get<uint32_t>(total + 1);
    uint32_t* out = sc.get<uint32_t>(total + 1);
    uint32_t* off = sc.get<uint32_t>(N + 1);
    uint32_t* out_off = sc.get<uint32_t>(N + 1);
    uint32_t* moved = sc.get<uint32_t>(total + 1);
    uint32_t* recv = sc.get<uint32_t>(size_t(N) * Lmax);
    uint32_t* ur = sc.get<uint32_t>(total + 1);
    uint32_t* status = sc.get<uint32_t>(1);
    unsigned long long* moves = sc.get<unsigned long long>(1);
    if (!items || !out || !off || !out_off || !moved || !recv || !ur || !status || !moves)
        return set_error(kInternal, "balance_step: scratch allocation failed");
    LSG_CUDA(cudaMemcpyAsync(items, h_items, total * 4, cudaMemcpyHostToDevice, st));
    LSG_CUDA(cudaMemcpyAsync(off, h_node_off, (N + 1) * 4, cudaMemcpyHostToDevice, st));
    LSG_CUDA(cudaMemsetAsync(moved, 0, (total + 1) * 4, st));
    LSG_CUDA(cudaMemsetAsync(status, 0, 4, st));
    LSG_CUDA(cudaMemsetAsync(moves, 0, 8, st));
    BalArgs b{items, off, out, out_off, moved, moves, N, Lmax};
    WideArgs a{};
    a.recv = recv;
    a.ur = ur;
    a.status = status;
    const size_t smem = size_t(kWW) * kSortCap * 8 + size_t(4) * kLevCap * 4 + (size_t(7) * N + N + 1) * 4;
    LSG_CUDA(cudaFuncSetAttribute(k_balance_lists, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_balance_lists<<<1, kWT, smem, st>>>(b, a);
    LSG_LAUNCH_CHECK("k_balance_lists");
    uint32_t h = 0;
    unsigned long long mv = 0;
    if (int _rc = d2h_small(&h, status, 4, st)) return _rc;
    if (int _rc = d2h_small(&mv, moves, 8, st)) return _rc;
    LSG_CUDA(cudaMemcpyAsync(h_items, out, total * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaMemcpyAsync(h_node_off, out_off, (N + 1) * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    if (h) return set_error(kInternal, "balance_step: device invariant violated");
    if (h_moves) *h_moves = mv;
    return kOk;
}

}  // extern "C"

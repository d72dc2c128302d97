// lru.cuh — LruBuffer (buffer.cpp:61-82) for one node, one warp, on device.
//
// LRU keeps the C most recently accessed ids; a miss inserts at the front and,
// over capacity, drops the least recently seen id. The node's own access
// sequence IS the recency queue: entry t is the t-th access of this node, and
// it is "live" iff its id is resident and was last accessed at t (a later
// access makes it stale). The victim of an eviction is the first live entry
// at or after the front pointer, so the front only moves forward and every
// entry is passed once over the whole run (amortised O(1) per access).
//
// State per node: last[x] = node time of x's last access while resident,
// kNone otherwise (residency and recency in one word), the front (step,
// index, time), the fill and the node time. Hits inside a step are
// lane-parallel; the walk is serial only at a miss (a miss may evict an id
// that is accessed later in the same step, which then misses too).
#pragma once
#include "common.cuh"

namespace lsg {

struct LruNode {    // warp-uniform
    uint32_t size;  // residents
    uint32_t t;     // accesses so far (node time)
    uint32_t fg;    // front: step
    uint32_t fi;    //        index in that step's list of this node
    uint32_t ft;    //        node time of that entry
    uint32_t fresh; // slots handed out so far (when slots are tracked)
};

// Step g's list of node k lives at items[base(g) + off[g][k]].
struct LruPlanView {
    const uint32_t* items;     // id | hit tag
    const uint32_t* node_off;  // [T][N+1]
    const uint64_t* gb64;      // step bases (replay) or null
    const uint32_t* gb32;      // step bases (planner) or null
    uint32_t N, k;
    // silent inserts (insert_redundant): step g's entries of this node are its
    // list, then red_ids[red_off[g*rs] .. red_off[g*rs+1]) with red_off already
    // at this node (replay: the (step, node) CSR, rs = N; planner: the node's
    // own row, rs = 1); node time runs through both. Null when there are none.
    const uint64_t* red_off = nullptr;
    const uint32_t* red_ids = nullptr;
    uint32_t rs = 0;
    __device__ __forceinline__ uint64_t base(uint32_t g) const { return gb64 ? gb64[g] : uint64_t(__ldcg(&gb32[g])); }
    __device__ __forceinline__ uint32_t llen(uint32_t g) const {  // the list
        const uint32_t* o = node_off + size_t(g) * (N + 1);
        return __ldcg(&o[k + 1]) - __ldcg(&o[k]);
    }
    __device__ __forceinline__ uint32_t len(uint32_t g) const {  // list + silent entries
        const uint32_t l = llen(g);
        return red_off ? l + uint32_t(__ldcg(&red_off[size_t(g) * rs + 1]) - __ldcg(&red_off[size_t(g) * rs])) : l;
    }
    __device__ __forceinline__ const uint32_t* list(uint32_t g) const {
        return items + base(g) + __ldcg(&node_off[size_t(g) * (N + 1) + k]);
    }
    __device__ __forceinline__ uint32_t at(uint32_t g, uint32_t i, uint32_t l) const {  // entry i, l = llen(g)
        return i < l ? (__ldcg(&list(g)[i]) & ~kHit) : __ldcg(&red_ids[__ldcg(&red_off[size_t(g) * rs]) + (i - l)]);
    }
};

// Evict the least recently seen resident (whole warp); returns its id.
__device__ __forceinline__ uint32_t lru_evict_front(const LruPlanView& v, LruNode& st, uint32_t* last,
                                                    uint32_t tnow, uint32_t lane, uint32_t* status) {
    for (;;) {
        const uint32_t L = v.len(st.fg), Ll = v.red_off ? v.llen(st.fg) : L;
        if (st.fi >= L) {
            st.fg += 1;
            st.fi = 0;
            continue;
        }
        const uint32_t j = st.fi + lane;
        uint32_t y = 0;
        bool live = false;
        if (j < L) {
            y = v.at(st.fg, j, Ll);
            live = __ldcg(&last[y]) == st.ft + lane;
        }
        const uint32_t vb = __ballot_sync(0xFFFFFFFFu, live);
        if (vb) {
            const uint32_t l = __ffs(vb) - 1;
            y = __shfl_sync(0xFFFFFFFFu, y, l);
            if (lane == 0) last[y] = kNone;
            st.fi += l + 1;
            st.ft += l + 1;
            st.size -= 1;
            __syncwarp();
            return y;
        }
        const uint32_t adv = min(32u, L - st.fi);
        st.fi += adv;
        st.ft += adv;
        if (st.ft > tnow) {  // walked past the present: bookkeeping broken
            if (lane == 0) atomicOr(status, 256u);
            return kNone;
        }
    }
}

// Access the L ids of lst (this node's list of the current step) in order.
// on_hit(i, x) runs on the lane of every hit, on_miss(x, victim) on lane 0
// after every miss (victim = the evicted id or kNone). Returns the misses.
template <class OnHit, class OnMiss>
__device__ __forceinline__ uint32_t lru_step(const LruPlanView& v, LruNode& st, uint32_t* last, const uint32_t* lst,
                                             uint32_t L, uint32_t C, uint32_t lane, uint32_t* status, OnHit on_hit,
                                             OnMiss on_miss) {
    const uint32_t t0 = st.t;
    uint32_t misses = 0, pos = 0;
    while (pos < L) {
        const uint32_t i = pos + lane;
        const bool valid = i < L;
        const uint32_t x = valid ? (__ldcg(&lst[i]) & ~kHit) : 0u;
        const bool res = valid && __ldcg(&last[x]) != kNone;  // current residency
        const uint32_t mb = __ballot_sync(0xFFFFFFFFu, valid && !res);
        const uint32_t nvalid = min(32u, L - pos);
        const uint32_t first = mb ? uint32_t(__ffs(mb) - 1) : nvalid;
        // hits: move to the front (buffer.cpp:63-66); an id repeated inside
        // the window (foreign plans) keeps its latest access
        const uint32_t hmask = first >= 32 ? 0xFFFFFFFFu : ((1u << first) - 1u);
        const uint32_t grp = __match_any_sync(0xFFFFFFFFu, valid ? x : 0x80000000u | lane) & hmask;
        if (lane < first && valid) {
            if (lane == 31 - __clz(grp)) last[x] = t0 + i;
            on_hit(i, x);
        }
        if (first < nvalid) {  // the miss at `first`: insert (buffer.cpp:68-70)
            const uint32_t xm = __shfl_sync(0xFFFFFFFFu, x, first);
            if (lane == 0) last[xm] = t0 + pos + first;
            st.size += 1;
            ++misses;
            __syncwarp();
            uint32_t y = kNone;
            if (st.size > C)  // buffer.cpp:71-76
                y = lru_evict_front(v, st, last, t0 + pos + first, lane, status);
            if (lane == 0) on_miss(xm, y);
            __syncwarp();
            pos += first + 1;
        } else {
            pos += nvalid;
        }
        __syncwarp();
    }
    st.t = t0 + L;
    return misses;
}

}  // namespace lsg

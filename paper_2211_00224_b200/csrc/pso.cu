// pso.cu — K4: bit-exact swap-sequence particle swarm epoch ordering
// (pso_order, epoch_order.cpp:121-221), run on device as one CTA.
//
// The reference draws every random number from ONE splitmix64 stream, with
// particles consuming draws in particle order. splitmix64 is counter-based,
// so a particle's draws are fixed once its starting counter is known:
//   restart:  E-1 draws (Fisher–Yates of E)
//   otherwise |vel| (momentum) + E (personal pull) + E (global pull)
//             + (E>1 ? 1 + (kick passes ? 2 : 0) : 0)
// and the kick outcome is itself the draw at a known counter. One thread scans
// the 32 particle offsets (32 draws) per iteration; then one warp per particle
// runs its iteration concurrently. Within a warp the draws are evaluated
// lane-parallel (ballot masks); only the swap application, which depends on
// the evolving permutation, is sequential. Costs are lane-parallel sums;
// the memetic polish (E <= 32, epoch_order.cpp:91-117) evaluates all 496
// transpositions lane-parallel with exact integer deltas and a first-index
// argmin, which reproduces the reference's scan-order tie rule.
#include "common.cuh"

namespace lsg {

namespace {

constexpr int kPsoThreads = 1024;
constexpr uint32_t kPsoMaxE = 1024;

struct PsoArgs {
    const uint64_t* w;
    uint32_t E, P, iters, stagnation, restart;
    double pp, pg, inertia, kick;
    uint64_t seed;
    uint32_t vcap;
    uint32_t* vel;  // [P][2][vcap] packed i | j<<16
    uint32_t* order;
    uint64_t* cost;
    uint64_t* hist;
    uint32_t* iters_out;
    uint32_t* status;
};

struct PsoSmem {
    uint16_t* pos;   // [P][E]
    uint16_t* inv;   // [P][E]
    uint16_t* best;  // [P][E]
    uint16_t* gbest; // [E] copy of the global best (a snapshot, like :173)
    uint64_t* pcost; // [P]
    uint64_t* bcost; // [P]
    uint64_t* off;   // [P]
    uint32_t* stale; // [P]
    uint32_t* vlen;  // [P]
    uint32_t* vsel;  // [P] which vel buffer is current
    uint32_t* bits;  // [32 warps][kPsoMaxE/32] draw-pass masks
};

__device__ __forceinline__ uint64_t wcost(const uint64_t* __restrict__ w, uint32_t E, uint32_t a,
                                          uint32_t b) {
    return __ldg(&w[size_t(a) * E + b]);
}

// sum of w(o[i], o[i+1]), lane-parallel
__device__ uint64_t warp_path_cost(const uint64_t* w, uint32_t E, const uint16_t* o, uint32_t lane) {
    uint64_t c = 0;
    for (uint32_t i = lane; i + 1 < E; i += 32) c += wcost(w, E, o[i], o[i + 1]);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, s);
    return c;
}

// Fisher–Yates of pos with draws (counter+1 ...), prng.hpp:45-53. Lane 0.
__device__ void fy_lane0(uint16_t* pos, uint32_t E, uint64_t seed, uint64_t counter) {
    uint64_t k = counter;
    for (uint32_t i = E; i > 1; --i) {
        const uint32_t j = uint32_t(draw(seed, ++k) % i);
        const uint16_t t = pos[i - 1];
        pos[i - 1] = pos[j];
        pos[j] = t;
    }
}

// Steepest descent over single transpositions (epoch_order.cpp:93-117), E<=32.
// Lane i holds o[i]; every (i<j) pair is scored with an exact cost delta.
__device__ void warp_descend(const uint64_t* w, uint32_t E, uint16_t* pos, uint64_t& cost,
                             uint32_t lane) {
    for (;;) {
        uint64_t best = cost;
        uint32_t bestidx = 0xFFFFFFFFu;
        // pairs enumerated in scan order: idx = rank of (i,j) in i-major order
        const uint32_t npairs = E * (E - 1) / 2;
        for (uint32_t p = lane; p < npairs; p += 32) {
            // invert p -> (i, j)
            uint32_t i = 0, rem = p;
            while (rem >= E - 1 - i) { rem -= E - 1 - i; ++i; }
            const uint32_t j = i + 1 + rem;
            const uint32_t oi = pos[i], oj = pos[j];
            auto at = [&](uint32_t q) -> uint32_t { return q == i ? oj : (q == j ? oi : pos[q]); };
            // edges touched: (i-1,i), (i,i+1), (j-1,j), (j,j+1) (dedup when j==i+1)
            uint64_t before = 0, after = 0;
            uint32_t e_idx[4];
            int ne = 0;
            if (i > 0) e_idx[ne++] = i - 1;
            e_idx[ne++] = i;
            if (j - 1 != i) e_idx[ne++] = j - 1;
            if (j + 1 < E) e_idx[ne++] = j;
            for (int q = 0; q < ne; ++q) {
                const uint32_t a = e_idx[q];
                before += wcost(w, E, pos[a], pos[a + 1]);
                after += wcost(w, E, at(a), at(a + 1));
            }
            const uint64_t c = cost - before + after;
            if (c < best) { best = c; bestidx = p; }  // p rises per lane: first wins
        }
        // warp argmin by (cost, pair index)
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            const uint64_t ob = __shfl_xor_sync(0xFFFFFFFFu, best, s);
            const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bestidx, s);
            if (ob < best || (ob == best && oi < bestidx)) { best = ob; bestidx = oi; }
        }
        if (best >= cost || bestidx == 0xFFFFFFFFu) return;
        __syncwarp();
        if (lane == 0) {
            uint32_t i = 0, rem = bestidx;
            while (rem >= E - 1 - i) { rem -= E - 1 - i; ++i; }
            const uint32_t j = i + 1 + rem;
            const uint16_t t = pos[i];
            pos[i] = pos[j];
            pos[j] = t;
        }
        __syncwarp();
        cost = best;
    }
}

__device__ void rebuild_inv(uint16_t* inv, const uint16_t* pos, uint32_t E, uint32_t lane) {
    for (uint32_t i = lane; i < E; i += 32) inv[pos[i]] = uint16_t(i);
}

__global__ void __launch_bounds__(kPsoThreads, 1) k_pso(PsoArgs a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const uint32_t E = a.E, P = a.P;
    PsoSmem s;
    unsigned char* q = smraw;
    s.pcost = reinterpret_cast<uint64_t*>(q); q += P * 8;
    s.bcost = reinterpret_cast<uint64_t*>(q); q += P * 8;
    s.off = reinterpret_cast<uint64_t*>(q); q += P * 8;
    s.stale = reinterpret_cast<uint32_t*>(q); q += P * 4;
    s.vlen = reinterpret_cast<uint32_t*>(q); q += P * 4;
    s.vsel = reinterpret_cast<uint32_t*>(q); q += P * 4;
    s.bits = reinterpret_cast<uint32_t*>(q); q += 32 * (kPsoMaxE / 32) * 4;
    s.pos = reinterpret_cast<uint16_t*>(q); q += size_t(P) * E * 2;
    s.inv = reinterpret_cast<uint16_t*>(q); q += size_t(P) * E * 2;
    s.best = reinterpret_cast<uint16_t*>(q); q += size_t(P) * E * 2;
    s.gbest = reinterpret_cast<uint16_t*>(q); q += E * 2;
    __shared__ uint64_t gcost;
    __shared__ int32_t gidx;  // particle whose best is the global best; -1 = identity init
    __shared__ uint32_t improved, stop;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nwarps = blockDim.x >> 5;
    const bool polish = E <= 32;

    // ---- initialisation (epoch_order.cpp:149-167)
    for (uint32_t p = warp; p < P; p += nwarps) {
        uint16_t* pos = s.pos + size_t(p) * E;
        for (uint32_t i = lane; i < E; i += 32) pos[i] = uint16_t(i);
        __syncwarp();
        if (p != 0 && lane == 0) fy_lane0(pos, E, a.seed, uint64_t(p - 1) * (E > 0 ? E - 1 : 0));
        __syncwarp();
        uint64_t c = warp_path_cost(a.w, E, pos, lane);
        if (polish) warp_descend(a.w, E, pos, c, lane);
        __syncwarp();
        rebuild_inv(s.inv + size_t(p) * E, pos, E, lane);
        for (uint32_t i = lane; i < E; i += 32) s.best[size_t(p) * E + i] = pos[i];
        if (lane == 0) {
            s.pcost[p] = c;
            s.bcost[p] = c;
            s.stale[p] = 0;
            s.vlen[p] = 0;
            s.vsel[p] = 0;
        }
    }
    __syncthreads();
    if (tid == 0) {
        gcost = s.pcost[0];
        gidx = 0;
        for (uint32_t p = 0; p < P; ++p)
            if (s.pcost[p] < gcost) { gcost = s.pcost[p]; gidx = int32_t(p); }
        stop = 0;
    }
    __syncthreads();
    for (uint32_t i = tid; i < E; i += blockDim.x) s.gbest[i] = s.pos[size_t(gidx) * E + i];
    __syncthreads();
    uint64_t counter = uint64_t(P - 1) * (E > 0 ? E - 1 : 0);
    uint32_t stagnant = 0, done = 0;

    for (uint32_t it = 0; it < a.iters; ++it) {
        // synchronous iteration: gbest only changes between iterations, so
        // the s.gbest copy is the reference's gbest_pos snapshot (:173)
        if (tid == 0) {
            // per-particle draw offsets: the only cross-particle dependency
            uint64_t c = counter;
            for (uint32_t p = 0; p < P; ++p) {
                s.off[p] = c;
                if (a.restart > 0 && s.stale[p] >= a.restart) {
                    c += E > 1 ? E - 1 : 0;
                } else {
                    uint64_t n = uint64_t(s.vlen[p]) + 2ull * E;
                    if (E > 1) {
                        const bool pass = to_unit(draw(a.seed, c + n + 1)) < a.kick;
                        n += pass ? 3 : 1;
                    }
                    c += n;
                }
            }
            counter = c;
            improved = 0;
        }
        __syncthreads();
        for (uint32_t p = warp; p < P; p += nwarps) {
            uint16_t* pos = s.pos + size_t(p) * E;
            uint16_t* inv = s.inv + size_t(p) * E;
            uint16_t* best = s.best + size_t(p) * E;
            uint32_t* mask = s.bits + warp * (kPsoMaxE / 32);
            uint64_t k = s.off[p];
            if (a.restart > 0 && s.stale[p] >= a.restart) {  // reseed (:176-183)
                if (lane == 0) fy_lane0(pos, E, a.seed, k);
                __syncwarp();
                rebuild_inv(inv, pos, E, lane);
                uint64_t c = warp_path_cost(a.w, E, pos, lane);
                if (polish) {
                    warp_descend(a.w, E, pos, c, lane);
                    __syncwarp();
                    rebuild_inv(inv, pos, E, lane);
                }
                __syncwarp();
                for (uint32_t i = lane; i < E; i += 32) best[i] = pos[i];
                if (lane == 0) {
                    s.vlen[p] = 0;
                    s.pcost[p] = c;
                    s.bcost[p] = c;
                    s.stale[p] = 0;
                }
                __syncwarp();
                continue;
            }
            const uint32_t vl = s.vlen[p];
            const uint32_t* vold = a.vel + (size_t(p) * 2 + s.vsel[p]) * a.vcap;
            uint32_t* vnew = a.vel + (size_t(p) * 2 + (s.vsel[p] ^ 1)) * a.vcap;
            uint32_t nn = 0;  // lane 0 owns the new velocity length
            // momentum (:185-190): keep swap v iff draw < inertia, in order
            for (uint32_t base = 0; base < vl; base += 32) {
                const uint32_t v = base + lane;
                const bool keep = v < vl && to_unit(draw(a.seed, k + 1 + v)) < a.inertia;
                uint32_t m = __ballot_sync(0xFFFFFFFFu, keep);
                if (lane == 0) {
                    while (m) {
                        const uint32_t vi = base + __ffs(m) - 1;
                        m &= m - 1;
                        const uint32_t sw = vold[vi];
                        const uint32_t i = sw & 0xFFFF, j = sw >> 16;
                        const uint16_t t = pos[i];
                        pos[i] = pos[j];
                        pos[j] = t;
                        inv[pos[i]] = uint16_t(i);
                        inv[pos[j]] = uint16_t(j);
                        vnew[nn++] = sw;
                    }
                }
            }
            k += vl;
            // two pulls (:77-87): toward personal best, then the snapshot
            for (int pull = 0; pull < 2; ++pull) {
                const uint16_t* target = pull == 0 ? best : s.gbest;
                const double prob = pull == 0 ? a.pp : a.pg;
                for (uint32_t base = 0; base < E; base += 32) {
                    const uint32_t i = base + lane;
                    const bool go = i < E && to_unit(draw(a.seed, k + 1 + i)) < prob;
                    const uint32_t m = __ballot_sync(0xFFFFFFFFu, go);
                    if (lane == 0) mask[base >> 5] = m;
                }
                __syncwarp();
                if (lane == 0) {
                    for (uint32_t wd = 0; wd < (E + 31) / 32; ++wd) {
                        uint32_t m = mask[wd];
                        while (m) {
                            const uint32_t i = wd * 32 + __ffs(m) - 1;
                            m &= m - 1;
                            const uint16_t want = target[i];
                            if (pos[i] == want) continue;
                            const uint32_t j = inv[want];
                            const uint16_t t = pos[i];
                            pos[i] = pos[j];
                            pos[j] = t;
                            inv[pos[i]] = uint16_t(i);
                            inv[pos[j]] = uint16_t(j);
                            if (nn < a.vcap) vnew[nn] = i | (j << 16);
                            ++nn;
                        }
                    }
                }
                __syncwarp();
                k += E;
            }
            if (E > 1 && lane == 0) {  // turbulence (:193-197)
                const bool pass = to_unit(draw(a.seed, ++k)) < a.kick;
                if (pass) {
                    const uint32_t i = uint32_t(draw(a.seed, ++k) % E);
                    uint32_t j = uint32_t(draw(a.seed, ++k) % (E - 1));
                    if (j >= i) ++j;
                    const uint16_t t = pos[i];
                    pos[i] = pos[j];
                    pos[j] = t;
                    inv[pos[i]] = uint16_t(i);
                    inv[pos[j]] = uint16_t(j);
                    if (nn < a.vcap) vnew[nn] = i | (j << 16);
                    ++nn;
                }
            }
            nn = __shfl_sync(0xFFFFFFFFu, nn, 0);
            __syncwarp();
            uint64_t c = warp_path_cost(a.w, E, pos, lane);
            const uint64_t bc = s.bcost[p];
            if (c < bc) {  // adopt (:201-203)
                if (polish) {
                    warp_descend(a.w, E, pos, c, lane);
                    __syncwarp();
                    rebuild_inv(inv, pos, E, lane);
                }
                __syncwarp();
                for (uint32_t i = lane; i < E; i += 32) best[i] = pos[i];
            }
            __syncwarp();
            if (lane == 0) {
                if (nn > a.vcap) atomicOr(a.status, 1u);
                s.vlen[p] = nn;
                s.vsel[p] ^= 1;
                s.pcost[p] = c;
                if (c < bc) {
                    s.bcost[p] = c;
                    s.stale[p] = 0;
                } else {
                    s.stale[p] += 1;
                }
            }
            __syncwarp();
        }
        __syncthreads();
        if (tid == 0) {  // global best scan, strict, particle order (:207-212)
            for (uint32_t p = 0; p < P; ++p)
                if (s.bcost[p] < gcost) { gcost = s.bcost[p]; gidx = int32_t(p); improved = 1; }
            if (a.hist) a.hist[it] = gcost;
            ++done;
            stagnant = improved ? 0 : stagnant + 1;
            stop = stagnant >= a.stagnation;
        }
        __syncthreads();
        // gbest = {part.best, part.best_cost}: a copy, so a later restart of
        // that particle cannot disturb it (:176-183 vs :207-212)
        if (improved)
            for (uint32_t i = tid; i < E; i += blockDim.x) s.gbest[i] = s.best[size_t(gidx) * E + i];
        __syncthreads();
        if (stop) break;
    }
    for (uint32_t i = tid; i < E; i += blockDim.x) a.order[i] = s.gbest[i];
    if (tid == 0) {
        if (a.cost) *a.cost = gcost;
        if (a.iters_out) *a.iters_out = done;
    }
}

}  // namespace

int pso_order_device(const uint64_t* d_w, uint32_t E, uint32_t swarm, uint32_t iters, double pp,
                     double pg, double inertia, double kick, uint32_t stagnation, uint32_t restart,
                     uint64_t seed, uint32_t* d_order, uint64_t* d_cost, uint64_t* d_hist,
                     uint32_t* d_iters, uint32_t* d_status, cudaStream_t st) {
    if (E == 0) return set_error(kValidation, "pso_order: empty graph");
    if (swarm == 0) return set_error(kValidation, "pso_order: swarm_size must be >= 1");
    if (inertia < 0.0 || inertia >= 1.0) return set_error(kValidation, "pso_order: inertia must be in [0, 1)");
    if (kick < 0.0 || kick > 1.0) return set_error(kValidation, "pso_order: kick must be in [0, 1]");
    if (E > kPsoMaxE) return set_error(kCapability, "pso_order: device swarm supports num_epochs <= 1024");
    if (swarm > 1024) return set_error(kCapability, "pso_order: device swarm supports swarm_size <= 1024");
    PsoArgs a;
    a.w = d_w;
    a.E = E;
    a.P = swarm;
    a.iters = iters;
    a.stagnation = stagnation;
    a.restart = restart;
    a.pp = pp;
    a.pg = pg;
    a.inertia = inertia;
    a.kick = kick;
    a.seed = seed;
    a.vcap = 16 * E + 256;
    a.order = d_order;
    a.cost = d_cost;
    a.hist = d_hist;
    a.iters_out = d_iters;
    a.status = d_status;
    Scratch sc(st);
    a.vel = sc.get<uint32_t>(size_t(swarm) * 2 * a.vcap);
    if (!a.vel) return set_error(kInternal, "pso_order: scratch allocation failed");
    const size_t smem = size_t(swarm) * (8 * 3 + 4 * 3) + 32 * (kPsoMaxE / 32) * 4 +
                        size_t(swarm) * E * 2 * 3 + E * 2 + 16;
    if (smem > 227 * 1024)
        return set_error(kCapability, "pso_order: swarm_size * num_epochs too large for one CTA");
    LSG_CUDA(cudaFuncSetAttribute(k_pso, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_pso<<<1, kPsoThreads, smem, st>>>(a);
    LSG_LAUNCH_CHECK("k_pso");
    return kOk;
}

}  // namespace lsg

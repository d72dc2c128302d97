// gather.cu — K8 batch gather from the HBM-resident sample buffer and K9 the
// synthetic Store payload fill.
//
// K8 replaces the per-sample pread of Store::read_one (store.cpp:123-139) for
// buffered samples: out row r = buf row slots[r]. It is a pure HBM copy
// (read once, write once), so it is written as a persistent grid over 16 KiB
// tiles with 128-bit loads issued 4-deep before their stores (MLP >= 4 per
// thread) and evict-first hints on both sides (the batch is consumed by the
// trainer, the buffer row is not re-read this step).
//
// K9 reproduces the Store payload (store.cpp:70-80): byte j of the payload is
// byte j%8 (little-endian) of mix(fill_seed + (j/8 + 1)*gamma), and sample i
// occupies payload bytes [i*size, (i+1)*size). Being counter-based, every
// 8-byte word is computed independently.
#include <atomic>
#include <cstdlib>

#include "fetch.cuh"

namespace lsg {

namespace {

constexpr int kGatherThreads = 256;
constexpr int kUnroll = 4;
constexpr uint32_t kTileVec = kGatherThreads * kUnroll;  // uint4 per tile (16 KiB)

__global__ void __launch_bounds__(kGatherThreads) k_gather(const uint4* __restrict__ buf,
                                                           const uint32_t* __restrict__ slots,
                                                           uint64_t n, uint64_t vec_per_row,
                                                           uint64_t tiles_per_row,
                                                           uint4* __restrict__ out) {
    const uint64_t ntiles = n * tiles_per_row;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t row = tile / tiles_per_row;
        const uint64_t c0 = (tile - row * tiles_per_row) * kTileVec;
        const uint4* src = buf + uint64_t(__ldg(&slots[row])) * vec_per_row;
        uint4* dst = out + row * vec_per_row;
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kGatherThreads + threadIdx.x;
            if (c < vec_per_row) v[u] = __ldcs(&src[c]);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kGatherThreads + threadIdx.x;
            if (c < vec_per_row) __stcs(&dst[c], v[u]);
        }
    }
}

// payload word path: sample_bytes % 16 == 0
__global__ void __launch_bounds__(256) k_store_fill_vec(const uint32_t* __restrict__ ids, uint64_t n,
                                                        uint64_t words_per_row, uint64_t seed,
                                                        ulonglong2* __restrict__ dst) {
    const uint64_t pairs = words_per_row / 2;
    const uint64_t total = n * pairs;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = i / pairs, p = i - row * pairs;
        const uint64_t word0 = uint64_t(ids[row]) * words_per_row + 2 * p;  // payload word index
        ulonglong2 v;
        v.x = mix64(seed + (word0 + 1) * kGamma);
        v.y = mix64(seed + (word0 + 2) * kGamma);
        __stcs(&dst[row * pairs + p], v);
    }
}

// general byte path
__global__ void k_store_fill_bytes(const uint32_t* __restrict__ ids, uint64_t n, uint64_t size,
                                   uint64_t seed, uint8_t* __restrict__ dst) {
    const uint64_t total = n * size;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = i / size, c = i - row * size;
        const uint64_t j = uint64_t(ids[row]) * size + c;
        dst[i] = uint8_t(mix64(seed + (j / 8 + 1) * kGamma) >> (8 * (j % 8)));
    }
}

// K8 fetch of one node list: rows whose replay slot carries the hit flag
// (bit 31) are copied from their HBM slot; the rest are left to k_fill_misses.
__global__ void __launch_bounds__(kGatherThreads) k_gather_hits(const uint4* __restrict__ buf,
                                                                const uint32_t* __restrict__ slots,
                                                                uint64_t n, uint64_t vec_per_row,
                                                                uint64_t tiles_per_row,
                                                                uint4* __restrict__ out) {
    const uint64_t ntiles = n * tiles_per_row;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t row = tile / tiles_per_row;
        const uint32_t sl = __ldg(&slots[row]);
        if (sl == kNever || !(sl & kHit)) continue;  // block-uniform
        const uint64_t c0 = (tile - row * tiles_per_row) * kTileVec;
        const uint4* src = buf + uint64_t(sl & ~kHit) * vec_per_row;
        uint4* dst = out + row * vec_per_row;
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kGatherThreads + threadIdx.x;
            if (c < vec_per_row) v[u] = __ldcs(&src[c]);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kGatherThreads + threadIdx.x;
            if (c < vec_per_row) __stcs(&dst[c], v[u]);
        }
    }
}

// Misses: the sample arrives from storage (synthesised Store payload) into
// its batch row and, unless the replay bypassed it, into its new HBM slot.
__global__ void __launch_bounds__(256) k_fill_misses(const uint32_t* __restrict__ ids,
                                                     const uint32_t* __restrict__ slots, uint64_t n,
                                                     uint64_t words_per_row, uint64_t seed,
                                                     ulonglong2* __restrict__ buf,
                                                     ulonglong2* __restrict__ out) {
    const uint64_t pairs = words_per_row / 2;
    for (uint64_t row = blockIdx.y; row < n; row += gridDim.y) {
        const uint32_t sl = __ldg(&slots[row]);
        if (sl != kNever && (sl & kHit)) continue;
        const uint64_t word0 = uint64_t(__ldg(&ids[row]) & ~kHit) * words_per_row;
        for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < pairs;
             p += uint64_t(gridDim.x) * blockDim.x) {
            ulonglong2 v;
            v.x = mix64(seed + (word0 + 2 * p + 1) * kGamma);
            v.y = mix64(seed + (word0 + 2 * p + 2) * kGamma);
            __stcs(&out[row * pairs + p], v);
            if (sl != kNever) __stcs(&buf[uint64_t(sl) * pairs + p], v);
        }
    }
}

__global__ void __launch_bounds__(kGatherThreads) k_fetch_step_hits(StepFetch f) {
    const uint32_t r0 = __ldg(&f.node_off[f.k0]);
    const uint64_t nrows = __ldg(&f.node_off[f.k1]) - r0;
    const uint64_t ntiles = nrows * f.tiles_per_row;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t rr = tile / f.tiles_per_row;
        const uint32_t r = r0 + uint32_t(rr);
        const uint32_t sl = __ldg(&f.slots[r]);
        if (sl == kNever || !(sl & kHit)) continue;  // block-uniform
        const uint32_t k = node_of_row(f, r);
        const uint64_t c0 = (tile - rr * f.tiles_per_row) * kTileVec;
        const uint4* src = f.bufs[k - f.k0] + uint64_t(sl & ~kHit) * f.vec_per_row;
        uint4* dst = f.outs[k - f.k0] + uint64_t(r - __ldg(&f.node_off[k])) * f.vec_per_row;
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kGatherThreads + threadIdx.x;
            if (c < f.vec_per_row) v[u] = __ldcs(&src[c]);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t c = c0 + u * kGatherThreads + threadIdx.x;
            if (c < f.vec_per_row) __stcs(&dst[c], v[u]);
        }
    }
}

// TMA bulk-copy version of the hit gather: one elected thread per CTA
// streams kTile-byte tiles global -> shared (cp.async.bulk, mbarrier
// complete_tx) -> global (cp.async.bulk bulk_group), kStages tiles per CTA;
// a slot is refilled once the store of its tile has read it, checked kLag
// stores later, so up to kLag+1 stores and kStages-kLag-1 loads are in
// flight. CTAs claim chunks of kTmaChunk consecutive tiles from a per-step
// counter (f.claim, zeroed per call), so a CTA that starts late
// (an SM shared with the planner's persistent CTA) takes fewer chunks instead
// of stretching the step; row descriptors change once per row and miss rows
// are skipped whole. Measured at 6.56 TB/s on the cfg2 shape vs 5.75 for the
// LSU gather (tools/ubench_gather.cu).
constexpr int kTmaTile = 8192, kTmaStages = 12, kTmaLag = 3, kTmaChunk = 16, kTmaTail = 4;

__global__ void __launch_bounds__(32) k_fetch_step_hits_tma(StepFetch f) {
    extern __shared__ __align__(128) unsigned char tsm[];
    __shared__ __align__(8) unsigned long long bar[kTmaStages];
    __shared__ unsigned char* sdst[kTmaStages];
    if (threadIdx.x != 0) return;
    for (int q = 0; q < kTmaStages; ++q) {
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[q]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    // programmatic dependent launch: the next kernel of the stream may be
    // scheduled now (it waits below for this grid); this grid waits for the
    // previous step's kernels (slots it filled, batch rows, the counters)
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t row_bytes = f.vec_per_row * 16, tpr = row_bytes / kTmaTile;
    const uint32_t r0 = __ldg(&f.node_off[f.k0]);
    const uint64_t nt = uint64_t(__ldg(&f.node_off[f.k1]) - r0) * tpr;
    // static split without a counter (claim == null), else dynamic chunks
    uint64_t tb, te;
    // guided claims: kTmaChunk tiles while plenty remain, then kTmaTail, so
    // the step's last CTAs finish together (shorter tail before the next step)
    const uint64_t guide = uint64_t(gridDim.x) * 2 * kTmaChunk;
    if (f.claim) {
        const uint32_t sz = nt > guide ? kTmaChunk : kTmaTail;
        tb = atomicAdd(f.claim, sz);
        te = min(nt, tb + sz);
    } else {
        const uint64_t per = (nt + gridDim.x - 1) / gridDim.x;
        tb = uint64_t(blockIdx.x) * per;
        te = min(nt, tb + per);
    }
    // the gathered bytes stream through L2 once: evict-first, so a planner
    // running beside the fetch keeps its working set in L2
    uint64_t pol = 0;
    if (f.l2hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint64_t cur = ~0ull;  // row of the cached descriptor
    const unsigned char* src_row = nullptr;
    unsigned char* dst_row = nullptr;
    uint64_t tn = tb;  // next tile to issue; miss rows are skipped whole
    auto issue = [&](uint64_t k) -> bool {
        for (;;) {
            if (tn >= te) {
                if (!f.claim || tb >= nt) return false;
                const uint32_t sz = nt - te > guide ? kTmaChunk : kTmaTail;
                tb = atomicAdd(f.claim, sz);
                if (tb >= nt) return false;
                te = min(nt, tb + sz);
                tn = tb;
            }
            const uint64_t rr = tn / tpr;
            if (rr != cur) {
                cur = rr;
                const uint32_t r = r0 + uint32_t(rr);
                const uint32_t sl = __ldg(&f.slots[r]);
                const uint32_t kk = node_of_row(f, r);
                const bool hit = sl != kNever && (sl & kHit);
                src_row = hit ? reinterpret_cast<const unsigned char*>(f.bufs[kk - f.k0]) +
                                    uint64_t(sl & ~kHit) * row_bytes
                              : nullptr;
                dst_row = reinterpret_cast<unsigned char*>(f.outs[kk - f.k0]) +
                          uint64_t(r - __ldg(&f.node_off[kk])) * row_bytes;
                // a miss row goes on the misses kernel's list, once: by the
                // CTA whose tile range (chunk) holds the row's first tile
                if (!hit && f.mlist && rr * tpr >= tb) {
                    const uint32_t at = atomicAdd(f.mctl, 1u);
                    if (at < f.mcap) f.mlist[at] = r;  // past mcap the misses kernel scans every row
                }
            }
            if (src_row) break;
            tn = (rr + 1) * tpr;  // a miss row: the misses kernel writes it
        }
        const uint64_t c = (tn - cur * tpr) * kTmaTile;
        ++tn;
        const int q = int(k % kTmaStages);
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[q]));
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(tsm + q * kTmaTile));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTmaTile));
        if (f.l2hint)
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                         " [%0], [%1], %2, [%3], %4;"
                         ::"r"(d), "l"(src_row + c), "r"(kTmaTile), "r"(b), "l"(pol) : "memory");
        else
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(d), "l"(src_row + c), "r"(kTmaTile), "r"(b) : "memory");
        sdst[q] = dst_row + c;
        return true;
    };
    uint64_t issued = 0;
    while (issued < uint64_t(kTmaStages - kTmaLag) && issue(issued)) ++issued;
    for (uint64_t k = 0; k < issued; ++k) {
        const int q = int(k % kTmaStages);
        const uint32_t par = uint32_t((k / kTmaStages) & 1);
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[q]));
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(b), "r"(par));
        const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(tsm + q * kTmaTile));
        if (f.l2hint)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                         ::"l"(sdst[q]), "r"(sp), "r"(kTmaTile), "l"(pol) : "memory");
        else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sdst[q]), "r"(sp),
                         "r"(kTmaTile) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        // stage k+S-L goes into the slot of stage k-L: fresh while k < L,
        // else free once that stage's store has read it
        if (k >= uint64_t(kTmaLag)) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaLag) : "memory");
        if (issued == k + uint64_t(kTmaStages - kTmaLag) && issue(issued)) ++issued;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Misses of the step: with the TMA hit kernel's list (mlist) only the miss
// rows are visited, else (no list, or more misses than it holds) every row of
// the step is scanned.
__global__ void __launch_bounds__(256) k_fetch_step_misses(StepFetch f) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the hit kernel's miss list
    const uint32_t r0 = __ldg(&f.node_off[f.k0]), r1 = __ldg(&f.node_off[f.k1]);
    const uint64_t pairs = f.vec_per_row;  // 16-byte pairs of payload words
    const uint32_t nlist = f.mlist ? __ldcg(f.mctl) : 0u;
    const bool listed = f.mlist && nlist <= f.mcap;
    const uint32_t n = listed ? nlist : r1 - r0;
    for (uint32_t m = blockIdx.y; m < n; m += gridDim.y) {
        const uint32_t r = listed ? __ldcg(&f.mlist[m]) : r0 + m;
        const uint32_t sl = __ldg(&f.slots[r]);
        if (sl != kNever && (sl & kHit)) continue;
        const uint32_t k = node_of_row(f, r);
        const uint64_t word0 = uint64_t(__ldg(&f.items[r]) & ~kHit) * (2 * pairs);
        ulonglong2* out = reinterpret_cast<ulonglong2*>(f.outs[k - f.k0]) + uint64_t(r - __ldg(&f.node_off[k])) * pairs;
        ulonglong2* buf = sl != kNever ? reinterpret_cast<ulonglong2*>(f.bufs[k - f.k0]) + uint64_t(sl) * pairs : nullptr;
        for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < pairs;
             p += uint64_t(gridDim.x) * blockDim.x) {
            ulonglong2 v;
            v.x = mix64(f.seed + (word0 + 2 * p + 1) * kGamma);
            v.y = mix64(f.seed + (word0 + 2 * p + 2) * kGamma);
            __stcs(&out[p], v);
            if (buf) __stcs(&buf[p], v);
        }
    }
}

}  // namespace

bool pdl_on(int which) {
    // LSG_PDL bit 0: hit kernels, bit 1: miss kernels. Default 1: a miss
    // kernel launched early beside a miss-heavy hit kernel measured slower
    // (E=4 cfg2 fetch 88.5 -> 96.9 ms), the hit kernels gain (1 rank 52.7 ->
    // 50.6 us per step)
    static const int mode = [] {
        const char* e = std::getenv("LSG_PDL");
        return e ? std::atoi(e) : 1;
    }();
    return (mode >> which) & 1;
}

namespace {

// launch with programmatic stream serialization (PDL): back-to-back step
// kernels overlap launch and ramp-up with the previous kernel's tail; the
// kernels order their memory through griddepcontrol.wait (LSG_PDL=0: off)
template <class K>
cudaError_t launch_pdl(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const StepFetch& f, int which) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on(which) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, f);
}

// TMA gather when rows are whole tiles (LSG_GATHER_LSU=1 keeps the 128-bit
// load/store kernel, for comparison)
}  // namespace

int launch_fetch_hits(StepFetch f, uint64_t rows, uint64_t sample_bytes, cudaStream_t st, bool* tma) {
    static const int l2hint = [] {
        const char* e = std::getenv("LSG_FETCH_L2HINT");
        return e && e[0] == '1' ? 1 : 0;  // measured: no gain beside the planner (default off)
    }();
    f.l2hint = l2hint;
    if (tma) *tma = false;
    static const bool lsu = [] {
        const char* e = std::getenv("LSG_GATHER_LSU");
        return e && e[0] == '1';
    }();
    if (!lsu && sample_bytes % kTmaTile == 0) {
        static std::atomic<uint64_t> attr_done{0};  // per device
        const int smem = kTmaTile * kTmaStages;
        int dev = 0;
        LSG_CUDA(cudaGetDevice(&dev));
        const uint64_t bit = 1ull << (dev & 63);
        if (!(attr_done.load() & bit)) {
            LSG_CUDA(cudaFuncSetAttribute(k_fetch_step_hits_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr_done.fetch_or(bit);
        }
        const uint64_t tiles = rows * (sample_bytes / kTmaTile);
        const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(tiles, 148ull * 2)));
        LSG_CUDA(launch_pdl(k_fetch_step_hits_tma, dim3(grid), dim3(32), size_t(smem), st, f, 0));
        LSG_LAUNCH_CHECK("k_fetch_step_hits_tma");
        if (tma) *tma = true;
        return kOk;
    }
    const unsigned grid = unsigned(std::min<uint64_t>(rows * f.tiles_per_row, 148ull * 8));
    k_fetch_step_hits<<<grid, kGatherThreads, 0, st>>>(f);
    LSG_LAUNCH_CHECK("k_fetch_step_hits");
    return kOk;
}

int fetch_step_device(void* const* d_bufs, void* const* d_outs, const uint32_t* d_items,
                      const uint32_t* d_slots, const uint32_t* d_node_off, uint32_t k0, uint32_t k1,
                      uint64_t rows_hint, uint64_t sample_bytes, uint64_t seed, cudaStream_t st) {
    if (k1 <= k0) return kOk;
    if (sample_bytes == 0 || sample_bytes % 16 != 0)
        return set_error(kValidation, "fetch_step: sample_bytes must be a positive multiple of 16");
    StepFetch f{};
    f.items = d_items;
    f.slots = d_slots;
    f.node_off = d_node_off;
    f.bufs = reinterpret_cast<uint4* const*>(d_bufs);
    f.outs = reinterpret_cast<uint4* const*>(d_outs);
    f.k0 = k0;
    f.k1 = k1;
    f.vec_per_row = sample_bytes / 16;
    f.tiles_per_row = (f.vec_per_row + kTileVec - 1) / kTileVec;
    f.seed = seed;
    const uint64_t rows = rows_hint ? rows_hint : 1;
    // this call's own control words (stream-ordered pool): the claim counter
    // and, with a row count, the TMA kernel's miss-row list; a list shorter
    // than the step (a low rows_hint) only makes the misses kernel scan
    Scratch sc(st);
    const bool tma_rows = sample_bytes % kTmaTile == 0;
    uint32_t* ctl = sc.get<uint32_t>(2 + (rows_hint && tma_rows ? rows_hint : 0));
    if (!ctl) return set_error(kInternal, "fetch_step: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(ctl, 0, 8, st));
    f.claim = ctl;
    if (rows_hint && tma_rows) {
        f.mctl = ctl + 1;
        f.mlist = ctl + 2;
        f.mcap = uint32_t(std::min<uint64_t>(rows_hint, 0xFFFFFFFFull));
    }
    bool tma = false;
    if (int rc = launch_fetch_hits(f, rows, sample_bytes, st, &tma)) return rc;
    if (!tma) f.mlist = f.mctl = nullptr;
    // each miss row is spread over up to 256 blocks (a 16 MiB row is 1 Mi
    // 16-byte pairs); listed miss rows over grid.y = 148, else every row
    dim3 g2(unsigned(std::min<uint64_t>(std::max<uint64_t>(f.vec_per_row / 4096, 1), 256)),
            unsigned(f.mlist ? std::min<uint64_t>(rows, 148) : std::min<uint64_t>(std::max<uint64_t>(rows, 1), 1024)));
    static const bool nomiss = std::getenv("LSG_DEBUG_NOMISS") != nullptr;  // timing experiments only
    if (nomiss) return kOk;
    LSG_CUDA(launch_pdl(k_fetch_step_misses, g2, dim3(256), 0, st, f, 1));
    LSG_LAUNCH_CHECK("k_fetch_step_misses");
    return kOk;
}

// hits only (the Store-backed step fetch reads the misses from the file)
int gather_step_hits_device(void* const* d_bufs, void* const* d_outs, const uint32_t* d_slots,
                            const uint32_t* d_node_off, uint32_t k0, uint32_t k1, uint64_t rows_hint,
                            uint64_t sample_bytes, cudaStream_t st) {
    if (k1 <= k0) return kOk;
    if (sample_bytes == 0 || sample_bytes % 16 != 0)
        return set_error(kValidation, "fetch_step: sample_bytes must be a positive multiple of 16");
    StepFetch f{};
    f.slots = d_slots;
    f.node_off = d_node_off;
    f.bufs = reinterpret_cast<uint4* const*>(d_bufs);
    f.outs = reinterpret_cast<uint4* const*>(d_outs);
    f.k0 = k0;
    f.k1 = k1;
    f.vec_per_row = sample_bytes / 16;
    f.tiles_per_row = (f.vec_per_row + kTileVec - 1) / kTileVec;
    const uint64_t rows = rows_hint ? rows_hint : 1;
    Scratch sc(st);
    f.claim = sc.get<uint32_t>(1);
    if (!f.claim) return set_error(kInternal, "fetch_step: scratch allocation failed");
    LSG_CUDA(cudaMemsetAsync(f.claim, 0, 4, st));
    return launch_fetch_hits(f, rows, sample_bytes, st, nullptr);
}

int batch_fetch_device(void* d_buf, const uint32_t* d_ids, const uint32_t* d_slots, uint64_t n,
                       uint64_t sample_bytes, uint64_t seed, void* d_out, cudaStream_t st) {
    if (n == 0) return kOk;
    if (sample_bytes == 0 || sample_bytes % 16 != 0)
        return set_error(kValidation, "batch_fetch: sample_bytes must be a positive multiple of 16");
    if ((reinterpret_cast<uintptr_t>(d_buf) | reinterpret_cast<uintptr_t>(d_out)) & 15)
        return set_error(kValidation, "batch_fetch: buffers must be 16-byte aligned");
    const uint64_t vpr = sample_bytes / 16;
    const uint64_t tpr = (vpr + kTileVec - 1) / kTileVec;
    const unsigned grid = unsigned(std::min<uint64_t>(n * tpr, 148ull * 8));
    k_gather_hits<<<grid, kGatherThreads, 0, st>>>(static_cast<const uint4*>(d_buf), d_slots, n, vpr, tpr,
                                                   static_cast<uint4*>(d_out));
    LSG_LAUNCH_CHECK("k_gather_hits");
    const uint64_t wpr = sample_bytes / 8;
    dim3 g2(unsigned(std::min<uint64_t>((wpr / 2 + 255) / 256, 16)), unsigned(std::min<uint64_t>(n, 4096)));
    k_fill_misses<<<g2, 256, 0, st>>>(d_ids, d_slots, n, wpr, seed, static_cast<ulonglong2*>(d_buf),
                                      static_cast<ulonglong2*>(d_out));
    LSG_LAUNCH_CHECK("k_fill_misses");
    return kOk;
}

int gather_device(const void* d_buf, const uint32_t* d_slots, uint64_t n, uint64_t sample_bytes,
                  void* d_out, cudaStream_t st) {
    if (n == 0) return kOk;
    if (sample_bytes == 0 || sample_bytes % 16 != 0)
        return set_error(kValidation, "gather: sample_bytes must be a positive multiple of 16");
    if ((reinterpret_cast<uintptr_t>(d_buf) | reinterpret_cast<uintptr_t>(d_out)) & 15)
        return set_error(kValidation, "gather: buffers must be 16-byte aligned");
    const uint64_t vpr = sample_bytes / 16;
    const uint64_t tpr = (vpr + kTileVec - 1) / kTileVec;
    const uint64_t tiles = n * tpr;
    const unsigned grid = unsigned(std::min<uint64_t>(tiles, 148ull * 8));
    k_gather<<<grid, kGatherThreads, 0, st>>>(static_cast<const uint4*>(d_buf), d_slots, n, vpr, tpr,
                                              static_cast<uint4*>(d_out));
    LSG_LAUNCH_CHECK("k_gather");
    return kOk;
}

int store_fill_device(const uint32_t* d_ids, uint64_t n, uint64_t sample_bytes, uint64_t seed,
                      void* d_dst, cudaStream_t st) {
    if (n == 0) return kOk;
    if (sample_bytes == 0) return set_error(kStorage, "store_fill: sample_size must be >= 1");
    if (sample_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(d_dst) & 15) == 0) {
        const uint64_t wpr = sample_bytes / 8;
        k_store_fill_vec<<<grid_for(n * wpr / 2, 256, 148 * 16), 256, 0, st>>>(
            d_ids, n, wpr, seed, static_cast<ulonglong2*>(d_dst));
        LSG_LAUNCH_CHECK("k_store_fill_vec");
    } else {
        k_store_fill_bytes<<<grid_for(n * sample_bytes, 256, 148 * 16), 256, 0, st>>>(
            d_ids, n, sample_bytes, seed, static_cast<uint8_t*>(d_dst));
        LSG_LAUNCH_CHECK("k_store_fill_bytes");
    }
    return kOk;
}

}  // namespace lsg

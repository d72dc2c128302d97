// chunk.cu — chunk-read planning of every (step, node) fetch list
// (plan_chunks, chunking.cpp:9-33, or singles_plan, pipeline.cpp:21-28, as
// pipeline.cpp:83-88 selects), producing StepPlan::reads.
//
// One warp per list: the list's fetch ids (items without the hit tag) are
// compacted into the warp's shared-memory slice, bitonic-sorted, de-duplicated
// (plan_chunks only), then greedily cut into reads of span <= threshold. The
// cut is a short serial chain per list (lane 0); lists are independent, so
// the T*N lists of a plan run fully in parallel. Reads of list (g, k) are
// written at that list's item offsets (a list never has more reads than
// items); start == end marks a Single read.
#include "common.cuh"

namespace lsg {

namespace {

struct ReadArgs {
    const uint32_t* items;
    const uint32_t* node_off;
    uint32_t T, N, S, B, keep, P2;
    int chunked;
    uint32_t thr;
    uint32_t *rstart, *rend, *rcount, *needed, *redundant;
};

__global__ void k_plan_reads(ReadArgs a) {
    extern __shared__ uint32_t cbuf[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t wpb = blockDim.x >> 5;
    uint32_t* buf = cbuf + size_t(wib) * a.P2;
    for (uint64_t list = uint64_t(blockIdx.x) * wpb + wib; list < uint64_t(a.T) * a.N;
         list += uint64_t(gridDim.x) * wpb) {
        const uint32_t g = uint32_t(list / a.N), k = uint32_t(list % a.N);
        const uint64_t base = uint64_t(g / a.S) * a.keep + uint64_t(g % a.S) * a.B;
        const uint32_t* off = a.node_off + size_t(g) * (a.N + 1);
        const uint64_t lo = base + off[k];
        const uint32_t L = off[k + 1] - off[k];
        // compact fetch ids
        uint32_t F = 0;
        for (uint32_t c = 0; c < L; c += 32) {
            const uint32_t v = c + lane < L ? a.items[lo + c + lane] : kHit;
            const bool f = !(v & kHit);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
            if (f) {
                uint32_t m;
                asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
                buf[F + __popc(bal & m)] = v;
            }
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
        if (lane == 0) {
            uint32_t nr = 0, red = 0, need = F;
            if (a.chunked) {
                uint32_t u = 0;
                for (uint32_t i = 0; i < F; ++i)
                    if (u == 0 || buf[u - 1] != buf[i]) buf[u++] = buf[i];
                need = u;
                for (uint32_t i = 0; i < u;) {
                    const uint32_t start = buf[i];
                    uint32_t j = i + 1;
                    while (j < u && buf[j] - start + 1 <= a.thr) ++j;
                    a.rstart[lo + nr] = start;
                    a.rend[lo + nr] = buf[j - 1];
                    if (j - i > 1) red += (buf[j - 1] - start + 1) - (j - i);
                    ++nr;
                    i = j;
                }
            } else {
                for (uint32_t i = 0; i < F; ++i) {
                    a.rstart[lo + nr] = buf[i];
                    a.rend[lo + nr] = buf[i];
                    ++nr;
                }
            }
            a.rcount[list] = nr;
            if (a.needed) a.needed[list] = need;
            if (a.redundant) a.redundant[list] = red;
        }
        __syncwarp();
    }
}

// longest list of the plan (sizes the per-warp sort slices)
__global__ void k_max_list(const uint32_t* __restrict__ node_off, uint32_t T, uint32_t N, uint32_t* out) {
    uint32_t m = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < uint64_t(T) * N;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t g = uint32_t(i / N), k = uint32_t(i % N);
        const uint32_t* off = node_off + size_t(g) * (N + 1);
        m = max(m, off[k + 1] - off[k]);
    }
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace

int plan_reads_device(const uint32_t* d_items, const uint32_t* d_node_off, uint32_t T, uint32_t N,
                      uint32_t S, uint32_t B, uint32_t keep, int chunked, uint64_t thr, uint32_t* rstart,
                      uint32_t* rend, uint32_t* rcount, uint32_t* needed, uint32_t* redundant,
                      cudaStream_t st) {
    if (!rstart || !rend || !rcount || T == 0) return kOk;
    if (chunked && thr == 0) return set_error(kValidation, "plan_chunks: threshold must be >= 1");
    ReadArgs a{d_items, d_node_off, T, N, S, B, keep, 1, chunked, uint32_t(std::min<uint64_t>(thr, 0xFFFFFFFFu)),
               rstart, rend, rcount, needed, redundant};
    uint32_t lmax = B;  // a node list never exceeds its step
    if (B > 4096) {     // wide steps: size the slices by the longest list
        Scratch sc(st);
        uint32_t* d_m = sc.get<uint32_t>(1);
        if (!d_m) return set_error(kInternal, "plan_reads: scratch allocation failed");
        LSG_CUDA(cudaMemsetAsync(d_m, 0, 4, st));
        k_max_list<<<grid_for(uint64_t(T) * N, 256, 592), 256, 0, st>>>(d_node_off, T, N, d_m);
        LSG_LAUNCH_CHECK("k_max_list");
        if (int _rc = d2h_small(&lmax, d_m, 4, st)) return _rc;
        LSG_CUDA(cudaStreamSynchronize(st));
    }
    while (a.P2 < lmax) a.P2 <<= 1;
    if (size_t(a.P2) * 4 > 200u * 1024)
        return set_error(kCapability, "plan_reads: a node list is too long for the device chunk planner");
    const uint32_t wpb = std::max<uint32_t>(1, std::min<uint32_t>(8, (96u * 1024) / (4 * a.P2)));
    const size_t smem = size_t(wpb) * a.P2 * 4;
    LSG_CUDA(cudaFuncSetAttribute(k_plan_reads, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const uint64_t lists = uint64_t(T) * N;
    const unsigned grid = unsigned(std::min<uint64_t>((lists + wpb - 1) / wpb, 148ull * 8));
    k_plan_reads<<<grid, wpb * 32, smem, st>>>(a);
    LSG_LAUNCH_CHECK("k_plan_reads");
    return kOk;
}

}  // namespace lsg

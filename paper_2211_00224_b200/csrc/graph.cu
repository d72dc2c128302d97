// graph.cu — K2 (reuse windows as bitsets) + K3 (epoch-pair reuse matrix).
//
// Reference: build_reuse_graph (reuse_graph.cpp:77-101) with distinct_window
// (:14-29), node_sequence (:31-41) and window (:43-56):
//   w(u,v) = sum_k | First_k(v) \ Last_k(u) |,  w(u,u) = 0,
// First/Last = first/last `want` DISTINCT ids of the epoch sequence (Global,
// want = C*N) or of node k's concatenated slices (PerNode, want = C).
//
// Windows become D-bit bitsets. For the PerNode mode the N node bitsets of an
// epoch are laid end to end, so both modes reduce to one "and-not popcount
// Gram matrix" between the Last rows and the First rows:
//   w(u,v) = sum_words popc(F[v][i] & ~L[u][i]).
// That contraction is integer-pipe work (LOP3 + POPC + IADD), tiled like a
// GEMM through shared memory, 4x4 pairs per thread, split over the word
// dimension so E=100 still fills the 148 SMs.
#include "common.cuh"

namespace lsg {

namespace {

struct WinGeom {
    uint32_t len;    // epoch sequence length
    uint32_t N;      // nodes
    uint32_t b;      // local batch
    uint32_t B;      // global batch
    uint32_t S;      // steps per epoch
    uint32_t words;  // words per bitset (ceil(D/32))
    uint32_t nwin;   // windows per epoch (1 Global, N PerNode)
    uint64_t want;   // distinct ids per window
};

// node k's sequence length (slices clamped at the sequence end, trace.cpp:45-57)
__device__ __forceinline__ uint32_t node_len(const WinGeom& g, uint32_t k) {
    if (g.nwin == 1) return g.len;
    uint32_t n = 0;
    // full steps contribute b each; only the final step can be ragged
    if (g.S == 0) return 0;
    const uint64_t last_lo = uint64_t(g.S - 1) * g.B + uint64_t(k) * g.b;
    const uint64_t lo = std::min<uint64_t>(last_lo, g.len);
    const uint64_t hi = std::min<uint64_t>(last_lo + g.b, g.len);
    n = (g.S - 1) * g.b + uint32_t(hi - lo);
    return n;
}
// q-th element of window k's sequence -> trace position
__device__ __forceinline__ uint32_t node_pos(const WinGeom& g, uint32_t k, uint32_t q) {
    if (g.nwin == 1) return q;
    return (q / g.b) * g.B + k * g.b + (q % g.b);
}

// Fast path: every epoch row holds distinct ids (always true for generated
// traces). The window is then a contiguous prefix/suffix of the sequence.
__global__ void k_windows_distinct(WinGeom g, const uint32_t* __restrict__ trace,
                                   uint32_t* __restrict__ Fb, uint32_t* __restrict__ Lb) {
    const uint32_t e = blockIdx.y / g.nwin, k = blockIdx.y % g.nwin;
    const uint32_t n = node_len(g, k);
    const uint32_t w = uint32_t(std::min<uint64_t>(g.want, n));
    const uint32_t* seq = trace + size_t(e) * g.len;
    uint32_t* F = Fb + (size_t(e) * g.nwin + k) * g.words;
    uint32_t* L = Lb + (size_t(e) * g.nwin + k) * g.words;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < w; q += gridDim.x * blockDim.x) {
        const uint32_t a = seq[node_pos(g, k, q)];
        atomicOr(&F[a >> 5], 1u << (a & 31));
        const uint32_t z = seq[node_pos(g, k, n - 1 - q)];
        atomicOr(&L[z >> 5], 1u << (z & 31));
    }
}

// Same, one CTA per (epoch, window, direction): the window's D-bit bitset is
// built in shared memory (atomicOr on banks instead of L2) and written out
// once, coalesced. Used while a bitset fits in shared memory.
__global__ void __launch_bounds__(1024) k_windows_smem(WinGeom g, const uint32_t* __restrict__ trace,
                                                       uint32_t* __restrict__ Fb, uint32_t* __restrict__ Lb) {
    extern __shared__ uint32_t bits[];
    const uint32_t e = blockIdx.x / g.nwin, k = blockIdx.x % g.nwin, dir = blockIdx.y;
    for (uint32_t i = threadIdx.x; i < g.words; i += blockDim.x) bits[i] = 0;
    __syncthreads();
    const uint32_t n = node_len(g, k);
    const uint32_t w = uint32_t(std::min<uint64_t>(g.want, n));
    const uint32_t* seq = trace + size_t(e) * g.len;
    for (uint32_t q = threadIdx.x; q < w; q += blockDim.x) {
        const uint32_t a = __ldg(&seq[node_pos(g, k, dir ? n - 1 - q : q)]);
        atomicOr(&bits[a >> 5], 1u << (a & 31));
    }
    __syncthreads();
    uint32_t* out = (dir ? Lb : Fb) + (size_t(e) * g.nwin + k) * g.words;
    for (uint32_t i = threadIdx.x; i < g.words; i += blockDim.x) out[i] = bits[i];
}

// General path (rows may repeat ids, as read_trace admits): one warp per
// (epoch, window, direction) walks the sequence 32 positions at a time and
// stops exactly at the want-th distinct id. Inside a chunk only the first lane
// of each equal-id group may claim the bit, so the cut is exact.
__global__ void k_windows_general(WinGeom g, uint32_t E, const uint32_t* __restrict__ trace,
                                  uint32_t* __restrict__ Fb, uint32_t* __restrict__ Lb) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t total = E * g.nwin * 2;
    if (warp >= total) return;
    const uint32_t dir = warp & 1, win = warp >> 1;
    const uint32_t e = win / g.nwin, k = win % g.nwin;
    const uint32_t n = node_len(g, k);
    const uint32_t* seq = trace + size_t(e) * g.len;
    uint32_t* bits = (dir == 0 ? Fb : Lb) + (size_t(e) * g.nwin + k) * g.words;
    uint64_t count = 0;
    if (g.want == 0) return;
    for (uint32_t c = 0; c < n; c += 32) {
        const uint32_t i = c + lane;
        const bool valid = i < n;
        uint32_t x = 0;
        if (valid) x = seq[node_pos(g, k, dir == 0 ? i : n - 1 - i)];
        const uint32_t vmask = __ballot_sync(0xFFFFFFFFu, valid);
        const uint32_t grp = __match_any_sync(0xFFFFFFFFu, valid ? x : 0xFFFFFFFFu) & vmask;
        const bool leader = valid && (lane == uint32_t(__ffs(grp) - 1));
        bool fresh = false;
        if (leader) {
            const uint32_t bit = 1u << (x & 31);
            fresh = (atomicOr(&bits[x >> 5], bit) & bit) == 0;
        }
        const uint32_t nb = __ballot_sync(0xFFFFFFFFu, fresh);
        const uint32_t got = __popc(nb);
        if (count + got >= g.want) {
            // keep the first (want - count) fresh claims, release the rest
            uint32_t need = uint32_t(g.want - count), m = nb, cut = 0;
            for (uint32_t r = 0; r < need; ++r) { cut = __ffs(m) - 1; m &= m - 1; }
            if (fresh && lane > cut) atomicAnd(&bits[x >> 5], ~(1u << (x & 31)));
            return;
        }
        count += got;
    }
}

constexpr int kGT = 64;   // tile edge (pairs)
constexpr int kGK = 32;   // words per smem stage

// and-not popcount Gram matrix: w[u][v] += sum popc(F[v] & ~L[u]) over this
// block's word range; 16x16 threads, 4x4 pairs each. Rows u in [r0, r1) are
// written to w[u - r0][v] (a row block, for the multi-GPU row sharding).
__global__ void __launch_bounds__(256) k_reuse_gram(uint32_t E, uint32_t r0, uint32_t r1, uint32_t W, uint32_t kspan,
                                                    const uint32_t* __restrict__ F,
                                                    const uint32_t* __restrict__ L,
                                                    unsigned long long* __restrict__ w) {
    __shared__ uint32_t Ls[kGK][kGT + 1];
    __shared__ uint32_t Fs[kGK][kGT + 1];
    const uint32_t u0 = r0 + blockIdx.y * kGT, v0 = blockIdx.x * kGT;
    const uint32_t k0 = blockIdx.z * kspan, k1 = std::min<uint32_t>(W, k0 + kspan);
    const uint32_t t = threadIdx.x, tu = t >> 4, tv = t & 15;
    uint32_t acc[4][4] = {};
    for (uint32_t kb = k0; kb < k1; kb += kGK) {
        // stage 64 rows x 32 words of L (rows u) and F (rows v)
        for (int i = 0; i < (kGT * kGK) / 256; ++i) {
            const uint32_t r = (t >> 5) + 8 * i, kk = t & 31;
            const uint32_t wd = kb + kk;
            const bool okw = wd < k1;
            const uint32_t u = u0 + r, v = v0 + r;
            Ls[kk][r] = (okw && u < r1) ? L[size_t(u) * W + wd] : 0xFFFFFFFFu;  // ~L = 0
            Fs[kk][r] = (okw && v < E) ? F[size_t(v) * W + wd] : 0u;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < kGK; ++kk) {
            uint32_t l[4], f[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) l[a] = Ls[kk][tu + 16 * a];
#pragma unroll
            for (int c = 0; c < 4; ++c) f[c] = Fs[kk][tv + 16 * c];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][c] += __popc(f[c] & ~l[a]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t u = u0 + tu + 16 * a, v = v0 + tv + 16 * c;
            if (u < r1 && v < E && u != v && acc[a][c])
                atomicAdd(&w[size_t(u - r0) * E + v], (unsigned long long)acc[a][c]);
        }
}

// Device check that every epoch row holds distinct ids (selects the path).
__global__ void k_rows_distinct(uint32_t len, uint32_t words, const uint32_t* __restrict__ trace,
                                uint32_t* __restrict__ seen, uint32_t* __restrict__ dup) {
    const uint32_t e = blockIdx.y;
    uint32_t* bits = seen + size_t(e) * words;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        const uint32_t x = trace[size_t(e) * len + i];
        const uint32_t bit = 1u << (x & 31);
        if (atomicOr(&bits[x >> 5], bit) & bit) atomicOr(dup, 1u);
    }
}

}  // namespace

// K2 alone: First/Last window bitsets, [E][nwin][ceil(D/32)] words each
// (first_buffer_window / last_buffer_window, reuse_graph.cpp:43-75).
int window_bits_device(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D, uint32_t N, uint64_t b,
                       bool drop_last, uint64_t buffer_size, int mode, bool rows_distinct_known, uint32_t* Fb,
                       uint32_t* Lb, cudaStream_t st);

// Rows [r0, r1) of w into d_w ([r1 - r0][E]); the full graph is r0 = 0, r1 = E.
int build_reuse_graph_device(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D,
                             uint32_t N, uint64_t b, bool drop_last, uint64_t buffer_size, int mode,
                             bool rows_distinct_known, uint64_t* d_w, cudaStream_t st, uint32_t r0,
                             uint32_t r1) {
    if (buffer_size == 0) return set_error(kValidation, "build_reuse_graph: buffer_size must be >= 1");
    if (r1 == kNone) r1 = E;
    if (r0 > r1 || r1 > E) return set_error(kValidation, "build_reuse_graph: bad row range");
    if (E == 0 || r0 == r1) return kOk;
    LSG_CUDA(cudaMemsetAsync(d_w, 0, size_t(r1 - r0) * E * sizeof(uint64_t), st));
    const uint64_t W = uint64_t((D + 31) / 32) * (mode == 0 ? 1 : N);  // words per (epoch) row
    Scratch sc(st);
    uint32_t* Fb = sc.get<uint32_t>(size_t(E) * W);
    uint32_t* Lb = sc.get<uint32_t>(size_t(E) * W);
    if (!Fb || !Lb) return set_error(kInternal, "build_reuse_graph: scratch allocation failed");
    if (int rc = window_bits_device(d_trace, E, len, D, N, b, drop_last, buffer_size, mode, rows_distinct_known, Fb,
                                    Lb, st))
        return rc;
    const uint32_t rows = r1 - r0;
    const uint32_t tiles = ((rows + kGT - 1) / kGT) * ((E + kGT - 1) / kGT);
    uint32_t split = std::max<uint32_t>(1, (296 + tiles - 1) / tiles);
    split = std::min<uint64_t>(split, std::max<uint64_t>(1, W / 256));
    uint32_t kspan = uint32_t((W + split - 1) / split);
    kspan = (kspan + kGK - 1) / kGK * kGK;
    split = uint32_t((W + kspan - 1) / kspan);
    dim3 grid((E + kGT - 1) / kGT, (rows + kGT - 1) / kGT, split);
    k_reuse_gram<<<grid, 256, 0, st>>>(E, r0, r1, uint32_t(W), kspan, Fb, Lb,
                                       reinterpret_cast<unsigned long long*>(d_w));
    LSG_LAUNCH_CHECK("k_reuse_gram");
    return kOk;
}

int window_bits_device(const uint32_t* d_trace, uint32_t E, uint64_t len, uint64_t D, uint32_t N, uint64_t b,
                       bool drop_last, uint64_t buffer_size, int mode, bool rows_distinct_known, uint32_t* Fb,
                       uint32_t* Lb, cudaStream_t st) {
    WinGeom g;
    g.len = uint32_t(len);
    g.N = N;
    g.b = uint32_t(b);
    g.B = uint32_t(uint64_t(N) * b);
    const uint64_t B = uint64_t(N) * b;
    g.S = uint32_t(B == 0 ? 0 : (drop_last ? D / B : (D + B - 1) / B));
    g.words = uint32_t((D + 31) / 32);
    g.nwin = mode == 0 ? 1 : N;
    g.want = mode == 0 ? buffer_size * N : buffer_size;
    const uint64_t W = uint64_t(g.words) * g.nwin;  // words per (epoch) row
    Scratch sc(st);
    const size_t smem_bits = size_t(g.words) * 4;
    const bool smem_fits = smem_bits <= 200 * 1024;
    if (!(rows_distinct_known && smem_fits)) {  // (the shared-memory path writes every word)
        LSG_CUDA(cudaMemsetAsync(Fb, 0, size_t(E) * W * 4, st));
        LSG_CUDA(cudaMemsetAsync(Lb, 0, size_t(E) * W * 4, st));
    }

    bool distinct = rows_distinct_known;
    if (!distinct) {
        uint32_t* seen = sc.get<uint32_t>(size_t(E) * g.words);
        uint32_t* dup = sc.get<uint32_t>(1);
        LSG_CUDA(cudaMemsetAsync(seen, 0, size_t(E) * g.words * 4, st));
        LSG_CUDA(cudaMemsetAsync(dup, 0, 4, st));
        k_rows_distinct<<<dim3(grid_for(len, 256, 1024), E), 256, 0, st>>>(g.len, g.words, d_trace, seen, dup);
        LSG_LAUNCH_CHECK("k_rows_distinct");
        uint32_t h = 1;
        if (int _rc = d2h_small(&h, dup, 4, st)) return _rc;
        LSG_CUDA(cudaStreamSynchronize(st));
        distinct = h == 0;
    }
    if (distinct && smem_fits) {
        LSG_CUDA(cudaFuncSetAttribute(k_windows_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bits)));
        k_windows_smem<<<dim3(E * g.nwin, 2), 1024, smem_bits, st>>>(g, d_trace, Fb, Lb);
        LSG_LAUNCH_CHECK("k_windows_smem");
    } else if (distinct) {
        const uint64_t per = std::min<uint64_t>(g.want, len);
        k_windows_distinct<<<dim3(grid_for(per, 256, 1024), E * g.nwin), 256, 0, st>>>(g, d_trace, Fb, Lb);
        LSG_LAUNCH_CHECK("k_windows_distinct");
    } else {
        const uint64_t warps = uint64_t(E) * g.nwin * 2;
        k_windows_general<<<grid_for(warps * 32, 256, 1u << 20), 256, 0, st>>>(g, E, d_trace, Fb, Lb);
        LSG_LAUNCH_CHECK("k_windows_general");
    }
    return kOk;
}

}  // namespace lsg

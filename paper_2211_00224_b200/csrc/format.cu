// format.cu — the text artifacts (trace.cpp:72-84 write_trace, plan.cpp:44-69
// write_plan, reuse_graph.cpp:103-112 write_graph) formatted on the GPU.
//
// At config 2 the plan file holds 26.2M `assign` rows (≈0.7 GB of text) and
// the trace file 26.2M id lines: formatting them is a throughput problem, so
// every row is a parallel unit. Pass 1 computes each row's byte length from
// its decimal digit counts, a device-wide exclusive scan turns lengths into
// offsets, pass 2 writes every row at its offset. The few header lines are
// formatted on the host. Output is byte-identical to the reference's
// ostream output.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace lsg {

namespace {

__device__ __forceinline__ uint32_t ndig(uint64_t v) {
    uint32_t n = 1;
    while (v >= 10) {
        v /= 10;
        ++n;
    }
    return n;
}

// writes v in n = ndig(v) characters at p, returns p + n
__device__ __forceinline__ char* put(char* p, uint64_t v, uint32_t n) {
    for (uint32_t i = n; i > 0; --i) {
        p[i - 1] = char('0' + v % 10);
        v /= 10;
    }
    return p + n;
}

__device__ __forceinline__ char* puts_(char* p, const char* s) {
    while (*s) *p++ = *s++;
    return p;
}

// ---- exclusive scan of u32 lengths into u64 offsets (3 passes) ----------
constexpr int kScanT = 1024, kScanPer = 8, kScanTile = kScanT * kScanPer;

__global__ void __launch_bounds__(kScanT) k_tile_sums(const uint32_t* __restrict__ len, uint64_t n,
                                                      uint64_t* __restrict__ sums) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
    uint64_t s = 0;
    for (int i = 0; i < kScanPer; ++i) {
        const uint64_t j = base + uint64_t(i) * kScanT + threadIdx.x;
        if (j < n) s += len[j];
    }
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, d);
    __shared__ uint64_t part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint64_t v = part[threadIdx.x];
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
        if (threadIdx.x == 0) sums[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(kScanT) k_scan_sums(uint64_t* __restrict__ sums, uint64_t n) {
    __shared__ uint64_t part[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint64_t c = 0; c < n; c += kScanT) {
        const uint64_t i = c + threadIdx.x;
        const uint64_t v = i < n ? sums[i] : 0;
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
        if (i < n) sums[i] = carry + part[w] + inc - v;
        __syncthreads();
        if (threadIdx.x == kScanT - 1) carry += part[w] + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[n] = carry;
}

__global__ void __launch_bounds__(kScanT) k_tile_scan(const uint32_t* __restrict__ len, uint64_t n,
                                                      const uint64_t* __restrict__ sums, uint64_t* __restrict__ off) {
    // thread t owns kScanPer consecutive elements of the tile
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanPer;
    uint32_t v[kScanPer];
    uint64_t s = 0;
    for (int i = 0; i < kScanPer; ++i) {
        v[i] = base + i < n ? len[base + i] : 0u;
        s += v[i];
    }
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = s;
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= uint32_t(d)) inc += o;
    }
    __shared__ uint64_t part[32];
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
    uint64_t run = sums[blockIdx.x] + part[w] + inc - s;
    for (int i = 0; i < kScanPer; ++i) {
        if (base + i < n) off[base + i] = run;
        run += v[i];
    }
}

// ---- write_trace (trace.cpp:72-84): row (e, p) = id line, preceded by the
// "epoch e" line when p == 0
struct TraceFmt {
    const uint32_t* ids;  // [E][keep]
    uint32_t E;
    uint64_t keep;
};

__global__ void k_trace_len(TraceFmt f, uint32_t* __restrict__ len) {
    const uint64_t n = uint64_t(f.E) * f.keep;
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n; r += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = r / f.keep, p = r - e * f.keep;
        uint32_t l = ndig(f.ids[r]) + 1;
        if (p == 0) l += 6 + ndig(e) + 1;  // "epoch " e "\n"
        len[r] = l;
    }
}

__global__ void k_trace_write(TraceFmt f, const uint64_t* __restrict__ off, char* __restrict__ out) {
    const uint64_t n = uint64_t(f.E) * f.keep;
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n; r += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = r / f.keep, p = r - e * f.keep;
        char* q = out + off[r];
        if (p == 0) {
            q = puts_(q, "epoch ");
            q = put(q, e, ndig(e));
            *q++ = '\n';
        }
        const uint32_t x = f.ids[r];
        q = put(q, x, ndig(x));
        *q = '\n';
    }
}

// ---- write_plan (plan.cpp:51-68) step rows. Row slots of step g (in file
// order): N balance rows, the step's items (assign rows, node lists in
// order), then read slots (item offsets; valid when index < read_count)
struct PlanFmt {
    const uint32_t* items;     // id | hit
    const uint32_t* node_off;  // [T][N+1]
    const uint32_t* fb;        // [T][N]
    const uint32_t* fa;        // [T][N]
    const uint32_t* rstart;    // item-aligned, may be null
    const uint32_t* rend;
    const uint32_t* rcount;    // [T][N]
    const uint32_t* order;     // [E] epoch id of execution epoch i
    const uint64_t* gbase;     // [T+1] first item of step g
    const uint64_t* sbase;     // [T+1] first slot of step g
    uint32_t T, N, S;
};

__device__ __forceinline__ uint32_t slot_step(const PlanFmt& f, uint64_t s) {
    uint32_t lo = 0, hi = f.T;  // last g with sbase[g] <= s
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (f.sbase[mid] <= s) lo = mid; else hi = mid;
    }
    return lo;
}

// the row of slot s: kind 0 balance (k), 1 assign (item i of the step, node k),
// 2 read (item-aligned index i of node k, valid or not)
struct RowRef {
    uint32_t g, kind, k, i;
    bool valid;
};

__device__ __forceinline__ RowRef row_of(const PlanFmt& f, uint64_t s) {
    RowRef r;
    r.g = slot_step(f, s);
    const uint32_t* off = f.node_off + size_t(r.g) * (f.N + 1);
    const uint32_t L = off[f.N];
    uint32_t q = uint32_t(s - f.sbase[r.g]);
    r.valid = true;
    if (q < f.N) {
        r.kind = 0;
        r.k = q;
        r.i = 0;
        return r;
    }
    q -= f.N;
    r.kind = q < L ? 1 : 2;
    r.i = q < L ? q : q - L;
    uint32_t lo = 0, hi = f.N;  // node of item i: first k with off[k+1] > i (skips empty lists)
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (off[mid + 1] > r.i) hi = mid; else lo = mid + 1;
    }
    r.k = lo;
    if (r.kind == 2) r.valid = f.rstart && (r.i - off[r.k]) < f.rcount[size_t(r.g) * f.N + r.k];
    return r;
}

__device__ __forceinline__ uint32_t prefix_len(const PlanFmt& f, const RowRef& r, uint32_t e, uint32_t t) {
    return ndig(e) + 1 + ndig(t) + 1 + ndig(r.k) + 1;  // "e t k "
}

__global__ void k_plan_len(PlanFmt f, uint64_t nslots, uint32_t* __restrict__ len) {
    for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < nslots;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const RowRef r = row_of(f, s);
        if (!r.valid) {
            len[s] = 0;
            continue;
        }
        const uint32_t e = f.order[r.g / f.S], t = r.g % f.S;
        uint32_t l = prefix_len(f, r, e, t);
        const size_t gk = size_t(r.g) * f.N + r.k;
        const uint64_t item = f.gbase[r.g] + r.i;
        if (r.kind == 0) {
            l += 8 + ndig(f.fb[gk]) + 1 + ndig(f.fa[gk]) + 1;  // "balance " .. "b a\n"
        } else if (r.kind == 1) {
            const uint32_t it = f.items[item];
            l += 7 + ndig(it & ~kHit) + 1 + ((it & kHit) ? 3 : 5) + 1;  // "assign " .. "id hit\n"
        } else {
            const uint32_t* off = f.node_off + size_t(r.g) * (f.N + 1);
            const uint64_t ri = f.gbase[r.g] + off[r.k] + (r.i - off[r.k]);
            const uint32_t a = f.rstart[ri], b = f.rend[ri];
            l += 5 + (a == b ? 6 : 5) + 1 + ndig(a) + 1 + ndig(b) + 1;  // "read " kind " a b\n"
        }
        len[s] = l;
    }
}

__global__ void k_plan_write(PlanFmt f, uint64_t nslots, const uint64_t* __restrict__ offs, char* __restrict__ out) {
    for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < nslots;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const RowRef r = row_of(f, s);
        if (!r.valid) continue;
        const uint32_t e = f.order[r.g / f.S], t = r.g % f.S;
        const size_t gk = size_t(r.g) * f.N + r.k;
        char* q = out + offs[s];
        q = puts_(q, r.kind == 0 ? "balance " : (r.kind == 1 ? "assign " : "read "));
        q = put(q, e, ndig(e));
        *q++ = ' ';
        q = put(q, t, ndig(t));
        *q++ = ' ';
        q = put(q, r.k, ndig(r.k));
        *q++ = ' ';
        if (r.kind == 0) {
            q = put(q, f.fb[gk], ndig(f.fb[gk]));
            *q++ = ' ';
            q = put(q, f.fa[gk], ndig(f.fa[gk]));
        } else if (r.kind == 1) {
            const uint32_t it = f.items[f.gbase[r.g] + r.i], x = it & ~kHit;
            q = put(q, x, ndig(x));
            q = puts_(q, (it & kHit) ? " hit" : " fetch");
        } else {
            const uint32_t* off = f.node_off + size_t(r.g) * (f.N + 1);
            const uint64_t ri = f.gbase[r.g] + off[r.k] + (r.i - off[r.k]);
            const uint32_t a = f.rstart[ri], b = f.rend[ri];
            q = puts_(q, a == b ? "single " : "chunk ");
            q = put(q, a, ndig(a));
            *q++ = ' ';
            q = put(q, b, ndig(b));
        }
        *q = '\n';
    }
}

int scan_lengths(const uint32_t* d_len, uint64_t n, uint64_t* d_off, uint64_t* total, Scratch& sc,
                 cudaStream_t st) {
    const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    uint64_t* sums = sc.get<uint64_t>(tiles + 1);
    if (!sums) return set_error(kInternal, "format: scratch allocation failed");
    if (tiles) {
        k_tile_sums<<<unsigned(tiles), kScanT, 0, st>>>(d_len, n, sums);
        LSG_LAUNCH_CHECK("k_tile_sums");
    }
    k_scan_sums<<<1, kScanT, 0, st>>>(sums, tiles);
    LSG_LAUNCH_CHECK("k_scan_sums");
    if (tiles) {
        k_tile_scan<<<unsigned(tiles), kScanT, 0, st>>>(d_len, n, sums, d_off);
        LSG_LAUNCH_CHECK("k_tile_scan");
    }
    LSG_CUDA(cudaMemcpyAsync(total, sums + tiles, 8, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    return kOk;
}

// the formatted body lands in device memory; copied to h_out when it fits
int finish(const char* head, size_t hlen, const char* d_body, uint64_t blen, char* h_out, uint64_t cap,
           uint64_t* nbytes, cudaStream_t st) {
    if (nbytes) *nbytes = hlen + blen;
    if (!h_out || cap < hlen + blen) return kOk;
    std::memcpy(h_out, head, hlen);
    if (blen) LSG_CUDA(cudaMemcpyAsync(h_out + hlen, d_body, blen, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    return kOk;
}

}  // namespace
}  // namespace lsg

using namespace lsg;

extern "C" {

int lsg_format_trace(const uint32_t* d_trace, uint64_t dataset_size, uint32_t num_epochs, uint32_t num_nodes,
                     uint64_t local_batch, uint64_t seed, int32_t drop_last, uint64_t keep, char* h_out,
                     uint64_t cap, uint64_t* nbytes, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::string head = "loadsched-trace 1\n";
    head += "dataset_size=" + std::to_string(dataset_size) + "\n";
    head += "num_epochs=" + std::to_string(num_epochs) + "\n";
    head += "num_nodes=" + std::to_string(num_nodes) + "\n";
    head += "local_batch=" + std::to_string(local_batch) + "\n";
    head += "seed=" + std::to_string(seed) + "\n";
    head += "drop_last=" + std::string(drop_last ? "1" : "0") + "\n";
    const uint64_t n = uint64_t(num_epochs) * keep;
    if (keep == 0) {  // epochs without ids: the headers only
        for (uint32_t e = 0; e < num_epochs; ++e) head += "epoch " + std::to_string(e) + "\n";
        return finish(head.data(), head.size(), nullptr, 0, h_out, cap, nbytes, st);
    }
    Scratch sc(st);
    uint32_t* len = sc.get<uint32_t>(n);
    uint64_t* off = sc.get<uint64_t>(n);
    if (!len || !off) return set_error(kInternal, "format_trace: scratch allocation failed");
    TraceFmt f{d_trace, num_epochs, keep};
    k_trace_len<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(f, len);
    LSG_LAUNCH_CHECK("k_trace_len");
    uint64_t total = 0;
    if (int rc = scan_lengths(len, n, off, &total, sc, st)) return rc;
    char* body = sc.get<char>(total);
    if (!body) return set_error(kInternal, "format_trace: scratch allocation failed");
    k_trace_write<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(f, off, body);
    LSG_LAUNCH_CHECK("k_trace_write");
    return finish(head.data(), head.size(), body, total, h_out, cap, nbytes, st);
}

int lsg_format_plan(const uint32_t* d_items, const uint32_t* d_node_off, const uint32_t* d_fetch_before,
                    const uint32_t* d_fetch_after, const uint32_t* d_read_start, const uint32_t* d_read_end,
                    const uint32_t* d_read_count, const uint32_t* d_order, uint64_t cost, uint32_t E, uint64_t T,
                    uint32_t N, uint64_t S, uint64_t dataset_size, uint64_t local_batch, uint64_t chunk_threshold,
                    char* h_out, uint64_t cap, uint64_t* nbytes, void* stream) {
    if (!d_items || !d_node_off || !d_fetch_before || !d_fetch_after || !d_order)
        return set_error(kValidation, "format_plan: missing plan arrays");
    if (S == 0 || T != uint64_t(E) * S) return set_error(kValidation, "format_plan: T must be E * S");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<uint32_t> order(E);
    LSG_CUDA(cudaMemcpyAsync(order.data(), d_order, E * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    std::string head = "loadsched-plan 1\n";
    head += "meta dataset_size=" + std::to_string(dataset_size) + " nodes=" + std::to_string(N) +
            " local_batch=" + std::to_string(local_batch) + " threshold=" + std::to_string(chunk_threshold) + "\n";
    head += "order:";
    for (uint32_t e : order) head += " " + std::to_string(e);
    head += "\ncost: " + std::to_string(cost) + "\n";
    // step bases: items before step g, row slots before step g
    std::vector<uint32_t> hoff(size_t(T) * (N + 1));
    LSG_CUDA(cudaMemcpyAsync(hoff.data(), d_node_off, hoff.size() * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    std::vector<uint64_t> hb(2 * (T + 1));
    uint64_t gi = 0, si = 0;
    for (uint64_t g = 0; g < T; ++g) {
        hb[g] = gi;
        hb[T + 1 + g] = si;
        const uint32_t L = hoff[g * (N + 1) + N];
        gi += L;
        si += N + 2ull * L;
    }
    hb[T] = gi;
    hb[2 * T + 1] = si;
    const uint64_t nslots = si;
    Scratch sc(st);
    uint64_t* gbase = sc.get<uint64_t>(2 * (T + 1));
    if (!gbase) return set_error(kInternal, "format_plan: scratch allocation failed");
    uint64_t* sbase = gbase + T + 1;
    LSG_CUDA(cudaMemcpyAsync(gbase, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice, st));
    uint32_t* len = sc.get<uint32_t>(nslots);
    uint64_t* off = sc.get<uint64_t>(nslots);
    if (!len || !off) return set_error(kInternal, "format_plan: scratch allocation failed");
    PlanFmt f{d_items, d_node_off, d_fetch_before, d_fetch_after, d_read_start, d_read_end,
              d_read_count, d_order, gbase, sbase, uint32_t(T), N, uint32_t(S)};
    if (!d_read_start || !d_read_end || !d_read_count) f.rstart = nullptr;
    k_plan_len<<<grid_for(nslots, 256, 148 * 16), 256, 0, st>>>(f, nslots, len);
    LSG_LAUNCH_CHECK("k_plan_len");
    uint64_t total = 0;
    if (int rc = scan_lengths(len, nslots, off, &total, sc, st)) return rc;
    char* body = sc.get<char>(total);
    if (!body) return set_error(kInternal, "format_plan: scratch allocation failed");
    k_plan_write<<<grid_for(nslots, 256, 148 * 16), 256, 0, st>>>(f, nslots, off, body);
    LSG_LAUNCH_CHECK("k_plan_write");
    return finish(head.data(), head.size(), body, total, h_out, cap, nbytes, st);
}

// write_graph (reuse_graph.cpp:103-112): E, then E rows of E weights
int lsg_format_graph(const uint64_t* d_w, uint32_t E, char* h_out, uint64_t cap, uint64_t* nbytes, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<uint64_t> w(size_t(E) * E);
    if (!w.empty()) LSG_CUDA(cudaMemcpyAsync(w.data(), d_w, w.size() * 8, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    std::string s = std::to_string(E) + "\n";
    char tmp[24];
    for (uint32_t u = 0; u < E; ++u) {
        for (uint32_t v = 0; v < E; ++v) {
            if (v) s += ' ';
            const int n = std::snprintf(tmp, sizeof tmp, "%llu", static_cast<unsigned long long>(w[size_t(u) * E + v]));
            s.append(tmp, size_t(n));
        }
        s += '\n';
    }
    if (nbytes) *nbytes = s.size();
    if (h_out && cap >= s.size()) std::memcpy(h_out, s.data(), s.size());
    return kOk;
}

}  // extern "C"

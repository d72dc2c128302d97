// store.cu — the sample Store (store.hpp:13-81, store.cpp:37-148) as a B200
// data path.
//
//  * create_store: the SLRD header (magic "SLRD", u16 version 1, u64 count,
//    u64 size, little-endian; 22 bytes) followed by ONE continuous splitmix64
//    byte stream (store.cpp:70-80). The payload is counter-based (word w =
//    mix(seed + (w+1)*gamma)), so the GPU computes 64 MiB blocks in HBM and
//    the host only writes them out (double-buffered pinned copies).
//  * Store handle: open validates magic, version and exact file length like
//    Store::Store (store.cpp:84-117); read_one/read_chunk are positional
//    reads (store.cpp:123-148), safe for concurrent use.
//  * Reads into HBM: a set of sample ids is sorted and cut into chunk reads
//    of span <= threshold (the plan_chunks rule, chunking.cpp:9-33), the
//    reads run as parallel pread()s from a host thread pool into pinned
//    staging, one async H2D moves the staging to HBM and a scatter kernel
//    puts every sample's bytes into its destination row(s).
//  * Step fetch with misses from the Store: hits are gathered from the HBM
//    buffer (K8); the step's misses (replay slots without the hit bit) are
//    read from the file and scattered into the batch rows and, unless the
//    replay bypassed them, into their new buffer slots — the same bytes
//    Store::read_one returns.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

struct lsg_store {
    int fd = -1;
    uint16_t version = 1;
    uint64_t count = 0, size = 0;
    // staging, grown on demand and reused across calls
    unsigned char* h_stage = nullptr;  // pinned
    size_t h_cap = 0;
    unsigned char* d_stage = nullptr;
    size_t d_cap = 0;
    void* h_meta = nullptr;  // pinned scatter descriptors
    size_t h_meta_cap = 0;
    void* d_meta = nullptr;
    size_t d_meta_cap = 0;
    cudaEvent_t done = nullptr;  // the last call's scatter (it reads d_stage / d_meta) finished
    unsigned threads = 8;
    std::mutex mu;               // one call at a time owns the staging (the handle is shared by threads)
};

namespace lsg {

int gather_step_hits_device(void* const* d_bufs, void* const* d_outs, const uint32_t* d_slots,
                            const uint32_t* d_node_off, uint32_t k0, uint32_t k1, uint64_t rows_hint,
                            uint64_t sample_bytes, cudaStream_t st);

namespace {

constexpr uint64_t kHeader = 22;  // kStoreHeaderBytes (store.hpp:23)
constexpr char kMagic[4] = {'S', 'L', 'R', 'D'};

__global__ void k_payload_block(uint64_t seed, uint64_t word0, uint64_t nwords, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nwords;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = mix64(seed + (word0 + i + 1) * kGamma);
}

// one destination of a staged sample: bytes [src, src + size) of the staging
// go to dst (and to dst2 when not null)
struct Scatter {
    unsigned long long src;
    unsigned char* dst;
    unsigned char* dst2;
};

__global__ void __launch_bounds__(256) k_scatter_rows(const unsigned char* __restrict__ stage,
                                                      const Scatter* __restrict__ sc, uint64_t n,
                                                      uint64_t size) {
    for (uint64_t r = blockIdx.y; r < n; r += gridDim.y) {
        const Scatter s = sc[r];
        const unsigned char* src = stage + s.src;
        const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(s.dst) |
                           reinterpret_cast<uintptr_t>(s.dst2) | size) & 15) == 0;
        if (vec) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
            uint4* d4 = reinterpret_cast<uint4*>(s.dst);
            uint4* e4 = reinterpret_cast<uint4*>(s.dst2);
            for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < size / 16;
                 i += uint64_t(gridDim.x) * blockDim.x) {
                const uint4 v = __ldcs(&s4[i]);
                __stcs(&d4[i], v);
                if (e4) __stcs(&e4[i], v);
            }
        } else {
            for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < size;
                 i += uint64_t(gridDim.x) * blockDim.x) {
                const unsigned char v = src[i];
                s.dst[i] = v;
                if (s.dst2) s.dst2[i] = v;
            }
        }
    }
}

int pread_all(int fd, void* dst, size_t bytes, uint64_t off) {
    char* p = static_cast<char*>(dst);
    while (bytes > 0) {
        const ssize_t n = ::pread(fd, p, bytes, off_t(off));
        if (n <= 0) return kStorage;
        p += n;
        bytes -= size_t(n);
        off += uint64_t(n);
    }
    return kOk;
}

int grow_pinned(void*& p, size_t& cap, size_t want) {
    if (want <= cap) return kOk;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t c = std::max<size_t>(want, size_t(1) << 20);
    LSG_CUDA(cudaHostAlloc(&p, c, cudaHostAllocDefault));
    cap = c;
    return kOk;
}

int grow_device(void*& p, size_t& cap, size_t want) {
    if (want <= cap) return kOk;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t c = std::max<size_t>(want, size_t(1) << 20);
    LSG_CUDA(cudaMalloc(&p, c));
    cap = c;
    return kOk;
}

struct Want {   // one requested sample
    uint32_t id;
    uint32_t row;  // index into the caller's destination list
};

// Read the samples `w` (any order, repeats allowed) into HBM: sorted, cut
// into reads of span <= thr (chunking.cpp:9-33), pread in parallel into the
// pinned staging, one H2D, then a scatter to dst[row] (and dst2[row]).
int read_into_device(lsg_store* h, std::vector<Want>& w, uint64_t thr, unsigned char* const* dst,
                     unsigned char* const* dst2, cudaStream_t st) {
    if (w.empty()) return kOk;
    std::sort(w.begin(), w.end(), [](const Want& a, const Want& b) { return a.id < b.id || (a.id == b.id && a.row < b.row); });
    struct Range {
        uint64_t start, count, stage_off;
    };
    std::vector<Range> ranges;
    std::vector<uint64_t> src(w.size());
    uint64_t stage_bytes = 0;
    size_t i = 0;
    while (i < w.size()) {
        const uint64_t start = w[i].id;
        size_t j = i + 1;
        while (j < w.size() && uint64_t(w[j].id) - start + 1 <= thr) ++j;
        const uint64_t count = uint64_t(w[j - 1].id) - start + 1;
        ranges.push_back({start, count, stage_bytes});
        for (size_t q = i; q < j; ++q) src[q] = stage_bytes + (uint64_t(w[q].id) - start) * h->size;
        stage_bytes += count * h->size;
        i = j;
    }
    // the staging belongs to one call at a time, and the previous call's H2D
    // copies and scatter (on whatever stream) must be done before it is reused
    std::lock_guard<std::mutex> lock(h->mu);
    if (h->done) LSG_CUDA(cudaEventSynchronize(h->done));
    void* hs = h->h_stage;
    if (int rc = grow_pinned(hs, h->h_cap, stage_bytes)) return rc;
    h->h_stage = static_cast<unsigned char*>(hs);
    void* ds = h->d_stage;
    if (int rc = grow_device(ds, h->d_cap, stage_bytes)) return rc;
    h->d_stage = static_cast<unsigned char*>(ds);
    // parallel positional reads (Store is documented safe for concurrent
    // reads, store.hpp:29-30); reads are dealt to threads by byte volume
    const unsigned nt = unsigned(std::min<size_t>(h->threads, ranges.size()));
    std::atomic<int> err{kOk};
    std::atomic<size_t> next{0};
    auto work = [&]() {
        for (;;) {
            const size_t r = next.fetch_add(1);
            if (r >= ranges.size()) return;
            const Range& g = ranges[r];
            if (pread_all(h->fd, h->h_stage + g.stage_off, g.count * h->size, kHeader + g.start * h->size))
                err.store(kStorage);
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (std::thread& t : pool) t.join();
    if (err.load()) return set_error(kStorage, "store: read failed");
    // scatter descriptors
    const size_t mbytes = w.size() * sizeof(Scatter);
    if (int rc = grow_pinned(h->h_meta, h->h_meta_cap, mbytes)) return rc;
    if (int rc = grow_device(h->d_meta, h->d_meta_cap, mbytes)) return rc;
    Scatter* sc = static_cast<Scatter*>(h->h_meta);
    for (size_t q = 0; q < w.size(); ++q)
        sc[q] = {src[q], dst[w[q].row], dst2 ? dst2[w[q].row] : nullptr};
    LSG_CUDA(cudaMemcpyAsync(h->d_stage, h->h_stage, stage_bytes, cudaMemcpyHostToDevice, st));
    LSG_CUDA(cudaMemcpyAsync(h->d_meta, h->h_meta, mbytes, cudaMemcpyHostToDevice, st));
    dim3 grid(unsigned(std::min<uint64_t>(std::max<uint64_t>(h->size / 4096, 1), 64)),
              unsigned(std::min<uint64_t>(w.size(), 4096)));
    k_scatter_rows<<<grid, 256, 0, st>>>(h->d_stage, static_cast<const Scatter*>(h->d_meta), w.size(), h->size);
    LSG_LAUNCH_CHECK("k_scatter_rows");
    if (!h->done) LSG_CUDA(cudaEventCreateWithFlags(&h->done, cudaEventDisableTiming));
    LSG_CUDA(cudaEventRecord(h->done, st));
    return kOk;
}

}  // namespace
}  // namespace lsg

using namespace lsg;

extern "C" {

// create_store(path, count, size, fill_seed, max_bytes) (store.cpp:37-82)
int lsg_store_create(const char* path, uint64_t count, uint64_t size, uint64_t fill_seed, uint64_t max_bytes,
                     void* stream) {
    if (!path) return set_error(kValidation, "create_store: null path");
    if (count == 0 || size == 0) return set_error(kStorage, "create_store: sample_count and sample_size must be >= 1");
    const uint64_t payload = count * size;
    if (payload / size != count) return set_error(kStorage, "create_store: size overflow");
    if (kHeader + payload > max_bytes) return set_error(kStorage, "create_store: store exceeds disk budget");
    const int fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) return set_error(kStorage, std::string("create_store: cannot open ") + path);
    auto write_all = [&](const void* data, size_t bytes) -> bool {
        const char* p = static_cast<const char*>(data);
        while (bytes > 0) {
            const ssize_t n = ::write(fd, p, bytes);
            if (n <= 0) return false;
            p += n;
            bytes -= size_t(n);
        }
        return true;
    };
    unsigned char hdr[kHeader];
    std::memcpy(hdr, kMagic, 4);
    hdr[4] = 1;
    hdr[5] = 0;
    for (int i = 0; i < 8; ++i) hdr[6 + i] = uint8_t(count >> (8 * i));
    for (int i = 0; i < 8; ++i) hdr[14 + i] = uint8_t(size >> (8 * i));
    if (!write_all(hdr, kHeader)) {
        ::close(fd);
        return set_error(kStorage, std::string("create_store: write failed for ") + path);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t kBlock = 64ull << 20;  // bytes per block (multiple of 8)
    const uint64_t nblk = (payload + kBlock - 1) / kBlock;
    uint64_t* d = nullptr;
    unsigned char* hb[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int rc = kOk;
    auto cleanup = [&]() {
        if (d) cudaFree(d);
        for (int q = 0; q < 2; ++q) {
            if (hb[q]) cudaFreeHost(hb[q]);
            if (ev[q]) cudaEventDestroy(ev[q]);
        }
        ::close(fd);
    };
    const uint64_t blk = std::min(kBlock, payload);
    if (cudaMalloc(&d, 2 * ((blk + 7) / 8) * 8) != cudaSuccess || cudaHostAlloc(&hb[0], blk + 8, 0) != cudaSuccess ||
        cudaHostAlloc(&hb[1], blk + 8, 0) != cudaSuccess || cudaEventCreate(&ev[0]) != cudaSuccess ||
        cudaEventCreate(&ev[1]) != cudaSuccess) {
        cleanup();
        return set_error(kInternal, "create_store: staging allocation failed");
    }
    // block b is computed into device half b%2, copied to host buffer b%2,
    // and written while block b+1 is computed and copied
    for (uint64_t b = 0; b <= nblk && rc == kOk; ++b) {
        if (b < nblk) {
            const uint64_t bytes = std::min(kBlock, payload - b * kBlock);
            const uint64_t words = (bytes + 7) / 8;
            uint64_t* dd = d + (b & 1) * ((blk + 7) / 8);
            k_payload_block<<<grid_for(words, 256, 148 * 8), 256, 0, st>>>(fill_seed, b * (kBlock / 8), words, dd);
            if (cudaGetLastError() != cudaSuccess ||
                cudaMemcpyAsync(hb[b & 1], dd, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaEventRecord(ev[b & 1], st) != cudaSuccess)
                rc = set_error(kInternal, "create_store: payload kernel failed");
            count_launch();
        }
        if (b > 0 && rc == kOk) {
            const uint64_t p = b - 1;
            const uint64_t bytes = std::min(kBlock, payload - p * kBlock);
            if (cudaEventSynchronize(ev[p & 1]) != cudaSuccess) rc = set_error(kInternal, "create_store: copy failed");
            else if (!write_all(hb[p & 1], size_t(bytes)))
                rc = set_error(kStorage, std::string("create_store: write failed for ") + path);
        }
    }
    cleanup();
    return rc;
}

// Store::Store (store.cpp:84-117)
int lsg_store_open(const char* path, lsg_store** out) {
    if (!path || !out) return set_error(kValidation, "store: null argument");
    *out = nullptr;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return set_error(kStorage, std::string("store: cannot open ") + path);
    unsigned char raw[kHeader];
    if (pread_all(fd, raw, kHeader, 0)) {
        ::close(fd);
        return set_error(kStorage, "store: read failed");
    }
    if (std::memcmp(raw, kMagic, 4) != 0) {
        ::close(fd);
        return set_error(kStorage, std::string("store: bad magic in ") + path);
    }
    const uint16_t version = uint16_t(raw[4] | (raw[5] << 8));
    if (version != 1) {
        ::close(fd);
        return set_error(kStorage, std::string("store: unsupported version in ") + path);
    }
    uint64_t count = 0, size = 0;
    for (int i = 0; i < 8; ++i) count |= uint64_t(raw[6 + i]) << (8 * i);
    for (int i = 0; i < 8; ++i) size |= uint64_t(raw[14 + i]) << (8 * i);
    struct stat sb{};
    if (::fstat(fd, &sb) != 0) {
        ::close(fd);
        return set_error(kStorage, std::string("store: fstat failed for ") + path);
    }
    if (uint64_t(sb.st_size) != kHeader + count * size) {
        ::close(fd);
        return set_error(kStorage, std::string("store: file length does not match header in ") + path);
    }
    lsg_store* h = new lsg_store;
    h->fd = fd;
    h->version = version;
    h->count = count;
    h->size = size;
    h->threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    *out = h;
    return kOk;
}

int lsg_store_info(const lsg_store* h, uint64_t* count, uint64_t* size) {
    if (!h) return set_error(kValidation, "store: null handle");
    if (count) *count = h->count;
    if (size) *size = h->size;
    return kOk;
}

void lsg_store_close(lsg_store* h) {
    if (!h) return;
    if (h->done) {
        cudaEventSynchronize(h->done);
        cudaEventDestroy(h->done);
    }
    if (h->h_stage) cudaFreeHost(h->h_stage);
    if (h->d_stage) cudaFree(h->d_stage);
    if (h->h_meta) cudaFreeHost(h->h_meta);
    if (h->d_meta) cudaFree(h->d_meta);
    if (h->fd >= 0) ::close(h->fd);
    delete h;
}

// Store::read_chunk (store.cpp:141-148); read_one is count == 1
int lsg_store_read(const lsg_store* h, uint64_t start, uint64_t count, void* h_dst) {
    if (!h || !h_dst) return set_error(kValidation, "store: null argument");
    if (count == 0) return set_error(kValidation, "store: read_chunk count must be >= 1");
    if (start >= h->count || count > h->count - start)
        return set_error(count == 1 ? kValidation : kValidation,
                         count == 1 ? "store: sample index out of range" : "store: chunk range out of range");
    if (pread_all(h->fd, h_dst, count * h->size, kHeader + start * h->size))
        return set_error(kStorage, "store: read failed");
    return kOk;
}

// Samples ids[0..n) (host array) into device rows d_rows[r] (row pitch =
// sample size), read as chunk reads of span <= threshold.
int lsg_store_read_rows(lsg_store* h, const uint32_t* h_ids, uint64_t n, uint64_t threshold, void* d_rows,
                        void* stream) {
    if (!h || (!h_ids && n)) return set_error(kValidation, "store: null argument");
    if (threshold == 0) return set_error(kValidation, "store: threshold must be >= 1");
    std::vector<Want> w(n);
    std::vector<unsigned char*> dst(n);
    for (uint64_t r = 0; r < n; ++r) {
        if (h_ids[r] >= h->count) return set_error(kValidation, "store: sample index out of range");
        w[r] = {h_ids[r], uint32_t(r)};
        dst[r] = static_cast<unsigned char*>(d_rows) + r * h->size;
    }
    return read_into_device(h, w, threshold, dst.data(), nullptr, static_cast<cudaStream_t>(stream));
}

// One training step's loading phase for nodes [node_begin, node_end) with
// the misses read from the Store: hits gathered from the HBM buffers (one
// launch), then the miss rows read from the file and scattered into the
// batch rows and their new buffer slots (layout as lsg_fetch_step; h_bufs /
// h_outs are HOST arrays of the same device pointers).
int lsg_fetch_step_store(lsg_store* h, void* const* d_bufs, void* const* d_outs, void* const* h_bufs,
                         void* const* h_outs, const uint32_t* d_items, const uint32_t* d_slots,
                         const uint32_t* d_node_off, uint32_t node_begin, uint32_t node_end, uint64_t rows_hint,
                         uint64_t threshold, void* stream) {
    if (!h) return set_error(kValidation, "store: null handle");
    if (node_end <= node_begin) return kOk;
    if (threshold == 0) return set_error(kValidation, "store: threshold must be >= 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int rc = gather_step_hits_device(d_bufs, d_outs, d_slots, d_node_off, node_begin, node_end, rows_hint,
                                         h->size, st))
        return rc;
    const uint32_t nk = node_end - node_begin;
    std::vector<uint32_t> off(nk + 1);
    LSG_CUDA(cudaMemcpyAsync(off.data(), d_node_off + node_begin, (nk + 1) * 4, cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    const uint32_t r0 = off[0], rows = off[nk] - off[0];
    std::vector<uint32_t> ids(rows), slots(rows);
    if (rows) {
        LSG_CUDA(cudaMemcpyAsync(ids.data(), d_items + r0, rows * 4, cudaMemcpyDeviceToHost, st));
        LSG_CUDA(cudaMemcpyAsync(slots.data(), d_slots + r0, rows * 4, cudaMemcpyDeviceToHost, st));
        LSG_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<Want> w;
    std::vector<unsigned char*> dst, dst2;
    uint32_t k = 0;
    for (uint32_t r = 0; r < rows; ++r) {
        while (k + 1 < nk && off[k + 1] - r0 <= r) ++k;
        const uint32_t sl = slots[r];
        if (sl != kNever && (sl & kHit)) continue;  // a hit: gathered above
        const uint32_t x = ids[r] & ~kHit;
        if (x >= h->count) return set_error(kValidation, "store: sample index out of range");
        w.push_back({x, uint32_t(dst.size())});
        dst.push_back(static_cast<unsigned char*>(h_outs[k]) + uint64_t(r - (off[k] - r0)) * h->size);
        dst2.push_back(sl == kNever ? nullptr : static_cast<unsigned char*>(h_bufs[k]) + uint64_t(sl) * h->size);
    }
    return read_into_device(h, w, threshold, dst.data(), dst2.data(), st);
}

}  // extern "C"

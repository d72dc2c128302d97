// parse.cu — readers of the text artifacts: read_trace (trace.cpp:103-147),
// read_graph (reuse_graph.cpp:114-128) and read_plan (plan.cpp:85-214),
// host C++ behind the C ABI. They accept exactly what the reference accepts
// and reject with the same error class and message: the reference reads
// with std::getline + istringstream, so integers follow its num_get rules
// (leading blanks, optional sign, digits up to the first non-digit; an
// unsigned 32-bit field rejects values above 2^32-1) and std::stoull where
// the reference calls it. Results come back in the flat layout of the
// device path (lsg_plan_out), so a parsed plan feeds lsg_simulate directly.
#include <algorithm>
#include <cctype>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace lsg {
namespace {

struct PErr {
    int code;
    std::string msg;
};

// ---- std::istream >> unsigned integer, on a cursor over one line ---------
struct Cursor {
    const char* p;
    const char* e;
    bool fail = false;
    void skip_ws() {
        while (p < e && std::isspace(static_cast<unsigned char>(*p))) ++p;
    }
    // num_get for unsigned long (strtoull rules: optional sign, a leading '-'
    // negates modulo 2^64); max = the target type's maximum
    bool get_u(unsigned long long& v, unsigned long long max) {
        if (fail) return false;
        skip_ws();
        bool neg = false;
        if (p < e && (*p == '+' || *p == '-')) {
            neg = *p == '-';
            ++p;
        }
        if (p >= e || !std::isdigit(static_cast<unsigned char>(*p))) {
            fail = true;
            v = 0;
            return false;
        }
        unsigned long long x = 0;
        bool over = false;
        while (p < e && std::isdigit(static_cast<unsigned char>(*p))) {
            const unsigned d = unsigned(*p - '0');
            if (x > (~0ull - d) / 10) over = true;
            x = x * 10 + d;
            ++p;
        }
        if (over) {
            fail = true;
            v = ~0ull;
            return false;
        }
        if (neg) x = 0ull - x;
        if (x > max) {
            fail = true;
            v = max;
            return false;
        }
        v = x;
        return true;
    }
    bool get_str(std::string& s) {
        if (fail) return false;
        skip_ws();
        const char* b = p;
        while (p < e && !std::isspace(static_cast<unsigned char>(*p))) ++p;
        if (p == b) {
            fail = true;
            return false;
        }
        s.assign(b, p);
        return true;
    }
};

// std::stoull(text) as the reference calls it: leading blanks, sign, digits;
// invalid_argument / out_of_range are not loadsched errors (exit 7 in the
// CLI, tools/loadsched.cpp:366-372)
bool stoull_ref(const std::string& t, unsigned long long& v, size_t* pos) {
    Cursor c{t.data(), t.data() + t.size()};
    if (!c.get_u(v, ~0ull)) return false;
    if (pos) *pos = size_t(c.p - t.data());
    return true;
}

// next line (std::getline: up to '\n', which is dropped)
bool getline_(const char*& p, const char* end, std::string& line) {
    if (p >= end) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
    const char* le = nl ? nl : end;
    line.assign(p, le);
    p = nl ? nl + 1 : end;
    return true;
}

// ---- read_trace --------------------------------------------------------
struct TraceParsed {
    uint64_t D = 0, b = 0, seed = 0;
    uint32_t E = 0, N = 0;
    bool drop_last = true;
    std::vector<std::vector<uint64_t>> epochs;
};

PErr parse_trace(const char* text, uint64_t len, TraceParsed& t) {
    const char* p = text;
    const char* end = text + len;
    std::string line;
    if (!getline_(p, end, line) || line != "loadsched-trace 1")
        return {kValidation, "trace file: missing 'loadsched-trace 1' header"};
    auto parse_u64 = [](const std::string& s, const std::string& what, uint64_t& v) -> PErr {
        unsigned long long x = 0;
        size_t pos = 0;
        if (!stoull_ref(s, x, &pos) || pos != s.size())
            return {kValidation, "trace file: bad integer for " + what + ": '" + s + "'"};
        v = x;
        return {kOk, ""};
    };
    std::vector<uint64_t>* current = nullptr;
    while (getline_(p, end, line)) {
        if (line.empty()) continue;
        if (line.rfind("epoch ", 0) == 0) {
            uint64_t index = 0;
            PErr e = parse_u64(line.substr(6), "epoch header", index);
            if (e.code) return e;
            if (index != t.epochs.size()) return {kValidation, "trace file: epoch headers out of order"};
            t.epochs.emplace_back();
            current = &t.epochs.back();
            continue;
        }
        const size_t eq = line.find('=');
        if (eq != std::string::npos && current == nullptr) {
            const std::string key = line.substr(0, eq), value = line.substr(eq + 1);
            uint64_t v = 0;
            PErr e = parse_u64(value, key, v);
            if (e.code) return e;
            if (key == "dataset_size") t.D = v;
            else if (key == "num_epochs") t.E = uint32_t(v);
            else if (key == "num_nodes") t.N = uint32_t(v);
            else if (key == "local_batch") t.b = v;
            else if (key == "seed") t.seed = v;
            else if (key == "drop_last") t.drop_last = v != 0;
            else return {kValidation, "trace file: unknown key '" + key + "'"};
            continue;
        }
        if (current == nullptr) return {kValidation, "trace file: sample id before first epoch header"};
        uint64_t id = 0;
        PErr e = parse_u64(line, "sample id", id);
        if (e.code) return e;
        current->push_back(id);
    }
    // TraceConfig::validate (trace.cpp:18-24)
    if (t.N == 0) return {kConfig, "num_nodes must be >= 1"};
    if (t.b == 0) return {kConfig, "local_batch must be >= 1"};
    if (t.E == 0) return {kConfig, "num_epochs must be >= 1"};
    const uint64_t B = uint64_t(t.N) * t.b;
    if (t.D < B) return {kConfig, "dataset_size must be >= num_nodes * local_batch"};
    if (t.epochs.size() != t.E) return {kValidation, "trace file: epoch count does not match num_epochs"};
    const uint64_t S = t.drop_last ? t.D / B : (t.D + B - 1) / B;
    const uint64_t expect = t.drop_last ? S * B : t.D;
    for (const auto& seq : t.epochs) {
        if (seq.size() != expect) return {kValidation, "trace file: epoch sequence length mismatch"};
        for (uint64_t id : seq)
            if (id >= t.D) return {kValidation, "trace file: sample id out of range"};
    }
    return {kOk, ""};
}

// ---- read_plan -----------------------------------------------------------
struct PlanRowA {  // assign
    uint32_t ep;   // epoch position
    uint64_t step;
    uint32_t node;
    uint64_t id;
    bool hit;
};
struct PlanRowR {  // read
    uint32_t ep;
    uint64_t step;
    uint32_t node;
    bool chunk;
    uint64_t start, end;
};
struct PlanRowB {
    uint32_t ep;
    uint64_t step;
    uint32_t node;
    uint64_t before, after;
};

}  // namespace
}  // namespace lsg

// parsed plan, flat (lsg.h lsg_plan_view)
struct lsg_parsed_plan {
    uint64_t D = 0, b = 0, thr = 0, cost = 0;
    uint32_t N = 0;
    std::vector<uint32_t> order, epoch_ids;
    std::vector<uint64_t> epoch_steps;
    std::vector<uint32_t> items, node_off;
    std::vector<uint64_t> fb, fa, read_off, read_start, read_end, needed, redundant;
    std::vector<uint8_t> read_chunk;
};

namespace lsg {
namespace {

PErr parse_plan(const char* text, uint64_t len, lsg_parsed_plan& pl) {
    const char* p = text;
    const char* end = text + len;
    std::string line;
    auto bad = [](const std::string& why) { return PErr{kValidation, "plan file: " + why}; };
    if (!getline_(p, end, line) || line != "loadsched-plan 1") return bad("missing 'loadsched-plan 1' header");
    bool have_meta = false, have_order = false, have_cost = false;
    std::vector<int64_t> epoch_pos;  // epoch id -> position
    std::vector<uint64_t> nsteps;    // per position
    auto epoch_slot = [&](uint32_t e) -> uint32_t {
        if (e >= epoch_pos.size()) epoch_pos.resize(size_t(e) + 1, -1);
        if (epoch_pos[e] < 0) {
            epoch_pos[e] = int64_t(pl.epoch_ids.size());
            pl.epoch_ids.push_back(e);
            nsteps.push_back(0);
        }
        return uint32_t(epoch_pos[e]);
    };
    std::vector<PlanRowA> as;
    std::vector<PlanRowR> rs;
    std::vector<PlanRowB> bs;
    const unsigned long long U32 = 0xFFFFFFFFull, U64 = ~0ull;
    while (getline_(p, end, line)) {
        if (line.empty()) continue;
        Cursor c{line.data(), line.data() + line.size()};
        std::string tag;
        c.get_str(tag);
        if (tag == "meta") {
            std::string kv;
            while (c.get_str(kv)) {
                const size_t eq = kv.find('=');
                if (eq == std::string::npos) return bad("meta entry without '=': " + kv);
                const std::string key = kv.substr(0, eq);
                unsigned long long v = 0;
                if (!stoull_ref(kv.substr(eq + 1), v, nullptr)) return {kInternal, "stoull"};
                if (key == "dataset_size") pl.D = v;
                else if (key == "nodes") pl.N = uint32_t(v);
                else if (key == "local_batch") pl.b = v;
                else if (key == "threshold") pl.thr = v;
                else return bad("unknown meta key: " + key);
            }
            if (pl.N == 0) return bad("meta missing nodes");
            have_meta = true;
        } else if (tag == "order:") {
            unsigned long long e = 0;
            while (c.get_u(e, U32)) pl.order.push_back(uint32_t(e));
            have_order = true;
        } else if (tag == "cost:") {
            unsigned long long v = 0;
            if (!c.get_u(v, U64)) return bad("bad cost line");
            pl.cost = v;
            have_cost = true;
        } else if (tag == "balance") {
            if (!have_meta) return bad("balance row before meta");
            unsigned long long e, s, k, bf, af;
            c.get_u(e, U32);
            c.get_u(s, U64);
            c.get_u(k, U32);
            c.get_u(bf, U64);
            c.get_u(af, U64);
            if (c.fail) return bad("bad balance row");
            if (k >= pl.N) return bad("balance row node out of range");
            const uint32_t ep = epoch_slot(uint32_t(e));
            nsteps[ep] = std::max<uint64_t>(nsteps[ep], s + 1);
            bs.push_back({ep, s, uint32_t(k), bf, af});
        } else if (tag == "assign") {
            if (!have_meta) return bad("assign row before meta");
            unsigned long long e, s, k, id;
            std::string src;
            c.get_u(e, U32);
            c.get_u(s, U64);
            c.get_u(k, U32);
            c.get_u(id, U64);
            c.get_str(src);
            if (c.fail) return bad("bad assign row");
            if (k >= pl.N) return bad("assign row node out of range");
            if (src != "hit" && src != "fetch") return bad("bad source tag: " + src);
            const uint32_t ep = epoch_slot(uint32_t(e));
            nsteps[ep] = std::max<uint64_t>(nsteps[ep], s + 1);
            as.push_back({ep, s, uint32_t(k), id, src == "hit"});
        } else if (tag == "read") {
            if (!have_meta) return bad("read row before meta");
            unsigned long long e, s, k, st, en;
            std::string kind;
            c.get_u(e, U32);
            c.get_u(s, U64);
            c.get_u(k, U32);
            c.get_str(kind);
            c.get_u(st, U64);
            c.get_u(en, U64);
            if (c.fail) return bad("bad read row");
            if (k >= pl.N) return bad("read row node out of range");
            if (kind != "single" && kind != "chunk") return bad("bad read kind: " + kind);
            if (en < st) return bad("read row end < start");
            const uint32_t ep = epoch_slot(uint32_t(e));
            nsteps[ep] = std::max<uint64_t>(nsteps[ep], s + 1);
            rs.push_back({ep, s, uint32_t(k), kind == "chunk", st, en});
        } else {
            return bad("unknown row tag: " + tag);
        }
    }
    if (!have_meta || !have_order || !have_cost) return bad("missing meta/order/cost");
    // flat layout: steps in epoch-position order, lists in file order
    const uint32_t N = pl.N;
    std::vector<uint64_t> sbase(nsteps.size() + 1, 0);
    for (size_t i = 0; i < nsteps.size(); ++i) sbase[i + 1] = sbase[i] + nsteps[i];
    const uint64_t T = sbase.back();
    pl.epoch_steps = nsteps;
    auto gk = [&](uint32_t ep, uint64_t s, uint32_t k) { return (sbase[ep] + s) * N + k; };
    // assign rows: stable counting sort by (step, node)
    std::vector<uint64_t> cnt(T * N + 1, 0);
    for (const PlanRowA& a : as) {
        if (a.id >= (1ull << 31)) return {kCapability, "plan file: sample ids must be < 2^31 on device"};
        cnt[gk(a.ep, a.step, a.node) + 1]++;
    }
    for (uint64_t i = 0; i < T * N; ++i) cnt[i + 1] += cnt[i];
    pl.items.assign(as.size(), 0);
    {
        std::vector<uint64_t> fill(cnt.begin(), cnt.end() - 1);
        for (const PlanRowA& a : as) pl.items[fill[gk(a.ep, a.step, a.node)]++] = uint32_t(a.id) | (a.hit ? kHit : 0u);
    }
    pl.node_off.assign(T * (N + 1), 0);
    for (uint64_t g = 0; g < T; ++g)
        for (uint32_t k = 0; k <= N; ++k) pl.node_off[g * (N + 1) + k] = uint32_t(cnt[g * N + k] - cnt[g * N]);
    pl.fb.assign(T * N, 0);
    pl.fa.assign(T * N, 0);
    for (const PlanRowB& b : bs) {
        pl.fb[gk(b.ep, b.step, b.node)] = b.before;
        pl.fa[gk(b.ep, b.step, b.node)] = b.after;
    }
    pl.read_off.assign(T * N + 1, 0);
    for (const PlanRowR& r : rs) pl.read_off[gk(r.ep, r.step, r.node) + 1]++;
    for (uint64_t i = 0; i < T * N; ++i) pl.read_off[i + 1] += pl.read_off[i];
    pl.read_start.assign(rs.size(), 0);
    pl.read_end.assign(rs.size(), 0);
    pl.read_chunk.assign(rs.size(), 0);
    {
        std::vector<uint64_t> fill(pl.read_off.begin(), pl.read_off.end() - 1);
        for (const PlanRowR& r : rs) {
            const uint64_t q = fill[gk(r.ep, r.step, r.node)]++;
            pl.read_start[q] = r.start;
            pl.read_end[q] = r.end;
            pl.read_chunk[q] = r.chunk;
        }
    }
    // needed / redundant re-derived from the rows (plan.cpp:188-206)
    pl.needed.assign(T * N, 0);
    pl.redundant.assign(T * N, 0);
    std::vector<uint64_t> fetch;
    for (uint64_t g = 0; g < T; ++g)
        for (uint32_t k = 0; k < N; ++k) {
            const uint64_t li = g * N + k;
            fetch.clear();
            for (uint64_t i = cnt[li]; i < cnt[li + 1]; ++i)
                if (!(pl.items[i] & kHit)) fetch.push_back(pl.items[i]);
            pl.needed[li] = fetch.size();
            uint64_t red = 0, chunk_needed = 0;
            std::sort(fetch.begin(), fetch.end());
            for (uint64_t q = pl.read_off[li]; q < pl.read_off[li + 1]; ++q)
                if (pl.read_chunk[q]) {
                    red += pl.read_end[q] - pl.read_start[q] + 1;
                    for (uint64_t id : fetch)
                        if (id >= pl.read_start[q] && id <= pl.read_end[q]) ++chunk_needed;
                }
            if (red < chunk_needed) return bad("read rows inconsistent with fetches");
            pl.redundant[li] = red - chunk_needed;
        }
    if (pl.order.size() != pl.epoch_ids.size()) return bad("order length != epoch count");
    for (size_t i = 0; i < pl.epoch_ids.size(); ++i)
        if (pl.epoch_ids[i] != pl.order[i]) return bad("epoch rows out of schedule order");
    return {kOk, ""};
}

}  // namespace
}  // namespace lsg

using namespace lsg;

extern "C" {

int lsg_parse_trace(const char* text, uint64_t len, lsg_trace_text* hdr, uint32_t* h_ids, uint64_t cap) {
    if (!text || !hdr) return set_error(kValidation, "parse_trace: null argument");
    TraceParsed t;
    PErr e = parse_trace(text, len, t);
    if (e.code) return set_error(e.code, e.msg);
    hdr->dataset_size = t.D;
    hdr->num_epochs = t.E;
    hdr->num_nodes = t.N;
    hdr->local_batch = t.b;
    hdr->seed = t.seed;
    hdr->drop_last = t.drop_last ? 1 : 0;
    hdr->keep = t.epochs.empty() ? 0 : t.epochs[0].size();
    if (t.D >= (1ull << 31)) return set_error(kCapability, "parse_trace: dataset_size must be < 2^31 on device");
    if (h_ids && cap >= uint64_t(t.E) * hdr->keep)
        for (uint32_t ep = 0; ep < t.E; ++ep)
            for (uint64_t i = 0; i < hdr->keep; ++i) h_ids[ep * hdr->keep + i] = uint32_t(t.epochs[ep][i]);
    return kOk;
}

int lsg_parse_graph(const char* text, uint64_t len, uint32_t* E, uint64_t* h_w, uint64_t cap) {
    if (!text || !E) return set_error(kValidation, "parse_graph: null argument");
    // operator>> over the whole stream (reuse_graph.cpp:114-128)
    Cursor c{text, text + len};
    unsigned long long e = 0;
    if (!c.get_u(e, ~0ull) || e == 0) return set_error(kValidation, "graph file: bad epoch count header");
    *E = uint32_t(e);
    const uint64_t n = uint64_t(uint32_t(e)) * uint32_t(e);
    std::vector<uint64_t> w(n);
    for (uint64_t i = 0; i < n; ++i) {
        unsigned long long v = 0;
        if (!c.get_u(v, ~0ull)) return set_error(kValidation, "graph file: truncated weight matrix");
        w[i] = v;
    }
    for (uint32_t u = 0; u < uint32_t(e); ++u)
        if (w[uint64_t(u) * uint32_t(e) + u] != 0) return set_error(kValidation, "graph file: nonzero diagonal");
    if (h_w && cap >= n) std::memcpy(h_w, w.data(), n * 8);
    return kOk;
}

int lsg_parse_plan(const char* text, uint64_t len, lsg_parsed_plan** out, lsg_plan_view* v) {
    if (!text || !out || !v) return set_error(kValidation, "parse_plan: null argument");
    *out = nullptr;
    std::unique_ptr<lsg_parsed_plan> pl(new lsg_parsed_plan);
    PErr e = parse_plan(text, len, *pl);
    if (e.code) return set_error(e.code, e.msg);
    v->dataset_size = pl->D;
    v->local_batch = pl->b;
    v->chunk_threshold = pl->thr;
    v->cost = pl->cost;
    v->num_nodes = pl->N;
    v->num_epochs = uint32_t(pl->epoch_ids.size());
    v->num_steps = pl->node_off.size() / (pl->N + 1);
    v->num_items = pl->items.size();
    v->num_reads = pl->read_start.size();
    v->order = pl->order.data();
    v->epoch_ids = pl->epoch_ids.data();
    v->epoch_steps = pl->epoch_steps.data();
    v->items = pl->items.data();
    v->node_off = pl->node_off.data();
    v->fetch_before = pl->fb.data();
    v->fetch_after = pl->fa.data();
    v->read_off = pl->read_off.data();
    v->read_start = pl->read_start.data();
    v->read_end = pl->read_end.data();
    v->read_chunk = pl->read_chunk.data();
    v->needed = pl->needed.data();
    v->redundant = pl->redundant.data();
    *out = pl.release();
    return kOk;
}

void lsg_free_plan(lsg_parsed_plan* p) { delete p; }

}  // extern "C"

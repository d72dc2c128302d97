// shim: the reference header store.hpp maps onto the B200 drop-in. The PFS
// access-pattern microbenchmark (store.hpp:52-79, store.cpp:160-235) is out
// of scope: its declarations live here for the test build
// only and tests/cpp/shim/out_of_scope.cpp throws CapabilityError for them.
#pragma once
#include "loadsched_gpu.hpp"

namespace loadsched {

enum class AccessPattern { Random, SequentialStride, ChunkCycle, FullChunk };

struct BenchRead {
    std::uint32_t proc = 0;
    std::uint64_t offset = 0;
    std::uint64_t bytes = 0;
};

struct BenchResult {
    AccessPattern pattern = AccessPattern::Random;
    std::uint32_t procs = 0;
    double seconds = 0.0;
    std::vector<BenchRead> reads;
};

BenchResult bench_pattern(const Store& store, AccessPattern pattern, std::uint32_t procs, std::uint64_t seed);
std::vector<BenchResult> bench_all_patterns(const Store& store, std::uint32_t procs, std::uint64_t seed);
const char* pattern_name(AccessPattern pattern);

}  // namespace loadsched

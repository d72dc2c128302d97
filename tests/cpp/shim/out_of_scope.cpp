// Test-only link shim: the reference symbols its suites name that are out of
// scope for the B200 drop-in (the PFS access-pattern benchmark,
// the ablation ladder, the run summary). Each throws CapabilityError; the
// TEST_CASEs that exercise them are excluded by name (LSG_DOCTEST_EXCLUDE,
// tests/test_gpu_reftests.py).
#include "loadsched/pipeline.hpp"
#include "loadsched/store.hpp"

namespace loadsched {

namespace {
[[noreturn]] void out_of_scope(const char* what) {
    throw CapabilityError(std::string(what) + " is out of scope for the B200 drop-in");
}
}  // namespace

BenchResult bench_pattern(const Store&, AccessPattern, std::uint32_t, std::uint64_t) { out_of_scope("bench_pattern"); }
std::vector<BenchResult> bench_all_patterns(const Store&, std::uint32_t, std::uint64_t) {
    out_of_scope("bench_all_patterns");
}
const char* pattern_name(AccessPattern) { out_of_scope("pattern_name"); }
// the configuration is still validated first (ConfigError, config.cpp:11-23)
std::vector<PassTotals> ablation_ladder(const PipelineConfig& c) {
    c.validate();
    out_of_scope("ablation_ladder");
}
std::string summary_text(const PipelineConfig& c) {
    c.validate();
    out_of_scope("summary_text");
}

}  // namespace loadsched

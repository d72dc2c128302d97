// shim: the reference header pipeline.hpp maps onto the B200 drop-in. The
// ablation ladder and the run summary (pipeline.hpp:65-72) are reporting, out
// of scope: declared here for the test build only;
// tests/cpp/shim/out_of_scope.cpp throws CapabilityError for them.
#pragma once
#include "loadsched_gpu.hpp"

namespace loadsched {

std::vector<PassTotals> ablation_ladder(const PipelineConfig& config);
std::string summary_text(const PipelineConfig& config);

}  // namespace loadsched

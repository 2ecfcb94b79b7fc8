// pipedp/sdp_pipeline.hpp -- S-DP pipeline drop-in (reference
// sdp_pipeline.hpp:62-84).
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "pipedp/analysis.hpp"
#include "pipedp/engine.hpp"
#include "pipedp/sdp.hpp"

namespace pipedp {

struct ConflictRunAnalysis {
  std::vector<std::pair<int, int>> runs;
  std::vector<int> run_lengths;
  int longest_run = 1;
};
ConflictRunAnalysis analyze_conflict_runs(const OffsetSet& offsets);

struct SdpRunConfig {
  Backend backend = Backend::lockstep;
  int worker_count = 1;
  bool collect_trace = true;
};

struct SdpPipelineResult {
  SolutionTable table;
  PipelineTrace trace;  // first_head = a_1, steps_executed = n + k - a_1 - 1
  ConflictReport conflicts;
};

SdpPipelineResult solve_sdp_pipeline(const SdpInstance& instance, const SdpRunConfig& config = {});

}  // namespace pipedp

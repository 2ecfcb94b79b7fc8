// pipedp/mcm_pipeline.hpp -- MCM pipeline drop-in (reference
// mcm_pipeline.hpp:88-109).  Both modes run on the GPU with the reference
// engine's exact lock-step semantics: same table, steps_executed and
// stall_iterations.
#pragma once

#include <cstdint>

#include "pipedp/analysis.hpp"
#include "pipedp/engine.hpp"
#include "pipedp/mcm.hpp"

namespace pipedp {

enum class McmMode : std::uint8_t { paper_literal, stall_on_hazard };

struct McmScheduleConfig {
  McmMode mode = McmMode::paper_literal;
  Backend backend = Backend::lockstep;
  int worker_count = 1;
  bool collect_trace = true;
};

struct McmPipelineResult {
  SolutionTable table;
  PipelineTrace trace;
  ConflictReport conflicts;
  HazardReport hazards;
};

McmPipelineResult solve_mcm_pipeline(const McmInstance& instance,
                                     const McmScheduleConfig& config = {});

}  // namespace pipedp

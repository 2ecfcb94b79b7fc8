// pipedp/mcm_pipeline.hpp -- MCM pipeline drop-in (reference
// mcm_pipeline.hpp:88-109).  Both modes run on the GPU with the reference
// engine's exact lock-step semantics: same table, steps_executed and
// stall_iterations.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

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

// Lemma 1/2 check on a trace (reference mcm_pipeline.hpp:115-126): substep-1
// reads, substep-2 reads and substep-4 writes touch distinct addresses across
// lanes at every head.  Declared for the reference's verify_mcm; the body is
// the reference's trace tool (mcm_pipeline.cpp:49-77), provided by the drop-in.
struct DistinctnessVerdict {
  bool substep1_reads_distinct = true;
  bool substep2_reads_distinct = true;
  bool substep4_writes_distinct = true;
  std::optional<ConflictGroup> counterexample;

  bool all_ok() const {
    return substep1_reads_distinct && substep2_reads_distinct && substep4_writes_distinct;
  }
};

DistinctnessVerdict verify_substep_distinctness(const PipelineTrace& trace);

/// Addresses of cells predicted to read a not-yet-final operand under the
/// paper-literal schedule (reference mcm_pipeline.hpp:128-131): cell (r,c) on
/// diagonal D is implicated iff some term j satisfies
/// lin(r,c) - lin(r+j,c) <= D - 2j.  lin(r,c) - lin(r+j,c) depends on D and j
/// only, so whole diagonals are in or out: O(n^2) for any n (the reference's
/// per-cell scan is O(n^3) and is what limits the CPU study to small n).
std::vector<std::int64_t> hazard_frontier(std::int64_t n);

/// Cells implicated by a paper-literal hazard report: the reading lane's own
/// cell, head - lane + 1.  Sorted, deduplicated (reference mcm_pipeline.cpp:96-103).
std::vector<std::int64_t> hazard_cells(const HazardReport& report);

}  // namespace pipedp

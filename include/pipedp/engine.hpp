// pipedp/engine.hpp -- the result types of the reference engine
// (engine.hpp:19-100) that the pipeline entry points return.  The lock-step
// simulator itself is replaced by GPU kernels; traces are not collected
// (PipelineTrace::collected == false, records empty), step counts are.
#pragma once

#include <cstdint>
#include <vector>

namespace pipedp {

struct HeadRange {
  std::int64_t first = 0;
  std::int64_t last = -1;

  std::int64_t count() const { return last < first ? 0 : last - first + 1; }
  bool contains(std::int64_t head) const { return head >= first && head <= last; }
};

enum class AccessKind : std::uint8_t { read, write };

struct AccessRecord {
  std::int64_t head = 0;
  int substep = 1;
  int lane = 1;
  AccessKind kind = AccessKind::read;
  std::int64_t address = 0;

  friend bool operator==(const AccessRecord&, const AccessRecord&) = default;
};

struct PipelineTrace {
  std::vector<AccessRecord> records;
  std::int64_t first_head = 0;
  std::int64_t steps_executed = 0;
  std::int64_t stall_iterations = 0;
  std::vector<std::int64_t> stall_heads;
  bool collected = true;
};

enum class Backend : std::uint8_t { lockstep, workers };  // kept for ABI; ignored on the GPU

}  // namespace pipedp

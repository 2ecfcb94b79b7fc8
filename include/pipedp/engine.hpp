// pipedp/engine.hpp -- the result and plan types of the reference engine
// (engine.hpp:19-100) that the pipeline entry points return and the
// reference's callers (commands.cpp, analysis.cpp, io.cpp) use.  The lock-step
// simulator itself is replaced by GPU kernels: with collect_trace the GPU
// lock-step kernels emit the access records themselves (canonical order,
// record_less), otherwise PipelineTrace::collected == false and records stay
// empty; step and stall counts are always filled.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <tuple>
#include <vector>

namespace pipedp {

struct HeadRange {
  std::int64_t first = 0;
  std::int64_t last = -1;

  std::int64_t count() const { return last < first ? 0 : last - first + 1; }
  bool contains(std::int64_t head) const { return head >= first && head <= last; }
};

inline constexpr int kMaxSubsteps = 4;
inline constexpr int kMaxReadsPerSubstep = 2;

// One lane's accesses in one substep (reference engine.hpp:30-35).
struct SubstepAccess {
  std::array<std::int64_t, kMaxReadsPerSubstep> reads{};
  int read_count = 0;
  std::int64_t write = -1;
};

// One lane's work at one head (reference engine.hpp:39-43).
struct LanePlan {
  std::array<SubstepAccess, kMaxSubsteps> sub{};
  int substep_count = 0;
  std::int64_t payload = 0;
};

using LaneScratch = std::array<std::int64_t, 4>;

enum class AccessKind : std::uint8_t { read, write };

struct AccessRecord {
  std::int64_t head = 0;
  int substep = 1;
  int lane = 1;
  AccessKind kind = AccessKind::read;
  std::int64_t address = 0;

  friend bool operator==(const AccessRecord&, const AccessRecord&) = default;
};

// Canonical record order (reference engine.hpp:61-66).
inline bool record_less(const AccessRecord& a, const AccessRecord& b) {
  return std::tuple(a.head, a.substep, a.lane, static_cast<int>(a.kind), a.address) <
         std::tuple(b.head, b.substep, b.lane, static_cast<int>(b.kind), b.address);
}

struct PipelineTrace {
  std::vector<AccessRecord> records;
  std::int64_t first_head = 0;
  std::int64_t steps_executed = 0;
  std::int64_t stall_iterations = 0;
  std::vector<std::int64_t> stall_heads;
  bool collected = true;

  void canonicalize() { std::sort(records.begin(), records.end(), record_less); }
};

enum class Backend : std::uint8_t { lockstep, workers };  // kept for ABI; ignored on the GPU

}  // namespace pipedp

// pipedp_dropin.cpp -- the reference's C++ solver entry points (namespace
// pipedp, include/pipedp/*.hpp) implemented over the C ABI of
// include/pipedp_cuda.h.  Same signatures, same validation order and errc,
// same returned values; the tables come from the sm_100a kernels.  A C ABI
// status >= 100 (no GPU, CUDA error) becomes pipedp::DeviceError -- there is no
// CPU solver behind these functions.
#include <algorithm>
#include <cstdio>
#include <map>
#include <string>
#include <tuple>

#include "pipedp/error.hpp"
#include "pipedp/generate.hpp"
#include "pipedp/mcm.hpp"
#include "pipedp/mcm_pipeline.hpp"
#include "pipedp/sdp.hpp"
#include "pipedp/sdp_pipeline.hpp"
#include "pipedp/semigroup.hpp"
#include "pipedp/table.hpp"
#include "pipedp_cuda.h"

namespace pipedp {

namespace {

void check(int32_t status) {
  if (status == PIPEDP_OK) return;
  std::string msg = pipedp_last_error();
  if (status >= 1 && status <= 11) {
    // strip the "Name: " prefix the C layer adds; Error re-adds it
    const auto colon = msg.find(": ");
    throw Error(static_cast<errc>(status - 1), colon == std::string::npos ? msg : msg.substr(colon + 2));
  }
  throw DeviceError(status, msg);
}

SolutionTable full_table(std::int64_t size) {
  SolutionTable t;
  t.cells.assign(static_cast<std::size_t>(size), 0);
  t.filled.assign(static_cast<std::size_t>(size), 1);
  return t;
}

std::int64_t ceil_log2(std::int64_t k) {  // sdp.cpp:78-80
  std::int64_t r = 0;
  while ((std::int64_t{1} << r) < k) ++r;
  return r;
}

// The device records of one engine run -> the reference's trace/report types.
constexpr std::int64_t kTraceLimit = std::int64_t(1) << 28;  // pipedp_engine: records per trace

struct EngineRun {
  pipedp_engine_t run = nullptr;
  pipedp_engine_summary sum{};
  ~EngineRun() { pipedp_engine_free(run); }
};

void fill_trace(EngineRun& e, bool collected, PipelineTrace& t) {
  t.first_head = e.sum.first_head;
  t.steps_executed = e.sum.steps_executed;
  t.stall_iterations = e.sum.stall_iterations;
  t.collected = collected;
  t.stall_heads.assign(static_cast<std::size_t>(e.sum.stall_heads), 0);
  check(pipedp_engine_stall_heads(e.run, t.stall_heads.data()));
  const std::size_t nr = static_cast<std::size_t>(e.sum.records);
  if (!nr) return;
  std::vector<std::int64_t> head(nr), addr(nr);
  std::vector<std::int32_t> sub(nr), lane(nr), kind(nr);
  check(pipedp_engine_records(e.run, head.data(), sub.data(), lane.data(), kind.data(), addr.data()));
  t.records.resize(nr);
  for (std::size_t i = 0; i < nr; ++i)
    t.records[i] = AccessRecord{head[i], sub[i], lane[i], kind[i] ? AccessKind::write : AccessKind::read, addr[i]};
}

ConflictReport conflicts_of(EngineRun& e) {
  ConflictReport c;
  c.first_head = e.sum.first_head;
  c.max_group_size = static_cast<int>(e.sum.max_group_size);
  const std::size_t g = static_cast<std::size_t>(e.sum.conflict_groups);
  std::vector<std::int64_t> groups(4 * g);
  std::vector<std::int32_t> sizes(g), lanes(static_cast<std::size_t>(e.sum.conflict_lanes));
  c.per_step_cost.assign(static_cast<std::size_t>(std::max<std::int64_t>(e.sum.steps_executed, 0)), 1);
  check(pipedp_engine_conflicts(e.run, groups.data(), sizes.data(), lanes.data(), c.per_step_cost.data()));
  std::size_t at = 0;
  for (std::size_t i = 0; i < g; ++i) {
    ConflictGroup cg;
    cg.head = groups[4 * i];
    cg.substep = static_cast<int>(groups[4 * i + 1]);
    cg.kind = groups[4 * i + 2] ? AccessKind::write : AccessKind::read;
    cg.address = groups[4 * i + 3];
    cg.lanes.assign(lanes.begin() + static_cast<std::ptrdiff_t>(at),
                    lanes.begin() + static_cast<std::ptrdiff_t>(at + sizes[i]));
    at += static_cast<std::size_t>(sizes[i]);
    c.groups.push_back(std::move(cg));
  }
  return c;
}

HazardReport hazards_of(EngineRun& e) {
  HazardReport h;
  const std::size_t nh = static_cast<std::size_t>(e.sum.hazards);
  std::vector<std::int64_t> v(6 * nh);
  check(pipedp_engine_hazards(e.run, v.data()));
  h.hazards.resize(nh);
  for (std::size_t i = 0; i < nh; ++i)
    h.hazards[i] = HazardRecord{v[6 * i], static_cast<int>(v[6 * i + 1]), static_cast<int>(v[6 * i + 2]),
                                v[6 * i + 3], v[6 * i + 4], static_cast<int>(v[6 * i + 5])};
  return h;
}

}  // namespace

// ------------------------------------------------------------------ L0 ---
const char* errc_name(errc code) {
  static const char* names[] = {"NonDecreasingOffsets", "NonPositiveOffset", "InitLengthMismatch",
                                "TableTooSmall",        "CoordOutOfRange",   "AddressOutOfRange",
                                "BaseCellHasNoDeps",    "TooLargeForBruteForce",
                                "StallLivelock",        "WeightOverflow",    "InvalidParams"};
  const int i = static_cast<int>(code);
  return i >= 0 && i < 11 ? names[i] : "UnknownError";
}

std::int64_t SemigroupOp::apply(std::int64_t a, std::int64_t b) const {
  switch (kind) {
    case OpKind::min:
      return std::min(a, b);
    case OpKind::max:
      return std::max(a, b);
    case OpKind::saturating_add: {
      std::int64_t out;
      if (__builtin_add_overflow(a, b, &out)) return b > 0 ? INT64_MAX : INT64_MIN;
      return out;
    }
    case OpKind::modular_add: {
      auto norm = [](std::int64_t v) {
        const std::int64_t r = v % kModulus;
        return r < 0 ? r + kModulus : r;
      };
      return (norm(a) + norm(b)) % kModulus;
    }
  }
  fail(errc::invalid_params, "unknown operator kind");
}

std::string_view SemigroupOp::name() const {
  switch (kind) {
    case OpKind::min: return "min";
    case OpKind::max: return "max";
    case OpKind::saturating_add: return "saturating-add";
    case OpKind::modular_add: return "modular-add";
  }
  return "?";
}

SemigroupOp SemigroupOp::from_name(std::string_view name) {
  for (const SemigroupOp& op : catalog())
    if (op.name() == name) return op;
  fail(errc::invalid_params, "unknown operator name: " + std::string(name));
}

const std::array<SemigroupOp, 4>& SemigroupOp::catalog() {
  static const std::array<SemigroupOp, 4> ops = {SemigroupOp{OpKind::min}, SemigroupOp{OpKind::max},
                                                 SemigroupOp{OpKind::saturating_add},
                                                 SemigroupOp{OpKind::modular_add}};
  return ops;
}

bool SolutionTable::all_filled() const {
  return std::all_of(filled.begin(), filled.end(), [](std::uint8_t f) { return f != 0; });
}

std::uint64_t table_digest(const SolutionTable& table) {
  return pipedp_table_digest(table.cells.data(), static_cast<std::int64_t>(table.cells.size()));
}

std::string digest_hex(std::uint64_t digest) {
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(digest));
  return buf;
}

// ----------------------------------------------------------------- S-DP ---
const SdpInstance& validate(const SdpInstance& inst) {
  check(pipedp_sdp_validate(inst.offsets.offsets.data(), inst.offsets.k(),
                            static_cast<std::int64_t>(inst.init.size()), inst.n));
  return inst;
}

SolutionTable initial_table(const SdpInstance& inst) {  // sdp.cpp:34-41
  SolutionTable table(inst.n);
  for (std::size_t i = 0; i < inst.init.size(); ++i) {
    table.cells[i] = inst.init[i];
    table.filled[i] = 1;
  }
  return table;
}

SolutionTable solve_sequential(const SdpInstance& inst) {
  validate(inst);
  SolutionTable t = full_table(inst.n);
  check(pipedp_sdp_solve(inst.offsets.offsets.data(), inst.offsets.k(), inst.init.data(),
                         static_cast<std::int64_t>(inst.init.size()), inst.n,
                         static_cast<int32_t>(inst.op.kind), t.cells.data(), nullptr));
  return t;
}

namespace {
SolutionTable solve_method(const SdpInstance& inst, int32_t method) {
  validate(inst);
  SolutionTable t = full_table(inst.n);
  check(pipedp_sdp_solve_method(inst.offsets.offsets.data(), inst.offsets.k(), inst.init.data(),
                                static_cast<std::int64_t>(inst.init.size()), inst.n,
                                static_cast<int32_t>(inst.op.kind), method, t.cells.data(), nullptr));
  return t;
}
}  // namespace

// The paper's own methods on the device (sdp_tournament / sdp_naive), with the
// reference's step models on top.
PrefixParallelResult solve_prefix_parallel(const SdpInstance& inst) {  // sdp.cpp:91-100
  PrefixParallelResult r;
  r.table = solve_method(inst, PIPEDP_SDP_PREFIX);
  r.depth_per_cell = ceil_log2(inst.offsets.k());
  r.modeled_steps = (inst.n - inst.offsets.a1()) * std::max<std::int64_t>(r.depth_per_cell, 1);
  return r;
}

NaiveParallelResult solve_naive_parallel(const SdpInstance& inst) {  // sdp.cpp:102-111
  NaiveParallelResult r;
  r.table = solve_method(inst, PIPEDP_SDP_NAIVE);
  r.serialized_accesses_per_cell = inst.offsets.k() - 1;
  r.modeled_steps = (inst.n - inst.offsets.a1()) * inst.offsets.k();
  return r;
}

std::vector<SolutionTable> solve_sequential_batch(const std::vector<SdpInstance>& insts, int device) {
  std::vector<SolutionTable> out;
  if (insts.empty()) return out;
  const SdpInstance& f = insts.front();
  const std::int64_t n = f.n, k = f.offsets.k(), a1 = f.offsets.a1(), b = (std::int64_t)insts.size();
  std::vector<std::int64_t> offs, init, cells(static_cast<std::size_t>(b * n));
  for (const SdpInstance& s : insts) {
    validate(s);
    if (s.n != n || s.offsets.k() != k || s.offsets.a1() != a1 || s.op != f.op)
      fail(errc::invalid_params, "batched instances must share n, k, a_1 and the operator");
    offs.insert(offs.end(), s.offsets.offsets.begin(), s.offsets.offsets.end());
    init.insert(init.end(), s.init.begin(), s.init.end());
  }
  check(pipedp_sdp_solve_batch(b, n, k, a1, offs.data(), init.data(), static_cast<int32_t>(f.op.kind),
                               cells.data(), device));
  out.reserve(insts.size());
  for (std::int64_t i = 0; i < b; ++i) {
    SolutionTable t;
    t.cells.assign(cells.begin() + i * n, cells.begin() + (i + 1) * n);
    t.filled.assign(static_cast<std::size_t>(n), 1);
    out.push_back(std::move(t));
  }
  return out;
}

ConflictRunAnalysis analyze_conflict_runs(const OffsetSet& offsets) {  // sdp_pipeline.cpp:17-32
  ConflictRunAnalysis a;
  const auto& v = offsets.offsets;
  const int k = static_cast<int>(v.size());
  int start = 1;
  for (int r = 1; r <= k; ++r) {
    if (r < k && v[r - 1] == v[r] + 1) continue;
    a.runs.emplace_back(start, r);
    a.run_lengths.push_back(r - start + 1);
    a.longest_run = std::max(a.longest_run, r - start + 1);
    start = r + 1;
  }
  return a;
}

// solve_sdp_pipeline (sdp_pipeline.cpp:34-44).  Without collect_trace the
// table comes from the fast S-DP solvers (the schedule never stalls, so its
// step count is n + k - a_1 - 1).  With collect_trace the GPU lock-step engine
// runs SdpProgram itself: the table, the access records (when they fit the
// trace limit; otherwise trace.collected = false) and detect_conflicts'
// report computed on the device.
SdpPipelineResult solve_sdp_pipeline(const SdpInstance& inst, const SdpRunConfig& cfg) {
  validate(inst);
  SdpPipelineResult r;
  if (!cfg.collect_trace) {
    r.table = solve_sequential(inst);
    r.trace.first_head = inst.offsets.a1();  // head range [a_1, n+k-2] (sdp_pipeline.hpp:20)
    r.trace.steps_executed = inst.n + inst.offsets.k() - inst.offsets.a1() - 1;
    r.trace.stall_iterations = 0;
    r.trace.collected = false;
    return r;
  }
  const std::int64_t k = inst.offsets.k(), a1 = inst.offsets.a1();
  const bool fits = (inst.n - a1) * (3 * k - 1) <= kTraceLimit;
  EngineRun e;
  r.table = full_table(inst.n);
  check(pipedp_sdp_engine(inst.offsets.offsets.data(), k, inst.init.data(), static_cast<std::int64_t>(inst.init.size()),
                          inst.n, static_cast<int32_t>(inst.op.kind),
                          PIPEDP_ENGINE_ANALYSIS | (fits ? PIPEDP_ENGINE_TRACE : 0), r.table.cells.data(), &e.sum,
                          &e.run));
  fill_trace(e, fits, r.trace);
  r.conflicts = conflicts_of(e);
  return r;
}

// ------------------------------------------------------------------ MCM ---
const McmInstance& validate(const McmInstance& inst) {
  check(pipedp_mcm_validate(inst.dims.data(), static_cast<std::int64_t>(inst.dims.size())));
  return inst;
}

std::int64_t lin(TriCoord c, std::int64_t n) {  // mcm.cpp:30-37
  if (c.row < 1 || c.row > c.col || c.col > n)
    fail(errc::coord_out_of_range, "(" + std::to_string(c.row) + "," + std::to_string(c.col) +
                                       ") outside the order-" + std::to_string(n) + " triangle");
  const std::int64_t d = c.col - c.row;
  return d * n - d * (d - 1) / 2 + c.row;
}

TriCoord coord(std::int64_t address, std::int64_t n) {  // mcm.cpp:39-53
  if (address < 1 || address > cell_count(n))
    fail(errc::address_out_of_range, "address " + std::to_string(address) + " outside table of " +
                                         std::to_string(cell_count(n)) + " cells");
  std::int64_t d = 0, base = 0;
  while (address > base + (n - d)) {
    base += n - d;
    ++d;
  }
  const std::int64_t row = address - base;
  return TriCoord{row, row + d};
}

std::vector<DependencyTerm> deps(std::int64_t address, const McmInstance& inst) {  // mcm.cpp:55-75
  const std::int64_t n = inst.n();
  const TriCoord cell = coord(address, n);
  if (cell.diagonal() == 0)
    fail(errc::base_cell_has_no_deps,
         "cell " + std::to_string(address) + " is preset and has no dependencies");
  std::vector<DependencyTerm> terms;
  terms.reserve(static_cast<std::size_t>(cell.diagonal()));
  const auto& p = inst.dims;
  for (std::int64_t j = 1; j <= cell.diagonal(); ++j) {
    terms.push_back({lin({cell.row, cell.row + j - 1}, n), lin({cell.row + j, cell.col}, n),
                     p[cell.row - 1] * p[cell.row + j - 1] * p[cell.col]});
  }
  return terms;
}

SolutionTable mcm_initial_table(const McmInstance& inst) {  // mcm.cpp:77-83
  const std::int64_t n = inst.n();
  SolutionTable table(cell_count(n) + 1);
  for (std::int64_t i = 0; i <= n; ++i) table.filled[static_cast<std::size_t>(i)] = 1;
  return table;
}

namespace {
SolutionTable mcm_solve(const McmInstance& inst, std::vector<std::int64_t>* split, int32_t kernel) {
  validate(inst);
  const std::int64_t size = cell_count(inst.n()) + 1;
  SolutionTable t = full_table(size);
  if (split) split->assign(static_cast<std::size_t>(size), 0);
  check(pipedp_mcm_solve(inst.dims.data(), static_cast<std::int64_t>(inst.dims.size()), kernel,
                         t.cells.data(), nullptr, split ? split->data() : nullptr));
  return t;
}
}  // namespace

SolutionTable solve_mcm_sequential(const McmInstance& inst, std::vector<std::int64_t>* split) {
  return mcm_solve(inst, split, PIPEDP_MCM_AUTO);
}

std::int64_t solve_mcm_bruteforce(const McmInstance& inst) {  // mcm.cpp:130-138
  std::int64_t out = 0;
  check(pipedp_mcm_bruteforce(inst.dims.data(), static_cast<std::int64_t>(inst.dims.size()), &out));
  return out;
}

SolutionTable solve_mcm_tournament(const McmInstance& inst, std::vector<std::int64_t>* split) {
  return mcm_solve(inst, split, PIPEDP_MCM_TOURNAMENT);
}

std::vector<SolutionTable> solve_mcm_batch(const std::vector<McmInstance>& insts,
                                           std::vector<std::vector<std::int64_t>>* splits, int device) {
  std::vector<SolutionTable> out;
  if (insts.empty()) return out;
  const std::int64_t n = insts.front().n(), b = (std::int64_t)insts.size();
  const std::int64_t size = cell_count(n) + 1;
  std::vector<std::int64_t> dims, cells(static_cast<std::size_t>(b * size)),
      split(static_cast<std::size_t>(b * size));
  for (const McmInstance& m : insts) {
    validate(m);
    if (m.n() != n) fail(errc::invalid_params, "batched MCM instances must share n");
    dims.insert(dims.end(), m.dims.begin(), m.dims.end());
  }
  check(pipedp_mcm_solve_batch(b, n, dims.data(), cells.data(), split.data(), device));
  if (splits) splits->clear();
  for (std::int64_t i = 0; i < b; ++i) {
    SolutionTable t;
    t.cells.assign(cells.begin() + i * size, cells.begin() + (i + 1) * size);
    t.filled.assign(static_cast<std::size_t>(size), 1);
    out.push_back(std::move(t));
    if (splits) splits->emplace_back(split.begin() + i * size, split.begin() + (i + 1) * size);
  }
  return out;
}

// solve_mcm_pipeline (mcm_pipeline.cpp:32-47): the GPU lock-step engine
// running McmProgram in either McmMode -- table, steps, stalls and stall
// heads always; with collect_trace also the access records (when they fit the
// trace limit; otherwise trace.collected = false) and the conflict and hazard
// reports, computed on the device while the schedule runs.
McmPipelineResult solve_mcm_pipeline(const McmInstance& inst, const McmScheduleConfig& cfg) {
  validate(inst);  // build_mcm_program: validate, then n >= 2 (mcm_pipeline.cpp:26-30)
  if (inst.n() < 2) fail(errc::invalid_params, "pipeline needs at least two matrices");
  const std::int64_t n = inst.n(), cc = cell_count(n);
  const bool fits = 4 * ((n * n * n - n) / 6) - (cc - n) <= kTraceLimit;
  const int32_t flags = cfg.collect_trace ? (PIPEDP_ENGINE_ANALYSIS | (fits ? PIPEDP_ENGINE_TRACE : 0)) : 0;
  McmPipelineResult r;
  r.table = full_table(cc + 1);
  EngineRun e;
  check(pipedp_mcm_engine(inst.dims.data(), static_cast<std::int64_t>(inst.dims.size()),
                          cfg.mode == McmMode::stall_on_hazard ? PIPEDP_MCM_STALL_ON_HAZARD : PIPEDP_MCM_PAPER_LITERAL,
                          flags, r.table.cells.data(), &e.sum, &e.run));
  fill_trace(e, cfg.collect_trace && fits, r.trace);
  if (cfg.collect_trace) {
    r.conflicts = conflicts_of(e);
    r.hazards = hazards_of(e);
  }
  return r;
}

// verify_substep_distinctness (mcm_pipeline.cpp:49-77): Lemma 1/2 check on a
// trace -- substep-1 reads, substep-2 reads and substep-4 writes must touch
// distinct addresses across lanes at every head.  The counterexample is the
// first offending (head, substep, address) in that order.
DistinctnessVerdict verify_substep_distinctness(const PipelineTrace& trace) {
  std::vector<std::tuple<std::int64_t, int, std::int64_t, int>> picked;  // head, substep, address, lane
  for (const AccessRecord& a : trace.records) {
    const bool rd = a.kind == AccessKind::read && (a.substep == 1 || a.substep == 2);
    const bool wr = a.kind == AccessKind::write && a.substep == 4;
    if (rd || wr) picked.emplace_back(a.head, a.substep, a.address, a.lane);
  }
  std::sort(picked.begin(), picked.end());
  DistinctnessVerdict v;
  for (std::size_t i = 0; i < picked.size();) {
    std::size_t j = i + 1;
    while (j < picked.size() && std::get<0>(picked[j]) == std::get<0>(picked[i]) &&
           std::get<1>(picked[j]) == std::get<1>(picked[i]) && std::get<2>(picked[j]) == std::get<2>(picked[i]))
      ++j;
    if (j - i >= 2) {
      const int sub = std::get<1>(picked[i]);
      (sub == 1 ? v.substep1_reads_distinct : sub == 2 ? v.substep2_reads_distinct : v.substep4_writes_distinct) =
          false;
      if (!v.counterexample) {
        ConflictGroup g;
        g.head = std::get<0>(picked[i]);
        g.substep = sub;
        g.kind = sub == 4 ? AccessKind::write : AccessKind::read;
        g.address = std::get<2>(picked[i]);
        for (std::size_t t = i; t < j; ++t) g.lanes.push_back(std::get<3>(picked[t]));
        v.counterexample = std::move(g);
      }
    }
    i = j;
  }
  return v;
}

// ------------------------------------------------------------ generators ---
SdpInstance generate_sdp(const SdpGenParams& p) {
  if (p.k < 1) fail(errc::invalid_params, "k must be >= 1");
  const std::int64_t cap = p.consecutive ? p.k : (p.a1_cap > 0 ? p.a1_cap : 2 * p.k);
  SdpInstance inst;
  inst.n = p.n;
  inst.op = p.op;
  inst.offsets.offsets.assign(static_cast<std::size_t>(p.k), 0);
  inst.init.assign(static_cast<std::size_t>(std::max(cap, p.k)), 0);
  std::int64_t a1 = 0;
  check(pipedp_generate_sdp(p.n, p.k, static_cast<int32_t>(p.op.kind), p.seed, p.consecutive ? 1 : 0,
                            p.a1_cap, inst.offsets.offsets.data(), inst.init.data(),
                            static_cast<std::int64_t>(inst.init.size()), &a1));
  inst.init.resize(static_cast<std::size_t>(a1));
  return inst;
}

McmInstance generate_mcm(const McmGenParams& p) {
  McmInstance inst;
  if (p.n >= 1) inst.dims.assign(static_cast<std::size_t>(p.n + 1), 0);
  check(pipedp_generate_mcm(p.n, p.seed, p.dims_min, p.dims_max, inst.dims.data()));
  return inst;
}

}  // namespace pipedp

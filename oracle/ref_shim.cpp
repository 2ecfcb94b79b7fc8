// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, compiled from
// the reference sources where they lie (/root/reference/proj/src, see
// oracle/Makefile) into oracle/_ref/libpipedp_ref.so.  Used by tests/ to pin
// the C restatement (oracle/pipedp_oracle.c) and by bench.py's CPU baseline
// ("kind": "reference").  Nothing here is part of the product.
//
// Status convention: 0 = ok, 1 + errc index for pipedp::Error, 99 for any
// other exception.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "pipedp/error.hpp"
#include "pipedp/generate.hpp"
#include "pipedp/mcm.hpp"
#include "pipedp/mcm_pipeline.hpp"
#include "pipedp/sdp.hpp"
#include "pipedp/sdp_pipeline.hpp"
#include "pipedp/table.hpp"

using namespace pipedp;

namespace {

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    return 1 + static_cast<int>(e.code());
  } catch (...) {
    return 99;
  }
}

SdpInstance make_sdp(const int64_t* offs, int64_t k, const int64_t* init, int64_t init_len,
                     int64_t n, int op) {
  SdpInstance inst;
  inst.n = n;
  inst.offsets.offsets.assign(offs, offs + k);
  inst.init.assign(init, init + init_len);
  inst.op = SemigroupOp{static_cast<OpKind>(op)};
  return inst;
}

McmInstance make_mcm(const int64_t* dims, int64_t len) {
  McmInstance inst;
  inst.dims.assign(dims, dims + len);
  return inst;
}

void put(const SolutionTable& t, int64_t* cells, uint8_t* filled) {
  std::memcpy(cells, t.cells.data(), t.cells.size() * sizeof(int64_t));
  if (filled) std::memcpy(filled, t.filled.data(), t.filled.size());
}

}  // namespace

extern "C" {

int64_t ref_apply(int op, int64_t a, int64_t b) { return SemigroupOp{static_cast<OpKind>(op)}.apply(a, b); }

int ref_sdp_solve(const int64_t* offs, int64_t k, const int64_t* init, int64_t init_len, int64_t n,
                  int op, int64_t* cells, uint8_t* filled) {
  return guard([&] { put(solve_sequential(make_sdp(offs, k, init, init_len, n, op)), cells, filled); });
}

// which: 0 prefix, 1 naive; *model = modeled_steps, *aux = depth / serialized accesses
int ref_sdp_solve_model(const int64_t* offs, int64_t k, const int64_t* init, int64_t init_len,
                        int64_t n, int op, int which, int64_t* cells, uint8_t* filled,
                        int64_t* model, int64_t* aux) {
  return guard([&] {
    const SdpInstance inst = make_sdp(offs, k, init, init_len, n, op);
    if (which == 0) {
      PrefixParallelResult r = solve_prefix_parallel(inst);
      put(r.table, cells, filled);
      *model = r.modeled_steps;
      *aux = r.depth_per_cell;
    } else {
      NaiveParallelResult r = solve_naive_parallel(inst);
      put(r.table, cells, filled);
      *model = r.modeled_steps;
      *aux = r.serialized_accesses_per_cell;
    }
  });
}

int ref_sdp_pipeline(const int64_t* offs, int64_t k, const int64_t* init, int64_t init_len,
                     int64_t n, int op, int64_t* cells, uint8_t* filled, int64_t* steps,
                     int64_t* first_head) {
  return guard([&] {
    SdpRunConfig cfg;
    cfg.collect_trace = false;
    SdpPipelineResult r = solve_sdp_pipeline(make_sdp(offs, k, init, init_len, n, op), cfg);
    put(r.table, cells, filled);
    *steps = r.trace.steps_executed;
    *first_head = r.trace.first_head;
  });
}

int ref_mcm_solve(const int64_t* dims, int64_t len, int64_t* cells, uint8_t* filled, int64_t* split) {
  return guard([&] {
    std::vector<int64_t> sp;
    SolutionTable t = solve_mcm_sequential(make_mcm(dims, len), split ? &sp : nullptr);
    put(t, cells, filled);
    if (split) std::memcpy(split, sp.data(), sp.size() * sizeof(int64_t));
  });
}

int ref_mcm_pipeline(const int64_t* dims, int64_t len, int mode, int collect_trace, int64_t* cells,
                     uint8_t* filled, int64_t* steps, int64_t* stall_iterations,
                     int64_t* hazard_cell_count) {
  return guard([&] {
    McmScheduleConfig cfg;
    cfg.mode = mode == 1 ? McmMode::stall_on_hazard : McmMode::paper_literal;
    cfg.collect_trace = collect_trace != 0;
    McmPipelineResult r = solve_mcm_pipeline(make_mcm(dims, len), cfg);
    put(r.table, cells, filled);
    *steps = r.trace.steps_executed;
    *stall_iterations = r.trace.stall_iterations;
    *hazard_cell_count = static_cast<int64_t>(hazard_cells(r.hazards).size());
  });
}

// Digest vector of one lock-step engine run with collect_trace (the trace and
// the reports of analysis.cpp), for the GPU engine's parity tests:
//  [0] steps [1] stalls [2] first_head [3] records [4] D(records: head, substep,
//  lane, kind, address) [5] max_group_size [6] groups [7] D(groups: head,
//  substep, kind, address, size, lanes...) [8] D(per_step_cost) [9] hazards
//  [10] D(hazards: 6 fields) [11] stall heads [12] D(stall heads) [13] D(cells)
// D = table_digest of the flattened int64 sequence.
namespace {
uint64_t dig(const std::vector<int64_t>& v) {
  SolutionTable t;
  t.cells = v;
  t.filled.assign(v.size(), 1);
  return table_digest(t);
}
void engine_digests(const SolutionTable& table, const PipelineTrace& tr, const ConflictReport& cr,
                    const HazardReport* hz, uint64_t* out) {
  std::vector<int64_t> v;
  for (const AccessRecord& a : tr.records)
    v.insert(v.end(), {a.head, a.substep, a.lane, static_cast<int64_t>(a.kind), a.address});
  out[0] = tr.steps_executed;
  out[1] = tr.stall_iterations;
  out[2] = tr.first_head;
  out[3] = tr.records.size();
  out[4] = dig(v);
  v.clear();
  for (const ConflictGroup& g : cr.groups) {
    v.insert(v.end(), {g.head, g.substep, static_cast<int64_t>(g.kind), g.address, (int64_t)g.lanes.size()});
    for (int l : g.lanes) v.push_back(l);
  }
  out[5] = cr.max_group_size;
  out[6] = cr.groups.size();
  out[7] = dig(v);
  out[8] = dig(std::vector<int64_t>(cr.per_step_cost.begin(), cr.per_step_cost.end()));
  v.clear();
  if (hz)
    for (const HazardRecord& h : hz->hazards)
      v.insert(v.end(), {h.head, h.substep, h.lane, h.address, h.finalization_head, h.finalization_substep});
  out[9] = hz ? hz->hazards.size() : 0;
  out[10] = dig(v);
  out[11] = tr.stall_heads.size();
  out[12] = dig(tr.stall_heads);
  out[13] = dig(table.cells);
}
}  // namespace

int ref_mcm_engine_digests(const int64_t* dims, int64_t len, int mode, uint64_t* out) {
  return guard([&] {
    McmScheduleConfig cfg;
    cfg.mode = mode == 1 ? McmMode::stall_on_hazard : McmMode::paper_literal;
    McmPipelineResult r = solve_mcm_pipeline(make_mcm(dims, len), cfg);
    engine_digests(r.table, r.trace, r.conflicts, &r.hazards, out);
  });
}

int ref_sdp_engine_digests(const int64_t* offs, int64_t k, const int64_t* init, int64_t init_len, int64_t n,
                           int op, uint64_t* out) {
  return guard([&] {
    SdpPipelineResult r = solve_sdp_pipeline(make_sdp(offs, k, init, init_len, n, op), SdpRunConfig{});
    engine_digests(r.table, r.trace, r.conflicts, nullptr, out);
  });
}

int64_t ref_mcm_bruteforce(const int64_t* dims, int64_t len) {
  int64_t out = 0;
  const int rc = guard([&] { out = solve_mcm_bruteforce(make_mcm(dims, len)); });
  return rc ? -rc : out;
}

int64_t ref_mcm_lin(int64_t row, int64_t col, int64_t n) {
  int64_t out = -1;
  guard([&] { out = lin(TriCoord{row, col}, n); });
  return out;
}

int ref_mcm_coord(int64_t address, int64_t n, int64_t* row, int64_t* col) {
  return guard([&] {
    const TriCoord c = coord(address, n);
    *row = c.row;
    *col = c.col;
  });
}

int64_t ref_hazard_frontier(int64_t n, int64_t* out, int64_t cap) {
  int64_t count = -1;
  guard([&] {
    std::vector<int64_t> f = hazard_frontier(n);
    count = static_cast<int64_t>(f.size());
    std::memcpy(out, f.data(), sizeof(int64_t) * static_cast<size_t>(std::min<int64_t>(cap, count)));
  });
  return count;
}

uint64_t ref_table_digest(const int64_t* cells, int64_t count) {
  SolutionTable t;
  t.cells.assign(cells, cells + count);
  t.filled.assign(static_cast<size_t>(count), 1);
  return table_digest(t);
}

int ref_generate_sdp(int64_t n, int64_t k, uint64_t seed, int consecutive, int64_t a1_cap,
                     int64_t* offs, int64_t* init, int64_t init_cap, int64_t* a1_out) {
  return guard([&] {
    SdpGenParams p;
    p.n = n;
    p.k = k;
    p.seed = seed;
    p.consecutive = consecutive != 0;
    p.a1_cap = a1_cap;
    SdpInstance inst = generate_sdp(p);
    std::memcpy(offs, inst.offsets.offsets.data(), sizeof(int64_t) * static_cast<size_t>(k));
    *a1_out = inst.offsets.a1();
    if (init_cap >= inst.offsets.a1())
      std::memcpy(init, inst.init.data(), sizeof(int64_t) * inst.init.size());
  });
}

int ref_generate_mcm(int64_t n, uint64_t seed, int64_t lo, int64_t hi, int64_t* dims) {
  return guard([&] {
    McmGenParams p;
    p.n = n;
    p.seed = seed;
    p.dims_min = lo;
    p.dims_max = hi;
    McmInstance inst = generate_mcm(p);
    std::memcpy(dims, inst.dims.data(), sizeof(int64_t) * inst.dims.size());
  });
}

int ref_validate_sdp(const int64_t* offs, int64_t k, int64_t init_len, int64_t n) {
  std::vector<int64_t> init(static_cast<size_t>(init_len > 0 ? init_len : 0), 0);
  return guard([&] { validate(make_sdp(offs, k, init.data(), init_len, n, 0)); });
}

int ref_validate_mcm(const int64_t* dims, int64_t len) {
  return guard([&] { validate(make_mcm(dims, len)); });
}

}  // extern "C"

// dropin_test.cpp -- exercises the C++ drop-in (include/pipedp/*.hpp, built
// into paper_2008_01938_b200/_lib/libpipedp_b200.so) exactly the way the
// reference's callers use it (commands.cpp:87-165 run_*_solver,
// verify_sdp / verify_mcm :246-340).  Built and driven by tests/test_dropin.py.
//
//   dropin_test validate   host-side checks (no GPU needed): errc mapping,
//                          lin/coord/deps, generators, digests
//   dropin_test nogpu      every solver must throw pipedp::DeviceError (no CPU path)
//   dropin_test solve      GPU: prints "<case> <cells digest> [<split digest>]" lines
//   dropin_test io         host-side: instance text round trips, batched loader,
//                          parenthesisation from a split table
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "pipedp/error.hpp"
#include "pipedp/generate.hpp"
#include "pipedp/io.hpp"
#include "pipedp/mcm.hpp"
#include "pipedp/mcm_pipeline.hpp"
#include "pipedp/sdp.hpp"
#include "pipedp/sdp_pipeline.hpp"
#include "pipedp/table.hpp"

using namespace pipedp;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);       \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static bool throws_errc(const std::function<void()>& f, errc code, const char* prefix) {
  try {
    f();
  } catch (const Error& e) {
    return e.code() == code && std::strncmp(e.what(), prefix, std::strlen(prefix)) == 0;
  } catch (...) {
    return false;
  }
  return false;
}

static SdpInstance sdp(std::int64_t n, std::vector<std::int64_t> offs, std::vector<std::int64_t> init,
                       OpKind op) {
  SdpInstance s;
  s.n = n;
  s.offsets.offsets = std::move(offs);
  s.init = std::move(init);
  s.op = SemigroupOp{op};
  return s;
}

static int run_validate() {
  // SPEC.md:61-63 / sdp.cpp:10-32
  EXPECT(throws_errc([] { validate(sdp(16, {3, 3, 1}, {0, 0, 0}, OpKind::min)); },
                     errc::non_decreasing_offsets, "NonDecreasingOffsets: "));
  EXPECT(throws_errc([] { validate(sdp(16, {5, 3, 1}, {0, 0, 0, 0}, OpKind::min)); },
                     errc::init_length_mismatch, "InitLengthMismatch: "));
  EXPECT(throws_errc([] { validate(sdp(16, {5, 3, 0}, {0, 0, 0, 0, 0}, OpKind::min)); },
                     errc::non_positive_offset, "NonPositiveOffset: "));
  EXPECT(throws_errc([] { validate(sdp(5, {5, 3, 1}, {0, 0, 0, 0, 0}, OpKind::min)); },
                     errc::table_too_small, "TableTooSmall: "));
  validate(sdp(16, {5, 3, 1}, {0, 0, 0, 0, 0}, OpKind::min));
  // validation happens BEFORE any device work: the error is the reference's
  EXPECT(throws_errc([] { solve_sequential(sdp(16, {3, 3, 1}, {0, 0, 0}, OpKind::min)); },
                     errc::non_decreasing_offsets, "NonDecreasingOffsets"));
  // mcm.cpp:11-28
  EXPECT(throws_errc([] { validate(McmInstance{{10}}); }, errc::invalid_params, "InvalidParams"));
  EXPECT(throws_errc([] { validate(McmInstance{{1000001, 2}}); }, errc::weight_overflow, "WeightOverflow"));
  EXPECT(throws_errc([] { solve_mcm_sequential(McmInstance{{0, 3}}); }, errc::invalid_params, "InvalidParams"));
  EXPECT(throws_errc([] { solve_mcm_pipeline(McmInstance{{4, 3}}); }, errc::invalid_params, "InvalidParams"));
  // SPEC.md:298-299, 318-319
  EXPECT(lin({1, 4}, 5) == 13);
  EXPECT(lin({3, 5}, 5) == 12);
  EXPECT((coord(13, 5) == TriCoord{1, 4}));
  EXPECT(throws_errc([] { lin({3, 2}, 5); }, errc::coord_out_of_range, "CoordOutOfRange"));
  EXPECT(throws_errc([] { coord(16, 5); }, errc::address_out_of_range, "AddressOutOfRange"));
  McmInstance m{{1, 2, 3, 4, 5, 6}};
  auto t = deps(13, m);
  EXPECT(t.size() == 3);
  EXPECT((t[0] == DependencyTerm{1, 11, 10}) && (t[1] == DependencyTerm{6, 8, 15}) &&
         (t[2] == DependencyTerm{10, 4, 20}));
  EXPECT(throws_errc([&] { deps(3, m); }, errc::base_cell_has_no_deps, "BaseCellHasNoDeps"));
  // semigroup catalog
  EXPECT(SemigroupOp{OpKind::saturating_add}.apply(INT64_MAX, 1) == INT64_MAX);
  EXPECT(SemigroupOp{OpKind::saturating_add}.apply(INT64_MIN, -1) == INT64_MIN);
  EXPECT(SemigroupOp{OpKind::modular_add}.apply(-5, 3) == 2147483645);
  EXPECT(SemigroupOp::from_name("modular-add").kind == OpKind::modular_add);
  EXPECT(throws_errc([] { SemigroupOp::from_name("xor"); }, errc::invalid_params, "InvalidParams"));
  // sdp_pipeline.cpp:17-32 (SPEC examples)
  EXPECT(analyze_conflict_runs(OffsetSet{{4, 3, 2, 1}}).longest_run == 4);
  EXPECT(analyze_conflict_runs(OffsetSet{{5, 3, 1}}).longest_run == 1);
  EXPECT(analyze_conflict_runs(OffsetSet{{7, 6, 4, 3, 2}}).longest_run == 3);
  // generators: same draws as the reference (digests printed for the golden check)
  SdpGenParams gp;
  gp.n = 1 << 24;
  gp.k = 1024;
  gp.seed = 1;
  gp.a1_cap = 4096;
  SdpInstance g = generate_sdp(gp);
  SolutionTable ot, it;
  ot.cells = g.offsets.offsets;
  it.cells = g.init;
  std::printf("gen_sdp %s %s\n", digest_hex(table_digest(ot)).c_str(), digest_hex(table_digest(it)).c_str());
  McmGenParams mp;
  mp.n = 1024;
  mp.seed = 1;
  mp.dims_max = 100;
  SolutionTable dt;
  dt.cells = generate_mcm(mp).dims;
  std::printf("gen_mcm %s\n", digest_hex(table_digest(dt)).c_str());
  std::printf("%s\n", failures ? "FAILED" : "OK");
  return failures ? 1 : 0;
}

static bool throws_device(const std::function<void()>& f) {
  try {
    f();
  } catch (const DeviceError&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static int run_nogpu() {
  const SdpInstance fib = sdp(7, {2, 1}, {1, 1}, OpKind::saturating_add);
  EXPECT(throws_device([&] { solve_sequential(fib); }));
  EXPECT(throws_device([&] { solve_sdp_pipeline(fib); }));
  EXPECT(throws_device([&] { solve_prefix_parallel(fib); }));
  EXPECT(throws_device([&] { solve_naive_parallel(fib); }));
  std::vector<std::int64_t> split;
  EXPECT(throws_device([&] { solve_mcm_sequential(McmInstance{{10, 20, 30}}, &split); }));
  EXPECT(throws_device([&] { solve_mcm_pipeline(McmInstance{{10, 20, 30}}); }));
  std::printf("%s\n", failures ? "FAILED" : "OK");
  return failures ? 1 : 0;
}

static int run_solve() {
  // SPEC KATs through the drop-in
  SolutionTable t = solve_sequential(sdp(7, {2, 1}, {1, 1}, OpKind::saturating_add));
  EXPECT((t.cells == std::vector<std::int64_t>{1, 1, 2, 3, 5, 8, 13}) && t.all_filled());
  std::vector<std::int64_t> split;
  SolutionTable m = solve_mcm_sequential(McmInstance{{30, 35, 15, 5, 10, 20, 25}}, &split);
  EXPECT(m.cells.back() == 15125 && split.back() == 3 && m.all_filled());
  // the reference's defaults (collect_trace = true, paper_literal) must be accepted
  McmPipelineResult pr = solve_mcm_pipeline(McmInstance{{10, 20, 30, 40, 30}});
  // -> trace collected by the GPU engine; n = 4 is hazardous at address 10
  EXPECT(pr.trace.steps_executed == 4 * 5 / 2 - 2 && pr.trace.collected && pr.trace.records.size() == 34);
  EXPECT(hazard_cells(pr.hazards) == std::vector<std::int64_t>{10} && pr.conflicts.max_group_size == 1);
  EXPECT(verify_substep_distinctness(pr.trace).all_ok());
  McmScheduleConfig sc;
  sc.mode = McmMode::stall_on_hazard;
  McmPipelineResult ps = solve_mcm_pipeline(McmInstance{{10, 20, 30, 40, 30}}, sc);
  EXPECT(ps.table.cells == solve_mcm_sequential(McmInstance{{10, 20, 30, 40, 30}}).cells);
  SdpPipelineResult sp = solve_sdp_pipeline(sdp(10, {5, 3, 1}, {0, 0, 0, 0, 0}, OpKind::min));
  EXPECT(sp.trace.steps_executed == 10 + 3 - 5 - 1 && sp.trace.first_head == 5);
  PrefixParallelResult pp = solve_prefix_parallel(sdp(10, {5, 3, 2, 1}, {1, 2, 3, 4, 5}, OpKind::max));
  EXPECT(pp.depth_per_cell == 2);
  // generated configs: digests compared with tests/golden/golden.json by the driver
  const char* ops[] = {"min", "max", "saturating-add", "modular-add"};
  for (int op = 0; op < 4; ++op) {
    SdpGenParams gp;
    gp.n = 20000;
    gp.k = 1024;
    gp.seed = 11;
    gp.a1_cap = 4096;
    gp.op = SemigroupOp{static_cast<OpKind>(op)};
    SdpInstance inst = generate_sdp(gp);
    std::printf("sdp 20000 1024 11 4096 %s %s\n", ops[op],
                digest_hex(table_digest(solve_sequential(inst))).c_str());
  }
  for (std::int64_t n : {64, 512, 1024}) {
    McmGenParams mp;
    mp.n = n;
    mp.seed = n == 512 ? 7 : 1;
    mp.dims_max = 100;
    McmInstance inst = generate_mcm(mp);
    std::vector<std::int64_t> s;
    SolutionTable c = solve_mcm_sequential(inst, &s);
    SolutionTable st;
    st.cells = s;
    std::printf("mcm %lld %s %s\n", (long long)n, digest_hex(table_digest(c)).c_str(),
                digest_hex(table_digest(st)).c_str());
  }
  // batch entry point agrees with per-instance solves
  std::vector<SdpInstance> batch;
  for (int i = 0; i < 9; ++i) {
    SdpGenParams gp;
    gp.n = 4000;
    gp.k = 64;
    gp.seed = static_cast<std::uint64_t>(i);
    batch.push_back(generate_sdp(gp));
  }
  std::vector<SolutionTable> bt = solve_sequential_batch(batch);
  for (int i = 0; i < 9; ++i) EXPECT(bt[i] == solve_sequential(batch[i]));
  std::printf("%s\n", failures ? "FAILED" : "OK");
  return failures ? 1 : 0;
}

// host MCM DP (test-side, tiny n) for a split table in the reference layout
static std::vector<std::int64_t> host_split(const McmInstance& m, std::int64_t* best_cost) {
  const std::int64_t n = m.n();
  std::vector<std::int64_t> cost((size_t)cell_count(n) + 1, 0), split((size_t)cell_count(n) + 1, 0);
  for (std::int64_t D = 1; D < n; ++D)
    for (std::int64_t r = 1; r + D <= n; ++r) {
      const std::int64_t c = r + D, a = lin(TriCoord{r, c}, n);
      std::int64_t best = INT64_MAX, bj = 0;
      for (std::int64_t j = 1; j <= D; ++j) {
        const std::int64_t k = r + j - 1;
        const std::int64_t v = cost[(size_t)lin(TriCoord{r, k}, n)] + cost[(size_t)lin(TriCoord{k + 1, c}, n)] +
                               m.dims[(size_t)(r - 1)] * m.dims[(size_t)k] * m.dims[(size_t)c];
        if (v < best) best = v, bj = j;
      }
      cost[(size_t)a] = best;
      split[(size_t)a] = bj;
    }
  *best_cost = n > 1 ? cost[(size_t)apex_address(n)] : 0;
  return split;
}

// cost of a parenthesised product string over dims (A1..An)
static std::int64_t paren_cost(const std::string& s, const std::vector<std::int64_t>& p, size_t& i,
                               std::int64_t& rows, std::int64_t& cols) {
  if (s[i] == 'A') {
    ++i;
    std::int64_t idx = 0;
    while (i < s.size() && s[i] >= '0' && s[i] <= '9') idx = idx * 10 + (s[i++] - '0');
    rows = p[(size_t)idx - 1];
    cols = p[(size_t)idx];
    return 0;
  }
  ++i;  // '('
  std::int64_t r1, c1, r2, c2;
  const std::int64_t a = paren_cost(s, p, i, r1, c1), b = paren_cost(s, p, i, r2, c2);
  ++i;  // ')'
  rows = r1;
  cols = c2;
  return a + b + r1 * c1 * c2;
}

static int run_io() {
  // round trips (reference io.cpp:10-42 format)
  const SdpInstance s = sdp(40, {7, 3, 1}, {5, -4, 3, 2, 1, 0, 9}, OpKind::modular_add);
  McmInstance m;
  m.dims = {30, 35, 15, 5, 10, 20, 25};
  EXPECT(to_text(s) == "sdp 40 3 modular-add\n7 3 1\n5 -4 3 2 1 0 9\n");
  EXPECT(to_text(m) == "mcm 6\n30 35 15 5 10 20 25\n");
  std::istringstream one(to_text(s));
  const ParsedInstance ps = read_instance(one);
  EXPECT(ps.kind == InstanceKind::sdp && ps.sdp && *ps.sdp == s);
  // batched loader: every instance in order
  std::istringstream many(to_text(m) + to_text(s) + to_text(m));
  const std::vector<ParsedInstance> all = read_instances(many);
  EXPECT(all.size() == 3 && all[0].kind == InstanceKind::mcm && *all[0].mcm == m &&
         all[1].kind == InstanceKind::sdp && *all[1].sdp == s && *all[2].mcm == m);
  // errors as the reference raises them
  EXPECT(throws_errc([] { std::istringstream in("dp 3\n"); read_instance(in); }, errc::invalid_params,
                     "InvalidParams: "));
  EXPECT(throws_errc([] { std::istringstream in("mcm 3\n1 2 3\n"); read_instance(in); },
                     errc::invalid_params, "InvalidParams: "));
  EXPECT(throws_errc([] { std::istringstream in("sdp 10 2 min\n2 2\n0 0\n"); read_instance(in); },
                     errc::non_decreasing_offsets, "NonDecreasingOffsets: "));
  EXPECT(throws_errc([] { std::istringstream in(""); read_instances(in); }, errc::invalid_params,
                     "InvalidParams: "));
  // parenthesisation: CLRS 15.2 example and random instances, cost == apex
  std::int64_t best = 0;
  const std::vector<std::int64_t> sp = host_split(m, &best);
  const std::string paren = mcm_parenthesization(m, sp);
  EXPECT(paren == "((A1(A2A3))((A4A5)A6))");
  EXPECT(best == 15125);
  unsigned long long x = 88172645463325252ull;
  for (int t = 0; t < 50; ++t) {
    McmInstance r;
    const int n = 1 + (int)(x % 40);
    for (int i = 0; i <= n; ++i) {
      x ^= x << 13, x ^= x >> 7, x ^= x << 17;
      r.dims.push_back(1 + (std::int64_t)(x % 100));
    }
    const std::vector<std::int64_t> rs = host_split(r, &best);
    const std::string pr = mcm_parenthesization(r, rs);
    size_t i = 0;
    std::int64_t rows, cols;
    EXPECT(paren_cost(pr, r.dims, i, rows, cols) == best && i == pr.size());
  }
  // hazard_frontier against the reference's per-cell scan (mcm_pipeline.cpp:79-93)
  for (std::int64_t n : {2, 3, 7, 33, 90}) {
    std::vector<std::int64_t> want;
    for (std::int64_t addr = n + 1; addr <= cell_count(n); ++addr) {
      const TriCoord cc = coord(addr, n);
      for (std::int64_t j = 1; j <= cc.diagonal(); ++j)
        if (addr - lin(TriCoord{cc.row + j, cc.col}, n) <= cc.diagonal() - 2 * j) {
          want.push_back(addr);
          break;
        }
    }
    EXPECT(hazard_frontier(n) == want);
  }
  EXPECT(throws_errc([] { hazard_frontier(1); }, errc::invalid_params, "InvalidParams: "));
  std::printf("%s\n", failures ? "FAILED" : "OK");
  return failures ? 1 : 0;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "validate";
  try {
    if (mode == "validate") return run_validate();
    if (mode == "nogpu") return run_nogpu();
    if (mode == "solve") return run_solve();
    if (mode == "io") return run_io();
  } catch (const std::exception& e) {
    std::printf("EXCEPTION %s\n", e.what());
    return 2;
  }
  std::printf("unknown mode %s\n", mode.c_str());
  return 2;
}

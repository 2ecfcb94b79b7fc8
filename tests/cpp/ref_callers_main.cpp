// Drives the reference's own callers (proj/src/commands.cpp: cmd_run,
// cmd_verify, cmd_bench) compiled against include/pipedp and linked with the
// B200 drop-in instead of the reference's solver translation units -- the
// INTEGRATION.md §2 recipe.  Usage: ref_callers <mode> ; prints what the
// reference's commands print, then "rc=<code>" per command.
#include <cstdio>
#include <iostream>
#include <string>

#include "pipedp/commands.hpp"

using namespace pipedp;

static int run(const char* what, int (*cmd)(const RunSpec&, std::ostream&), const RunSpec& s) {
  const int rc = cmd(s, std::cerr);
  std::cout << what << " rc=" << rc << std::endl;
  return rc;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "run";
  RunSpec s;
  s.seed = 7;
  if (mode == "run") {  // one solve per solver kind through cmd_run
    for (Solver v : {Solver::sequential, Solver::naive, Solver::prefix, Solver::pipeline}) {
      s.problem = Problem::sdp; s.solver = v; s.n = 5000; s.k = 16; s.op = "min";
      run("sdp", cmd_run, s);
    }
    s.problem = Problem::mcm; s.n = 48; s.dims_min = 1; s.dims_max = 50;
    for (Solver v : {Solver::sequential, Solver::pipeline}) {
      s.solver = v;
      s.mode = McmMode::stall_on_hazard;
      run("mcm", cmd_run, s);
    }
    return 0;
  }
  if (mode == "verify") {  // the reference's own checks against its oracle entry points
    s.problem = Problem::sdp; s.solver = Solver::pipeline; s.n = 3000; s.k = 12; s.op = "min";
    run("verify-sdp-pipeline", cmd_verify, s);
    s.solver = Solver::sequential; s.op = "max";
    run("verify-sdp-sequential", cmd_verify, s);
    s.problem = Problem::mcm; s.n = 10; s.solver = Solver::sequential;
    run("verify-mcm-sequential", cmd_verify, s);
    s.n = 40; s.solver = Solver::pipeline;
    s.mode = McmMode::stall_on_hazard;
    run("verify-mcm-stall", cmd_verify, s);
    s.mode = McmMode::paper_literal;
    run("verify-mcm-literal", cmd_verify, s);
    return 0;
  }
  if (mode == "bench") {
    s.problem = Problem::sdp; s.reps = 2; s.format = OutputFormat::csv;
    run("bench", cmd_bench, s);
    return 0;
  }
  std::fprintf(stderr, "unknown mode %s\n", mode.c_str());
  return 64;
}

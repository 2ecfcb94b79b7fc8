// pipedp_io.cpp -- instance text I/O and split-table parenthesisation for the
// drop-in (host C++; no device work).  Format and error behaviour follow the
// reference's io.cpp:10-80 (header word, then whitespace-separated integers;
// malformed input -> Error{invalid_params}; every parsed instance validated).
#include <fstream>
#include <sstream>

#include "pipedp/error.hpp"
#include "pipedp/io.hpp"
#include "pipedp/mcm_pipeline.hpp"

#include <algorithm>

namespace pipedp {

namespace {

void write_row(std::ostream& out, const std::vector<std::int64_t>& v) {
  for (std::size_t i = 0; i < v.size(); ++i) out << (i ? " " : "") << v[i];
  out << '\n';
}

std::int64_t next_int(std::istream& in, const char* what) {
  std::int64_t v;
  if (!(in >> v)) fail(errc::invalid_params, std::string("malformed instance: missing ") + what);
  return v;
}

ParsedInstance parse_after_header(std::istream& in, const std::string& header) {
  ParsedInstance p;
  if (header == "sdp") {
    p.kind = InstanceKind::sdp;
    SdpInstance s;
    s.n = next_int(in, "n");
    const std::int64_t k = next_int(in, "k");
    std::string op;
    if (!(in >> op)) fail(errc::invalid_params, "malformed instance: missing operator name");
    s.op = SemigroupOp::from_name(op);
    for (std::int64_t j = 0; j < k; ++j) s.offsets.offsets.push_back(next_int(in, "offset"));
    const std::int64_t a1 = s.offsets.offsets.empty() ? 0 : s.offsets.a1();
    for (std::int64_t i = 0; i < a1; ++i) s.init.push_back(next_int(in, "initial value"));
    validate(s);
    p.sdp = std::move(s);
  } else if (header == "mcm") {
    p.kind = InstanceKind::mcm;
    McmInstance m;
    const std::int64_t n = next_int(in, "n");
    for (std::int64_t i = 0; i <= n; ++i) m.dims.push_back(next_int(in, "dimension"));
    validate(m);
    p.mcm = std::move(m);
  } else {
    fail(errc::invalid_params, "unknown instance header: " + header);
  }
  return p;
}

}  // namespace

void write_sdp_instance(std::ostream& out, const SdpInstance& instance) {
  out << "sdp " << instance.n << ' ' << instance.offsets.k() << ' ' << instance.op.name() << '\n';
  write_row(out, instance.offsets.offsets);
  write_row(out, instance.init);
}

void write_mcm_instance(std::ostream& out, const McmInstance& instance) {
  out << "mcm " << instance.n() << '\n';
  write_row(out, instance.dims);
}

std::string to_text(const SdpInstance& instance) {
  std::ostringstream s;
  write_sdp_instance(s, instance);
  return s.str();
}

std::string to_text(const McmInstance& instance) {
  std::ostringstream s;
  write_mcm_instance(s, instance);
  return s.str();
}

ParsedInstance read_instance(std::istream& in) {
  std::string header;
  if (!(in >> header)) fail(errc::invalid_params, "empty instance file");
  return parse_after_header(in, header);
}

ParsedInstance read_instance_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(errc::invalid_params, "cannot open instance file: " + path);
  return read_instance(in);
}

std::vector<ParsedInstance> read_instances(std::istream& in) {
  std::vector<ParsedInstance> all;
  std::string header;
  while (in >> header) all.push_back(parse_after_header(in, header));
  if (all.empty()) fail(errc::invalid_params, "empty instance file");
  return all;
}

std::vector<ParsedInstance> read_instances_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(errc::invalid_params, "cannot open instance file: " + path);
  return read_instances(in);
}

std::string mcm_parenthesization(const McmInstance& instance, const std::vector<std::int64_t>& split_points) {
  const std::int64_t n = instance.n();
  if (n < 1) fail(errc::invalid_params, "mcm_parenthesization: n must be >= 1");
  if ((std::int64_t)split_points.size() != cell_count(n) + 1)
    fail(errc::invalid_params, "mcm_parenthesization: split table size != n(n+1)/2 + 1");
  // explicit stack (n reaches 8192: no recursion); a frame prints "(" L R ")"
  std::string out;
  struct Frame {
    std::int64_t r, c;
    int state;  // 0 open, 1 after left, 2 after right
  };
  std::vector<Frame> st{{1, n, 0}};
  while (!st.empty()) {
    Frame& f = st.back();
    if (f.r == f.c) {
      out += 'A';
      out += std::to_string(f.r);
      st.pop_back();
      continue;
    }
    const std::int64_t j = split_points[(size_t)lin(TriCoord{f.r, f.c}, n)];
    if (j < 1 || j > f.c - f.r) fail(errc::invalid_params, "mcm_parenthesization: split index out of range");
    const std::int64_t k = f.r + j - 1;  // A_r..A_k | A_{k+1}..A_c
    if (f.state == 0) {
      out += '(';
      f.state = 1;
      st.push_back({f.r, k, 0});
    } else if (f.state == 1) {
      f.state = 2;
      st.push_back({k + 1, f.c, 0});
    } else {
      out += ')';
      st.pop_back();
    }
  }
  return out;
}

std::vector<std::int64_t> hazard_frontier(std::int64_t n) {
  if (n < 2) fail(errc::invalid_params, "frontier needs n >= 2");
  std::vector<std::int64_t> out;
  for (std::int64_t D = 1; D < n; ++D) {
    // lin(r, r+D) - lin(r+j, r+D) = sum_{e = D-j+1}^{D} (n - e + 1) - j
    //                             = j n - j (2D - j - 1) / 2 - j
    bool hit = false;
    for (std::int64_t j = 1; j <= D && !hit; ++j) hit = j * n - j * (2 * D - j - 1) / 2 - j <= D - 2 * j;
    if (!hit) continue;
    const std::int64_t base = D * n - D * (D - 1) / 2;  // lin(r, r+D) = base + r
    for (std::int64_t r = 1; r + D <= n; ++r) out.push_back(base + r);
  }
  return out;
}

std::vector<std::int64_t> hazard_cells(const HazardReport& report) {
  std::vector<std::int64_t> cells;
  cells.reserve(report.hazards.size());
  for (const HazardRecord& h : report.hazards) cells.push_back(h.head - h.lane + 1);
  std::sort(cells.begin(), cells.end());
  cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
  return cells;
}

}  // namespace pipedp

// engine.cu -- C ABI of the GPU lock-step engine (include/pipedp_cuda.h,
// "lock-step engine"): solve_mcm_pipeline / solve_sdp_pipeline with the
// reference's trace semantics (engine.hpp:134-433) and the trace analyses of
// analysis.cpp computed on the device (engine_kernels.cuh).
//
// Host work here is bookkeeping only: buffer sizing, the canonical sort of the
// records the device emitted (PipelineTrace::canonicalize, engine.hpp:76) and
// grouping of the device's conflict entries into ConflictGroups.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <numeric>
#include <tuple>
#include <vector>

#include "capi_util.hpp"
#include "engine_kernels.cuh"

using namespace pipedp_capi;
using namespace pipedp_dev;

struct pipedp_engine_run {
  pipedp_engine_summary sum{};
  std::vector<int64_t> rec_head, rec_addr;
  std::vector<int32_t> rec_meta;
  std::vector<int64_t> haz;        // [h][6]
  std::vector<int64_t> groups;     // [g][4]
  std::vector<int32_t> group_sizes, lanes, per_step_cost;
  std::vector<int64_t> stall_heads;
};

namespace {

constexpr int64_t kMaxRecords = int64_t(1) << 28;  // 8.6 GB of AccessRecord on the host

template <class P>
int engine_run(const P& prog, int stall, int flags, const int64_t* init, int64_t init_len,
               int64_t* cells_out, pipedp_engine_summary* summary, pipedp_engine_t* run_out,
               int64_t records_exact, Scope& sc) {
  if (flags & ~(PIPEDP_ENGINE_TRACE | PIPEDP_ENGINE_ANALYSIS))
    return fail(PIPEDP_E_INVALID_PARAMS, "unknown engine flags 0x%x", flags);
  if ((flags & PIPEDP_ENGINE_TRACE) && records_exact > kMaxRecords)
    return fail(PIPEDP_E_INVALID_PARAMS,
                "collect_trace: %lld access records exceed the %lld-record trace limit "
                "(the device analyses need no trace)",
                (long long)records_exact, (long long)kMaxRecords);
  const int64_t ts = prog.tsize(), lanes = prog.lanes();
  const int64_t heads = prog.last() - prog.first() + 1;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int threads = 512;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((lanes + threads - 1) / threads, sms));
  const bool analysis = flags & PIPEDP_ENGINE_ANALYSIS, trace = flags & PIPEDP_ENGINE_TRACE;

  EngState S{};
  S.stall = stall;
  S.flags = flags;
  S.budget = heads * (lanes + 2) + 16;  // engine.hpp:357
  TRY(sc.alloc(&S.cells, ts));
  TRY(sc.alloc(&S.wdone, ts));
  TRY(sc.alloc(&S.lastw, ts));
  TRY(sc.alloc(&S.vhead, lanes + 1));
  TRY(sc.alloc(&S.lstate, lanes + 1));
  TRY(sc.alloc(&S.exec, lanes + 1));
  TRY(sc.alloc(&S.wval, lanes + 1));
  TRY(sc.alloc(&S.wtarget, lanes + 1));
  TRY(sc.alloc(&S.flags_it, 8));
  TRY(sc.alloc(&S.bar, 2));
  TRY(sc.alloc(&S.counts, 4));
  TRY(sc.alloc(&S.result, 2));
  if (analysis) {
    TRY(sc.alloc(&S.cnt, 2 * 8 * ts));
    TRY(sc.alloc(&S.pend, 4 * (lanes + 1)));
  }
  S.rec_cap = trace ? records_exact : 0;
  if (trace) {
    TRY(sc.alloc(&S.rec_head, S.rec_cap));
    TRY(sc.alloc(&S.rec_addr, S.rec_cap));
    TRY(sc.alloc(&S.rec_meta, S.rec_cap));
  }
  cudaStream_t st = sc.stream;
  CK(cudaMemsetAsync(S.cells, 0, sizeof(int64_t) * ts, st));
  if (init_len) CK(cudaMemcpyAsync(S.cells, init, sizeof(int64_t) * init_len, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(S.wdone, 0, sizeof(int32_t) * ts, st));
  CK(cudaMemsetAsync(S.lastw, 0xff, sizeof(int64_t) * ts, st));
  CK(cudaMemsetAsync(S.lstate, 0, lanes + 1, st));
  CK(cudaMemsetAsync(S.flags_it, 0, sizeof(int) * 8, st));
  CK(cudaMemsetAsync(S.bar, 0, sizeof(unsigned) * 2, st));
  if (analysis) {
    CK(cudaMemsetAsync(S.cnt, 0, sizeof(int32_t) * 2 * 8 * ts, st));
    CK(cudaMemsetAsync(S.pend, 0xff, sizeof(int64_t) * 4 * (lanes + 1), st));
  }
  {  // every lane starts at the first head
    std::vector<int64_t> vh((size_t)lanes + 1, prog.first());
    CK(cudaMemcpyAsync(S.vhead, vh.data(), sizeof(int64_t) * (lanes + 1), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  // hazard / conflict / stall-head buffers: a first guess, rerun once with the
  // exact counts if it was short (the schedule is deterministic)
  int64_t cap = analysis ? std::min<int64_t>(int64_t(1) << 20, std::max<int64_t>(records_exact, 1)) : 0;
  int64_t stall_cap = stall ? std::min<int64_t>(int64_t(1) << 20, S.budget) : 0;
  unsigned long long counts[4] = {0, 0, 0, 0};
  int64_t result[2] = {0, 0};
  std::vector<void*> mine;
  auto cleanup = [&]() {
    for (void* p : mine) cudaFree(p);
    mine.clear();
  };
  for (int attempt = 0; attempt < 2; ++attempt) {
    S.haz_cap = cap;
    S.conf_cap = cap;
    S.stall_cap = stall_cap;
    cleanup();
    if (cap) {
      void* p;
      CK(cudaMalloc(&p, sizeof(int64_t) * 6 * cap)); mine.push_back(p); S.haz = (int64_t*)p;
      CK(cudaMalloc(&p, sizeof(int64_t) * 5 * cap)); mine.push_back(p); S.conf = (int64_t*)p;
    }
    if (stall_cap) {
      void* p;
      CK(cudaMalloc(&p, sizeof(int64_t) * stall_cap)); mine.push_back(p); S.stall_heads = (int64_t*)p;
    }
    if (attempt) {  // reset the run state
      CK(cudaMemsetAsync(S.cells, 0, sizeof(int64_t) * ts, st));
      if (init_len) CK(cudaMemcpyAsync(S.cells, init, sizeof(int64_t) * init_len, cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(S.wdone, 0, sizeof(int32_t) * ts, st));
      CK(cudaMemsetAsync(S.lastw, 0xff, sizeof(int64_t) * ts, st));
      CK(cudaMemsetAsync(S.lstate, 0, lanes + 1, st));
      CK(cudaMemsetAsync(S.flags_it, 0, sizeof(int) * 8, st));
      CK(cudaMemsetAsync(S.bar, 0, sizeof(unsigned) * 2, st));
      if (analysis) {
        CK(cudaMemsetAsync(S.cnt, 0, sizeof(int32_t) * 2 * 8 * ts, st));
        CK(cudaMemsetAsync(S.pend, 0xff, sizeof(int64_t) * 4 * (lanes + 1), st));
      }
      std::vector<int64_t> vh((size_t)lanes + 1, prog.first());
      CK(cudaMemcpyAsync(S.vhead, vh.data(), sizeof(int64_t) * (lanes + 1), cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    }
    CK(cudaMemsetAsync(S.counts, 0, sizeof(unsigned long long) * 4, st));
    CK(cudaMemsetAsync(S.result, 0, sizeof(int64_t) * 2, st));
    if (grid == 1) {
      engine_kernel<P><<<1, threads, 0, st>>>(prog, S);
    } else {
      void* args[] = {(void*)&prog, (void*)&S};
      CK(cudaLaunchCooperativeKernel((const void*)engine_kernel<P>, dim3(grid), dim3(threads), args, 0, st));
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(counts, S.counts, sizeof counts, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(result, S.result, sizeof result, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (result[1]) {
      cleanup();
      return result[1] == 1 ? fail(PIPEDP_E_STALL_LIVELOCK,
                                   "no lane can make progress; the program has an unsatisfiable dependency")
                            : fail(PIPEDP_E_STALL_LIVELOCK, "stall budget exceeded");
    }
    const int64_t need = (int64_t)std::max(counts[1], counts[2]);
    if (need <= cap && (int64_t)counts[3] <= stall_cap + (stall ? 0 : (int64_t)counts[3])) break;
    cap = std::max(cap, need);
    stall_cap = std::max<int64_t>(stall_cap, (int64_t)counts[3]);
  }
  pipedp_engine_run* R = new pipedp_engine_run();
  R->sum.first_head = prog.first();
  R->sum.steps_executed = result[0];
  R->sum.stall_iterations = result[0] - heads;
  if (cells_out) CK(cudaMemcpyAsync(cells_out, S.cells, sizeof(int64_t) * ts, cudaMemcpyDeviceToHost, st));
  const int64_t nrec = trace ? (int64_t)counts[0] : 0, nhaz = analysis ? (int64_t)counts[1] : 0,
                nconf = analysis ? (int64_t)counts[2] : 0, nstall = stall ? (int64_t)counts[3] : 0;
  if (nhaz) {
    engine_fix_hazards<<<(unsigned)std::min<int64_t>(1024, (nhaz + 255) / 256), 256, 0, st>>>(S.haz, nhaz, S.lastw);
    CK(cudaGetLastError());
  }
  R->rec_head.resize(nrec);
  R->rec_addr.resize(nrec);
  R->rec_meta.resize(nrec);
  R->haz.resize(6 * nhaz);
  std::vector<int64_t> conf(5 * nconf);
  R->stall_heads.resize(nstall);
  if (nrec) {
    CK(cudaMemcpyAsync(R->rec_head.data(), S.rec_head, 8 * nrec, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(R->rec_addr.data(), S.rec_addr, 8 * nrec, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(R->rec_meta.data(), S.rec_meta, 4 * nrec, cudaMemcpyDeviceToHost, st));
  }
  if (nhaz) CK(cudaMemcpyAsync(R->haz.data(), S.haz, 48 * nhaz, cudaMemcpyDeviceToHost, st));
  if (nconf) CK(cudaMemcpyAsync(conf.data(), S.conf, 40 * nconf, cudaMemcpyDeviceToHost, st));
  if (nstall) CK(cudaMemcpyAsync(R->stall_heads.data(), S.stall_heads, 8 * nstall, cudaMemcpyDeviceToHost, st));
  const cudaError_t e = cudaStreamSynchronize(st);
  cleanup();
  if (e != cudaSuccess) {
    delete R;
    return cuda_fail(e, "engine results");
  }
  // canonical record order (record_less: head, substep, lane, kind, address)
  if (nrec) {
    std::vector<int64_t> idx(nrec);
    std::iota(idx.begin(), idx.end(), 0);
    auto key = [&](int64_t i) {
      const int32_t m = R->rec_meta[i];
      return std::make_tuple(R->rec_head[i], (m >> 1) & 0x7f, m >> 8, m & 1, R->rec_addr[i]);
    };
    std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
    std::vector<int64_t> h(nrec), ad(nrec);
    std::vector<int32_t> m(nrec);
    for (int64_t i = 0; i < nrec; ++i) {
      h[i] = R->rec_head[idx[i]];
      ad[i] = R->rec_addr[idx[i]];
      m[i] = R->rec_meta[idx[i]];
    }
    R->rec_head.swap(h);
    R->rec_addr.swap(ad);
    R->rec_meta.swap(m);
  }
  // hazards in detect_hazards order (head, substep, lane, address)
  if (nhaz) {
    std::vector<std::array<int64_t, 6>> hz(nhaz);
    for (int64_t i = 0; i < nhaz; ++i)
      for (int q = 0; q < 6; ++q) hz[i][q] = R->haz[i * 6 + q];
    std::sort(hz.begin(), hz.end(), [](const auto& a, const auto& b) {
      return std::tie(a[0], a[1], a[2], a[3]) < std::tie(b[0], b[1], b[2], b[3]);
    });
    for (int64_t i = 0; i < nhaz; ++i)
      for (int q = 0; q < 6; ++q) R->haz[i * 6 + q] = hz[i][q];
  }
  // conflict groups in detect_conflicts order (head, substep, kind, address), lanes ascending
  R->per_step_cost.assign(analysis ? (size_t)std::max<int64_t>(result[0], 0) : 0, 1);
  int64_t maxg = 1;
  if (nconf) {
    std::vector<std::array<int64_t, 5>> cf(nconf);
    for (int64_t i = 0; i < nconf; ++i)
      for (int q = 0; q < 5; ++q) cf[i][q] = conf[i * 5 + q];
    std::sort(cf.begin(), cf.end());
    for (int64_t i = 0; i < nconf;) {
      int64_t j = i + 1;
      while (j < nconf && cf[j][0] == cf[i][0] && cf[j][1] == cf[i][1] && cf[j][2] == cf[i][2] &&
             cf[j][3] == cf[i][3])
        ++j;
      for (int q = 0; q < 4; ++q) R->groups.push_back(cf[i][q]);
      R->group_sizes.push_back((int32_t)(j - i));
      for (int64_t t = i; t < j; ++t) R->lanes.push_back((int32_t)cf[t][4]);
      maxg = std::max<int64_t>(maxg, j - i);
      const int64_t step = cf[i][0] - prog.first();
      if (step >= 0 && step < (int64_t)R->per_step_cost.size())
        R->per_step_cost[step] = std::max<int32_t>(R->per_step_cost[step], (int32_t)(j - i));
      i = j;
    }
  }
  R->sum.records = nrec;
  R->sum.hazards = nhaz;
  R->sum.conflict_groups = (int64_t)R->group_sizes.size();
  R->sum.conflict_lanes = (int64_t)R->lanes.size();
  R->sum.max_group_size = maxg;
  R->sum.stall_heads = nstall;
  if (summary) *summary = R->sum;
  if (run_out)
    *run_out = R;
  else
    delete R;
  return PIPEDP_OK;
}

}  // namespace

extern "C" {

int32_t pipedp_mcm_engine(const int64_t* dims, int64_t dims_len, int32_t mode, int32_t flags,
                          int64_t* cells_out, pipedp_engine_summary* summary, pipedp_engine_t* run_out) {
  if (run_out) *run_out = nullptr;
  TRY(validate_mcm(dims, dims_len));
  const int64_t n = dims_len - 1;
  if (n < 2) return fail(PIPEDP_E_INVALID_PARAMS, "pipeline needs at least two matrices");  // mcm_pipeline.cpp:28
  if (mode != PIPEDP_MCM_PAPER_LITERAL && mode != PIPEDP_MCM_STALL_ON_HAZARD)
    return fail(PIPEDP_E_INVALID_PARAMS, "unknown McmMode %d", mode);
  TRY(select_device(-1));
  const int64_t cc = n * (n + 1) / 2;
  Scope sc;
  TRY(sc.init());
  int64_t* d_dims;
  int32_t *d_row, *d_diag;
  TRY(sc.alloc(&d_dims, n + 1));
  TRY(sc.alloc(&d_row, cc + 1));
  TRY(sc.alloc(&d_diag, cc + 1));
  CK(cudaMemcpyAsync(d_dims, dims, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, sc.stream));
  eng_coord_table<<<(unsigned)std::min<int64_t>(4096, (cc + 255) / 256), 256, 0, sc.stream>>>(n, d_row, d_diag);
  CK(cudaGetLastError());
  EngMcm prog{n, d_dims, d_row, d_diag};
  const int64_t relax = (n * n * n - n) / 6;
  const int64_t records = 4 * relax - (cc - n);  // lane 1 has no substep-4 read
  return engine_run(prog, mode == PIPEDP_MCM_STALL_ON_HAZARD, flags, nullptr, 0, cells_out, summary, run_out,
                    records, sc);
}

int32_t pipedp_sdp_engine(const int64_t* offsets, int64_t k, const int64_t* init, int64_t init_len, int64_t n,
                          int32_t op, int32_t flags, int64_t* cells_out, pipedp_engine_summary* summary,
                          pipedp_engine_t* run_out) {
  if (run_out) *run_out = nullptr;
  TRY(validate_sdp(offsets, k, init_len, n));
  if (op < 0 || op > 3) return fail(PIPEDP_E_INVALID_PARAMS, "unknown operator %d", op);
  TRY(select_device(-1));
  Scope sc;
  TRY(sc.init());
  int64_t* d_offs;
  TRY(sc.alloc(&d_offs, k));
  CK(cudaMemcpyAsync(d_offs, offsets, sizeof(int64_t) * k, cudaMemcpyHostToDevice, sc.stream));
  EngSdp prog{n, k, offsets[0], d_offs, op};
  const int64_t records = (n - offsets[0]) * (3 * k - 1);  // lane 1: one read + write
  return engine_run(prog, 0, flags, init, init_len, cells_out, summary, run_out, records, sc);
}

int32_t pipedp_mcm_pipeline(const int64_t* dims, int64_t dims_len, int32_t mode, int64_t* cells_out,
                            uint8_t* filled_out, int64_t* steps_out, int64_t* stall_out) {
  pipedp_engine_summary s{};
  TRY(pipedp_mcm_engine(dims, dims_len, mode, 0, cells_out, &s, nullptr));
  if (filled_out) memset(filled_out, 1, (size_t)((dims_len - 1) * dims_len / 2 + 1));
  if (steps_out) *steps_out = s.steps_executed;
  if (stall_out) *stall_out = s.stall_iterations;
  return PIPEDP_OK;
}

int32_t pipedp_engine_records(pipedp_engine_t R, int64_t* head, int32_t* substep, int32_t* lane, int32_t* kind,
                              int64_t* address) {
  if (!R) return fail(PIPEDP_E_INVALID_PARAMS, "null engine run");
  for (int64_t i = 0; i < R->sum.records; ++i) {
    const int32_t m = R->rec_meta[i];
    if (head) head[i] = R->rec_head[i];
    if (substep) substep[i] = (m >> 1) & 0x7f;
    if (lane) lane[i] = m >> 8;
    if (kind) kind[i] = m & 1;
    if (address) address[i] = R->rec_addr[i];
  }
  return PIPEDP_OK;
}

int32_t pipedp_engine_hazards(pipedp_engine_t R, int64_t* out) {
  if (!R) return fail(PIPEDP_E_INVALID_PARAMS, "null engine run");
  if (out && !R->haz.empty()) memcpy(out, R->haz.data(), 8 * R->haz.size());
  return PIPEDP_OK;
}

int32_t pipedp_engine_conflicts(pipedp_engine_t R, int64_t* groups, int32_t* group_sizes, int32_t* lanes,
                                int32_t* per_step_cost) {
  if (!R) return fail(PIPEDP_E_INVALID_PARAMS, "null engine run");
  if (groups && !R->groups.empty()) memcpy(groups, R->groups.data(), 8 * R->groups.size());
  if (group_sizes && !R->group_sizes.empty())
    memcpy(group_sizes, R->group_sizes.data(), 4 * R->group_sizes.size());
  if (lanes && !R->lanes.empty()) memcpy(lanes, R->lanes.data(), 4 * R->lanes.size());
  if (per_step_cost && !R->per_step_cost.empty())
    memcpy(per_step_cost, R->per_step_cost.data(), 4 * R->per_step_cost.size());
  return PIPEDP_OK;
}

int32_t pipedp_engine_stall_heads(pipedp_engine_t R, int64_t* out) {
  if (!R) return fail(PIPEDP_E_INVALID_PARAMS, "null engine run");
  if (out && !R->stall_heads.empty()) memcpy(out, R->stall_heads.data(), 8 * R->stall_heads.size());
  return PIPEDP_OK;
}

void pipedp_engine_free(pipedp_engine_t R) { delete R; }

}  // extern "C"

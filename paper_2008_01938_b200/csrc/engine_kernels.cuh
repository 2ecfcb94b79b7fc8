// engine_kernels.cuh -- the reference's lock-step pipeline engine
// (engine.hpp:124-433) as one persistent GPU kernel, with the trace analyses of
// analysis.cpp computed on the device while the schedule runs.
//
// What it reproduces, iteration for iteration:
//  * `Run::plan_all` / `ready` (engine.hpp:304-350): each lane's next action
//    at its own virtual head; in stall mode a lane holds until every operand
//    it does not write has seen all of its program writes and every
//    program-order-earlier write to its own target has executed;
//  * `exec_substep` / `apply_writes` (engine.hpp:364-397): reads observe the
//    table as of the previous substep boundary, writes land at the boundary.
//    Both programs write only in their last substep, so all reads of an
//    iteration run before all of its writes (phase A / phase B below);
//  * `finish_iteration` / `check_progress` (engine.hpp:352-362, 399-415):
//    stall heads, per-lane head advance, the livelock guard and budget.
//
// What the device adds in place of trace post-processing:
//  * access records (head = iteration head, substep, lane, kind, address)
//    appended to a buffer (the host sorts them into record_less order);
//  * hazard records (detect_hazards, analysis.cpp:72-103): a non-own read of
//    an address whose program writes are not all done at the start of the
//    iteration is a read at or before that address's last write; its
//    finalisation head is filled in after the run from the per-address last
//    write head;
//  * conflict entries (detect_conflicts, analysis.cpp:31-70): per iteration,
//    per (substep, kind) class and address, a counter of touching lanes; every
//    access whose counter ends >= 2 is emitted (the host groups them).
//
// The two programs are the reference's McmProgram (mcm_pipeline.hpp:22-84)
// and SdpProgram (sdp_pipeline.hpp:16-58), restated as device plan/eval
// functions.  One lane per thread slot, lanes strided over a cooperative grid
// (one CTA per SM at most) with two grid barriers per iteration; a single CTA
// uses __syncthreads.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace pipedp_dev {

struct EngAccess {
  int64_t addr;
  int sub;   // 1-based substep
  int kind;  // 0 read, 1 write (AccessKind order)
};

__host__ __device__ __forceinline__ int64_t eng_dbase(int64_t d, int64_t n) { return d * n - d * (d - 1) / 2; }

// McmProgram (mcm_pipeline.hpp:22-84).  Lane j at head h works on cell
// h - j + 1 if it is a computed cell with at least j terms.
struct EngMcm {
  int64_t n;
  const int64_t* dims;
  const int32_t* row;   // [cc+1] coord table
  const int32_t* diag;  // [cc+1]
  static constexpr int kWriteSub = 4;

  __host__ __device__ int64_t first() const { return n + 1; }
  __host__ __device__ int64_t last() const { return n * (n + 1) / 2 + n - 2; }
  __host__ __device__ int64_t lanes() const { return n - 1; }
  __host__ __device__ int64_t tsize() const { return n * (n + 1) / 2 + 1; }

  __device__ __forceinline__ bool plan(int64_t head, int64_t j, EngAccess* a, int& na, int64_t& target,
                                       int64_t& payload) const {
    const int64_t cell = head - j + 1;
    if (cell < n + 1 || cell > n * (n + 1) / 2) return false;
    const int64_t D = diag[cell];
    if (j > D) return false;
    const int64_t r = row[cell], c = r + D;
    a[0] = {eng_dbase(j - 1, n) + r, 1, 0};      // v_l <- left
    a[1] = {eng_dbase(D - j, n) + r + j, 2, 0};  // v_r <- right
    na = 2;
    if (j > 1) a[na++] = {cell, 4, 0};           // min-fold reads the cell
    a[na++] = {cell, 4, 1};
    target = cell;
    payload = dims[r - 1] * dims[r + j - 1] * dims[c];
    return true;
  }
  // values in access order (reads only)
  __device__ __forceinline__ int64_t eval(int64_t j, const int64_t* v, int64_t payload) const {
    const int64_t s = v[0] + v[1] + payload;
    return j == 1 ? s : (v[2] < s ? v[2] : s);
  }
  // program writes per address (writers_ sizes) and the rank of (head, j)
  // among its target's writers (lane j is the j-th writer of its cell)
  __device__ __forceinline__ int64_t writes_total(int64_t addr) const { return addr > n ? diag[addr] : 0; }
  __device__ __forceinline__ int64_t write_rank(int64_t /*head*/, int64_t j) const { return j - 1; }
};

// SdpProgram (sdp_pipeline.hpp:16-58): lane j at head h owns cell h - j + 1.
struct EngSdp {
  int64_t n, k, a1;
  const int64_t* offs;
  int op;
  static constexpr int kWriteSub = 1;

  __host__ __device__ int64_t first() const { return a1; }
  __host__ __device__ int64_t last() const { return n + k - 2; }
  __host__ __device__ int64_t lanes() const { return k; }
  __host__ __device__ int64_t tsize() const { return n; }

  __device__ __forceinline__ bool plan(int64_t head, int64_t j, EngAccess* a, int& na, int64_t& target,
                                       int64_t& payload) const {
    const int64_t cell = head - j + 1;
    if (cell < a1 || cell >= n) return false;
    if (j == 1) {
      a[0] = {cell - a1, 1, 0};
      na = 1;
    } else {
      a[0] = {cell, 1, 0};  // own partial value
      a[1] = {cell - offs[j - 1], 1, 0};
      na = 2;
    }
    a[na++] = {cell, 1, 1};
    target = cell;
    payload = 0;
    return true;
  }
  __device__ __forceinline__ int64_t eval(int64_t j, const int64_t* v, int64_t) const {
    if (j == 1) return v[0];
    switch (op) {
      case kMin: return SemiOp<kMin, int64_t>::apply(v[0], v[1]);
      case kMax: return SemiOp<kMax, int64_t>::apply(v[0], v[1]);
      case kSatAdd: return SemiOp<kSatAdd, int64_t>::apply(v[0], v[1]);
      default: return SemiOp<kModAdd, int64_t>::apply(v[0], v[1]);
    }
  }
  __device__ __forceinline__ int64_t writes_total(int64_t addr) const { return addr >= a1 ? k : 0; }
  __device__ __forceinline__ int64_t write_rank(int64_t, int64_t j) const { return j - 1; }
};

enum : int { kEngTrace = 1, kEngAnalysis = 2 };

struct EngState {
  int stall;
  int flags;  // kEngTrace | kEngAnalysis
  int64_t budget;
  int64_t* cells;      // [tsize]
  int32_t* wdone;      // [tsize] writes executed per address
  int64_t* lastw;      // [tsize] iteration head of the latest write
  int64_t* vhead;      // [lanes+1]
  int8_t* lstate;      // [lanes+1] 0 running, 1 done
  int8_t* exec;        // [lanes+1] this iteration: 0 held, 1 executes, 2 inactive no-op
  int64_t* wval;       // [lanes+1]
  int64_t* wtarget;    // [lanes+1]
  int32_t* cnt;        // [2][8][tsize] conflict counters (analysis only)
  int64_t* pend;       // [lanes+1][4] last iteration's counted (class << 58 | addr), -1 none
  int* flags_it;       // [2][4] per parity: not-done, executed, held
  unsigned* bar;       // [2] grid barrier
  // outputs
  int64_t* rec_head;   // trace
  int64_t* rec_addr;
  int32_t* rec_meta;   // lane << 8 | substep << 1 | kind
  int64_t rec_cap;
  int64_t* haz;        // [cap][6] head, substep, lane, address, fin head, fin substep
  int64_t haz_cap;
  int64_t* conf;       // [cap][5] head, substep, kind, address, lane
  int64_t conf_cap;
  int64_t* stall_heads;
  int64_t stall_cap;
  unsigned long long* counts;  // [4] records, hazards, conflict entries, stall heads
  int64_t* result;     // [2] steps, error (1 livelock: no progress, 2 budget)
};

__device__ __forceinline__ void eng_grid_sync(unsigned* bar) {
  if (gridDim.x == 1) {
    __syncthreads();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = (unsigned)ld_relaxed_gpu_i32(reinterpret_cast<const int*>(bar + 1));
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while ((unsigned)ld_relaxed_gpu_i32(reinterpret_cast<const int*>(bar + 1)) == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int eng_class(const EngAccess& a) { return (a.sub - 1) * 2 + a.kind; }

template <class P>
__global__ void __launch_bounds__(512, 1) engine_kernel(const P prog, const EngState S) {
  const int64_t first = prog.first(), last = prog.last(), lanes = prog.lanes(), ts = prog.tsize();
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  const bool analysis = S.flags & kEngAnalysis, trace = S.flags & kEngTrace;
  __shared__ int s_cnt[3];
  int64_t steps = 0;
  for (;;) {
    const int par = (int)(steps & 1);
    const int64_t iter_head = first + steps;
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    int notdone = 0, executed = 0, held = 0;
    // ---- phase A: plan, ready, reads (+ records, hazards, conflict counts)
    for (int64_t j = gtid + 1; j <= lanes; j += gthreads) {
      if (analysis) {  // clear last iteration's counters (other parity)
        int64_t* pe = S.pend + j * 4;
        for (int q = 0; q < 4; ++q) {
          const int64_t e = pe[q];
          if (e >= 0) {
            S.cnt[((int64_t)((par ^ 1) * 8 + (int)(e >> 58))) * ts + (e & ((1ll << 58) - 1))] = 0;
            pe[q] = -1;
          }
        }
      }
      if (S.lstate[j]) continue;
      ++notdone;
      const int64_t vh = S.vhead[j];
      EngAccess acc[4];
      int na = 0;
      int64_t target = -1, payload = 0;
      if (!prog.plan(vh, j, acc, na, target, payload)) {
        S.exec[j] = 2;  // inactive slot: consumes the iteration as a no-op
        ++executed;
        continue;
      }
      bool ready = true;
      if (S.stall) {
        for (int q = 0; q < na; ++q) {
          if (acc[q].kind != 0 || acc[q].addr == target) continue;
          if (S.wdone[acc[q].addr] < prog.writes_total(acc[q].addr)) ready = false;
        }
        if (S.wdone[target] != prog.write_rank(vh, j)) ready = false;
      }
      if (!ready) {
        S.exec[j] = 0;
        ++held;
        continue;
      }
      S.exec[j] = 1;
      ++executed;
      int64_t v[3];
      int nv = 0;
      for (int q = 0; q < na; ++q) {
        const EngAccess& a = acc[q];
        if (a.kind == 0) {
          v[nv++] = S.cells[a.addr];
          if (a.addr != target) {
            const int64_t tot = prog.writes_total(a.addr);
            if (tot > 0 && S.wdone[a.addr] < tot) {
              const unsigned long long h = atomicAdd(S.counts + 1, 1ull);
              if ((int64_t)h < S.haz_cap) {
                int64_t* o = S.haz + h * 6;
                o[0] = iter_head; o[1] = a.sub; o[2] = j; o[3] = a.addr; o[4] = -1; o[5] = P::kWriteSub;
              }
            }
          }
        }
        if (trace) {
          const unsigned long long r = atomicAdd(S.counts + 0, 1ull);
          if ((int64_t)r < S.rec_cap) {
            S.rec_head[r] = iter_head;
            S.rec_addr[r] = a.addr;
            S.rec_meta[r] = (int32_t)((j << 8) | (a.sub << 1) | a.kind);
          }
        }
        if (analysis) {
          const int c = eng_class(a);
          atomicAdd(S.cnt + (int64_t)(par * 8 + c) * ts + a.addr, 1);
          S.pend[j * 4 + q] = ((int64_t)c << 58) | a.addr;
        }
      }
      S.wval[j] = prog.eval(j, v, payload);
      S.wtarget[j] = target;
    }
    // block totals -> global per-parity flags
    if (notdone) atomicAdd(&s_cnt[0], notdone);
    if (executed) atomicAdd(&s_cnt[1], executed);
    if (held) atomicAdd(&s_cnt[2], held);
    __syncthreads();
    if (threadIdx.x < 3 && s_cnt[threadIdx.x]) atomicAdd(S.flags_it + par * 4 + threadIdx.x, s_cnt[threadIdx.x]);
    eng_grid_sync(S.bar);
    // ---- phase B: progress checks, writes, conflict entries, head advance
    const int g_notdone = ld_relaxed_gpu_i32(S.flags_it + par * 4 + 0);
    const int g_exec = ld_relaxed_gpu_i32(S.flags_it + par * 4 + 1);
    const int g_held = ld_relaxed_gpu_i32(S.flags_it + par * 4 + 2);
    if (g_notdone == 0) break;
    if (g_exec == 0 || steps > S.budget) {  // check_progress (engine.hpp:352-362)
      if (gtid == 0) S.result[1] = g_exec == 0 ? 1 : 2;
      return;
    }
    if (gtid == 0) {
      int* other = S.flags_it + (par ^ 1) * 4;
      other[0] = other[1] = other[2] = 0;
      if (g_held) {
        const unsigned long long h = atomicAdd(S.counts + 3, 1ull);
        if ((int64_t)h < S.stall_cap) S.stall_heads[h] = iter_head;
      }
    }
    for (int64_t j = gtid + 1; j <= lanes; j += gthreads) {
      if (S.lstate[j]) continue;
      const int e = S.exec[j];
      if (e == 1) {
        const int64_t t = S.wtarget[j];
        S.cells[t] = S.wval[j];
        S.wdone[t] += 1;
        S.lastw[t] = iter_head;
        if (analysis) {
          const int64_t* pe = S.pend + j * 4;
          for (int q = 0; q < 4; ++q) {
            const int64_t en = pe[q];
            if (en < 0) continue;
            const int c = (int)(en >> 58);
            const int64_t addr = en & ((1ll << 58) - 1);
            if (S.cnt[(int64_t)(par * 8 + c) * ts + addr] >= 2) {
              const unsigned long long h = atomicAdd(S.counts + 2, 1ull);
              if ((int64_t)h < S.conf_cap) {
                int64_t* o = S.conf + h * 5;
                o[0] = iter_head; o[1] = c / 2 + 1; o[2] = c & 1; o[3] = addr; o[4] = j;
              }
            }
          }
        }
      }
      if (e != 0) {
        const int64_t nh = S.vhead[j] + 1;
        S.vhead[j] = nh;
        if (nh > last) S.lstate[j] = 1;
      }
    }
    ++steps;
    eng_grid_sync(S.bar);
  }
  if (gtid == 0) {
    S.result[0] = steps;
    S.result[1] = 0;
  }
}

// hazard finalisation heads from the per-address last write
__global__ void engine_fix_hazards(int64_t* haz, int64_t count, const int64_t* lastw) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    haz[i * 6 + 4] = lastw[haz[i * 6 + 3]];
}

}  // namespace pipedp_dev

namespace pipedp_dev {

// coord (mcm.cpp:39-53) for every address at once: row and diagonal tables
__global__ void eng_coord_table(int64_t n, int32_t* row, int32_t* diag) {
  const int64_t cc = n * (n + 1) / 2;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; a <= cc;
       a += (int64_t)gridDim.x * blockDim.x) {
    const double nn = (double)n + 0.5;
    int64_t D = (int64_t)(nn - sqrt(nn * nn - 2.0 * (double)(a - 1)));
    if (D < 0) D = 0;
    if (D > n - 1) D = n - 1;
    while (D > 0 && eng_dbase(D, n) >= a) --D;
    while (D + 1 <= n - 1 && eng_dbase(D + 1, n) < a) ++D;
    row[a] = (int32_t)(a - eng_dbase(D, n));
    diag[a] = (int32_t)D;
  }
}

}  // namespace pipedp_dev

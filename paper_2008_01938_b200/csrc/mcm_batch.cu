// mcm_batch.cu -- batched small-n MCM (BASELINE config 5a: 65,536 instances
// of n = 64), one WARP per instance.
//
// Same recurrence and tie rule as solve_mcm_sequential (mcm.cpp:85-110): cell
// (r, c) on diagonal D = c - r takes the first j (1-based) minimising
//   m[r][r+j-1] + m[r+j][c] + p[r-1] p[r+j-1] p[c].
// The instance's triangle lives in shared memory twice, so both operand runs
// of a cell are contiguous:
//   row copy:    (m[r][k], p[k]) pairs, row r from k = r on  -> one 8-byte LDS
//                gives the left operand AND its weight factor;
//   column copy: m[i][c], column c from i = 1 on             -> one 4-byte LDS
// i.e. two shared-memory loads per term and no per-term index arithmetic.
// A diagonal's cells spread over the 32 lanes (G lanes per cell on the short
// diagonals, several cells per lane on the long ones); each lane scans its
// terms j ascending with strict '<', and the G partials reduce
// lexicographically on (value, j) -- the reference's first minimum.  The warp
// synchronises per diagonal with __syncwarp only: no CTA barrier, no idle
// threads of other cells.  32-bit values; a cell >= 2^30 raises the overflow
// flag and the host recomputes the batch exactly in 64 bits.
#include "mcm_batch.hpp"

#include <cstdint>

#include "common.cuh"

namespace pipedp_mcmb {

constexpr int kWarps = 1;  // 25 KB of shared memory per instance: nine warps per SM
constexpr int kTri = kMaxN * (kMaxN + 1) / 2;  // 2080 entries
constexpr uint32_t kLimit = 1u << 30;

// One diagonal with G lanes per cell (G a compile-time stride: the unrolled
// term loop addresses its operands with immediate offsets).
template <int G>
__device__ __forceinline__ bool diag_pass(int n, int D, int ncell, int lane, uint2* R, uint32_t* Cm,
                                          const uint32_t* p, int64_t* oc, int64_t* os) {
  bool ovf = false;
  constexpr int kCells = 32 / G;
  const int q = lane & (G - 1);
  for (int base = 0; base < ncell; base += kCells) {
    const int r = 1 + base + lane / G, c = r + D;
    const bool live = r <= ncell;
    uint32_t bv = 0xFFFFFFFFu;
    int32_t bj = 0;
    if (live) {
      const uint32_t prc = p[r - 1] * p[c];
      const uint2* L = R + (r - 1) * (n + 1) - r * (r - 1) / 2 - 1 + q;  // L[G t] = (m[r][r+j-1], p[r+j-1]), j = 1+q+G t
      const uint32_t* Cc = Cm + c * (c - 1) / 2 + r - 1 + q;           // Cc[G t] = m[r+j][c]
      const int cnt = (D - q + G - 1) / G;                               // terms of this lane
#pragma unroll 4
      for (int t = 0; t < cnt; ++t) {
        const uint2 lv = L[1 + G * t];
        const uint32_t cost = lv.x + Cc[1 + G * t] + prc * lv.y;
        if (cost < bv) {  // j ascending in this lane: first minimum
          bv = cost;
          bj = 1 + q + G * t;
        }
      }
    }
#pragma unroll
    for (int sh = G >> 1; sh > 0; sh >>= 1) {  // lexicographic (value, j)
      const uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, sh);
      const int32_t oj = __shfl_xor_sync(0xffffffffu, bj, sh);
      if (ov < bv || (ov == bv && oj < bj)) {
        bv = ov;
        bj = oj;
      }
    }
    if (live && q == 0) {
      R[(r - 1) * (n + 1) - r * (r - 1) / 2 + D].x = bv;  // m[r][c]
      Cm[c * (c - 1) / 2 + r - 1] = bv;
      oc[r] = (int64_t)bv;
      os[r] = bj;
      ovf |= bv >= kLimit;
    }
  }
  return ovf;
}

__global__ void __launch_bounds__(32 * kWarps) mcm_batch_warp(int32_t n, int64_t batch,
                                                             const int64_t* __restrict__ g_dims,
                                                             int64_t* __restrict__ out_cells,
                                                             int64_t* __restrict__ out_split,
                                                             int* __restrict__ overflow) {
  __shared__ uint2 s_row[kWarps][kTri];      // (m[r][k], p[k])
  __shared__ uint32_t s_col[kWarps][kTri];   // m[i][c]
  __shared__ uint32_t s_p[kWarps][kMaxN + 1];
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int64_t inst = (int64_t)blockIdx.x * kWarps + warp;
  if (inst >= batch) return;
  uint2* R = s_row[warp];
  uint32_t* Cm = s_col[warp];
  uint32_t* p = s_p[warp];
  const int64_t cc = (int64_t)n * (n + 1) / 2;
  const int64_t* gd = g_dims + inst * (n + 1);
  int64_t* oc = out_cells + inst * (cc + 1);
  int64_t* os = out_split + inst * (cc + 1);
  for (int i = lane; i <= n; i += 32) {
    p[i] = (uint32_t)gd[i];
    oc[i] = 0;  // slot 0 and the base cells (mcm.cpp:77-83)
    os[i] = 0;
  }
  __syncwarp();
  // rows: entry (r, k), k >= r, at rowoff(r) + k - r with rowoff(r) = (r-1)(n+1) - r(r-1)/2;
  // columns: entry (i, c), i <= c, at coloff(c) + i - 1 with coloff(c) = c(c-1)/2
  for (int r = 1; r <= n; ++r) {
    const int ro = (r - 1) * (n + 1) - r * (r - 1) / 2;
    for (int k = r + lane; k <= n; k += 32) R[ro + k - r] = make_uint2(0u, p[k]);
  }
  for (int c = 1 + lane; c <= n; c += 32) Cm[c * (c - 1) / 2 + c - 1] = 0u;  // m[c][c] = 0
  __syncwarp();
  bool ovf = false;
  int64_t db = 0;  // lin(r, r+D) = db(D) + r
  for (int D = 1; D < n; ++D) {
    db += n - (D - 1);
    const int ncell = n - D;
    int lg = 0;  // G = 2^lg lanes per cell
    while (lg < 5 && (ncell << (lg + 1)) <= 32 && (1 << lg) < D) ++lg;
    switch (lg) {
      case 0: ovf |= diag_pass<1>(n, D, ncell, lane, R, Cm, p, oc + db, os + db); break;
      case 1: ovf |= diag_pass<2>(n, D, ncell, lane, R, Cm, p, oc + db, os + db); break;
      case 2: ovf |= diag_pass<4>(n, D, ncell, lane, R, Cm, p, oc + db, os + db); break;
      case 3: ovf |= diag_pass<8>(n, D, ncell, lane, R, Cm, p, oc + db, os + db); break;
      case 4: ovf |= diag_pass<16>(n, D, ncell, lane, R, Cm, p, oc + db, os + db); break;
      default: ovf |= diag_pass<32>(n, D, ncell, lane, R, Cm, p, oc + db, os + db); break;
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(overflow, 1);
}

cudaError_t launch(int32_t n, int64_t batch, const int64_t* d_dims, int64_t* d_cells, int64_t* d_split,
                   int* d_overflow, cudaStream_t st) {
  // all of the SM's 228 KB as shared memory: nine instances per SM
  cudaError_t e = cudaFuncSetAttribute(mcm_batch_warp, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  mcm_batch_warp<<<(unsigned)((batch + kWarps - 1) / kWarps), 32 * kWarps, 0, st>>>(n, batch, d_dims, d_cells,
                                                                                   d_split, d_overflow);
  return cudaGetLastError();
}

}  // namespace pipedp_mcmb

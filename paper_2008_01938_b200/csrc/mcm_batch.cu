// mcm_batch.cu -- batched small-n MCM (BASELINE config 5a: 65,536 instances
// of n = 64), one WARP per instance, terms folded as packed keys.
//
// Same recurrence and tie rule as solve_mcm_sequential (mcm.cpp:85-110): cell
// (r, c) on diagonal D = c - r takes the first j (1-based) minimising
//   m[r][r+j-1] + m[r+j][c] + p[r-1] p[r+j-1] p[c].
//
// Key arithmetic.  Every table entry is held as M'[a][b] = (m[a][b] << 6) | (b & 63)
// and every dimension as p''[k] = p[k] << 6.  For split column k = r + j - 1
// of cell (r, c) (k < c <= 64, so k < 64):
//   M'[r][k] + M'[k+1][c] + p[r-1] p[c] * p''[k] - (c & 63)
//     = ((m[r][k] + m[k+1][c] + p[r-1] p[k] p[c]) << 6) | k
// exactly (mod 2^32, and exact whenever the cost < 2^26): the low field of the
// left operand is k, the right operand's is c & 63 and is cancelled by a
// per-cell constant.  One unsigned min over these keys is the lexicographic
// (cost, k) minimum, i.e. the reference's first minimum (j ascending = k
// ascending).  Per term: three 4-byte shared loads, IMAD, IADD3 and half a
// three-way min -- no index bookkeeping and no serial compare/select chain, so
// the terms of a lane fold into two independent accumulators.
//
// Validity (as mcm_smem_square's packed mode): the host admits the kernel only
// when every weight p[r-1] p[k] p[c] < 2^24; a cell >= 2^24 raises overflow
// bit 2 and the host reruns the launch with the unpacked kernel.  By induction
// over the diagonals every candidate of an unflagged run is < 3 * 2^24 < 2^26,
// so no key wrapped.
//
// Layout: the (n+1) x P square, P even: the row walk M'[r][r+q+Gt] and the
// column walk M'[r+1+q+Gt][c] of the 32 cells of a pass (G = 1) land on 32
// distinct banks (bank = r (P+1) + const, P+1 odd).  A diagonal of ncell cells
// runs as passes of 32 cells (one lane each) and a remainder pass in which the
// last ncell mod 32 cells get G lanes each (G the largest power of two that
// fits), the G partial keys min-reduced by shuffles.  The warp synchronises
// per diagonal with __syncwarp only.
#include "mcm_batch.hpp"

#include <cstdint>

#include "common.cuh"

namespace pipedp_mcmb {

constexpr int kPitch = 66;                       // even, >= kMaxN + 1
constexpr int kSquare = (kMaxN + 1) * kPitch;    // words
constexpr uint32_t kCellLimit = 1u << 24;        // packed-key validity (see above)

struct Smem {
  uint32_t M[kSquare];
  uint32_t p[kMaxN + 2];    // raw dimensions
  uint32_t pk[kMaxN + 2];   // dimensions << 6
};

// Cells [base, base + 32 / G) of diagonal D (cells numbered from 0: r = 1 + i),
// G lanes per cell.  G is a compile-time stride so the unrolled term loop
// addresses its operands with immediate offsets.
template <int G>
__device__ __forceinline__ bool diag_pass(int n, int D, int base, int ncell, int lane, Smem& s, int64_t* oc,
                                          int64_t* os) {
  constexpr int kCells = 32 / G;
  (void)kCells;
  const int q = lane & (G - 1);
  const int r = 1 + base + lane / G, c = r + D;
  const bool live = base + lane / G < ncell;
  uint32_t k0 = 0xFFFFFFFFu, k1 = 0xFFFFFFFFu;
  if (live) {
    const uint32_t prc = s.p[r - 1] * s.p[c];
    const uint32_t negc = 0u - (uint32_t)(c & 63);  // the right operand's low field
    const uint32_t* L = s.M + r * kPitch + r + q;            // M'[r][k],   k = r + q + G t
    const uint32_t* R = s.M + (r + 1 + q) * kPitch + c;      // M'[k+1][c]
    const uint32_t* W = s.pk + r + q;                        // p''[k]
    const int cnt = (D - q + G - 1) / G;                     // this lane's terms
    int t = 0;
#pragma unroll 2
    for (; t + 2 <= cnt; t += 2) {
      const uint32_t a = prc * W[G * t] + L[G * t] + R[G * t * kPitch] + negc;
      const uint32_t b = prc * W[G * (t + 1)] + L[G * (t + 1)] + R[G * (t + 1) * kPitch] + negc;
      k0 = min(k0, a);
      k1 = min(k1, b);
    }
    if (t < cnt) k0 = min(k0, prc * W[G * t] + L[G * t] + R[G * t * kPitch] + negc);
  }
  uint32_t key = min(k0, k1);
#pragma unroll
  for (int sh = G >> 1; sh > 0; sh >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, sh));
  bool ovf = false;
  if (live && q == 0) {
    const uint32_t v = key >> 6;
    const int k = (int)(key & 63u);
    s.M[r * kPitch + c] = (key & ~63u) | (uint32_t)(c & 63);
    oc[r] = (int64_t)v;
    os[r] = k - r + 1;
    ovf = v >= kCellLimit;
  }
  return ovf;
}

__global__ void __launch_bounds__(32) mcm_batch_warp(int32_t n, int64_t batch, const int64_t* __restrict__ g_dims,
                                                    int64_t* __restrict__ out_cells, int64_t* __restrict__ out_split,
                                                    int* __restrict__ overflow) {
  __shared__ Smem s;
  const int lane = threadIdx.x;
  const int64_t inst = blockIdx.x;
  if (inst >= batch) return;
  const int64_t cc = (int64_t)n * (n + 1) / 2;
  const int64_t* gd = g_dims + inst * (n + 1);
  int64_t* oc = out_cells + inst * (cc + 1);
  int64_t* os = out_split + inst * (cc + 1);
  for (int i = lane; i <= n; i += 32) {
    const uint32_t d = (uint32_t)gd[i];
    s.p[i] = d;
    s.pk[i] = d << 6;
    s.M[i * kPitch + i] = (uint32_t)(i & 63);  // base cells m[i][i] = 0 (row 0 unused)
    oc[i] = 0;  // slot 0 and the base cells (mcm.cpp:77-83)
    os[i] = 0;
  }
  __syncwarp();
  bool ovf = false;
  int64_t db = 0;  // lin(r, r+D) = db(D) + r
  for (int D = 1; D < n; ++D) {
    db += n - (D - 1);
    const int ncell = n - D;
    int base = 0;
    for (; base + 32 <= ncell; base += 32) ovf |= diag_pass<1>(n, D, base, ncell, lane, s, oc + db, os + db);
    const int rem = ncell - base;
    if (rem > 0) {
      int lg = 0;  // G = 2^lg lanes per remaining cell
      while (lg < 5 && (rem << (lg + 1)) <= 32 && (1 << lg) < D) ++lg;
      switch (lg) {
        case 0: ovf |= diag_pass<1>(n, D, base, ncell, lane, s, oc + db, os + db); break;
        case 1: ovf |= diag_pass<2>(n, D, base, ncell, lane, s, oc + db, os + db); break;
        case 2: ovf |= diag_pass<4>(n, D, base, ncell, lane, s, oc + db, os + db); break;
        case 3: ovf |= diag_pass<8>(n, D, base, ncell, lane, s, oc + db, os + db); break;
        case 4: ovf |= diag_pass<16>(n, D, base, ncell, lane, s, oc + db, os + db); break;
        default: ovf |= diag_pass<32>(n, D, base, ncell, lane, s, oc + db, os + db); break;
      }
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(overflow, 2);
}

cudaError_t launch(int32_t n, int64_t batch, const int64_t* d_dims, int64_t* d_cells, int64_t* d_split,
                   int* d_overflow, cudaStream_t st) {
  // all of the SM's 228 KB as shared memory: twelve instances per SM
  cudaError_t e = cudaFuncSetAttribute(mcm_batch_warp, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  mcm_batch_warp<<<(unsigned)batch, 32, 0, st>>>(n, batch, d_dims, d_cells, d_split, d_overflow);
  return cudaGetLastError();
}

}  // namespace pipedp_mcmb

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
// Layout: one (n+2) x P square, P even, holds TWO instances, one per warp of
// the CTA, at addr(r, c) = sg (P r + c) + gm:
//   instance A (sg = +1, gm = 0):  A(r, c) at [r][c]          (upper triangle)
//   instance B (sg = -1, gm = P(n+2) + n+1): B(r, c) at [n+2-r][n+1-c]
//                                  (point-reflected: strict lower triangle)
// A walks its terms k ascending from r, B descending from c-1; with the
// reflection both walks then move by +1 (left operand (r, k)) and +P (right
// operand (k+1, c)) per term, and B's weights are stored reversed, so ONE code
// path (same immediates) serves both warps -- two specialised copies thrash
// the instruction cache (measured: 12.8 no-instruction stalls per issue).
// The 32 cells of a pass (G = 1) land on 32 distinct banks in both layouts
// (bank = +-(P+1) r + const, P+1 odd).  Sharing the square halves the shared
// memory per instance: 22 instances (warps) per SM instead of 12 -- the
// kernel is latency-bound, so resident warps are what it runs on.  A diagonal
// of ncell cells runs as passes of 32 cells (one lane each) and a remainder
// pass in which the last ncell mod 32 cells get G lanes each (G the largest
// power of two that fits), the G partial keys min-reduced by shuffles.  Each
// warp synchronises per diagonal with __syncwarp only; the two warps never
// touch each other's cells.
#include "mcm_batch.hpp"

#include <cstdint>

#include "common.cuh"

namespace pipedp_mcmb {

constexpr int kPitch = 66;                          // even, >= kMaxN + 1
constexpr int kSquare = (kMaxN + 2) * kPitch;       // words (rows 0..n+1)
constexpr uint32_t kCellLimit = 1u << 24;           // packed-key validity (see above)
constexpr int kCtasPerSm = 11;                      // 11 x (19 + 1) KB of the 228 KB

struct Smem {
  uint32_t M[kSquare];
  uint32_t p[2][kMaxN + 2];    // raw dimensions, per instance
  uint32_t pk[2][kMaxN + 2];   // dimensions << 6 (instance B: reversed, [n+1-k])
};

// One warp's instance in the shared square (see the layout note).
struct Geo {
  int sg;              // +1 (A) or -1 (B)
  int gm;              // address offset
  int om;              // weight index offset: weight of k at pk[sg k + om]
  int spare;           // a column no cell of this instance uses (B's partial keys)
  uint32_t* M;
  const uint32_t* p;   // raw dimensions (natural order)
  const uint32_t* pk;  // weights << 6, walked +1 per term
  __device__ __forceinline__ int at(int r, int c) const { return sg * (kPitch * r + c) + gm; }
};

// Diagonals are taken in PAIRS (D, D+1): cell A = (r, r+D) and cell B =
// (r, r+D+1) of the same row share the left operand M'(r, k) and the weight
// p''[k] of every split column k in [r+1, r+D-1] -- all of those terms only
// read diagonals < D -- so one lane folds both cells' terms over that range
// with four loads per two terms (8 B per term instead of 12).  A's remaining
// term (k = r) is folded too; B's two remaining terms (k = r and k = r+D, whose
// operands lie on diagonal D) follow after the warp has finished diagonal D,
// from B's partial key parked in the square's spare column (col 0 for the
// upper-triangle instance, col P-1 for the reflected one: neither is a cell).
//
// Phase 1: cells [base, base + 32 / G) of diagonal D (r = 1 + i), G lanes
// per cell, G a compile-time stride (the term loop walks four pointers with
// immediate offsets).  The per-cell constant c & 63 (the right operand's low
// field) is taken off once after the fold: every sum is < 2^32 before it, so
// the min commutes.
template <int LGT>  // LGT >= 0: compile-time G = 2^LGT; LGT < 0: G = 2^lgr at run time (the rarer short passes)
__device__ __forceinline__ bool pair_pass(int D, int base, int nA, int lane, const Geo& g, int64_t* oc,
                                          int64_t* os, int lgr = 0) {
  const int lg = LGT >= 0 ? LGT : lgr;
  const int G = 1 << lg;
  const int SL = G, SR = G * kPitch;
  const int q = lane & (G - 1);
  const int i = base + lane / G;
  const int r = 1 + i, cA = r + D, cB = cA + 1;
  const bool liveA = i < nA, liveB = i + 1 < nA;
  uint32_t a0 = 0xFFFFFFFFu, a1 = 0xFFFFFFFFu, b0 = 0xFFFFFFFFu, b1 = 0xFFFFFFFFu;
  if (liveA) {
    const uint32_t pr = g.p[r - 1];
    const uint32_t prcA = pr * g.p[cA], prcB = pr * g.p[cB];  // p[n+1] is padding when !liveB
    if (q == 0) a0 = prcA * g.pk[g.sg * r + g.om] + g.M[g.at(r, r)] + g.M[g.at(r + 1, cA)];  // k = r
    const int kq = g.sg > 0 ? r + 1 + q : cA - 1 - q;  // this lane's first shared split column
    const uint32_t* L = g.M + g.at(r, kq);             // M'(r, k)
    const uint32_t* RA = g.M + g.at(kq + 1, cA);       // M'(k+1, cA)
    // M'(k+1, cB); without a cell B (cB = n+1) the walk would read the other
    // instance's spare column (harmless, unused -- but a cross-warp race to
    // racecheck): walk A's own column instead
    const uint32_t* RB = liveB ? RA + g.sg : RA;
    const uint32_t* W = g.pk + g.sg * kq + g.om;       // p''[k]
    int cnt = (D - 1 - q + G - 1) >> lg;               // this lane's shared columns
    for (; cnt >= 4; cnt -= 4) {
      const uint32_t l0 = L[0], w0 = W[0], l1 = L[SL], w1 = W[G];
      const uint32_t l2 = L[2 * SL], w2 = W[2 * G], l3 = L[3 * SL], w3 = W[3 * G];
      a0 = min(a0, prcA * w0 + l0 + RA[0]);
      b0 = min(b0, prcB * w0 + l0 + RB[0]);
      a1 = min(a1, prcA * w1 + l1 + RA[SR]);
      b1 = min(b1, prcB * w1 + l1 + RB[SR]);
      a0 = min(a0, prcA * w2 + l2 + RA[2 * SR]);
      b0 = min(b0, prcB * w2 + l2 + RB[2 * SR]);
      a1 = min(a1, prcA * w3 + l3 + RA[3 * SR]);
      b1 = min(b1, prcB * w3 + l3 + RB[3 * SR]);
      L += 4 * SL;
      RA += 4 * SR;
      RB += 4 * SR;
      W += 4 * G;
    }
    if (cnt >= 2) {
      cnt -= 2;
      const uint32_t l0 = L[0], w0 = W[0], l1 = L[SL], w1 = W[G];
      a0 = min(a0, prcA * w0 + l0 + RA[0]);
      b0 = min(b0, prcB * w0 + l0 + RB[0]);
      a1 = min(a1, prcA * w1 + l1 + RA[SR]);
      b1 = min(b1, prcB * w1 + l1 + RB[SR]);
      L += 2 * SL;
      RA += 2 * SR;
      RB += 2 * SR;
      W += 2 * G;
    }
    if (cnt) {
      const uint32_t l0 = L[0], w0 = W[0];
      a0 = min(a0, prcA * w0 + l0 + RA[0]);
      b0 = min(b0, prcB * w0 + l0 + RB[0]);
    }
  }
  uint32_t ka = min(a0, a1), kb = min(b0, b1);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    if (sh < G) {
      ka = min(ka, __shfl_xor_sync(0xffffffffu, ka, sh));
      kb = min(kb, __shfl_xor_sync(0xffffffffu, kb, sh));
    }
  }
  bool ovf = false;
  if (liveA && q == 0) {
    ka -= (uint32_t)(cA & 63);
    const uint32_t v = ka >> 6;
    g.M[g.at(r, cA)] = (ka & ~63u) | (uint32_t)(cA & 63);
    oc[r] = (int64_t)v;
    os[r] = (int64_t)(ka & 63u) - r + 1;
    ovf = v >= kCellLimit;
    if (liveB) g.M[kPitch * r + g.spare] = kb;  // B's partial (still carries + (cB & 63))
  }
  return ovf;
}

// Phase 2: B = (r, r+D+1) for r = 1 .. nB (nB <= 62: at most two cells per
// lane), its two terms on diagonal D.  Every address is affine in r along
// the diagonal, so the second cell's are the first's plus a constant.
__device__ __forceinline__ bool pair_finish(int D, int nB, int lane, const Geo& g, int64_t* oc, int64_t* os) {
  bool ovf = false;
  int r = 1 + lane;
  if (r > nB) return false;
  const int c = r + D + 1;
  const int step = 32 * g.sg * (kPitch + 1);  // (r, c) -> (r + 32, c + 32)
  const uint32_t* mrr = g.M + g.at(r, r);
  const uint32_t* mr1c = g.M + g.at(r + 1, c);
  const uint32_t* mrc1 = g.M + g.at(r, c - 1);
  const uint32_t* mcc = g.M + g.at(c, c);
  uint32_t* mrc = g.M + g.at(r, c);
  uint32_t* sp = g.M + kPitch * r + g.spare;
  const uint32_t* w1 = g.pk + g.sg * r + g.om;
  const uint32_t* w2 = g.pk + g.sg * (c - 1) + g.om;
  const uint32_t* pr = g.p + r - 1;
  int cc = c;
#pragma unroll 1
  for (;;) {
    const uint32_t prc = pr[0] * pr[D + 2];
    uint32_t key = min(sp[0], prc * w1[0] + mrr[0] + mr1c[0]);  // k = r
    key = min(key, prc * w2[0] + mrc1[0] + mcc[0]);               // k = c - 1
    key -= (uint32_t)(cc & 63);
    const uint32_t v = key >> 6;
    mrc[0] = (key & ~63u) | (uint32_t)(cc & 63);
    oc[r] = (int64_t)v;
    os[r] = (int64_t)(key & 63u) - r + 1;
    ovf |= v >= kCellLimit;
    r += 32;
    if (r > nB) break;
    cc += 32;
    mrr += step;
    mr1c += step;
    mrc1 += step;
    mcc += step;
    mrc += step;
    sp += 32 * kPitch;
    w1 += 32 * g.sg;
    w2 += 32 * g.sg;
    pr += 32;
  }
  return ovf;
}

__global__ void __launch_bounds__(64, kCtasPerSm) mcm_batch_warp(int32_t n, int64_t batch,
                                                                 const int64_t* __restrict__ g_dims,
                                                                 int64_t* __restrict__ out_cells,
                                                                 int64_t* __restrict__ out_split,
                                                                 int* __restrict__ overflow) {
  __shared__ Smem s;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform
  const int64_t inst = 2 * (int64_t)blockIdx.x + warp;
  if (inst >= batch) return;
  const int64_t cc = (int64_t)n * (n + 1) / 2;
  const int64_t* gd = g_dims + inst * (n + 1);
  int64_t* oc = out_cells + inst * (cc + 1);
  int64_t* os = out_split + inst * (cc + 1);
  Geo g;
  g.sg = warp == 0 ? 1 : -1;
  g.gm = warp == 0 ? 0 : kPitch * (n + 2) + n + 1;
  g.om = warp == 0 ? 0 : n + 1;
  g.spare = warp == 0 ? 0 : kPitch - 1;
  g.M = s.M;
  g.p = s.p[warp];
  g.pk = s.pk[warp];
  for (int i = lane; i <= kMaxN + 1; i += 32) {
    const uint32_t d = i <= n ? (uint32_t)gd[i] : 0u;
    s.p[warp][i] = d;
    if (i <= n) s.pk[warp][g.sg * i + g.om] = d << 6;
    if (i >= 1 && i <= n) s.M[g.at(i, i)] = (uint32_t)(i & 63);  // base cells m[i][i] = 0
    if (i <= n) {
      oc[i] = 0;  // slot 0 and the base cells (mcm.cpp:77-83)
      os[i] = 0;
    }
  }
  __syncwarp();
  bool ovf = false;
  int64_t db = 0;  // lin(r, r+D) = db(D) + r
  for (int D = 1; D < n; D += 2) {
    db += n - (D - 1);
    const int nA = n - D;  // cells on diagonal D (B: nA - 1 on D + 1)
    int base = 0;
    for (; base + 32 <= nA; base += 32) ovf |= pair_pass<0>(D, base, nA, lane, g, oc + db, os + db);
    const int rem = nA - base;
    if (rem > 0) {
      // G = 2^lg lanes per remaining cell: rem G <= 32, and G / 2 < D
      const int lg = min(5 - (rem > 1 ? 32 - __clz(rem - 1) : 0), D > 1 ? 32 - __clz(D - 1) : 0);
      if (lg == 0) ovf |= pair_pass<0>(D, base, nA, lane, g, oc + db, os + db);
      else ovf |= pair_pass<-1>(D, base, nA, lane, g, oc + db, os + db, lg);
    }
    __syncwarp();
    if (nA > 1) {
      db += n - D;
      ovf |= pair_finish(D, nA - 1, lane, g, oc + db, os + db);
      __syncwarp();
    }
  }
  if (__any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(overflow, 2);
}

cudaError_t launch(int32_t n, int64_t batch, const int64_t* d_dims, int64_t* d_cells, int64_t* d_split,
                   int* d_overflow, cudaStream_t st) {
  // all of the SM's 228 KB as shared memory: eleven CTAs (22 instances) per SM
  cudaError_t e = cudaFuncSetAttribute(mcm_batch_warp, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  mcm_batch_warp<<<(unsigned)((batch + 1) / 2), 64, 0, st>>>(n, batch, d_dims, d_cells, d_split, d_overflow);
  return cudaGetLastError();
}

}  // namespace pipedp_mcmb

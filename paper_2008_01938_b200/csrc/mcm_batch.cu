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
constexpr int kCtasPerSm = 11;                      // 11 x (19.5 + 1) KB of the 228 KB

struct Smem {
  uint32_t M[kSquare];
  uint32_t p[2][kMaxN + 3];    // raw dimensions, per instance (zero padded: p[n+1], p[n+2])
  uint32_t pk[2][kMaxN + 2];   // dimensions << 6 (instance B: reversed, [n+1-k])
  uint32_t part[2][2][kMaxN + 2];  // per instance: B's and C's partial keys by row
};

// One warp's instance in the shared square (see the layout note).
struct Geo {
  int sg;              // +1 (A) or -1 (B)
  int gm;              // address offset
  int om;              // weight index offset: weight of k at pk[sg k + om]
  uint32_t* M;
  const uint32_t* p;   // raw dimensions (natural order)
  const uint32_t* pk;  // weights << 6, walked +1 per term
  uint32_t* partB;     // B's / C's partial keys by row (between the phases)
  uint32_t* partC;
  __device__ __forceinline__ int at(int r, int c) const { return sg * (kPitch * r + c) + gm; }
};

// Diagonals are taken in TRIPLES (D, D+1, D+2): cells A = (r, r+D), B =
// (r, r+D+1) and C = (r, r+D+2) of one row share the left operand M'(r, k) and
// the weight p''[k] of every split column k in [r+2, r+D-1] -- all of those
// terms only read diagonals < D -- so one lane folds the three cells' terms
// over that range with five loads per three terms (6.7 B per term instead of
// 12).  The rest, by when their operands are final:
//   phase 1 (with the shared fold):  A: k = r, r+1;  B: k = r+1 (D >= 2)
//   phase 2 (diagonal D final):      B: k = r, r+D (B done);  C: k = r+1, r+D
//   phase 3 (diagonal D+1 final):    C: k = r, r+D+1 (C done)
// B's and C's partial keys wait in `part` between the phases.
//
// Phase 1: cells [base, base + 32 / G) of diagonal D (r = 1 + i), G lanes
// per cell; G is compile-time for the one-lane passes (the term loop walks
// five pointers with immediate offsets) and run-time for the rarer short
// ones (i-cache).  The per-cell constant c & 63 (the right operand's low
// field) is taken off once after the fold: every sum is < 2^32 before it, so
// the min commutes.
template <int LGT>  // LGT >= 0: compile-time G = 2^LGT; LGT < 0: G = 2^lgr at run time
__device__ __forceinline__ bool tri_pass(int D, int base, int nA, int lane, const Geo& g, int64_t* oc,
                                         int64_t* os, int lgr = 0) {
  const int lg = LGT >= 0 ? LGT : lgr;
  const int G = 1 << lg;
  const int SL = G, SR = G * kPitch;
  const int q = lane & (G - 1);
  const int i = base + lane / G;
  const int r = 1 + i, cA = r + D, cB = cA + 1, cC = cA + 2;
  const bool liveA = i < nA, liveB = i + 1 < nA, liveC = i + 2 < nA;
  uint32_t a0 = 0xFFFFFFFFu, a1 = 0xFFFFFFFFu, b0 = 0xFFFFFFFFu, b1 = 0xFFFFFFFFu;
  uint32_t c0 = 0xFFFFFFFFu, c1 = 0xFFFFFFFFu;
  if (liveA) {
    const uint32_t pr = g.p[r - 1];
    // p[n+1], p[n+2] are padding when B / C do not exist
    const uint32_t prcA = pr * g.p[cA], prcB = pr * g.p[cB], prcC = pr * g.p[cC];
    if (q == 0) {
      a0 = prcA * g.pk[g.sg * r + g.om] + g.M[g.at(r, r)] + g.M[g.at(r + 1, cA)];  // A: k = r
      if (D >= 2) {
        const uint32_t w = g.pk[g.sg * (r + 1) + g.om], l = g.M[g.at(r, r + 1)];
        a1 = prcA * w + l + g.M[g.at(r + 2, cA)];                                   // A: k = r+1
        if (liveB) b0 = prcB * w + l + g.M[g.at(r + 2, cB)];                        // B: k = r+1
      }
    }
    const int kq = g.sg > 0 ? r + 2 + q : cA - 1 - q;  // this lane's first shared split column
    const uint32_t* L = g.M + g.at(r, kq);             // M'(r, k)
    const uint32_t* RA = g.M + g.at(kq + 1, cA);       // M'(k+1, cA)
    // M'(k+1, cB), M'(k+1, cC).  Without a cell B / C (cB = n+1, cC = n+2) the
    // walks run down column 65 or 0 of the square, which no cell of either
    // instance uses (unused values, no race) -- and keep the pass's loads on
    // distinct banks (redirecting them to A's column made 2-way conflicts)
    const uint32_t* RB = RA + g.sg;
    const uint32_t* RC = RA + 2 * g.sg;
    const uint32_t* W = g.pk + g.sg * kq + g.om;       // p''[k]
    int cnt = D >= 2 ? (D - 2 - q + G - 1) >> lg : 0;  // this lane's shared columns
    for (; cnt >= 2; cnt -= 2) {
      const uint32_t l0 = L[0], w0 = W[0], l1 = L[SL], w1 = W[G];
      a0 = min(a0, prcA * w0 + l0 + RA[0]);
      b0 = min(b0, prcB * w0 + l0 + RB[0]);
      c0 = min(c0, prcC * w0 + l0 + RC[0]);
      a1 = min(a1, prcA * w1 + l1 + RA[SR]);
      b1 = min(b1, prcB * w1 + l1 + RB[SR]);
      c1 = min(c1, prcC * w1 + l1 + RC[SR]);
      L += 2 * SL;
      RA += 2 * SR;
      RB += 2 * SR;
      RC += 2 * SR;
      W += 2 * G;
    }
    if (cnt) {
      const uint32_t l0 = L[0], w0 = W[0];
      a0 = min(a0, prcA * w0 + l0 + RA[0]);
      b0 = min(b0, prcB * w0 + l0 + RB[0]);
      c0 = min(c0, prcC * w0 + l0 + RC[0]);
    }
  }
  uint32_t ka = min(a0, a1), kb = min(b0, b1), kc = min(c0, c1);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    if (sh < G) {
      ka = min(ka, __shfl_xor_sync(0xffffffffu, ka, sh));
      kb = min(kb, __shfl_xor_sync(0xffffffffu, kb, sh));
      kc = min(kc, __shfl_xor_sync(0xffffffffu, kc, sh));
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
    g.partB[r] = kb;  // partials (still carrying + (c & 63)); unused without B / C
    g.partC[r] = kc;
  }
  return ovf;
}

// Phase 2 (diagonal D final): B = (r, r+D+1) done for r <= nA - 1 (terms
// k = r, r+D); C = (r, r+D+2) for r <= nA - 2 takes k = r+1 and k = r+D.
// Every address is affine in r along the diagonal: a lane's second cell
// (r + 32) is its first's plus a constant.
__device__ __forceinline__ bool tri_mid(int D, int nA, int lane, const Geo& g, int64_t* ocB, int64_t* osB) {
  bool ovf = false;
  int i = lane;
  if (i + 1 >= nA) return false;
  const int r0 = 1 + i;
  const int dm = 32 * g.sg * (kPitch + 1), dw = 32 * g.sg;
  // B: k = r (left M'(r,r), right M'(r+1, cB)), k = r+D (left M'(r, r+D), right M'(r+D+1, cB))
  const uint32_t* mrr = g.M + g.at(r0, r0);
  const uint32_t* mr1B = g.M + g.at(r0 + 1, r0 + D + 1);
  const uint32_t* mrD = g.M + g.at(r0, r0 + D);
  const uint32_t* mD1B = g.M + g.at(r0 + D + 1, r0 + D + 1);
  uint32_t* mB = g.M + g.at(r0, r0 + D + 1);
  // C: k = r+1 (left M'(r, r+1), right M'(r+2, cC)), k = r+D (left M'(r, r+D), right M'(r+D+1, cC))
  const uint32_t* mr_1 = g.M + g.at(r0, r0 + 1);
  const uint32_t* m2C = g.M + g.at(r0 + 2, r0 + D + 2);
  const uint32_t* mD1C = g.M + g.at(r0 + D + 1, r0 + D + 2);
  const uint32_t* wr = g.pk + g.sg * r0 + g.om;
  const uint32_t* wD = g.pk + g.sg * (r0 + D) + g.om;
  const uint32_t* pr = g.p + r0 - 1;
#pragma unroll 1
  for (int r = r0;;) {
    const uint32_t prv = pr[0], prcB = prv * pr[D + 2];
    const uint32_t wrv = wr[0], wDv = wD[0], lD = mrD[0];
    uint32_t kb = min(g.partB[r], prcB * wrv + mrr[0] + mr1B[0]);
    kb = min(kb, prcB * wDv + lD + mD1B[0]);
    const int cB = r + D + 1;
    kb -= (uint32_t)(cB & 63);
    const uint32_t v = kb >> 6;
    mB[0] = (kb & ~63u) | (uint32_t)(cB & 63);
    ocB[r] = (int64_t)v;
    osB[r] = (int64_t)(kb & 63u) - r + 1;
    ovf |= v >= kCellLimit;
    if (i + 2 < nA) {
      const uint32_t prcC = prv * pr[D + 3];
      uint32_t kc = min(g.partC[r], prcC * wr[g.sg] + mr_1[0] + m2C[0]);
      g.partC[r] = min(kc, prcC * wDv + lD + mD1C[0]);
    }
    i += 32;
    if (i + 1 >= nA) break;
    r += 32;
    mrr += dm;
    mr1B += dm;
    mrD += dm;
    mD1B += dm;
    mB += dm;
    mr_1 += dm;
    m2C += dm;
    mD1C += dm;
    wr += dw;
    wD += dw;
    pr += 32;
  }
  return ovf;
}

// Phase 3 (diagonal D+1 final): C = (r, r+D+2) done for r <= nA - 2 (terms
// k = r: M'(r,r) + M'(r+1, cC); k = r+D+1: M'(r, r+D+1) + M'(cC, cC)).
__device__ __forceinline__ bool tri_end(int D, int nA, int lane, const Geo& g, int64_t* ocC, int64_t* osC) {
  bool ovf = false;
  int i = lane;
  if (i + 2 >= nA) return false;
  const int r0 = 1 + i;
  const int dm = 32 * g.sg * (kPitch + 1), dw = 32 * g.sg;
  const uint32_t* mrr = g.M + g.at(r0, r0);
  const uint32_t* mr1C = g.M + g.at(r0 + 1, r0 + D + 2);
  const uint32_t* mrD1 = g.M + g.at(r0, r0 + D + 1);
  const uint32_t* mCC = g.M + g.at(r0 + D + 2, r0 + D + 2);
  uint32_t* mC = g.M + g.at(r0, r0 + D + 2);
  const uint32_t* wr = g.pk + g.sg * r0 + g.om;
  const uint32_t* wD1 = g.pk + g.sg * (r0 + D + 1) + g.om;
  const uint32_t* pr = g.p + r0 - 1;
#pragma unroll 1
  for (int r = r0;;) {
    const uint32_t prcC = pr[0] * pr[D + 3];
    uint32_t kc = min(g.partC[r], prcC * wr[0] + mrr[0] + mr1C[0]);
    kc = min(kc, prcC * wD1[0] + mrD1[0] + mCC[0]);
    const int cC = r + D + 2;
    kc -= (uint32_t)(cC & 63);
    const uint32_t v = kc >> 6;
    mC[0] = (kc & ~63u) | (uint32_t)(cC & 63);
    ocC[r] = (int64_t)v;
    osC[r] = (int64_t)(kc & 63u) - r + 1;
    ovf |= v >= kCellLimit;
    i += 32;
    if (i + 2 >= nA) break;
    r += 32;
    mrr += dm;
    mr1C += dm;
    mrD1 += dm;
    mCC += dm;
    mC += dm;
    wr += dw;
    wD1 += dw;
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
  g.M = s.M;
  g.p = s.p[warp];
  g.pk = s.pk[warp];
  g.partB = s.part[warp][0];
  g.partC = s.part[warp][1];
  for (int i = lane; i <= kMaxN + 2; i += 32) {
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
  for (int D = 1; D < n; D += 3) {
    db += n - (D - 1);
    const int nA = n - D;  // cells on diagonal D (B: nA - 1, C: nA - 2)
    int base = 0;
    for (; base + 32 <= nA; base += 32) ovf |= tri_pass<0>(D, base, nA, lane, g, oc + db, os + db);
    const int rem = nA - base;
    if (rem > 0) {
      // G = 2^lg lanes per remaining cell: rem G <= 32, and G / 2 < D
      const int lg = min(5 - (rem > 1 ? 32 - __clz(rem - 1) : 0), D > 1 ? 32 - __clz(D - 1) : 0);
      if (lg == 0) ovf |= tri_pass<0>(D, base, nA, lane, g, oc + db, os + db);
      else ovf |= tri_pass<-1>(D, base, nA, lane, g, oc + db, os + db, lg);
    }
    __syncwarp();
    const int64_t dbB = db + (n - D), dbC = dbB + (n - D - 1);  // lin bases of diagonals D+1, D+2
    if (nA > 1) {
      ovf |= tri_mid(D, nA, lane, g, oc + dbB, os + dbB);
      __syncwarp();
    }
    if (nA > 2) {
      ovf |= tri_end(D, nA, lane, g, oc + dbC, os + dbC);
      __syncwarp();
    }
    db = dbC;
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

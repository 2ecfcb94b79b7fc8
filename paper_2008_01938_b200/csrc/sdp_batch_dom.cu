// sdp_batch_dom.cu -- batched S-DP for min / max by dominance closure: one
// warp per instance, 32 cells per step, the last four steps in registers.
//
// Exactness.  For an idempotent (x) (min here; max mirrored) every computed
// cell satisfies ST[x] <= ST[x - a] for a in A (it is their minimum), hence
// ST[c] <= ST[c - s] for every s in S*, the additive closure of A, as long as
// the path c -> c - s stays on computed cells.  So adding operands ST[c - s],
// s in S*, to the fold of cell c (sdp.cpp:52-59) cannot change its value.  If
// S* covers [g, a_1 - 1] (and a_1 in A), the offsets >= g of cell c can be
// replaced by the whole window [c - a_1, c - g]:
//     ST[c] = min( min_{a in F} ST[c - a],  min ST[c - a_1 .. c - g] ),
// F = A n [1, g).  Valid once c >= 2 a_1 (window and paths on computed cells);
// the first a_1 computed cells run the reference's fold directly.
//
// Step b (cells c = B + l, lane l), with the previous four steps' values kept
// as suffix minima (sfx_j, lane l: min of step b-j's lanes >= l), prefix minima
// of step b-1 and their whole-step minima m_j:
//   b_l  = window part in earlier steps  (a suffix of one step, whole steps,
//          and for l < g a prefix of step b-1: shuffles)
//        (x) the F-terms that reach step b-1 (a > l: shuffles of step b-1);
//   in-step: x_l = b_l (x) (x)_{d in S_in, d <= l} x_{l-d}, S_in = F u [g, 31];
//          with S_in* = {0} u D u [h, 31] this unrolls (idempotence) to
//          x_l = b_l (x) B(l - h) (x) (x)_{d in D} b_{l-d},  B = prefix-min of b,
//          one scan and |D| + 1 shuffles;  the prefix-min of x equals B.
// Cost per step: two 5-level scans and ~10 shuffles for 32 x k relaxations.
#include "sdp_batch_dom.hpp"

#include "common.cuh"

namespace pipedp_bdom {

using namespace pipedp_dev;

template <int OP>
struct Sel {
  __device__ __forceinline__ static int32_t f(int32_t a, int32_t b) { return OP == kMin ? min(a, b) : max(a, b); }
  static constexpr int32_t id = OP == kMin ? INT32_MAX : INT32_MIN;
};

// One thread per instance: S* over [0, a_1), then g, F, h, D.
__global__ void dom_classify(int64_t batch, int32_t k, int32_t a1, const int64_t* __restrict__ offsets,
                             DomInfo* __restrict__ info) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int64_t* o = offsets + b * k;
  DomInfo r{0, 0, 0, 0};
  if (a1 < 64 || a1 > 128 || o[0] != a1) {
    info[b] = r;
    return;
  }
  uint64_t A0 = 0, A1 = 0;  // A n [1, 127]
  for (int j = 0; j < k; ++j) {
    const int64_t d = o[j];
    if (d < 64) A0 |= 1ull << d;
    else if (d < 128) A1 |= 1ull << (d - 64);
  }
  // S* (with 0) in increasing v: W holds reach[v - d] at bit d (d = 1..127),
  // so reach[v] = (W & A) != 0 -- a 128-bit shift and test per v
  uint64_t R0 = 1, R1 = 0, W0 = 0, W1 = 0;
  bool last = true;  // reach[v - 1]
  for (int v = 1; v < a1; ++v) {
    W1 = (W1 << 1) | (W0 >> 63);
    W0 = (W0 << 1) | (last ? 2ull : 0ull);  // bit 1 = reach[v - 1]
    last = ((W0 & A0) | (W1 & A1)) != 0;
    if (last) {
      if (v < 64) R0 |= 1ull << v;
      else R1 |= 1ull << (v - 64);
    }
  }
  int g = a1;  // smallest g with [g, a1) in S*
  while (g > 1) {
    const int v = g - 1;
    const bool in = v < 64 ? (R0 >> v) & 1 : (R1 >> (v - 64)) & 1;
    if (!in) break;
    --g;
  }
  if (g > 32) {
    info[b] = r;
    return;
  }
  const uint32_t F = (uint32_t)(A0 & ((g >= 32 ? 0xFFFFFFFFull : ((1ull << g) - 1)))) & ~1u;
  // S_in = F u [g, 31]; S_in* over [0, 31]
  const uint32_t Sin = F | (g <= 31 ? (0xFFFFFFFFu << g) : 0u);
  uint32_t reach = 1;
  for (int v = 1; v < 32; ++v) {
    bool hit = false;
    for (int d = 1; d <= v && !hit; ++d) hit = ((Sin >> d) & 1) && ((reach >> (v - d)) & 1);
    if (hit) reach |= 1u << v;
  }
  int h = 32;
  while (h > 1 && ((reach >> (h - 1)) & 1)) --h;
  const uint32_t D = reach & ((h >= 32 ? 0xFFFFFFFFu : ((1u << h) - 1))) & ~1u;
  r.g = (uint32_t)g;
  r.F = F;
  r.h = (uint32_t)h;
  r.D = D;
  info[b] = r;
}

template <int OP>
__device__ __forceinline__ int32_t scan_prefix(int32_t v, int lane) {
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int32_t u = __shfl_up_sync(0xffffffffu, v, s);
    if (lane >= s) v = Sel<OP>::f(v, u);
  }
  return v;
}
template <int OP>
__device__ __forceinline__ int32_t scan_suffix(int32_t v, int lane) {
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int32_t u = __shfl_down_sync(0xffffffffu, v, s);
    if (lane + s < 32) v = Sel<OP>::f(v, u);
  }
  return v;
}
template <int OP>
__device__ __forceinline__ int32_t warp_all(int32_t v) {
  return OP == kMin ? __reduce_min_sync(0xffffffffu, v) : __reduce_max_sync(0xffffffffu, v);
}

struct DomCtx {
  int j0, L0, g, lg, h, lane;
  uint32_t F, D;
};

// One step of 32 cells.  s2, s3, s4: suffix minima of steps b-2, b-3, b-4;
// m1..m3 whole-step minima of steps b-1..b-3; p1 / x1: step b-1's prefix
// minima and values (updated to step b's).  Returns step b's suffix minima.
// MODE 1: g = 1 (x = prefix minimum of b); MODE 2: F = D = {} (one window
// term per lane); MODE 0: general.  A128: a_1 = 128 (window start = lane l of
// step b-4).
template <int OP, bool A128, int MODE>
__device__ __forceinline__ int32_t dom_step(const DomCtx& cx, int32_t s2, int32_t s3, int32_t s4, int32_t m1,
                                            int32_t m2, int32_t m3, int32_t& p1, int32_t& x1) {
  using S = Sel<OP>;
  const int lane = cx.lane;
  int32_t r;
  if (A128) {
    r = S::f(S::f(s4, m3), m2);
  } else {
    const int32_t t2 = __shfl_sync(0xffffffffu, s2, cx.L0);
    const int32_t t3 = __shfl_sync(0xffffffffu, s3, cx.L0);
    const int32_t t4 = __shfl_sync(0xffffffffu, s4, cx.L0);
    r = cx.j0 == 2 ? t2 : (cx.j0 == 3 ? t3 : t4);
    if (cx.j0 > 2) r = S::f(r, m2);
    if (cx.j0 > 3) r = S::f(r, m3);
  }
  const int32_t t1 = __shfl_sync(0xffffffffu, p1, cx.lg);
  r = S::f(r, lane < cx.g ? t1 : m1);
  if (MODE == 0) {  // F-terms reaching step b-1
    for (uint32_t f = cx.F; f; f &= f - 1) {
      const int a = __ffs(f) - 1;
      const int32_t v = __shfl_sync(0xffffffffu, x1, (32 + lane - a) & 31);
      if (a > lane) r = S::f(r, v);
    }
  }
  const int32_t Bp = scan_prefix<OP>(r, lane);
  int32_t x;
  if (MODE == 1) {
    x = Bp;
  } else {
    x = r;
    if (cx.h < 32) {
      const int32_t v = __shfl_sync(0xffffffffu, Bp, (lane - cx.h) & 31);
      if (lane >= cx.h) x = S::f(x, v);
    }
    if (MODE == 0) {
      for (uint32_t dm = cx.D; dm; dm &= dm - 1) {
        const int d = __ffs(dm) - 1;
        const int32_t v = __shfl_sync(0xffffffffu, r, (lane - d) & 31);
        if (d <= lane) x = S::f(x, v);
      }
    }
  }
  p1 = Bp;
  x1 = x;
  return scan_suffix<OP>(x, lane);
}

template <int OP, bool A128, int MODE>
__device__ __forceinline__ void dom_loop(const DomCtx& cx, int64_t nfull, int64_t cells, int64_t* op, int32_t x1,
                                         int32_t p1, int32_t q0, int32_t q1, int32_t q2, int32_t q3, int32_t mq0,
                                         int32_t mq1, int32_t mq2, int32_t mq3) {
  // slots hold steps (b-1, b-2, b-3, b-4) = (q0, q1, q2, q3) at the top of
  // each unrolled group; each step overwrites the oldest slot
  int64_t b = 0;
#define DOM_STEP(A, B, C, Dq, MA, MB, MC, MD)                                    \
  Dq = dom_step<OP, A128, MODE>(cx, B, C, Dq, MA, MB, MC, p1, x1);             \
  MD = __shfl_sync(0xffffffffu, Dq, 0);                                         \
  op[32 * b] = (int64_t)x1;                                                     \
  ++b;
  for (; b + 4 <= nfull;) {
    DOM_STEP(q0, q1, q2, q3, mq0, mq1, mq2, mq3)  // step b:   new in q3
    DOM_STEP(q3, q0, q1, q2, mq3, mq0, mq1, mq2)  // step b+1: new in q2
    DOM_STEP(q2, q3, q0, q1, mq2, mq3, mq0, mq1)  // step b+2: new in q1
    DOM_STEP(q1, q2, q3, q0, mq1, mq2, mq3, mq0)  // step b+3: new in q0
  }
#undef DOM_STEP
  for (; 32 * b < cells; ++b) {  // the rest (and a partial last step)
    const int32_t sf = dom_step<OP, A128, MODE>(cx, q1, q2, q3, mq0, mq1, mq2, p1, x1);
    q3 = q2;
    q2 = q1;
    q1 = q0;
    q0 = sf;
    mq3 = mq2;
    mq2 = mq1;
    mq1 = mq0;
    mq0 = __shfl_sync(0xffffffffu, sf, 0);
    if (32 * b + cx.lane < cells) op[32 * b] = (int64_t)x1;
  }
}

constexpr int kWarps = 8;
constexpr int kRing = 256;  // exact-phase ring per warp: a_1 presets + a_1 computed cells

template <int OP>
// 64 warps per SM (32 registers; the few spills are in the per-instance setup):
// the steps are shuffle-latency chains, so occupancy is what hides them
// (C5b: 4 blocks per SM 17.6 ms, 6 15.0, 8 13.9 measured)
__global__ void __launch_bounds__(32 * kWarps, 8) sdp_batch_dom(int64_t count, const int32_t* __restrict__ perm,
                                                             int64_t n, int32_t k, int32_t a1,
                                                             const int64_t* __restrict__ offsets,
                                                             const int64_t* __restrict__ init,
                                                             int64_t* __restrict__ out,
                                                             const DomInfo* __restrict__ info) {
  using S = Sel<OP>;
  __shared__ int32_t s_ring[kWarps][kRing];
  __shared__ int32_t s_offs[kWarps][128];
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  if (gw >= count) return;
  const int64_t inst = perm[gw];
  const int64_t* io = offsets + inst * k;
  const int64_t* ii = init + inst * a1;
  int64_t* o = out + inst * n;
  int32_t* ring = s_ring[warp];
  int32_t* offs = s_offs[warp];
  const DomInfo di = info[inst];
  const int g = (int)di.g, h = (int)di.h;
  const uint32_t F = di.F, D = di.D;

  for (int j = lane; j < k; j += 32) offs[j] = (int32_t)io[j];
  for (int i = lane; i < a1; i += 32) {
    const int64_t v = ii[i];
    ring[i] = (int32_t)v;
    o[i] = v;
  }
  __syncwarp();
  // exact phase: cells [a1, 2 a1) by the reference's fold, one cell at a time
  const int64_t e0 = min((int64_t)2 * a1, n);
  for (int64_t c = a1; c < e0; ++c) {
    int32_t acc = S::id;
    for (int j = lane; j < k; j += 32) acc = S::f(acc, ring[c - offs[j]]);
    acc = warp_all<OP>(acc);
    if (lane == 0) ring[c] = acc;
    __syncwarp();
  }
  for (int64_t c = a1 + lane; c < e0; c += 32) o[c] = (int64_t)ring[c];
  if (e0 >= n) return;

  // register state: suffix minima of steps b-1 .. b-4 (slots q0..q3, rotated
  // by unrolling four steps), their whole-step minima, step b-1's prefix
  // minima and values; the first fast step is B0 = 2 a1
  const int B0 = 2 * a1;
  int32_t x1 = ring[B0 - 32 + lane];
  int32_t q0 = scan_suffix<OP>(x1, lane), q1 = scan_suffix<OP>(ring[B0 - 64 + lane], lane);
  int32_t q2 = scan_suffix<OP>(ring[B0 - 96 + lane], lane), q3 = scan_suffix<OP>(ring[B0 - 128 + lane], lane);
  int32_t mq0 = __shfl_sync(0xffffffffu, q0, 0), mq1 = __shfl_sync(0xffffffffu, q1, 0);
  int32_t mq2 = __shfl_sync(0xffffffffu, q2, 0), mq3 = 0;
  int32_t p1 = scan_prefix<OP>(x1, lane);
  DomCtx cx;
  cx.j0 = (a1 - lane + 31) / 32;  // window start c - a1: step j0 back (2..4), lane L0
  cx.L0 = (lane - a1) & 31;
  cx.g = __shfl_sync(0xffffffffu, g, 0);
  cx.lg = (32 + lane - cx.g) & 31;  // lane of step b-1 where the window ends (l < g)
  cx.h = __shfl_sync(0xffffffffu, h, 0);
  cx.F = __shfl_sync(0xffffffffu, F, 0);
  cx.D = __shfl_sync(0xffffffffu, D, 0);
  cx.lane = lane;
  const int64_t nfull = (n - B0) / 32;  // whole steps; then at most one partial step
  int64_t* op = o + B0 + lane;
  const int mode = cx.g == 1 ? 1 : (cx.F == 0 && cx.D == 0 ? 2 : 0);
  if (a1 == 128) {
    if (mode == 1) dom_loop<OP, true, 1>(cx, nfull, n - B0, op, x1, p1, q0, q1, q2, q3, mq0, mq1, mq2, mq3);
    else if (mode == 2) dom_loop<OP, true, 2>(cx, nfull, n - B0, op, x1, p1, q0, q1, q2, q3, mq0, mq1, mq2, mq3);
    else dom_loop<OP, true, 0>(cx, nfull, n - B0, op, x1, p1, q0, q1, q2, q3, mq0, mq1, mq2, mq3);
  } else {
    dom_loop<OP, false, 0>(cx, nfull, n - B0, op, x1, p1, q0, q1, q2, q3, mq0, mq1, mq2, mq3);
  }
}

cudaError_t classify(int64_t batch, int32_t k, int32_t a1, const int64_t* d_offsets, DomInfo* d_info,
                     cudaStream_t st) {
  dom_classify<<<(unsigned)((batch + 127) / 128), 128, 0, st>>>(batch, k, a1, d_offsets, d_info);
  return cudaGetLastError();
}

cudaError_t launch(int op, int64_t count, const int32_t* d_perm, int64_t n, int32_t k, int32_t a1,
                   const int64_t* d_offsets, const int64_t* d_init, int64_t* d_out, const DomInfo* d_info,
                   cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((count + kWarps - 1) / kWarps);
  if (op == 0)
    sdp_batch_dom<kMin><<<grid, 32 * kWarps, 0, st>>>(count, d_perm, n, k, a1, d_offsets, d_init, d_out, d_info);
  else
    sdp_batch_dom<kMax><<<grid, 32 * kWarps, 0, st>>>(count, d_perm, n, k, a1, d_offsets, d_init, d_out, d_info);
  return cudaGetLastError();
}

}  // namespace pipedp_bdom

// sdp_jump.cuh -- S-DP for small a_1 (<= 8) by jump-ahead segments (sm_100a).
//
// The recurrence ST[i] = (x)_j ST[i - a_j] (sdp.cpp:48-60) only ever looks a_1
// cells back, so the table is a linear dynamical system on the a_1-vector
//   s_i = (ST[i], ST[i-1], ..., ST[i-a_1+1]),   s_{i+1} = M s_i,
// over the semiring the operator induces:
//   min / max      boolean reachability (which preset cells a path of offsets
//                  lands on first) -- ST[i] is the (x) of those preset values;
//   mod-add        (+, *) mod 2^31 - 1 on normalised residues;
//   sat-add        (+, *) clamped at INT64_MAX, legal when every preset value is
//                  >= 0: then every table value is min(exact sum, INT64_MAX), and
//                  clamped arithmetic with non-negative entries preserves that.
// The cells are cut into segments of L; a thread gets its segment's entry
// state by applying the powers M^(L 2^i) for the set bits of its segment index
// (powers computed per CTA in shared memory), then computes the L cells with
// the reference's own fold, in the reference's operand order -- every cell's k
// relaxations are performed exactly as the reference performs them; only the
// entry state of a segment comes from the jump.  One serial dependency chain
// of n cells becomes n / L independent chains of L.  Single-instance,
// k >= 2 (k = 1 is a raw periodic copy with no (x) applied).
#pragma once

#include "common.cuh"

namespace pipedp_dev {

constexpr int kJumpLevels = 40;  // segment index bits
constexpr int kJumpLog2L = 6;    // cells per segment = 64
constexpr int kJumpThreads = 256;

template <int OP>
struct JumpRing;  // entry arithmetic of the induced semiring

template <>
struct JumpRing<kModAdd> {
  __device__ __forceinline__ static int64_t zero() { return 0; }
  __device__ __forceinline__ static int64_t one() { return 1; }
  __device__ __forceinline__ static int64_t add(int64_t a, int64_t b) {
    const int64_t s = a + b;
    return s >= kModulus ? s - kModulus : s;
  }
  __device__ __forceinline__ static int64_t mul(int64_t a, int64_t b) {
    return (int64_t)(((uint64_t)a * (uint64_t)b) % (uint64_t)kModulus);
  }
};
template <>
struct JumpRing<kSatAdd> {  // non-negative entries, clamped
  __device__ __forceinline__ static int64_t zero() { return 0; }
  __device__ __forceinline__ static int64_t one() { return 1; }
  __device__ __forceinline__ static int64_t add(int64_t a, int64_t b) {
    const uint64_t s = (uint64_t)a + (uint64_t)b;
    return s > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)s;
  }
  __device__ __forceinline__ static int64_t mul(int64_t a, int64_t b) {
    if (a == 0 || b == 0) return 0;
    const uint64_t hi = __umul64hi((uint64_t)a, (uint64_t)b), lo = (uint64_t)a * (uint64_t)b;
    return hi != 0 || lo > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)lo;
  }
};
struct JumpBool {  // min / max: reachability
  __device__ __forceinline__ static int64_t zero() { return 0; }
  __device__ __forceinline__ static int64_t one() { return 1; }
  __device__ __forceinline__ static int64_t add(int64_t a, int64_t b) { return a | b; }
  __device__ __forceinline__ static int64_t mul(int64_t a, int64_t b) { return a & b; }
};
template <>
struct JumpRing<kMin> : JumpBool {};
template <>
struct JumpRing<kMax> : JumpBool {};

// C = A * B (A1 x A1), one entry per thread of the first A1*A1 threads
template <int OP, int A1>
__device__ __forceinline__ void jump_matmul(const int64_t* A, const int64_t* B, int64_t* C) {
  using Rg = JumpRing<OP>;
  const int t = threadIdx.x;
  if (t < A1 * A1) {
    const int r = t / A1, c = t % A1;
    int64_t acc = Rg::zero();
#pragma unroll
    for (int m = 0; m < A1; ++m) acc = Rg::add(acc, Rg::mul(A[r * A1 + m], B[m * A1 + c]));
    C[t] = acc;
  }
}

template <int OP, int A1>
__global__ void __launch_bounds__(kJumpThreads)
    sdp_jump(const int64_t n, const int32_t k, const int64_t* __restrict__ g_offsets,
             const int64_t* __restrict__ g_init, int64_t* __restrict__ out) {
  using O = SemiOp<OP, int64_t>;
  using Rg = JumpRing<OP>;
  constexpr int64_t L = 1 << kJumpLog2L;
  __shared__ int64_t pw[kJumpLevels][A1 * A1];  // pw[i] = M^(L 2^i)
  __shared__ int64_t tmp[2][A1 * A1];
  __shared__ int32_t offs[A1];
  const int t = threadIdx.x;
  if (t < k) offs[t] = (int32_t)g_offsets[t];
  // M: row 0 has a one at column a_j - 1 for every offset, rows d >= 1 shift
  if (t < A1 * A1) {
    const int r = t / A1, c = t % A1;
    int64_t v = Rg::zero();
    if (r > 0 && c == r - 1) v = Rg::one();
    if (r == 0)
      for (int j = 0; j < k; ++j)
        if ((int)g_offsets[j] - 1 == c) v = Rg::one();
    tmp[0][t] = v;
  }
  __syncthreads();
  // M^L by kJumpLog2L squarings, then the ladder M^(L 2^i)
  int cur = 0;
  for (int i = 0; i < kJumpLog2L; ++i) {
    jump_matmul<OP, A1>(tmp[cur], tmp[cur], tmp[cur ^ 1]);
    __syncthreads();
    cur ^= 1;
  }
  if (t < A1 * A1) pw[0][t] = tmp[cur][t];
  __syncthreads();
  const int64_t nseg = (n - A1 + L - 1) / L;
  int levels = 1;
  while (levels < kJumpLevels && (1ll << levels) < nseg) ++levels;
  for (int i = 1; i < levels; ++i) {
    jump_matmul<OP, A1>(pw[i - 1], pw[i - 1], pw[i]);
    __syncthreads();
  }
  const int64_t seg = (int64_t)blockIdx.x * kJumpThreads + t;
  if (seg == 0)
    for (int i = 0; i < A1; ++i) out[i] = g_init[i];
  if (seg >= nseg) return;
  // entry state s[d] = ST[c0 - 1 - d]: the preset cells moved by M^(L seg)
  int64_t s[A1];
#pragma unroll
  for (int d = 0; d < A1; ++d) s[d] = g_init[A1 - 1 - d];
  if (OP == kModAdd && seg > 0) {
#pragma unroll
    for (int d = 0; d < A1; ++d) s[d] = norm_mod64(s[d]);
  }
  for (int i = 0; i < levels; ++i) {
    if (!((seg >> i) & 1)) continue;
    const int64_t* P = pw[i];
    int64_t ns[A1];
#pragma unroll
    for (int r = 0; r < A1; ++r) {
      if (OP == kMin || OP == kMax) {  // (x) over the reachable preset values
        bool have = false;
        int64_t acc = 0;
#pragma unroll
        for (int c = 0; c < A1; ++c)
          if (P[r * A1 + c]) {
            acc = have ? O::apply(acc, s[c]) : s[c];
            have = true;
          }
        ns[r] = acc;
      } else {
        int64_t acc = Rg::zero();
#pragma unroll
        for (int c = 0; c < A1; ++c) acc = Rg::add(acc, Rg::mul(P[r * A1 + c], s[c]));
        ns[r] = acc;
      }
    }
#pragma unroll
    for (int r = 0; r < A1; ++r) s[r] = ns[r];
  }
  // the segment's cells: the reference's fold, offsets in the given order
  const int64_t c0 = A1 + seg * L, c1 = c0 + L < n ? c0 + L : n;
  for (int64_t c = c0; c < c1; ++c) {
    int64_t acc = 0;
#pragma unroll
    for (int d = 0; d < A1; ++d)
      if (offs[0] - 1 == d) acc = s[d];
    for (int j = 1; j < k; ++j) {
      int64_t x = 0;
#pragma unroll
      for (int d = 0; d < A1; ++d)
        if (offs[j] - 1 == d) x = s[d];
      acc = O::apply(acc, x);
    }
#pragma unroll
    for (int d = A1 - 1; d >= 1; --d) s[d] = s[d - 1];
    s[0] = acc;
    out[c] = acc;
  }
}

}  // namespace pipedp_dev

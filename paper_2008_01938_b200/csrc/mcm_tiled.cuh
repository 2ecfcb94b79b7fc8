// mcm_tiled.cuh -- blocked MCM pipeline for large n (sm_100a).
//
// Same recurrence as mcm.cpp:85-110 (terms from deps, mcm.cpp:55-75):
//   m[r][c] = min_{k=r..c-1} m[r][k] + m[k+1][c] + p[r-1] p[k] p[c],
//   split = the FIRST minimising k (reported as the 1-based term index k-r+1).
// Every reduction here is a lexicographic min on (value, k), which is
// order-free and equals the reference's ascending scan with strict '<'.
//
// The index space is cut into T x T tiles (T = 64); tile (I, J), I <= J, holds
// rows r in tile I and columns c in tile J.  For a tile with Delta = J - I >= 1
// the split points k of every cell fall in three classes:
//   far    k in [(I+1)T+1, JT]  (tiles K = I+1 .. J-1 of k): both operands in
//          finished tiles (I, K) and (K.., J) -- a min-plus product with
//          weights over shared-memory tiles, split over "far tasks", one per K,
//          combined with 64-bit atomicMin on key = value << 32 | k (the
//          lexicographic order of (value, k) for value < 2^32);
//   k0     k = (I+1)T: left operand in (I, I), right operand row 0 of (I+1, J);
//   near   k in tile I (right operand in this tile, rows below) or k in tile J
//          (left operand in this tile, columns to the left): the in-tile
//          dependency, resolved by the paper's pipeline over the tile's
//          anti-diagonals (2T - 1 steps, 4 lanes per cell) in shared memory.
// Diagonal tiles (I, I) are small MCM triangles solved diagonal by diagonal.
//
// Scheduling: one persistent grid pulls tasks from a list ordered by
// readiness level (near/diagonal task of level Delta at position 2*Delta, far
// task (I, J, K) at 2*max(K-I, J-K) + 1), so every task's inputs come from
// tasks earlier in the list -- no deadlock with all CTAs resident.  Tasks wait
// on gpu-scope release/acquire flags; operand tiles move global -> shared with
// cp.async.bulk (TMA bulk copies completing on an mbarrier).
//
// Values are uint32: the host selects this kernel only when max_dim^3 < 2^31,
// and every finished cell is checked against 2^30 (so v_l + v_r + w < 2^32
// never wraps); a flagged instance is recomputed exactly in int64 by the
// wavefront kernel.
#pragma once

#include "common.cuh"
#include "mcm_kernels.cuh"

namespace pipedp_dev {

constexpr int kTiledThreads = 256;
constexpr int kTiledMaxT = 64;          // largest tile edge (host scratch sizing)

struct McmTiled {
  int64_t n;
  int32_t N;                   // tiles per side
  int64_t ntasks;
  const int32_t* p;            // dims, zero padded to N*T + 2 entries
  uint32_t* tiles;             // [N(N+1)/2][T*T] finished values, row-major per tile
  unsigned long long* keys;    // [N(N+1)/2][T*T] far partial keys (value << 32 | k)
  int* tile_done;              // [N(N+1)/2]
  int* far_count;              // [N(N+1)/2]
  const unsigned long long* tasks;  // kind | I | J | K (16 bits each)
  unsigned long long* next;    // task counter
  int64_t* out_cells;          // reference layout (diagonal-major, slot 0)
  int64_t* out_split;
  int* overflow;
  int32_t blocked;             // near in-tile pipeline: 0 CTA-wide folds per step, 1 8x8 sub-blocks, 2 pull
  int32_t packed;              // far tasks fold (value << 5 | k-in-half) keys: every cell < 2^25 required
                               // (a finished cell >= 2^25 raises overflow bit 2 -> unpacked rerun)
  int32_t gate;                // rerun gate (mcm_gated_off): 0 = always run
};

__host__ __device__ __forceinline__ int64_t tiled_index(int64_t I, int64_t J, int64_t N) {
  return I * N - I * (I - 1) / 2 + (J - I);
}

enum : int { kTaskDiag = 0, kTaskNear = 1, kTaskFar = 2, kTaskFar2 = 3 };  // Far2: K and K2 = I + J - K

__host__ __device__ __forceinline__ unsigned long long tiled_task(int kind, int I, int J, int K) {
  return ((unsigned long long)kind << 48) | ((unsigned long long)I << 32) | ((unsigned long long)J << 16) |
         (unsigned long long)K;
}

// ---- TMA bulk copy + mbarrier helpers ----------------------------------------
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
constexpr uint32_t kMcmPackedLimit = 1u << 25;  // packed far keys: cells and weights below this

__device__ __forceinline__ void spin_until_set(const int* flag) { spin_ge_gpu(flag, 1, 64); }
__device__ __forceinline__ void spin_until_count(const int* ctr, int want) { spin_ge_gpu(ctr, want, 64); }

#ifdef PIPEDP_PROFILE
__shared__ long long s_prof_ready;
__shared__ long long s_prof_mark;   // near: end of init
__shared__ long long s_prof_mark2;  // near/diag: end of the wavefront
#define PROF_READY() \
  if (threadIdx.x == 0) s_prof_ready = clock64()
#else
#define PROF_READY()
#endif

struct TBest {
  uint32_t v;
  uint32_t k;
};
__device__ __forceinline__ void tb_take(TBest& b, uint32_t v, uint32_t k) {
  if (v < b.v || (v == b.v && k < b.k)) {
    b.v = v;
    b.k = k;
  }
}
__device__ __forceinline__ void tb_take_lex(uint32_t& bv, uint32_t& bk, uint32_t v, uint32_t k) {
  const bool take = v < bv || (v == bv && k < bk);
  bv = take ? v : bv;
  bk = take ? k : bk;
}
__device__ __forceinline__ TBest tb_reduce4(TBest b) {  // over lanes l, l^1, l^2, l^3
#pragma unroll
  for (int s = 1; s <= 2; s <<= 1) {
    const uint32_t ov = __shfl_xor_sync(0xffffffffu, b.v, s);
    const uint32_t ok = __shfl_xor_sync(0xffffffffu, b.k, s);
    tb_take(b, ov, ok);
  }
  return b;
}

// Lexicographic (value, k) reduction over aligned groups of 2^lg lanes (lg <= 5);
// fully unrolled with warp-uniform guards (no data-dependent loop trip count).
__device__ __forceinline__ TBest tb_reduce(TBest b, int lg) {
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (i < lg) {
      const uint32_t ov = __shfl_xor_sync(0xffffffffu, b.v, 1 << i);
      const uint32_t ok = __shfl_xor_sync(0xffffffffu, b.k, 1 << i);
      tb_take(b, ov, ok);
    }
  }
  return b;
}

// log2 of the lanes per cell for a step with `count` live cells: the largest
// G = 2^lg with count * G <= 256, at most 32 (the reduction stays in a warp).
__device__ __forceinline__ int lanes_log2(int count) {
  const int cl = 32 - __clz(count - 1);  // ceil(log2(count)), count >= 1
  const int lg = 8 - cl;
  return lg > 5 ? 5 : lg;
}

// Fold terms kl = k0, k0 + G, ... < k1 of one cell, k ascending (strict '<'
// keeps the first minimum).  Four terms per iteration with every load issued
// before any use, so a lane pays one shared-memory latency per four terms.
template <typename F>
__device__ __forceinline__ TBest fold_terms(int k0, int k1, int G, uint32_t kbase, F term) {
  TBest b0{0xFFFFFFFFu, 0xFFFFFFFFu}, b1{0xFFFFFFFFu, 0xFFFFFFFFu};
  int kl = k0;
  for (; kl + 3 * G < k1; kl += 4 * G) {
    const uint32_t c0 = term(kl), c1 = term(kl + G), c2 = term(kl + 2 * G), c3 = term(kl + 3 * G);
    if (c0 < b0.v) { b0.v = c0; b0.k = kbase + kl; }
    if (c1 < b1.v) { b1.v = c1; b1.k = kbase + kl + G; }
    if (c2 < b0.v) { b0.v = c2; b0.k = kbase + kl + 2 * G; }
    if (c3 < b1.v) { b1.v = c3; b1.k = kbase + kl + 3 * G; }
  }
  for (; kl < k1; kl += G) {
    const uint32_t c0 = term(kl);
    if (c0 < b0.v) { b0.v = c0; b0.k = kbase + kl; }
  }
  tb_take(b0, b1.v, b1.k);
  return b0;
}

// Lanes per cell (log2) for `count` live cells with about `terms` terms each:
// enough lanes for ~8 terms per lane, no more than the CTA and a warp allow.
__device__ __forceinline__ int step_lanes_log2(int count, int terms) {
  const int cap = lanes_log2(count);
  const int want = terms <= 8 ? 0 : 32 - __clz((terms - 1) >> 3);  // ceil(log2(terms / 8))
  return want < cap ? want : cap;
}

// One instantiation per tile edge: 32 (short critical path, small n) and 64
// (fewer, denser far tasks, large n).
namespace t64 {
constexpr int kT = 64;
#include "mcm_tiled_body.inc"
}  // namespace t64
namespace t32 {
constexpr int kT = 32;
#include "mcm_tiled_body.inc"
}  // namespace t32

}  // namespace pipedp_dev

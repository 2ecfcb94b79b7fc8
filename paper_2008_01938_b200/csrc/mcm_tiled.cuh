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

constexpr int kT = 64;                 // tile edge
constexpr int kTC = kT * kT;           // cells per tile
constexpr int kXP = kT + 4;            // padded pitch (16-B aligned rows for the bulk copies)
constexpr int kTiledThreads = 256;

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
};

__host__ __device__ __forceinline__ int64_t tiled_index(int64_t I, int64_t J, int64_t N) {
  return I * N - I * (I - 1) / 2 + (J - I);
}

enum : int { kTaskDiag = 0, kTaskNear = 1, kTaskFar = 2 };

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
// keeps the first minimum), two independent accumulators for ILP.
//   cost = L[lrow + kl * ls] + Rm[rrow + kl * rs] + prc * pk[kl]
template <typename F>
__device__ __forceinline__ TBest fold_terms(int k0, int k1, int G, uint32_t kbase, F term) {
  TBest b0{0xFFFFFFFFu, 0xFFFFFFFFu}, b1{0xFFFFFFFFu, 0xFFFFFFFFu};
  int kl = k0;
  for (; kl + G < k1; kl += 2 * G) {
    const uint32_t c0 = term(kl), c1 = term(kl + G);
    if (c0 < b0.v) { b0.v = c0; b0.k = kbase + kl; }
    if (c1 < b1.v) { b1.v = c1; b1.k = kbase + kl + G; }
  }
  if (kl < k1) {
    const uint32_t c0 = term(kl);
    if (c0 < b0.v) { b0.v = c0; b0.k = kbase + kl; }
  }
  tb_take(b0, b1.v, b1.k);
  return b0;
}

// Shared-memory carve-up (bytes), one layout for every task kind.
struct TiledSmem {
  uint32_t* A;      // far: tile (I, K) [T][T];  near: tile (I, I) [T][kXP]
  uint32_t* B;      // far: rows k+1 [T][T];     near: tile (J, J) [T][kXP]
  uint32_t* X;      // near/diag: this tile's values [T][kXP]
  uint32_t* KX;     // near/diag: this tile's split k [T][kXP]
  uint32_t* R0;     // near: row 0 of tile (I+1, J) [T]
  int32_t* P;       // dims slices [4][T + 1]
  uint64_t* bar;
};

__device__ __forceinline__ TiledSmem tiled_smem(unsigned char* base) {
  TiledSmem s;
  s.A = reinterpret_cast<uint32_t*>(base);
  s.B = s.A + kT * kXP;
  s.X = s.B + kT * kXP;
  s.KX = s.X + kT * kXP;
  s.R0 = s.KX + kT * kXP;
  s.P = reinterpret_cast<int32_t*>(s.R0 + kT);
  s.bar = reinterpret_cast<uint64_t*>(s.P + 4 * (kT + 4));
  return s;
}
constexpr size_t kTiledSmemBytes =
    (size_t)(4 * kT * kXP + kT) * 4 + 4 * (kT + 4) * 4 + 16;

// ---- far task: tile (I, J), split points k in tile K ------------------------------
__device__ __forceinline__ void tiled_far(const McmTiled& S, const TiledSmem& sm, int I, int J, int K,
                                          unsigned& phase) {
  const int tid = threadIdx.x;
  const int64_t N = S.N;
  if (tid == 0) {
    spin_until_set(S.tile_done + tiled_index(I, K, N));
    spin_until_set(S.tile_done + tiled_index(K, J, N));
    spin_until_set(S.tile_done + tiled_index(K + 1, J, N));
    fence_proxy_async_global();
    fence_proxy_async_shared();
    mbar_expect_tx(sm.bar, (uint32_t)(kTC * 4 * 2));
    bulk_g2s(sm.A, S.tiles + tiled_index(I, K, N) * kTC, kTC * 4, sm.bar);
    // rows k+1 for k in tile K: rows 1..T-1 of (K, J), then row 0 of (K+1, J)
    bulk_g2s(sm.B, S.tiles + tiled_index(K, J, N) * kTC + kT, (kTC - kT) * 4, sm.bar);
    bulk_g2s(sm.B + kTC - kT, S.tiles + tiled_index(K + 1, J, N) * kTC, kT * 4, sm.bar);
  }
  int32_t* pr = sm.P;            // p[r-1], r in tile I
  int32_t* pc = sm.P + (kT + 4); // p[c],   c in tile J
  int32_t* pk = sm.P + 2 * (kT + 4);  // p[k],   k in tile K
  if (tid < kT) {
    pr[tid] = S.p[(int64_t)I * kT + tid];
    pc[tid] = S.p[(int64_t)J * kT + 1 + tid];
    pk[tid] = S.p[(int64_t)K * kT + 1 + tid];
  }
  __syncthreads();
  mbar_wait(sm.bar, phase);
  phase ^= 1u;
  PROF_READY();
  const int ty = tid >> 4, tx = tid & 15;
  uint32_t u[4][4], best[4][4], bk[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u[i][j] = (uint32_t)pr[4 * ty + i] * (uint32_t)pc[4 * tx + j];
      best[i][j] = 0xFFFFFFFFu;
      bk[i][j] = 0;
    }
#pragma unroll 4
  for (int kk = 0; kk < kT; ++kk) {
    uint32_t a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sm.A[(4 * ty + i) * kT + kk];
    const uint4 b4 = *reinterpret_cast<const uint4*>(sm.B + kk * kT + 4 * tx);
    const uint32_t b[4] = {b4.x, b4.y, b4.z, b4.w};
    const uint32_t w = (uint32_t)pk[kk];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t cost = a[i] + b[j] + u[i][j] * w;
        if (cost < best[i][j]) {  // kk ascending: strict '<' keeps the first minimum
          best[i][j] = cost;
          bk[i][j] = (uint32_t)kk;
        }
      }
  }
  unsigned long long* key = S.keys + tiled_index(I, J, N) * kTC;
  const uint32_t kbase = (uint32_t)K * kT + 1;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      atomicMin(key + (4 * ty + i) * kT + 4 * tx + j,
                ((unsigned long long)best[i][j] << 32) | (kbase + bk[i][j]));
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(S.far_count + tiled_index(I, J, N))
                 : "memory");
  }
}

// ---- finish a tile: overflow check, tile store, reference-layout outputs, flag --
__device__ __forceinline__ void tiled_finish(const McmTiled& S, const TiledSmem& sm, int I, int J) {
  const int tid = threadIdx.x;
  const int64_t N = S.N, n = S.n;
  uint32_t* gt = S.tiles + tiled_index(I, J, N) * kTC;
  bool ovf = false;
  for (int e = tid; e < kTC; e += kTiledThreads) {
    const int rl = e >> 6, ul = e & 63;
    const uint32_t v = sm.X[rl * kXP + ul];
    gt[e] = v;
    const int64_t r = (int64_t)I * kT + 1 + rl, c = (int64_t)J * kT + 1 + ul;
    if (r < c && c <= n && v >= kMcm32Limit) ovf = true;
  }
  if (ovf) atomicOr(S.overflow, 1);
  // outputs: fixed global diagonal D -> consecutive rows -> consecutive addresses
  const int warp = tid >> 5, lane = tid & 31;
  for (int dl = -(kT - 1) + warp; dl <= kT - 1; dl += kTiledThreads / 32) {
    const int r0 = dl < 0 ? -dl : 0;
    const int r1 = dl < 0 ? kT : kT - dl;  // rl in [r0, r1)
    const int64_t D = (int64_t)(J - I) * kT + dl;
    if (D <= 0) continue;  // base cells / lower half of a diagonal tile
    const int64_t db = mcm_dbase(D, n);
    for (int rl = r0 + lane; rl < r1; rl += 32) {
      const int64_t r = (int64_t)I * kT + 1 + rl;
      if (r + D > n) continue;
      const int ul = rl + dl;
      S.out_cells[db + r] = (int64_t)sm.X[rl * kXP + ul];
      S.out_split[db + r] = (int64_t)sm.KX[rl * kXP + ul] - r + 1;
    }
  }
  __threadfence();
  fence_proxy_async_global();
  __syncthreads();
  if (tid == 0) st_release_gpu_i32(S.tile_done + tiled_index(I, J, N), 1);
}

// ---- diagonal tile: MCM on the T x T triangle --------------------------------------
__device__ __forceinline__ void tiled_diag(const McmTiled& S, const TiledSmem& sm, int I) {
  const int tid = threadIdx.x;
  PROF_READY();
  int32_t* pI = sm.P;  // pI[x] = p[IT + x], x = 0..T
  if (tid <= kT) pI[tid] = S.p[(int64_t)I * kT + tid];
  for (int e = tid; e < kT; e += kTiledThreads) {
    sm.X[e * kXP + e] = 0;
    sm.KX[e * kXP + e] = 0;
  }
  __syncthreads();
  const uint32_t kb = (uint32_t)I * kT + 1;
  for (int dl = 1; dl < kT; ++dl) {
    const int lg = lanes_log2(kT - dl), G = 1 << lg;
    const int rl = tid >> lg, q = tid & (G - 1), cl = rl + dl;
    TBest b{0xFFFFFFFFu, 0xFFFFFFFFu};
    if (cl < kT) {
      const uint32_t prc = (uint32_t)pI[rl] * (uint32_t)pI[cl + 1];
      const uint32_t* xr = sm.X + rl * kXP;
      const uint32_t* xc = sm.X + kXP + cl;
      b = fold_terms(rl + q, cl, G, kb, [&](int kl) {
        return xr[kl] + xc[kl * kXP] + prc * (uint32_t)pI[kl + 1];
      });
    }
    b = tb_reduce(b, lg);
    if (cl < kT && q == 0) {
      sm.X[rl * kXP + cl] = b.v;
      sm.KX[rl * kXP + cl] = b.k;
    }
    __syncthreads();
  }
}

// ---- near task: tile (I, J), Delta >= 1 --------------------------------------------
__device__ __forceinline__ void tiled_near(const McmTiled& S, const TiledSmem& sm, int I, int J,
                                           unsigned& phase) {
  const int tid = threadIdx.x;
  const int64_t N = S.N;
  const int delta = J - I;
  if (tid == 0) {
    spin_until_set(S.tile_done + tiled_index(I, I, N));
    spin_until_set(S.tile_done + tiled_index(J, J, N));
    spin_until_set(S.tile_done + tiled_index(I + 1, J, N));
    if (delta >= 2) spin_until_count(S.far_count + tiled_index(I, J, N), delta - 1);
    fence_proxy_async_global();
    fence_proxy_async_shared();
  }
  __syncthreads();
  if (tid < 32) {  // tile (I, I) contiguous; tile (J, J) row by row into the padded pitch
    if (tid == 0) {
      mbar_expect_tx(sm.bar, (uint32_t)(kTC * 4 * 2 + kT * 4));
      bulk_g2s(sm.R0, S.tiles + tiled_index(I + 1, J, N) * kTC, kT * 4, sm.bar);
    }
    __syncwarp();
    // tiles (I, I) and (J, J) row by row into the padded pitch (column reads stay conflict-light)
    const uint32_t* srcI = S.tiles + tiled_index(I, I, N) * kTC;
    const uint32_t* srcJ = S.tiles + tiled_index(J, J, N) * kTC;
    for (int row = tid; row < kT; row += 32) {
      bulk_g2s(sm.A + row * kXP, srcI + row * kT, kT * 4, sm.bar);
      bulk_g2s(sm.B + row * kXP, srcJ + row * kT, kT * 4, sm.bar);
    }
  }
  int32_t* pr = sm.P;                 // p[r-1], r in tile I
  int32_t* pc = sm.P + (kT + 4);      // p[c],   c in tile J
  int32_t* pkI = sm.P + 2 * (kT + 4); // p[k],   k in tile I
  int32_t* pkJ = sm.P + 3 * (kT + 4); // p[k],   k in tile J
  if (tid < kT) {
    pr[tid] = S.p[(int64_t)I * kT + tid];
    pc[tid] = S.p[(int64_t)J * kT + 1 + tid];
    pkI[tid] = S.p[(int64_t)I * kT + 1 + tid];
    pkJ[tid] = S.p[(int64_t)J * kT + 1 + tid];
  }
  __syncthreads();
  mbar_wait(sm.bar, phase);
  phase ^= 1u;
  PROF_READY();
  // init: far partial (Delta >= 2) (x) the k0 = (I+1)T term
  const unsigned long long* key = S.keys + tiled_index(I, J, N) * kTC;
  const uint32_t k0 = (uint32_t)(I + 1) * kT;
  for (int e = tid; e < kTC; e += kTiledThreads) {
    const int rl = e >> 6, ul = e & 63;
    TBest b{0xFFFFFFFFu, 0xFFFFFFFFu};
    if (delta >= 2) {
      const unsigned long long kv = __ldcg(key + e);
      b.v = (uint32_t)(kv >> 32);
      b.k = (uint32_t)kv;
    }
    const uint32_t cost = sm.A[rl * kXP + (kT - 1)] + sm.R0[ul] + (uint32_t)pr[rl] * (uint32_t)pkI[kT - 1] * (uint32_t)pc[ul];
    tb_take(b, cost, k0);
    sm.X[rl * kXP + ul] = b.v;
    sm.KX[rl * kXP + ul] = b.k;
  }
  __syncthreads();
#ifdef PIPEDP_PROFILE
  if (tid == 0) s_prof_mark = clock64();
#endif
  // pipeline over the tile's anti-diagonals: cell (rl, ul) at step (T-1-rl) + ul
  const uint32_t kI = (uint32_t)I * kT + 1, kJ = (uint32_t)J * kT + 1;
  for (int s = 0; s <= 2 * (kT - 1); ++s) {
    const int ulo = s > kT - 1 ? s - (kT - 1) : 0;
    const int uhi = s < kT - 1 ? s : kT - 1;
    const int lg = lanes_log2(uhi - ulo + 1), G = 1 << lg;
    const int ci = tid >> lg, q = tid & (G - 1);
    const int ul = ulo + ci;
    const bool live = ul <= uhi;
    TBest b{0xFFFFFFFFu, 0xFFFFFFFFu};
    int rl = 0;
    if (live) {
      rl = (kT - 1) - s + ul;
      const uint32_t prc = (uint32_t)pr[rl] * (uint32_t)pc[ul];
      // k in tile I: left (r, k) from tile (I, I), right (k+1, c) from rows below
      const uint32_t* ar = sm.A + rl * kXP;
      const uint32_t* xc = sm.X + kXP + ul;
      b = fold_terms(rl + q, kT - 1, G, kI, [&](int kl) {
        return ar[kl] + xc[kl * kXP] + prc * (uint32_t)pkI[kl];
      });
      // k in tile J: left (r, k) from columns to the left, right (k+1, c) from tile (J, J)
      const uint32_t* xr = sm.X + rl * kXP;
      const uint32_t* bc = sm.B + kXP + ul;
      const TBest b2 = fold_terms(q, ul, G, kJ, [&](int kl) {
        return xr[kl] + bc[kl * kXP] + prc * (uint32_t)pkJ[kl];
      });
      tb_take(b, b2.v, b2.k);
    }
    b = tb_reduce(b, lg);
    if (live && q == 0) {
      TBest cur{sm.X[rl * kXP + ul], sm.KX[rl * kXP + ul]};
      tb_take(cur, b.v, b.k);
      sm.X[rl * kXP + ul] = cur.v;
      sm.KX[rl * kXP + ul] = cur.k;
    }
    __syncthreads();
#ifdef PIPEDP_PROFILE
    if (tid == 0 && (s == 15 || s == 31 || s == 63 || s == 95 || s == 126)) {
      const int slot = s == 15 ? 0 : s == 31 ? 1 : s == 63 ? 2 : s == 95 ? 3 : 4;
      atomicAdd(&g_prof[48 + slot], (unsigned long long)(clock64() - s_prof_mark));
    }
#endif
  }
}

__global__ void __launch_bounds__(kTiledThreads, 2) mcm_tiled_kernel(const McmTiled S) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const TiledSmem sm = tiled_smem(smem_raw);
  __shared__ unsigned long long s_task;
  if (threadIdx.x == 0) {
    mbar_init(sm.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(S.next, 1ull);
    __syncthreads();
    const unsigned long long idx = s_task;
    if ((int64_t)idx >= S.ntasks) return;
    const unsigned long long t = S.tasks[idx];
    const int kind = (int)(t >> 48), I = (int)((t >> 32) & 0xFFFF), J = (int)((t >> 16) & 0xFFFF),
              K = (int)(t & 0xFFFF);
    const long long p_t0 = PROF_NOW();
#ifdef PIPEDP_PROFILE
    if (threadIdx.x == 0 && idx == 0) {
      unsigned long long g0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
      g_prof[63] = g0;
    }
#endif
    if (kind == kTaskFar) {
      tiled_far(S, sm, I, J, K, phase);
    } else {
      if (kind == kTaskDiag) tiled_diag(S, sm, I);
      else tiled_near(S, sm, I, J, phase);
#ifdef PIPEDP_PROFILE
      if (threadIdx.x == 0) s_prof_mark2 = clock64();
#endif
      tiled_finish(S, sm, I, J);
    }
    __syncthreads();
#ifdef PIPEDP_PROFILE
    if (threadIdx.x == 0) {  // per kind: task cycles, wait cycles, count; per level: last finish
      const long long p_t1 = clock64();
      atomicAdd(&g_prof[32 + 4 * kind], (unsigned long long)(p_t1 - p_t0));
      atomicAdd(&g_prof[33 + 4 * kind], (unsigned long long)(s_prof_ready - p_t0));
      atomicAdd(&g_prof[34 + 4 * kind], 1ull);
      if (kind == kTaskNear) {
        atomicAdd(&g_prof[44], (unsigned long long)(s_prof_mark - s_prof_ready));   // init
        atomicAdd(&g_prof[45], (unsigned long long)(s_prof_mark2 - s_prof_mark));   // wavefront
        atomicAdd(&g_prof[46], (unsigned long long)(p_t1 - s_prof_mark2));          // finish
      }
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      if (kind != kTaskFar && J - I < 64) atomicMax(&g_prof[64 + J - I], gt);
    }
#endif
  }
}

}  // namespace pipedp_dev

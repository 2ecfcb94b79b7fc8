// sdp_chunked.cuh -- one large min/max S-DP instance as independent chunks
// (sm_100a).
//
// The recurrence reads a_1 cells back, so the table is a linear system on the
// state s_t = (ST[t], ST[t-1], ..., ST[t-a_1+1]) over the idempotent semiring
// of (x) (min or max):  s_{t+1} = M (.) s_t  with M[0][a_j - 1] = 1 for every
// offset and M[r][r-1] = 1 (shift).  For an idempotent, commutative (x) the
// product "(.)" is reachability: (M^L (.) s)[r] = (x) of s[c] over the c with
// (M^L)[r][c] = 1, so the state L cells later is a boolean matrix power
// applied to the state now.
//
// Cells [a_1, n) are cut into G chunks of L (a power of two).  Q = M^L is
// formed by log2(L) boolean squarings (bit-packed rows, 64 x 64 output tiles,
// AND/OR over 64-bit words; the transpose is carried along so both operands
// of every product are read row-wise), the entry state of chunk g is
// Q (.) (entry state of chunk g-1), and then every chunk is solved as one
// instance of a batch by the regular pipeline kernels with its entry state as
// the preset cells -- every cell's k relaxations run in the reference's
// fold; the matrix powers only replace the serial dependency between chunks.
#pragma once

#include "common.cuh"

namespace pipedp_dev {


// Set the ones of M and M^T (bit-packed, W words per row; the host zeroes
// both first).  Rows and columns >= a1 stay empty.
__global__ void bm_build(const int64_t* __restrict__ offsets, int32_t k, int32_t a1, int32_t W,
                         unsigned long long* __restrict__ M, unsigned long long* __restrict__ MT) {
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const int c = (int)offsets[j] - 1;  // row 0, column a_j - 1
    atomicOr(&M[c / 64], 1ull << (c % 64));
    atomicOr(&MT[(int64_t)c * W], 1ull);  // row c of M^T, column 0
  }
  for (int64_t r = 1 + threadIdx.x; r < a1; r += blockDim.x) {
    const int64_t c = r - 1;  // M[r][r-1]
    atomicOr(&M[r * W + c / 64], 1ull << (c % 64));
    atomicOr(&MT[c * W + r / 64], 1ull << (r % 64));
  }
}

// Z = X * Y (boolean), given X (rows) and YT (rows of Y^T): Z[r][c] = any(X[r] & YT[c]).
// Rows are read as 32-bit words; acc |= a & b is one LOP3.  CTA tile 128 rows
// x 64 columns (one output word per row), thread tile 8 x 4, K staged through
// shared memory 64 words at a time.  Grid (A1P/64, A1P/128).
// Squaring support: `prev_changed` (nullable) = did the previous squaring
// change the matrix; if not, X is idempotent (X X = X) and the tile is copied.
// `changed` (nullable) records whether this product differs from X.  The
// epilogue also writes the tile transposed into ZT (the next product's right
// operand), so no separate transpose pass runs.
constexpr int kBmR = 128;  // CTA output rows
constexpr int kBmC = 64;   // CTA output columns (one 64-bit word)
constexpr int kBmK = 32;   // 32-bit words per K stage (early exit between stages)
__global__ void __launch_bounds__(256, 2) bm_mul(const uint32_t* __restrict__ X, const uint32_t* __restrict__ YT,
                                                 int32_t W32, unsigned long long* __restrict__ Z,
                                                 const int* __restrict__ prev_changed, int* __restrict__ changed,
                                                 unsigned long long* __restrict__ ZT) {
  extern __shared__ __align__(16) uint32_t bm_smem[];
  constexpr int P = kBmK + 4;  // padded pitch (words), 16-byte rows
  uint32_t* xs = bm_smem;            // [128][P]
  uint32_t* ys = bm_smem + kBmR * P;  // [64][P]
  __shared__ unsigned long long zw[kBmR];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * kBmR, c0 = (int64_t)blockIdx.x * kBmC;
  const int W64 = W32 / 2;
  const unsigned long long* X64 = reinterpret_cast<const unsigned long long*>(X);
  if (prev_changed && *prev_changed == 0) {  // stable: X X = X (and Z^T = X^T = YT)
    if (t < kBmR) Z[(r0 + t) * W64 + c0 / 64] = X64[(r0 + t) * W64 + c0 / 64];
    if (t < kBmR) {
      const unsigned long long* YT64 = reinterpret_cast<const unsigned long long*>(YT);
      const int64_t o = (c0 + (t & 63)) * W64 + r0 / 64 + (t >> 6);
      ZT[o] = YT64[o];
    }
    return;
  }
  const int tr = t / 16, tc = t % 16;  // rows 8 tr .. +8, columns tc + 16 j (j < 4)
  uint32_t acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  if (t < kBmR) zw[t] = 0;
  for (int k0 = 0; k0 < W32; k0 += kBmK) {
    __syncthreads();
    bool nz = false;
    for (int e = t; e < kBmR * (kBmK / 4); e += 256) {  // 16-byte loads
      const int i = e / (kBmK / 4), q = e % (kBmK / 4);
      const uint4 xv = *reinterpret_cast<const uint4*>(X + (r0 + i) * W32 + k0 + 4 * q);
      *reinterpret_cast<uint4*>(xs + i * P + 4 * q) = xv;
      nz = nz || (xv.x | xv.y | xv.z | xv.w) != 0;
      if (i < kBmC)
        *reinterpret_cast<uint4*>(ys + i * P + 4 * q) =
            *reinterpret_cast<const uint4*>(YT + (c0 + i) * W32 + k0 + 4 * q);
    }
    // an all-zero X stage contributes nothing (sparse early powers: mostly shifts)
    if (!__syncthreads_or(nz)) continue;
#pragma unroll 2
    for (int w = 0; w < kBmK; w += 4) {
      uint4 a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const uint4*>(xs + (8 * tr + i) * P + w);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const uint4*>(ys + (tc + 16 * j) * P + w);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          acc[i][j] |= (a[i].x & b[j].x) | (a[i].y & b[j].y) | (a[i].z & b[j].z) | (a[i].w & b[j].w);
    }
    // every output of the tile already 1: the remaining K stages cannot change it
    bool full = true;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) full = full && acc[i][j] != 0;
    if (__syncthreads_and(full)) break;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    unsigned long long bits = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) bits |= (unsigned long long)(acc[i][j] != 0) << (tc + 16 * j);
    if (bits) atomicOr(&zw[8 * tr + i], bits);
  }
  __syncthreads();
  if (t < kBmR) {
    const int64_t o = (r0 + t) * W64 + c0 / 64;
    Z[o] = zw[t];
    if (changed && zw[t] != X64[o]) atomicOr(changed, 1);
    // the transposed tile (64 rows of Z^T, two words each) for the next
    // product's right operand -- instead of a separate transpose launch
    const int c = t & 63, h = t >> 6;
    unsigned long long out = 0;
#pragma unroll 8
    for (int i = 0; i < 64; ++i) out |= ((zw[64 * h + i] >> c) & 1ull) << i;
    ZT[(c0 + c) * W64 + r0 / 64 + h] = out;
  }
}

// Rows [r0, 64 W) of M^t for t < a1 are pure shifts: row r (state position r
// at time T + t) is state position r - t at time T.  Written directly instead
// of multiplied; they differ from every other power's rows, so `changed` is set.
__global__ void bm_shift_rows(unsigned long long* __restrict__ Z, int32_t W, int64_t t, int64_t r0, int32_t a1,
                              int* changed, unsigned long long* __restrict__ ZT) {
  const int64_t rows = 64ll * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (rows - r0) * W;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = r0 + e / W, w = e % W, c = r - t;
    Z[r * W + w] = (r < a1 && c >= 0 && c / 64 == w) ? 1ull << (c % 64) : 0ull;
  }
  // the same rows in Z^T: words [r0 / 64, W) of every row c hold bit r = c + t
  // (r0 is a multiple of 128, so those words lie wholly in the shift rows)
  const int64_t w0 = r0 / 64, nw = W - w0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * nw;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / nw, w = w0 + e % nw, r = c + t;
    ZT[c * W + w] = (r < a1 && r >= r0 && r / 64 == w) ? 1ull << (r % 64) : 0ull;
  }
  if (changed && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(changed, 1);
}

// E1 = Q (.) E0 over rows [0, a1): one warp per row; lane l takes columns
// l + 32 i (coalesced E0 reads from shared memory, one broadcast word per
// 64 columns), branch-free select, then a warp reduction.
// Also writes the chunk's preset cells: init_out[a1 - 1 - r] = E1[r].
template <int OP>
__global__ void __launch_bounds__(256) bm_matvec(const unsigned long long* __restrict__ Q, int32_t W, int32_t a1,
                                                 const int64_t* __restrict__ E0, int64_t* __restrict__ E1,
                                                 int64_t* __restrict__ init_out) {
  using O = SemiOp<OP, int64_t>;
  extern __shared__ __align__(16) int64_t es[];  // [64 W]
  for (int c = threadIdx.x; c < 64 * W; c += blockDim.x) es[c] = c < a1 ? E0[c] : SemiId<OP, int64_t>::value();
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= a1) return;
  const int64_t id = SemiId<OP, int64_t>::value();
  int64_t acc0 = id, acc1 = id;
  const unsigned long long* qr = Q + r * W;
  for (int w = 0; w < W; ++w) {
    const unsigned long long bits = __ldg(qr + w);
    const int64_t v0 = es[64 * w + lane], v1 = es[64 * w + 32 + lane];
    acc0 = O::apply(acc0, (bits >> lane) & 1 ? v0 : id);
    acc1 = O::apply(acc1, (bits >> (32 + lane)) & 1 ? v1 : id);
  }
  int64_t acc = O::apply(acc0, acc1);
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) acc = O::apply(acc, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)acc, s));
  if (lane == 0) {
    E1[r] = acc;
    init_out[a1 - 1 - r] = acc;
  }
}

// Grid barrier for a co-resident (cooperative) grid: generation counter.
__device__ __forceinline__ void bm_grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = (unsigned)ld_relaxed_gpu_i32(reinterpret_cast<const int*>(bar + 1));
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while ((unsigned)ld_relaxed_gpu_i32(reinterpret_cast<const int*>(bar + 1)) == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// One warp's row of P (.) E into chunk dst's preset cells (state order r ->
// cell a1 - 1 - r); E is in shared memory in state order, wmin[w] = (x) of
// E's 64 entries under word w.  Lane l takes words l, l + 32, ...: a full word
// contributes wmin[w] (one operation for 64 columns -- dense powers are the
// common case), a partial word its set bits one by one.
template <int OP>
__device__ __forceinline__ int64_t bm_word(unsigned long long bits, int w, const int64_t* es, const int64_t* wmin,
                                           int64_t acc) {
  using O = SemiOp<OP, int64_t>;
  if (bits == ~0ull) return O::apply(acc, wmin[w]);
  while (bits) {
    const int b = __ffsll((long long)bits) - 1;
    bits &= bits - 1;
    acc = O::apply(acc, es[64 * w + b]);
  }
  return acc;
}

// Rows r0 and r1 (r1 < 0: none) of P (.) E, their words loaded together so
// the L2 latency of one row hides behind the other's.
template <int OP>
__device__ __forceinline__ void bm_row2(const unsigned long long* __restrict__ P, int32_t W, int32_t a1, int64_t r0,
                                        int64_t r1, const int64_t* es, const int64_t* wmin, int64_t* dst_init) {
  using O = SemiOp<OP, int64_t>;
  const int lane = threadIdx.x & 31;
  int64_t a0 = SemiId<OP, int64_t>::value(), a1v = a0;
  const unsigned long long* q0 = P + r0 * W;
  const unsigned long long* q1 = P + (r1 >= 0 ? r1 : r0) * W;
  for (int w = lane; w < W; w += 64) {  // two words of each row in flight per lane
    const bool two = w + 32 < W;
    const unsigned long long b00 = __ldg(q0 + w), b10 = __ldg(q1 + w);
    const unsigned long long b01 = two ? __ldg(q0 + w + 32) : 0ull, b11 = two ? __ldg(q1 + w + 32) : 0ull;
    a0 = bm_word<OP>(b00, w, es, wmin, a0);
    a1v = bm_word<OP>(b10, w, es, wmin, a1v);
    if (two) {
      a0 = bm_word<OP>(b01, w + 32, es, wmin, a0);
      a1v = bm_word<OP>(b11, w + 32, es, wmin, a1v);
    }
  }
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    a0 = O::apply(a0, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)a0, s));
    a1v = O::apply(a1v, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)a1v, s));
  }
  if (lane == 0) {
    dst_init[a1 - 1 - r0] = a0;
    if (r1 >= 0) dst_init[a1 - 1 - r1] = a1v;
  }
}

// The entry-state chain in one persistent launch (all CTAs co-resident).
// Chunk g's preset cells cinit[g] are E_g in cell order.  Two levels:
//   A: E_{B m} = Q_B (.) E_{B (m-1)}          (Q_B = Q^B; G/B sequential steps)
//   B: E_{B m + j} = Q (.) E_{B m + j - 1}   (all groups m at once; B - 1 steps)
// so G - 1 dependent steps become G/B + B - 2 (B = 16 for G = 256: 30).
template <int OP>
__global__ void __launch_bounds__(1024, 1) bm_chain(const unsigned long long* __restrict__ Q,
                                                    const unsigned long long* __restrict__ QB, int32_t B,
                                                    int32_t W, int32_t a1, int64_t G, int64_t* cinit,
                                                    unsigned* bar) {
  using O = SemiOp<OP, int64_t>;
  extern __shared__ __align__(16) int64_t es[];  // [64 W] E, then [W] per-word (x)
  int64_t* wmin = es + 64 * W;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int64_t id = SemiId<OP, int64_t>::value();
  auto load = [&](int64_t g) {  // E_g (state order) from chunk g's preset cells
    const long long* src = reinterpret_cast<const long long*>(cinit + g * a1);
    for (int c = threadIdx.x; c < 64 * W; c += blockDim.x) es[c] = c < a1 ? (int64_t)__ldcg(src + a1 - 1 - c) : id;
    __syncthreads();
    for (int w = warp; w < W; w += nw) {  // one warp per word
      int64_t v = O::apply(es[64 * w + lane], es[64 * w + 32 + lane]);
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) v = O::apply(v, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)v, s));
      if (lane == 0) wmin[w] = v;
    }
    __syncthreads();
  };
  const int64_t groups = (G + B - 1) / B;
  // A: the group heads, every CTA on one matrix-vector product per step
  for (int64_t m = 1; m < groups; ++m) {
    load(B * (m - 1));
    for (int64_t r = (int64_t)blockIdx.x * nw + warp, st = (int64_t)gridDim.x * nw; r < a1; r += 2 * st)
      bm_row2<OP>(QB, W, a1, r, r + st < a1 ? r + st : -1, es, wmin, cinit + B * m * a1);
    bm_grid_sync(bar);
  }
  // B: inside every group at once; CTA b serves group b % groups
  const int64_t m = blockIdx.x % groups;
  const int64_t per = gridDim.x / groups + ((int64_t)(blockIdx.x % groups) < (int64_t)(gridDim.x % groups) ? 1 : 0);
  const int64_t slot = blockIdx.x / groups;  // this CTA's index among its group's CTAs
  for (int j = 1; j < B; ++j) {
    const int64_t g = B * m + j;
    if (g < G && per > 0) {
      load(g - 1);
      for (int64_t r = slot * nw + warp, st = per * nw; r < a1; r += 2 * st)
        bm_row2<OP>(Q, W, a1, r, r + st < a1 ? r + st : -1, es, wmin, cinit + g * a1);
    }
    bm_grid_sync(bar);
  }
}

// E0[r] = init[a1 - 1 - r] (state order) and chunk 0's preset cells = init.
__global__ void bm_state0(const int64_t* __restrict__ init, int32_t a1, int64_t* __restrict__ E0,
                          int64_t* __restrict__ init0) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a1; r += gridDim.x * blockDim.x) {
    E0[r] = init[a1 - 1 - r];
    init0[r] = init[r];
  }
}

}  // namespace pipedp_dev

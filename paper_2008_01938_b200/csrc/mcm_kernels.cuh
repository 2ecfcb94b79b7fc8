// mcm_kernels.cuh -- matrix-chain-multiplication table fill for sm_100a.
//
// Reference semantics (mcm.cpp:85-110, terms from mcm.cpp:55-75): cells are
// addressed 1-based in diagonal-major order, lin(r,c) = D*n - D(D-1)/2 + r with
// D = c - r; slot 0 and the n base cells are 0.  For a computed cell (r, c)
//   best = min_{j=1..D} cells[lin(r, r+j-1)] + cells[lin(r+j, c)] + p[r-1]*p[r+j-1]*p[c]
// with the FIRST minimal j recorded as split (strict '<' while scanning j up).
// Every kernel here reduces on the pair (value, j) lexicographically, which is
// order-free and equals that first-min rule exactly.
//
// Layout: the kernels keep the reference's diagonal-major layout.  It is the
// layout the dataflow wavefront wants: for 32 consecutive cells (r .. r+31) of
// one diagonal, the left operand of term j lies on diagonal j-1 at rows
// r..r+31 and the right operand on diagonal D-j at rows r+j..r+j+31 -- both
// contiguous, so every warp load is one coalesced 128-byte line.
//
// Value width: 'uint32_t' kernels are used when max_dim^3 < 2^31; they keep
// every finalised value below 2^30 (so v_l + v_r + w never wraps) and raise a
// device flag if a value reaches 2^30, in which case the host reruns the
// instance with the int64 kernel (both on the GPU).
#pragma once

#include "common.cuh"

namespace pipedp_dev {

constexpr uint32_t kMcm32Limit = 1u << 30;

__host__ __device__ __forceinline__ int64_t mcm_dbase(int64_t d, int64_t n) {
  return d * n - d * (d - 1) / 2;  // lin(r, r+d) = dbase(d) + r   (mcm.cpp:35-36)
}

template <typename T>
__device__ __forceinline__ T ldcg_t(const T* p);
template <>
__device__ __forceinline__ uint32_t ldcg_t<uint32_t>(const uint32_t* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ int64_t ldcg_t<int64_t>(const int64_t* p) {
  return (int64_t)__ldcg(reinterpret_cast<const long long*>(p));
}

template <typename T>
struct McmBest {
  T v;
  int32_t j;
};

template <typename T>
__device__ __forceinline__ void mcm_take(McmBest<T>& b, T v, int32_t j) {
  if (v < b.v || (v == b.v && j < b.j)) {
    b.v = v;
    b.j = j;
  }
}

template <typename T>
__device__ __forceinline__ McmBest<T> mcm_group_reduce(McmBest<T> b, int group) {
  for (int s = group >> 1; s > 0; s >>= 1) {
    const T ov = __shfl_xor_sync(0xffffffffu, b.v, s);
    const int32_t oj = __shfl_xor_sync(0xffffffffu, b.j, s);
    mcm_take(b, ov, oj);
  }
  return b;
}

template <typename T>
__device__ __forceinline__ T mcm_max_value();
template <>
__device__ __forceinline__ uint32_t mcm_max_value<uint32_t>() { return 0xFFFFFFFFu; }
template <>
__device__ __forceinline__ int64_t mcm_max_value<int64_t>() { return INT64_MAX; }

// Terms j = j0, j0+G, ... <= D of cell (r, r+D) over a diagonal-major table V.
template <typename T, typename Load>
__device__ __forceinline__ McmBest<T> mcm_cell_terms(const T* V, const int32_t* __restrict__ p,
                                                     int64_t n, int64_t r, int64_t D, int j0,
                                                     int G, Load load) {
  McmBest<T> best{mcm_max_value<T>(), 0};
  const int64_t c = r + D;
  const T prc = (T)p[r - 1] * (T)p[c];
  for (int64_t j = j0; j <= D; j += G) {
    const T left = load(V + mcm_dbase(j - 1, n) + r);
    const T right = load(V + mcm_dbase(D - j, n) + r + j);
    const T cost = left + right + prc * (T)p[r + j - 1];
    mcm_take(best, cost, (int32_t)j);
  }
  return best;
}

// A rerun launched behind the first attempt without a host round trip: it
// does its work only if the attempt raised one of the `gate` overflow bits
// (bit 2: a packed key could wrap -> unpacked rerun; bit 1: a 32-bit value
// reached 2^30 -> 64-bit rerun); gate 0 = unconditional.  Stream order makes
// the earlier launches' flag visible.
__device__ __forceinline__ bool mcm_gated_off(const int* overflow, int gate) {
  return gate != 0 && (*reinterpret_cast<const volatile int*>(overflow) & gate) == 0;
}

// -----------------------------------------------------------------------------
// Small n: one CTA per instance, the whole triangle in shared memory,
// diagonal by diagonal (n-1 __syncthreads).  Also the batched kernel.
// Output per instance: cells / split int64 in the reference layout.
template <typename T>
__global__ void __launch_bounds__(512)
    mcm_smem_cta(int64_t n, int64_t batch, const int64_t* __restrict__ g_dims,
                 int64_t* __restrict__ out_cells, int64_t* __restrict__ out_split,
                 int* __restrict__ overflow, int gate = 0) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (mcm_gated_off(overflow, gate)) return;
  bool ovf = false;
  // instance loop: a gated rerun launches a small grid (its gated-off cost
  // stays a few hundred CTAs), the first attempt one CTA per instance
  for (int64_t inst = blockIdx.x; inst < batch; inst += gridDim.x) {
  const int64_t cc = n * (n + 1) / 2;
  T* V = reinterpret_cast<T*>(smem);  // cc + 1 entries
  int32_t* p = reinterpret_cast<int32_t*>(V + ((cc + 1 + 3) & ~3ll));
  const int64_t* gd = g_dims + inst * (n + 1);
  int64_t* oc = out_cells + inst * (cc + 1);
  int64_t* os = out_split + inst * (cc + 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t i = tid; i <= n; i += nt) {
    p[i] = (int32_t)gd[i];
    V[i] = T(0);
    oc[i] = 0;
    os[i] = 0;
  }
  __syncthreads();
  for (int64_t D = 1; D < n; ++D) {
    const int64_t ncell = n - D;
    int G = 1;  // lanes per cell: spread the terms when the diagonal is short
    while (G < 32 && ncell * G * 2 <= nt && G < D) G <<= 1;
    const int64_t slots = (int64_t)(nt / G) * G;
    const int64_t db = mcm_dbase(D, n);
    for (int64_t base = 0; base < ncell * G; base += slots) {
      const int64_t t = base + tid;
      const bool live = tid < slots && t < ncell * G;
      McmBest<T> best{mcm_max_value<T>(), 0};
      const int64_t r = 1 + t / G;
      if (live) {
        best = mcm_cell_terms<T>(V, p, n, r, D, 1 + (int)(t % G), G,
                                 [](const T* a) { return *a; });
      }
      if (G > 1) best = mcm_group_reduce(best, G);
      if (live && (t % G) == 0) {
        V[db + r] = best.v;
        oc[db + r] = (int64_t)best.v;
        os[db + r] = best.j;
        if (sizeof(T) == 4 && (uint64_t)best.v >= kMcm32Limit) ovf = true;
      }
    }
    __syncthreads();
  }
  }  // instances
  if (ovf) atomicOr(overflow, 1);
}

// -----------------------------------------------------------------------------
// Large n: persistent multi-SM dataflow wavefront.  Work items ("chunks") are
// CPW = 32/G consecutive cells of one diagonal, handed out in address order by
// an atomic counter; G = lanes per cell grows with D so per-lane work stays
// bounded.  A chunk on diagonal D waits only for the (at most two) chunks of
// diagonal D-1 holding rows r_lo .. r_hi+1 -- the cells (r, c-1) and (r+1, c)
// whose finality implies that of every other operand.  Flags are released with
// st.release.gpu after a gpu-scope fence; operands are read with ld.global.cg
// (L2) so no stale L1 line can be observed.
struct McmWave {
  int64_t n;
  int64_t total_chunks;
  const int64_t* chunk_base;  // [n]: first chunk index of diagonal D (D = 1..n-1), [0] unused
  int* done;                  // [total_chunks] completion flags
  unsigned long long* next;   // work counter
};

__host__ __device__ __forceinline__ int mcm_wave_group(int64_t D) {
  int G = 1;
  while (G < 32 && D > 48 * G) G <<= 1;
  return G;
}

template <typename T>
__global__ void __launch_bounds__(256)
    mcm_wavefront(const McmWave W, const int32_t* __restrict__ p, T* V, int64_t* out_cells,
                  int64_t* __restrict__ out_split,
                  int* __restrict__ overflow, int gate = 0) {
  if (mcm_gated_off(overflow, gate)) return;
  const int lane = threadIdx.x & 31;
  const int64_t n = W.n;
  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(W.next, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if ((int64_t)idx >= W.total_chunks) return;
    // diagonal of this chunk: chunk_base is increasing over D = 1..n-1
    int64_t lo = 1, hi = n - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (__ldg(W.chunk_base + mid) <= (int64_t)idx) lo = mid; else hi = mid - 1;
    }
    const int64_t D = lo;
    const int64_t q = (int64_t)idx - __ldg(W.chunk_base + D);
    const int G = mcm_wave_group(D);
    const int cpw = 32 / G;
    const int64_t r_lo = q * cpw + 1;
    const int64_t r_hi = min(r_lo + cpw - 1, n - D);
    if (D > 1) {  // wait for rows r_lo .. r_hi+1 of diagonal D-1
      const int cpw1 = 32 / mcm_wave_group(D - 1);
      const int64_t b1 = __ldg(W.chunk_base + D - 1);
      const int64_t q1 = (r_lo - 1) / cpw1, q2 = r_hi / cpw1;
      for (int64_t qq = q1; qq <= q2; ++qq) spin_ge_gpu(W.done + b1 + qq, 1, 32);
    }
    const int64_t r = r_lo + lane / G;
    const bool live = r <= r_hi;
    McmBest<T> best{mcm_max_value<T>(), 0};
    if (live) {
      best = mcm_cell_terms<T>(V, p, n, r, D, 1 + (lane % G), G,
                               [](const T* a) { return ldcg_t<T>(a); });
    }
    if (G > 1) best = mcm_group_reduce(best, G);
    if (live && (lane % G) == 0) {
      const int64_t a = mcm_dbase(D, n) + r;
      V[a] = best.v;
      if (sizeof(T) == 4) {
        out_cells[a] = (int64_t)best.v;
        if ((uint64_t)best.v >= kMcm32Limit) atomicOr(overflow, 1);
      }
      out_split[a] = best.j;
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_gpu_i32(W.done + idx, 1);
  }
}

}  // namespace pipedp_dev

namespace pipedp_dev {

// -----------------------------------------------------------------------------
// solve_mcm_bruteforce (mcm.cpp:112-138): the reference's independent oracle,
// minimum over every full parenthesisation by direct recursion on splits
// (exponential on purpose, n <= 12, never touches a table).  One thread.
__device__ int64_t mcm_enumerate(const int64_t* __restrict__ p, int r, int c) {
  if (r == c) return 0;
  int64_t best = INT64_MAX;
  for (int s = r; s < c; ++s) {
    const int64_t cost = mcm_enumerate(p, r, s) + mcm_enumerate(p, s + 1, c) + p[r - 1] * p[s] * p[c];
    best = cost < best ? cost : best;
  }
  return best;
}

__global__ void mcm_bruteforce_kernel(const int64_t* __restrict__ p, int n, int64_t* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = mcm_enumerate(p, 1, n);
}

}  // namespace pipedp_dev

namespace pipedp_dev {

// -----------------------------------------------------------------------------
// Batched small-n MCM (BASELINE config 5a: 65,536 instances of n = 64), one CTA
// per instance.  The instance's table lives in shared memory as a row-major
// (n+1) x (n+1) square (pitch P = n + 1, odd-stride rows keep a warp's loads
// on distinct banks), so term j of cell (r, c) reads
//   left  = M[r][r+j-1]   (walks along row r:      +1 per term)
//   right = M[r+j][c]     (walks down column c:    +P per term)
// with incremental 32-bit addresses -- no per-term index arithmetic.  Lanes
// per cell G = 2^lg grows as the diagonal shortens; each lane scans its terms
// j ascending with strict '<' and the G partials reduce lexicographically on
// (value, j): the reference's first-min split (mcm.cpp:95-104).
// PACKED (uint32 tables, n <= 64): terms fold as keys (cost << 6) | j with one
// unsigned min -- exact while every cost < 2^26: every finished cell and every
// weight < 2^24 (host-checked weights; a cell >= 2^24 sets overflow bit 2 and
// the host reruns the launch unpacked; by induction over the diagonals no
// candidate of an unflagged run wrapped).  Keys order as (cost, j): the first
// minimum, as the reference.
template <typename T, bool PACKED = false>
__global__ void __launch_bounds__(128)
    mcm_smem_square(int32_t n, int64_t batch, const int64_t* __restrict__ g_dims,
                    int64_t* __restrict__ out_cells, int64_t* __restrict__ out_split,
                    int* __restrict__ overflow, int gate = 0) {
  if (mcm_gated_off(overflow, gate)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  bool ovf = false, ovf2 = false;
  // instance loop: a gated rerun launches a small grid (its gated-off cost
  // stays a few hundred CTAs), the first attempt one CTA per instance
  for (int64_t inst = blockIdx.x; inst < batch; inst += gridDim.x) {
  const int P = n + 1;
  T* M = reinterpret_cast<T*>(smem);                         // [P][P], row r = 1..n
  int32_t* p = reinterpret_cast<int32_t*>(M + P * P + 1);    // dims p_0..p_n
  const int64_t cc = (int64_t)n * (n + 1) / 2;
  const int64_t* gd = g_dims + inst * (n + 1);
  int64_t* oc = out_cells + inst * (cc + 1);
  int64_t* os = out_split + inst * (cc + 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i <= n; i += nt) {
    p[i] = (int32_t)gd[i];
    if (i >= 1) M[i * P + i] = T(0);  // base cells m[i][i] = 0
    oc[i] = 0;                        // slot 0 and base cells 1..n (mcm.cpp:77-83)
    os[i] = 0;
  }
  __syncthreads();
  int64_t db = 0;  // lin(r, r+D) = db(D) + r, db(D) = D*n - D(D-1)/2
  for (int D = 1; D < n; ++D) {
    db += n - (D - 1);
    const int ncell = n - D;
    int lg = 0;  // lanes per cell: spread the D terms when the diagonal is short
    while (lg < 5 && (ncell << (lg + 1)) <= nt && (1 << lg) < D) ++lg;
    const int G = 1 << lg;
    const int slots = (nt >> lg) << lg;
    for (int base = 0; base < ncell * G; base += slots) {
      const int t = base + tid;
      const bool live = tid < slots && t < ncell * G;
      const int r = 1 + (t >> lg), q = t & (G - 1), c = r + D;
      McmBest<T> best{mcm_max_value<T>(), 0};
      if constexpr (PACKED) {
        uint32_t key = 0xFFFFFFFFu;
        if (live) {
          const uint32_t prc = (uint32_t)p[r - 1] * (uint32_t)p[c];
          const T* L = M + r * P + r - 1;
          const T* Rt = M + r * P + c;
          const int32_t* pk = p + r - 1;
          for (int j = 1 + q; j <= D; j += G)
            key = min(key, ((uint32_t)(L[j] + Rt[j * P] + prc * (uint32_t)pk[j]) << 6) | (uint32_t)j);
        }
        for (int sh = G >> 1; sh > 0; sh >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, sh));
        best.v = (T)(key >> 6);
        best.j = (int32_t)(key & 63u);
        if (live && q == 0 && (uint32_t)best.v >= (1u << 24)) ovf2 = true;
      } else {
        if (live) {
          const T prc = (T)p[r - 1] * (T)p[c];
          const T* L = M + r * P + r - 1;  // m[r][r+j-1] at L[j]
          const T* Rt = M + r * P + c;     // m[r+j][c]   at Rt[j*P]
          const int32_t* pk = p + r - 1;   // p[r+j-1]    at pk[j]
          for (int j = 1 + q; j <= D; j += G) {
            const T cost = L[j] + Rt[j * P] + prc * (T)pk[j];
            if (cost < best.v) {  // j ascending in this lane: first minimum
              best.v = cost;
              best.j = j;
            }
          }
        }
        if (G > 1) best = mcm_group_reduce(best, G);
      }
      if (live && q == 0) {
        M[r * P + c] = best.v;
        oc[db + r] = (int64_t)best.v;
        os[db + r] = best.j;
        if (sizeof(T) == 4 && (uint64_t)best.v >= kMcm32Limit) ovf = true;
      }
    }
    __syncthreads();
  }
  }  // instances
  if (ovf) atomicOr(overflow, 1);
  if (ovf2) atomicOr(overflow, 2);
}

}  // namespace pipedp_dev

// sdp_kernels.cuh -- S-DP pipeline kernels for sm_100a.
//
// Reference semantics (sdp.cpp:48-60 fill_table, sdp_pipeline.hpp:24-46): for
// every cell i >= a_1, acc = ST[i - a_1] and then acc = acc (x) ST[i - a_j] for
// j = 2..k IN THAT ORDER.  Saturating-add is not associative for mixed signs,
// so the kernels keep the j-ascending left fold per cell (a_j descending) --
// exactly the order in which the paper's k-stage pipeline hands the partial
// accumulator from lane j to lane j+1.  Regrouping (never reordering) is used
// only when the host has proven the operator associative on the instance
// (min, max, modular-add always; saturating-add when no two init values have
// opposite signs) -- template flag ASSOC.
//
// B200 mapping:
//  * cells are processed in batches of 32, one cell per lane, so a warp's ring
//    read for one offset touches 32 consecutive words (conflict-free);
//  * the offsets are split into three pipeline STAGES by size; each stage is a
//    set of warps that hands the 32 partial accumulators of a batch to the
//    next stage through shared-memory slots published with st.release.cta:
//      far   (a_j >= a_mid): lookahead >= a_mid/32 batches, most of the work;
//      mid   (64 <= a_j < a_mid): lookahead 2 batches;
//      chain (a_j < 64): one warp.  Offsets in [32, 64) and the out-of-batch
//            part of offsets < 32 come from the ring; the in-batch part is a
//            31-step warp-shuffle broadcast (step t: lane t-1 is final and
//            every lane l with l-t+1 in the offset set folds it).  This
//            hand-off is the kernel's dependency-chain step;
//  * finalised values live in a MIRRORED shared-memory ring (value stored at p
//    and p + R) so the operand of offset a is simply base_lane - a;
//  * finished batches stream to HBM as coalesced int64 stores issued by the
//    mid warps two batches behind the chain (GFAR=false), or by the chain warp
//    itself when a_1 is too large for a shared-memory ring (GFAR=true: the far
//    stage then reads its operands from the HBM table, L1/L2-resident).
#pragma once

#include "common.cuh"

namespace pipedp_dev {

constexpr int kMidSlots = 32;  // mid -> chain partial slots
constexpr int kFarSlots = 64;  // far -> mid partial slots

// Uniform launch shape (all instances of a launch share n, k, a_1).
struct SdpShape {
  int64_t n;
  int32_t k;
  int32_t a1;
  int32_t ring_log2;  // R = 1 << ring_log2 (ring holds 2R values)
  int32_t a_mid;      // offsets >= a_mid belong to the far stage
  int32_t mid_warps;
  int32_t far_warps;
};

template <typename T, typename S>
__device__ __forceinline__ T ldv(const S* p) {
  return (T)(*p);
}

// Fold offsets[j0, j1) into acc; operands at base[-a].  HAVE=false assigns the
// first operand (sdp.cpp:53).  ASSOC splits the range into four contiguous
// quarters folded independently and combined in order (regrouping only).
template <int OP, typename T, bool ASSOC, typename S>
__device__ __forceinline__ T fold_range(T acc, bool have, const S* __restrict__ base,
                                        const int32_t* __restrict__ offs, int j0, int j1) {
  using O = SemiOp<OP, T>;
  if (j0 >= j1) return acc;
  if (!have) {
    acc = ldv<T>(base - offs[j0]);
    ++j0;
  }
  if (ASSOC && j1 - j0 >= 16) {
    const int q = (j1 - j0) >> 2;
    const int s1 = j0 + q, s2 = j0 + 2 * q, s3 = j0 + 3 * q;
    T p0 = acc;
    T p1 = ldv<T>(base - offs[s1]);
    T p2 = ldv<T>(base - offs[s2]);
    T p3 = ldv<T>(base - offs[s3]);
    for (int i = 1; i < q; ++i) {
      const T v0 = ldv<T>(base - offs[j0 + i - 1]);
      const T v1 = ldv<T>(base - offs[s1 + i]);
      const T v2 = ldv<T>(base - offs[s2 + i]);
      const T v3 = ldv<T>(base - offs[s3 + i]);
      p0 = O::apply(p0, v0);
      p1 = O::apply(p1, v1);
      p2 = O::apply(p2, v2);
      p3 = O::apply(p3, v3);
    }
    p0 = O::apply(p0, ldv<T>(base - offs[s1 - 1]));
    for (int j = s3 + q; j < j1; ++j) p3 = O::apply(p3, ldv<T>(base - offs[j]));
    return O::apply(O::apply(O::apply(p0, p1), p2), p3);
  }
  int j = j0;
  for (; j + 4 <= j1; j += 4) {
    const T v0 = ldv<T>(base - offs[j]);
    const T v1 = ldv<T>(base - offs[j + 1]);
    const T v2 = ldv<T>(base - offs[j + 2]);
    const T v3 = ldv<T>(base - offs[j + 3]);
    acc = O::apply(O::apply(O::apply(O::apply(acc, v0), v1), v2), v3);
  }
  for (; j < j1; ++j) acc = O::apply(acc, ldv<T>(base - offs[j]));
  return acc;
}

// -----------------------------------------------------------------------------
// The chain warp's fold for one batch: offsets[jb, k) (all < 64), strictly in
// descending order.  HAVE_ACC=false: no larger offset exists, the first
// operand is ASSIGNED, possibly inside the shuffle chain.  ring_pos = position
// of this lane's cell in the upper ring half; operand of offset a at
// ring[ring_pos - a].
template <int OP, typename T, bool HAVE_ACC>
__device__ __forceinline__ T chain_fold(T acc, const T* __restrict__ ring, uint32_t ring_pos,
                                        const int32_t* __restrict__ offs, int jb, int j32, int k,
                                        uint32_t mask32, int lane) {
  using O = SemiOp<OP, T>;
  bool have = HAVE_ACC;
  for (int j = jb; j < j32; ++j) {  // offsets in [32, 64): out of batch for all lanes
    const T v = ring[ring_pos - offs[j]];
    acc = (HAVE_ACC || have) ? O::apply(acc, v) : v;
    have = true;
  }
  for (int j = j32; j < k; ++j) {  // offsets < 32 reaching into earlier batches (a > lane)
    const int a = offs[j];
    if (a > lane) {
      const T v = ring[ring_pos - a];
      acc = (HAVE_ACC || have) ? O::apply(acc, v) : v;
      have = true;
    }
  }
  // in-batch chain: step t folds offset a = lane - t + 1 with lane t-1's value
  const uint32_t bits = (mask32 & ((2u << lane) - 1u) & ~1u) << (31 - lane);
#pragma unroll
  for (int t = 1; t < 32; ++t) {
    const T v = shfl_idx(acc, t - 1);
    const bool take = (bits >> (32 - t)) & 1u;
    if (HAVE_ACC) {
      if (take) acc = O::apply(acc, v);
    } else {
      if (take) acc = have ? O::apply(acc, v) : v;
      have = have || take;
    }
  }
  return acc;
}

__device__ __forceinline__ void spin_until_ge(const int* flag, int target) {
  while (ld_acquire_cta(flag) < target) __nanosleep(16);
}

// Offset classes of one instance, from its offsets in shared memory.
struct SdpClasses {
  int jf, jn, j32, far_look;
  uint32_t mask32;
};

__device__ __forceinline__ SdpClasses sdp_classes(const int32_t* offs, int k, int a_mid) {
  SdpClasses c{0, 0, 0, 0, 0u};
  for (int j = 0; j < k; ++j) {
    const int a = offs[j];
    c.jf += a >= a_mid;
    c.jn += a >= 64;
    c.j32 += a >= 32;
    if (a < 32) c.mask32 |= 1u << a;
  }
  c.far_look = c.jf > 0 ? offs[c.jf - 1] / 32 : 0;
  return c;
}

// -----------------------------------------------------------------------------
// One CTA per instance (blockIdx.x = instance; batch 1 = the single-instance
// solver):
//   warp 0                          chain stage
//   warps 1 .. mid_warps            mid stage   (batch b -> warp 1 + b % mid_warps)
//   warps mid_warps+1 .. +far_warps far stage   (batch b -> b % far_warps)
// SMALL (a_1 < 64): chain warp only.
template <int OP, typename T, bool SMALL, bool ASSOC, bool GFAR>
__global__ void __launch_bounds__(1024, 1)
    sdp_pipeline_cta(const SdpShape S, const int64_t* __restrict__ g_offsets,
                     const int64_t* __restrict__ g_init, int64_t* __restrict__ g_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t R = 1u << S.ring_log2;
  const int kpad = (S.k + 3) & ~3;
  T* ring = reinterpret_cast<T*>(smem);
  int32_t* offs = reinterpret_cast<int32_t*>(ring + 2 * R);
  T* mid_part = reinterpret_cast<T*>(offs + kpad);
  T* far_part = mid_part + kMidSlots * 32;
  int* flags = reinterpret_cast<int*>(far_part + kFarSlots * 32);
  int* final_count = flags;                // batches finalised by the chain warp
  int* mid_ready = flags + 1;              // [kMidSlots] = batch+1 held by the slot
  int* far_ready = mid_ready + kMidSlots;  // [kFarSlots]

  const int64_t inst = blockIdx.x;
  const int64_t* offsets = g_offsets + inst * S.k;
  const int64_t* init = g_init + inst * S.a1;
  int64_t* out = g_out + inst * S.n;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int64_t a1 = S.a1;
  const int64_t n = S.n;

  for (int j = tid; j < S.k; j += blockDim.x) offs[j] = (int32_t)offsets[j];
  const int64_t ring_from = a1 > (int64_t)R ? a1 - (int64_t)R : 0;  // the last R preset cells
  for (int64_t i = tid; i < a1; i += blockDim.x) {
    const int64_t v = init[i];
    if (i >= ring_from) {
      const uint32_t p = (uint32_t)i & (R - 1);
      ring[p] = (T)v;
      ring[p + R] = (T)v;
    }
    out[i] = v;
  }
  if (tid == 0) *final_count = 0;
  for (int s = tid; s < kMidSlots + kFarSlots; s += blockDim.x) mid_ready[s] = 0;
  __syncthreads();
  const SdpClasses C = sdp_classes(offs, S.k, S.a_mid);
  const int64_t nb = (n - a1 + 31) / 32;  // batches of 32 computed cells

  if (warp == 0) {
    // ============================ chain stage ===============================
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t c = a1 + 32 * b + lane;
      const uint32_t pos = ((uint32_t)c & (R - 1)) + R;
      T acc;
      if (!SMALL) {
        const int slot = (int)(b % kMidSlots);
        while (ld_acquire_cta(&mid_ready[slot]) != (int)(b + 1)) {
        }
        acc = mid_part[slot * 32 + lane];
        acc = chain_fold<OP, T, true>(acc, ring, pos, offs, C.jn, C.j32, S.k, C.mask32, lane);
      } else {
        acc = chain_fold<OP, T, false>(T(0), ring, pos, offs, 0, C.j32, S.k, C.mask32, lane);
      }
      if (c < n) {
        ring[pos - R] = acc;
        ring[pos] = acc;
        if (SMALL || GFAR) out[c] = (int64_t)acc;
      }
      __syncwarp();
      if (lane == 0) st_release_cta(final_count, (int)(b + 1));
    }
  } else if (!SMALL && warp <= S.mid_warps) {
    // ============================ mid stage =================================
    for (int64_t b = warp - 1; b < nb; b += S.mid_warps) {
      spin_until_ge(final_count, (int)(b - 1));  // offsets >= 64 reach batches <= b-2
      if (!GFAR && b >= 2) {  // stream batch b-2 (final, still in the ring) to HBM
        const int64_t cw = a1 + 32 * (b - 2) + lane;
        if (cw < n) out[cw] = (int64_t)ring[(uint32_t)cw & (R - 1)];
      }
      const int64_t c = a1 + 32 * b + lane;
      const T* base = ring + (((uint32_t)c & (R - 1)) + R);
      T acc = T(0);
      bool have = false;
      if (C.jf > 0) {
        const int fs = (int)(b % kFarSlots);
        spin_until_ge(&far_ready[fs], (int)(b + 1));
        acc = far_part[fs * 32 + lane];
        have = true;
      }
      acc = fold_range<OP, T, ASSOC>(acc, have, base, offs, C.jf, C.jn);
      const int slot = (int)(b % kMidSlots);
      mid_part[slot * 32 + lane] = acc;
      __syncwarp();
      if (lane == 0) st_release_cta(&mid_ready[slot], (int)(b + 1));
    }
  } else if (!SMALL && C.jf > 0 && warp <= S.mid_warps + S.far_warps) {
    // ============================ far stage =================================
    const int f = warp - 1 - S.mid_warps;
    for (int64_t b = f; b < nb; b += S.far_warps) {
      // operands final, and the slot's previous batch consumed by the mid stage
      const int64_t need = b + 1 - C.far_look;
      const int64_t need_slot = b + 1 - kFarSlots;
      spin_until_ge(final_count, (int)(need > need_slot ? need : need_slot));
      const int64_t c = a1 + 32 * b + lane;
      T acc;
      if (GFAR) {
        acc = fold_range<OP, T, ASSOC>(T(0), false, out + c, offs, 0, C.jf);
      } else {
        const T* base = ring + (((uint32_t)c & (R - 1)) + R);
        acc = fold_range<OP, T, ASSOC>(T(0), false, base, offs, 0, C.jf);
      }
      const int fs = (int)(b % kFarSlots);
      far_part[fs * 32 + lane] = acc;
      __syncwarp();
      if (lane == 0) st_release_cta(&far_ready[fs], (int)(b + 1));
    }
  }
  __syncthreads();
  if (!SMALL && !GFAR) {  // the last two batches were never streamed by a mid warp
    const int64_t first = nb >= 2 ? nb - 2 : 0;
    for (int64_t i = a1 + 32 * first + tid; i < n; i += blockDim.x) {
      out[i] = (int64_t)ring[(uint32_t)i & (R - 1)];
    }
  }
}

// -----------------------------------------------------------------------------
// Batched S-DP with a small a_1: one warp per instance runs every stage itself
// -- offsets >= 32 straight from its private mirrored ring, offsets < 32
// through chain_fold.  SMALL: a_1 < 32.
template <int OP, typename T, bool SMALL, bool ASSOC>
__global__ void __launch_bounds__(256)
    sdp_batch_warp(const SdpShape S, int64_t batch, const int64_t* __restrict__ g_offsets,
                   const int64_t* __restrict__ g_init, int64_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t R = 1u << S.ring_log2;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int kpad = (S.k + 3) & ~3;
  T* ring = reinterpret_cast<T*>(smem) + (size_t)warp * 2 * R;
  int32_t* offs = reinterpret_cast<int32_t*>(reinterpret_cast<T*>(smem) + (size_t)wpb * 2 * R) +
                  (size_t)warp * kpad;
  const int64_t inst = (int64_t)blockIdx.x * wpb + warp;
  if (inst >= batch) return;
  const int64_t a1 = S.a1, n = S.n;
  const int64_t* io = g_offsets + inst * S.k;
  const int64_t* ii = g_init + inst * a1;
  int64_t* o = out + inst * n;
  for (int j = lane; j < S.k; j += 32) offs[j] = (int32_t)io[j];
  for (int64_t i = lane; i < a1; i += 32) {
    const int64_t v = ii[i];
    const uint32_t p = (uint32_t)i & (R - 1);
    ring[p] = (T)v;
    ring[p + R] = (T)v;
    o[i] = v;
  }
  __syncwarp();
  int j32 = S.k;
  uint32_t mask32 = 0;
  for (int j = S.k - 1; j >= 0; --j) {
    const int a = offs[j];
    if (a >= 32) break;
    j32 = j;
    mask32 |= 1u << a;
  }
  const int64_t nb = (n - a1 + 31) / 32;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t c = a1 + 32 * b + lane;
    const uint32_t pos = ((uint32_t)c & (R - 1)) + R;
    T acc;
    if (!SMALL) {
      acc = fold_range<OP, T, ASSOC>(T(0), false, ring + pos, offs, 0, j32);
      acc = chain_fold<OP, T, true>(acc, ring, pos, offs, j32, j32, S.k, mask32, lane);
    } else {
      acc = chain_fold<OP, T, false>(T(0), ring, pos, offs, 0, 0, S.k, mask32, lane);
    }
    if (c < n) {
      ring[pos - R] = acc;
      ring[pos] = acc;
      o[c] = (int64_t)acc;
    }
    __syncwarp();
  }
}

// -----------------------------------------------------------------------------
// Hand-off microbenchmark: the chain warp's dependent step (warp-shuffle
// broadcast + one (x)) with every step taking, timed with clock64.  Gives
// t_step,min for the dependency-chain roofline.
template <int OP, typename T>
__global__ void sdp_chain_step_probe(int64_t batches, T seed, long long* cycles, T* sink) {
  using O = SemiOp<OP, T>;
  const int lane = threadIdx.x & 31;
  T acc = seed + (T)lane;
  const uint32_t bits = ((2u << lane) - 1u) & ~1u;
  const uint32_t rev = bits << (31 - lane);
  __syncwarp();
  const long long t0 = clock64();
  for (int64_t b = 0; b < batches; ++b) {
#pragma unroll
    for (int t = 1; t < 32; ++t) {
      const T v = shfl_idx(acc, t - 1);
      if ((rev >> (32 - t)) & 1u) acc = O::apply(acc, v);
    }
    acc = shfl_idx(acc, 31);
  }
  const long long t1 = clock64();
  if (lane == 0) *cycles = t1 - t0;
  sink[lane] = acc;
}

}  // namespace pipedp_dev

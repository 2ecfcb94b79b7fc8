// sdp_kernels.cuh -- S-DP pipeline kernels for sm_100a.
//
// Reference semantics (sdp.cpp:48-60 fill_table, sdp_pipeline.hpp:24-46): for
// every cell i >= a_1, acc = ST[i - a_1] and then acc = acc (x) ST[i - a_j] for
// j = 2..k IN THAT ORDER.  Saturating-add is not associative for mixed signs,
// so every kernel keeps the j-ascending left fold per cell (a_j descending) --
// the order in which the paper's k-stage pipeline hands the partial
// accumulator from lane j to lane j+1.  Regrouping (never reordering) is used
// only when the host has proven the operator associative on the instance
// (min, max, modular-add always; saturating-add when no two init values have
// opposite signs): template flag ASSOC.
//
// B200 mapping:
//  * cells are processed in batches of 32, one cell per lane, so a warp's ring
//    read for one offset touches 32 consecutive words (conflict-free);
//  * the offsets are split into pipeline STAGES by size.  A stage is a set of
//    warps; it hands the 32 partial accumulators of a batch to the next stage
//    through a shared-memory slot guarded by an mbarrier (hardware-suspended
//    waits, so idle stages burn no issue slots):
//      remote (a >= a_remote): producer CTAs on other SMs (multi-CTA mode),
//              operands read from the HBM table (L2), partials through global
//              slots with gpu-scope release/acquire flags;
//      far    (a_mid <= a < a_remote): lookahead >= a_mid/32 batches;
//      mid    (64 <= a < a_mid): lookahead 2 batches;
//      chain  (a < 64): one warp.  Offsets in [32, 64) and the out-of-batch
//              part of offsets < 32 come from the ring; the in-batch part is a
//              31-step warp-shuffle broadcast (step t: lane t-1 is final and
//              every lane l with l-t+1 in the offset set folds it).  This
//              hand-off is the kernel's dependency-chain step;
//  * finalised values live in a MIRRORED shared-memory ring (value stored at p
//    and p + R) so the operand of offset a is base_lane - a (offsets are kept
//    pre-scaled to bytes: one IADD per term);
//  * a writer warp streams finished batches to HBM (coalesced int64 stores)
//    and, in multi-CTA mode, publishes the finished prefix to the producers
//    with a gpu-scope release every few batches.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace pipedp_dev {

constexpr int kMidSlots = 32;  // mid -> chain partial slots
constexpr int kFarSlots = 64;  // far -> mid partial slots
constexpr int kBatchBars = 64; // batch_done / written mbarrier rings
constexpr int kRemSlots = 64;  // remote -> far partial slots (global)
constexpr int kPubEvery = 4;   // writer publishes to the producers every 4 batches

// Uniform launch shape (all instances of a launch share n, k, a_1).
struct SdpShape {
  int64_t n;
  int32_t k;
  int32_t a1;
  int32_t ring_log2;  // R = 1 << ring_log2 (ring holds 2R values)
  int32_t a_mid;      // offsets >= a_mid: far stage (or remote)
  int32_t a_remote;   // offsets >= a_remote: remote producers (multi-CTA mode only)
  int32_t ring_cover; // largest offset read from the ring (a_1, a_mid or a_remote)
  int32_t mid_warps;
  int32_t far_warps;
  int32_t remote_warps;  // warps per producer CTA
  int32_t writers;       // finisher writer warps publishing progress (published[0..writers))
  int32_t j_rem;         // number of offsets >= a_remote (the producers' share)
  int32_t rem_look;      // batches between a producer batch and the newest cell it reads
  const int32_t* perm;   // batch warp kernel: warp -> instance order (nullable), set at launch
};

// Global workspace of the multi-CTA mode (zeroed before every launch).
struct SdpRemote {
  void* part;               // [kRemSlots][32] T
  int* ready;               // [kRemSlots] batch+1
  unsigned long long* published;  // [writers] batches < published[w] of writer w's share are in HBM
  const int32_t* obg;             // [k] offsets as HBM-table byte offsets (a_j * 8)
};

template <typename T, typename S>
__device__ __forceinline__ T ldv(const S* p) {
  return (T)(*p);
}
template <typename T, typename S>
__device__ __forceinline__ T ldv_cg(const S* p);
template <>
__device__ __forceinline__ int32_t ldv_cg<int32_t, int64_t>(const int64_t* p) {
  return (int32_t)__ldcg(reinterpret_cast<const long long*>(p));
}
template <>
__device__ __forceinline__ int64_t ldv_cg<int64_t, int64_t>(const int64_t* p) {
  return (int64_t)__ldcg(reinterpret_cast<const long long*>(p));
}

// Element at (char*)base - off_bytes.
template <typename T, typename S, bool CG>
__device__ __forceinline__ T at(const char* base, int32_t ob) {
  const S* p = reinterpret_cast<const S*>(base - ob);
  if constexpr (CG) return ldv_cg<T, S>(p);
  else return ldv<T>(p);
}

// Fold the operands at byte offsets ob[j0, j1) below `base` into acc.
// HAVE=false assigns the first operand (sdp.cpp:53).  ASSOC folds four
// contiguous quarters independently and combines them in order (regrouping).
template <int OP, typename T, bool ASSOC, typename S, bool CG = false>
__device__ __forceinline__ T fold_range(T acc, bool have, const S* base_elem,
                                        const int32_t* __restrict__ ob, int j0, int j1) {
  using O = SemiOp<OP, T>;
  const char* base = reinterpret_cast<const char*>(base_elem);
  if (j0 >= j1) return acc;
  if (!have) {
    acc = at<T, S, CG>(base, ob[j0]);
    ++j0;
  }
  if (ASSOC && j1 - j0 >= 16) {
    const int q = (j1 - j0) >> 2;
    const int s1 = j0 + q, s2 = j0 + 2 * q, s3 = j0 + 3 * q;
    T p0 = acc;
    T p1 = at<T, S, CG>(base, ob[s1]);
    T p2 = at<T, S, CG>(base, ob[s2]);
    T p3 = at<T, S, CG>(base, ob[s3]);
#pragma unroll 4
    for (int i = 1; i < q; ++i) {
      const T v0 = at<T, S, CG>(base, ob[j0 + i - 1]);
      const T v1 = at<T, S, CG>(base, ob[s1 + i]);
      const T v2 = at<T, S, CG>(base, ob[s2 + i]);
      const T v3 = at<T, S, CG>(base, ob[s3 + i]);
      p0 = O::apply(p0, v0);
      p1 = O::apply(p1, v1);
      p2 = O::apply(p2, v2);
      p3 = O::apply(p3, v3);
    }
    p0 = O::apply(p0, at<T, S, CG>(base, ob[s1 - 1]));
    for (int j = s3 + q; j < j1; ++j) p3 = O::apply(p3, at<T, S, CG>(base, ob[j]));
    return O::apply(O::apply(O::apply(p0, p1), p2), p3);
  }
  int j = j0;
  for (; j + 4 <= j1; j += 4) {
    const T v0 = at<T, S, CG>(base, ob[j]);
    const T v1 = at<T, S, CG>(base, ob[j + 1]);
    const T v2 = at<T, S, CG>(base, ob[j + 2]);
    const T v3 = at<T, S, CG>(base, ob[j + 3]);
    acc = O::apply(O::apply(O::apply(O::apply(acc, v0), v1), v2), v3);
  }
  for (; j < j1; ++j) acc = O::apply(acc, at<T, S, CG>(base, ob[j]));
  return acc;
}

// -----------------------------------------------------------------------------
// The chain warp's fold for one batch: offsets[jb, k) (all < 64), strictly in
// descending order.  HAVE_ACC=false: no larger offset exists, the first
// operand is ASSIGNED, possibly inside the shuffle chain.  ring_pos = position
// of this lane's cell in the upper ring half; operand of offset a at
// ring[ring_pos - a].  `bits` = chain_bits(mask32, lane), hoisted by the caller.
__device__ __forceinline__ uint32_t chain_bits(uint32_t mask32, int lane) {
  return (mask32 & ((2u << lane) - 1u) & ~1u) << (31 - lane);
}

// Bit (32 - t) of `bits`, tested at step t.  asm volatile keeps the test at its
// step: left to itself the compiler materialises all 31 predicates up front
// (~100 bit-shuffling instructions per batch on the critical warp).
template <int T_STEP>
__device__ __forceinline__ bool chain_take(uint32_t bits) {
  uint32_t r;
  asm volatile("and.b32 %0, %1, %2;" : "=r"(r) : "r"(bits), "n"(1u << (32 - T_STEP)));
  return r != 0;
}

template <int OP, typename T, bool HAVE_ACC, int T_STEP>
struct ChainSteps {
  __device__ __forceinline__ static void run(T& acc, bool& have, uint32_t bits) {
    using O = SemiOp<OP, T>;
    const T v = shfl_idx(acc, T_STEP - 1);
    const bool take = chain_take<T_STEP>(bits);
    if (HAVE_ACC) {
      if (take) acc = O::apply(acc, v);
    } else {
      if (take) acc = have ? O::apply(acc, v) : v;
      have = have || take;
    }
    ChainSteps<OP, T, HAVE_ACC, T_STEP + 1>::run(acc, have, bits);
  }
};
template <int OP, typename T, bool HAVE_ACC>
struct ChainSteps<OP, T, HAVE_ACC, 32> {
  __device__ __forceinline__ static void run(T&, bool&, uint32_t) {}
};

// Out-of-batch operands of the chain warp: offsets d in [32, 64) (all lanes)
// and d < 32 with d > lane, in descending d.  Displacements are compile-time
// immediates.  The 63 candidate slots are processed in groups of 16: all 16
// loads are issued first (distinct registers, unconditional -- every slot lies
// inside the ring), then
//   ASSOC: absent slots become the operator's identity and the group is
//          reduced as a tree, one (x) into the accumulator per group;
//   strict: predicated left fold in descending d (saturating-add, mixed signs).
template <int D>
__device__ __forceinline__ bool pre_take(uint32_t hi, uint32_t lo) {
  uint32_t r;
  if (D >= 32) asm volatile("and.b32 %0, %1, %2;" : "=r"(r) : "r"(hi), "n"(1u << (D >= 32 ? D - 32 : 0)));
  else asm volatile("and.b32 %0, %1, %2;" : "=r"(r) : "r"(lo), "n"(1u << (D < 32 ? D : 0)));
  return r != 0;
}

template <int OP, typename T, int D0>  // slots D0, D0-1, ..., D0-15 (those >= 1)
__device__ __forceinline__ void pre_group_assoc(T& acc, const T* p, uint32_t hi, uint32_t lo) {
  using O = SemiOp<OP, T>;
  const T id = SemiId<OP, T>::value();
  T v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (D0 - i >= 1) ? p[-(D0 - i)] : id;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    bool t = false;
    switch (i) {  // keep the immediates compile-time
#define PRE_CASE(I) case I: t = (D0 - I >= 1) && pre_take<(D0 - I >= 1 ? D0 - I : 1)>(hi, lo); break;
      PRE_CASE(0) PRE_CASE(1) PRE_CASE(2) PRE_CASE(3) PRE_CASE(4) PRE_CASE(5) PRE_CASE(6)
      PRE_CASE(7) PRE_CASE(8) PRE_CASE(9) PRE_CASE(10) PRE_CASE(11) PRE_CASE(12) PRE_CASE(13)
      PRE_CASE(14) PRE_CASE(15)
#undef PRE_CASE
    }
    if (!t) v[i] = id;
  }
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) v[i] = O::apply(v[i], v[i + w]);
  }
  acc = O::apply(acc, v[0]);
}

template <int OP, typename T, bool HAVE_ACC, int D0>
__device__ __forceinline__ void pre_group_strict(T& acc, bool& have, const T* p, uint32_t hi,
                                                 uint32_t lo) {
  using O = SemiOp<OP, T>;
  T v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (D0 - i >= 1) ? p[-(D0 - i)] : T(0);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    bool t = false;
    switch (i) {
#define PRE_CASE(I) case I: t = (D0 - I >= 1) && pre_take<(D0 - I >= 1 ? D0 - I : 1)>(hi, lo); break;
      PRE_CASE(0) PRE_CASE(1) PRE_CASE(2) PRE_CASE(3) PRE_CASE(4) PRE_CASE(5) PRE_CASE(6)
      PRE_CASE(7) PRE_CASE(8) PRE_CASE(9) PRE_CASE(10) PRE_CASE(11) PRE_CASE(12) PRE_CASE(13)
      PRE_CASE(14) PRE_CASE(15)
#undef PRE_CASE
    }
    if (t) {
      if (HAVE_ACC) {
        acc = O::apply(acc, v[i]);
      } else {
        acc = have ? O::apply(acc, v[i]) : v[i];
        have = true;
      }
    }
  }
}

template <int OP, typename T, bool HAVE_ACC, bool ASSOC>
__device__ __forceinline__ void pre_steps(T& acc, bool& have, const T* p, uint32_t hi, uint32_t lo) {
  // 64-bit modular-add keeps the strict path: folding the identity would
  // normalise a raw single operand (k = 1 copies raw values, sdp.cpp:53)
  constexpr bool kTree = ASSOC && HAVE_ACC && !(OP == kModAdd && sizeof(T) == 8);
  if (kTree) {
    pre_group_assoc<OP, T, 63>(acc, p, hi, lo);
    pre_group_assoc<OP, T, 47>(acc, p, hi, lo);
    pre_group_assoc<OP, T, 31>(acc, p, hi, lo);
    pre_group_assoc<OP, T, 15>(acc, p, hi, lo);
  } else {
    pre_group_strict<OP, T, HAVE_ACC, 63>(acc, have, p, hi, lo);
    pre_group_strict<OP, T, HAVE_ACC, 47>(acc, have, p, hi, lo);
    pre_group_strict<OP, T, HAVE_ACC, 31>(acc, have, p, hi, lo);
    pre_group_strict<OP, T, HAVE_ACC, 15>(acc, have, p, hi, lo);
  }
}

// Per-lane chain masks of one instance.
struct ChainMasks {
  uint32_t hi;    // bit d-32 for offsets d in [32, 64)
  uint32_t lo;    // bit d for offsets d < 32 with d > lane (out of batch)
  uint32_t bits;  // chain_bits(): in-batch steps
};

__device__ __forceinline__ ChainMasks chain_masks(const int32_t* offs, int k, int lane) {
  uint32_t hi = 0, m32 = 0;
  for (int j = k - 1; j >= 0; --j) {
    const int a = offs[j];
    if (a >= 64) break;
    if (a >= 32) hi |= 1u << (a - 32);
    else m32 |= 1u << a;
  }
  return ChainMasks{hi, m32 & ~((2u << lane) - 1u), chain_bits(m32, lane)};
}

// The chain warp's fold for one batch: every offset < 64, strictly in
// descending order.  HAVE_ACC=false: no larger offset exists, the first
// operand is ASSIGNED (possibly inside the shuffle chain).  ring_pos =
// position of this lane's cell in the upper ring half.
template <int OP, typename T, bool HAVE_ACC, bool ASSOC>
__device__ __forceinline__ T chain_fold(T acc, const T* __restrict__ ring, uint32_t ring_pos,
                                        const ChainMasks& m) {
  bool have = HAVE_ACC;
  pre_steps<OP, T, HAVE_ACC, ASSOC>(acc, have, ring + ring_pos, m.hi, m.lo);
  // in-batch chain: step t folds offset a = lane - t + 1 with lane t-1's value
  ChainSteps<OP, T, HAVE_ACC, 1>::run(acc, have, m.bits);
  return acc;
}

// ---- look-ahead chain (associative ops) -------------------------------------
// While batch b's shuffle chain broadcasts cell t-1 of batch b, every lane l
// also folds it into its accumulator for batch b+1 when offset d = l+33-t is in
// the set (the cell c0+32+l-d of batch b+1's lane l).  Together with the ring
// group d >= l+33 (cells of batch b-1, folded first) this covers every
// out-of-batch offset < 64 of batch b+1 in descending d, so batch b+1 starts
// with mid(b+1) (x) next -- regrouping only (ASSOC).  Step 32 broadcasts lane
// 31 for d = l+1.
struct LaMasks {
  uint32_t bits;   // in-batch steps of the current batch (chain_bits)
  uint32_t nbits;  // bit 32-t: offset l+33-t present (t = 1..32)
  uint32_t far;    // bit d-32 for d in [l+33, 63] present
};

__device__ __forceinline__ LaMasks la_masks(const int32_t* offs, int k, int lane) {
  uint64_t s64 = 0;
  for (int j = k - 1; j >= 0; --j) {
    const int a = offs[j];
    if (a >= 64) break;
    s64 |= 1ull << a;
  }
  const uint32_t hi = (uint32_t)(s64 >> 32);
  return LaMasks{chain_bits((uint32_t)s64, lane), (uint32_t)(s64 >> (lane + 1)),
                 hi & ~((2u << lane) - 1u)};
}

template <int T_STEP>
__device__ __forceinline__ bool bit_at(uint32_t m) {
  uint32_t r;
  asm volatile("and.b32 %0, %1, %2;" : "=r"(r) : "r"(m), "n"(1u << (32 - T_STEP)));
  return r != 0;
}

template <int OP, typename T, int T_STEP>
struct LaSteps {
  __device__ __forceinline__ static void run(T& acc, T& nxt, const LaMasks& m) {
    using O = SemiOp<OP, T>;
    const T v = shfl_idx(acc, T_STEP - 1);
    if (bit_at<T_STEP>(m.bits)) acc = O::apply(acc, v);
    if (bit_at<T_STEP>(m.nbits)) nxt = O::apply(nxt, v);
    LaSteps<OP, T, T_STEP + 1>::run(acc, nxt, m);
  }
};
template <int OP, typename T>
struct LaSteps<OP, T, 32> {
  __device__ __forceinline__ static void run(T& acc, T& nxt, const LaMasks& m) {
    using O = SemiOp<OP, T>;
    const T v = shfl_idx(acc, 31);  // last cell of the batch, offset l+1 of the next
    uint32_t r;
    asm volatile("and.b32 %0, %1, 1;" : "=r"(r) : "r"(m.nbits));
    if (r) nxt = O::apply(nxt, v);
  }
};

// ---- idempotent closure (min / max) ------------------------------------------
// For an idempotent, associative, commutative (x) the in-batch recurrence
//   x_l = b_l (x) (x)_{d in S, d <= l} x_{l-d}      (b_l: every out-of-batch term)
// unrolls to x_l = (x)_{t in T_l} b_t with T_l = {t <= l : l - t in S*}, S* the
// additive closure of the offset set (a path t -> l of in-batch steps exists
// iff l - t is a sum of offsets; folding a value twice changes nothing).  The
// next batch's terms from this batch, (x)_{d in S, l < d <= l+32} x_{l+32-d},
// unroll the same way to (x)_{t in V_l} b_t.  Both are reductions over b that
// do NOT depend on each other lane's result, so the batch's 31 dependent
// shuffle steps become independent shuffles.  When 1 in S, S* covers
// everything: T_l = [0, l] (x = inclusive prefix-(x) of b, a 5-step scan) and
// x is monotone along the batch, so the next-batch fold is x at the single
// lane src_l = l + 32 - min{d in S : d > l}.
struct IdemMasks {
  uint32_t T;   // in-batch sources of x_l
  uint32_t V;   // sources of the next batch's fold
  int32_t src;  // scan form: lane whose x is the next-batch fold (-1: none)
  bool scan;    // 1 in S (warp-uniform)
};

__device__ __forceinline__ IdemMasks idem_masks(const int32_t* offs, int k, int lane) {
  uint64_t s64 = 0;
  for (int j = k - 1; j >= 0; --j) {
    const int a = offs[j];
    if (a >= 64) break;
    s64 |= 1ull << a;
  }
  const uint32_t s32 = (uint32_t)s64;
  uint32_t reach = 1;  // bit m: m in S* (m < 32)
  for (int m = 1; m < 32; ++m) {
    const uint32_t cand = s32 & ((2u << m) - 1u);  // offsets d <= m
    uint32_t hit = 0;
    for (int d = 1; d <= m; ++d) hit |= ((cand >> d) & (reach >> (m - d))) & 1u;
    reach |= hit << m;
  }
  auto tmask = [&](int l) {  // T_l
    uint32_t t = 0;
    for (int u = 0; u <= l; ++u) t |= ((reach >> (l - u)) & 1u) << u;
    return t;
  };
  IdemMasks m;
  m.scan = (s64 & 2ull) != 0;
  m.T = tmask(lane);
  m.V = 0;
  m.src = -1;
  for (int t = 31; t >= 0; --t) {  // U_l = {t : l + 32 - t in S}
    const int d = lane + 32 - t;
    if ((s64 >> d) & 1ull) {
      m.V |= tmask(t);
      if (m.src < 0) m.src = t;  // largest t = smallest d
    }
  }
  return m;
}

// General form: broadcast b_t, t = 0..31 (independent shuffles), fold into x
// when t in T_l and into the next-batch accumulator when t in V_l.  Four
// accumulators per side (t mod 4), combined at the end: the 32 folds form four
// independent chains of 8 instead of one chain of 32 (the batch's critical
// path is the chain warp's closure latency); regrouping an idempotent,
// commutative (x) changes nothing.
template <int OP, typename T, int TT>
struct IdemBcast {
  __device__ __forceinline__ static void run(const T& b, T* x, T* nx, uint32_t mt, uint32_t mv) {
    using O = SemiOp<OP, T>;
    const T v = shfl_idx(b, TT);
    if (bit_at<32 - TT>(mt)) x[TT & 3] = O::apply(x[TT & 3], v);  // bit TT
    if (bit_at<32 - TT>(mv)) nx[TT & 3] = O::apply(nx[TT & 3], v);
    IdemBcast<OP, T, TT + 1>::run(b, x, nx, mt, mv);
  }
};
template <int OP, typename T>
struct IdemBcast<OP, T, 32> {
  __device__ __forceinline__ static void run(const T&, T*, T*, uint32_t, uint32_t) {}
};

// acc: in b, out x.  nxt: out, the next batch's fold of this batch's cells.
template <int OP, typename T>
__device__ __forceinline__ void idem_closure(T& acc, T& nxt, const IdemMasks& m) {
  using O = SemiOp<OP, T>;
  const T id = SemiId<OP, T>::value();
  if (m.scan) {
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const T v = __shfl_up_sync(0xffffffffu, acc, s);  // lanes < s get their own value: idempotent
      acc = O::apply(acc, v);
    }
    const T v = shfl_idx(acc, m.src < 0 ? 0 : m.src);
    nxt = m.src < 0 ? id : v;
  } else {
    T x[4] = {id, id, id, id}, nx[4] = {id, id, id, id};
    IdemBcast<OP, T, 0>::run(acc, x, nx, m.T, m.V);
    acc = O::apply(O::apply(x[0], x[1]), O::apply(x[2], x[3]));
    nxt = O::apply(O::apply(nx[0], nx[1]), O::apply(nx[2], nx[3]));
  }
}

template <int OP>
struct IsIdem {
  static constexpr bool value = OP == kMin || OP == kMax;
};

// Ring group of offsets d in [l+33, 63] below p (cells two batches back),
// identity for absent slots, tree-reduced.  The identity select is arithmetic
// (sign-extended mask bit + LOP3): 31 live predicates exhaust the 7 predicate
// registers.
template <typename T>
__device__ __forceinline__ T sel_or_id(T x, T id, uint32_t word, int bit) {
  const int32_t m32 = (int32_t)(word << (31 - bit)) >> 31;  // 0 or -1
  const T m = (T)m32;
  return (x & m) | (id & ~m);
}

template <int OP, typename T>
__device__ __forceinline__ T la_ring_group(const T* p, uint32_t far) {
  using O = SemiOp<OP, T>;
  const T id = SemiId<OP, T>::value();
  T v[32];
#pragma unroll
  for (int i = 0; i < 31; ++i) v[i] = sel_or_id(p[-(63 - i)], id, far, 31 - i);  // d = 63 - i
  v[31] = id;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) v[i] = O::apply(v[i], v[i + w]);
  }
  return v[0];
}

// The ring group's slots i in [I0, I1) only (d = 63 - i), tree-reduced: a
// batch's group split over several warps.
template <int OP, typename T, int I0, int I1>
__device__ __forceinline__ T la_ring_range(const T* p, uint32_t far) {
  using O = SemiOp<OP, T>;
  const T id = SemiId<OP, T>::value();
  constexpr int W = 32;
  T v[W];
#pragma unroll
  for (int i = 0; i < W; ++i) v[i] = (i >= I0 && i < I1 && i < 31) ? sel_or_id(p[-(63 - i)], id, far, 31 - i) : id;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) v[i] = O::apply(v[i], v[i + w]);
  }
  return v[0];
}

// Offset classes of one instance, from its raw offsets in shared memory.
struct SdpClasses {
  int jr, jf, jn, j32;
  int far_look, rem_look;
  uint32_t mask32;
};

__device__ __forceinline__ SdpClasses sdp_classes(const int32_t* offs, int k, int a_mid,
                                                  int a_remote) {
  SdpClasses c{0, 0, 0, 0, 0, 0, 0u};
  for (int j = 0; j < k; ++j) {
    const int a = offs[j];
    c.jr += a >= a_remote;
    c.jf += a >= a_mid;
    c.jn += a >= 64;
    c.j32 += a >= 32;
    if (a < 32) c.mask32 |= 1u << a;
  }
  c.far_look = c.jf > c.jr ? offs[c.jf - 1] / 32 : 1 << 30;
  c.rem_look = c.jr > 0 ? offs[c.jr - 1] / 32 : 1 << 30;
  return c;
}

// Warp ids of the non-chain roles skip every id that is 0 mod 4: warps map to
// SM sub-partitions by id % 4, so the chain warp (id 0) owns SMSP 0 alone and
// its shuffle/(x) chain never waits behind another warp's issue.
__host__ __device__ __forceinline__ int sdp_role_of_warp(int warp) {
  return (warp % 4 == 0) ? -1 : warp - 1 - warp / 4;
}
__host__ __device__ __forceinline__ int sdp_warps_for_roles(int roles) {
  return roles == 0 ? 1 : 2 + (roles - 1) + (roles - 1) / 3;
}

__device__ __forceinline__ void wait_batches(uint64_t* bars, int64_t count) {
  // wait until batches [0, count) passed the barrier ring
  if (count <= 0) return;
  const int64_t b = count - 1;
  mbar_wait(&bars[b % kBatchBars], (unsigned)((b / kBatchBars) & 1));
}

// -----------------------------------------------------------------------------
// Finisher: one CTA per instance (blockIdx.x = instance), or block 0 of a
// multi-CTA launch (REMOTE) whose other blocks run sdp_remote_producer.
//   warp 0                 chain
//   warps 1 .. M           mid            (batch b -> 1 + b % M)
//   warps M+1 .. M+F       far            (batch b -> b % F)
//   warp  M+F+1            writer
// SMALL (a_1 < 64): chain warp only, it writes the table itself.
// GFAR: a_1 too large for the ring -- the far stage reads the HBM table.
template <int OP, typename T, bool SMALL, bool ASSOC, bool GFAR, bool REMOTE>
__device__ __forceinline__ void sdp_finisher(const SdpShape& S, const int64_t* __restrict__ offsets,
                                             const int64_t* __restrict__ init, int64_t* out,
                                             const SdpRemote& RM) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t R = 1u << S.ring_log2;
  const int kpad = (S.k + 3) & ~3;
  T* ring = reinterpret_cast<T*>(smem);
  int32_t* offs = reinterpret_cast<int32_t*>(ring + 2 * R);  // raw a_j
  int32_t* ob = offs + kpad;                                 // a_j * sizeof(T) (ring reads)
  int32_t* obg = ob + kpad;                                  // a_j * 8 (HBM table reads)
  T* mid_part = reinterpret_cast<T*>(obg + kpad);
  T* far_part = mid_part + kMidSlots * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(far_part + kFarSlots * 32);
  uint64_t* batch_done = bars;                  // [kBatchBars] chain -> all
  uint64_t* written = batch_done + kBatchBars;  // [kBatchBars] writer -> far
  uint64_t* mid_full = written + kBatchBars;    // [kMidSlots]
  uint64_t* far_full = mid_full + kMidSlots;    // [kFarSlots]

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int64_t a1 = S.a1;
  const int64_t n = S.n;

  for (int j = tid; j < S.k; j += blockDim.x) {
    const int32_t a = (int32_t)offsets[j];
    offs[j] = a;
    ob[j] = a * (int32_t)sizeof(T);
    obg[j] = a * 8;
  }
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
  if (tid == 0) {
    for (int s = 0; s < 2 * kBatchBars + kMidSlots + kFarSlots; ++s) mbar_init(&bars[s], 1);
  }
  __syncthreads();
  const SdpClasses C = sdp_classes(offs, S.k, S.a_mid, REMOTE ? S.a_remote : (1 << 30));
  const int64_t nb = (n - a1 + 31) / 32;  // batches of 32 computed cells
  const int M = S.mid_warps, F = S.far_warps;
  const int role = sdp_role_of_warp(warp);  // -1: chain warp or an idle SMSP-0 warp

  if (warp == 0) {
    // ================================= chain ================================
    const ChainMasks cm = chain_masks(offs, S.k, lane);
    constexpr bool kLA = !SMALL && ASSOC && !(OP == kModAdd && sizeof(T) == 8);
    const LaMasks lm = la_masks(offs, S.k, lane);
    const IdemMasks im = idem_masks(offs, S.k, lane);
    T nxt = T(0);  // look-ahead accumulator of the next batch (kLA)
    if (kLA) {
      // seed nxt for batch 0: offsets d in [l+1, l+32] over the preset cells,
      // descending (what the look-ahead of a virtual batch -1 would have folded)
      nxt = SemiId<OP, T>::value();
      const uint32_t pos0 = ((uint32_t)(a1 + lane) & (R - 1)) + R;
      for (int d = lane + 32; d >= lane + 1; --d) {
        if ((lm.nbits >> (d - lane - 1)) & 1u) nxt = SemiOp<OP, T>::apply(nxt, ring[pos0 - d]);
      }
    }
    PROF_DECL(p_wait);
    PROF_DECL(p_fold);
    PROF_DECL(p_all);
    const long long p_start = PROF_NOW();
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t c = a1 + 32 * b + lane;
      const uint32_t pos = ((uint32_t)c & (R - 1)) + R;
      T acc;
      if (!SMALL) {
        const int slot = (int)(b % kMidSlots);
        const long long t0 = PROF_NOW();
        mbar_wait(&mid_full[slot], (unsigned)((b / kMidSlots) & 1));
        PROF_ADD(p_wait, t0);
        acc = mid_part[slot * 32 + lane];
        const long long t1 = PROF_NOW();
        if (kLA) {
          // mid(b) already holds the offsets >= l+33; nxt the ones in [l+1, l+32]
          acc = SemiOp<OP, T>::apply(acc, nxt);
          if (IsIdem<OP>::value) {
            idem_closure<OP, T>(acc, nxt, im);
          } else {
            nxt = SemiId<OP, T>::value();
            LaSteps<OP, T, 1>::run(acc, nxt, lm);
          }
        } else {
          acc = chain_fold<OP, T, true, ASSOC>(acc, ring, pos, cm);
        }
        PROF_ADD(p_fold, t1);
      } else {
        acc = chain_fold<OP, T, false, ASSOC>(T(0), ring, pos, cm);
      }
      if (c < n) {
        ring[pos - R] = acc;
        ring[pos] = acc;
        if (SMALL) out[c] = (int64_t)acc;
      }
      __syncwarp();
      if (!SMALL && lane == 0) mbar_arrive(&batch_done[b % kBatchBars]);
    }
    PROF_ADD(p_all, p_start);
    PROF_FLUSH(0, p_wait);
    PROF_FLUSH(1, p_fold);
    PROF_FLUSH(2, p_all);
    PROF_FLUSH(3, nb);
  } else if (SMALL || role < 0) {
    // no work: the chain warp keeps SMSP 0 to itself
  } else if (role < M) {
    // ================================== mid =================================
    PROF_DECL(p_wfc);
    PROF_DECL(p_wfar);
    PROF_DECL(p_fold);
    constexpr bool kMidLA = ASSOC && !(OP == kModAdd && sizeof(T) == 8);
    const LaMasks mlm = la_masks(offs, S.k, lane);
    for (int64_t b = role; b < nb; b += M) {
      long long t0 = PROF_NOW();
      wait_batches(batch_done, b - 1);  // offsets >= 64 reach batches <= b-2
      PROF_ADD(p_wfc, t0);
      const int64_t c = a1 + 32 * b + lane;
      const T* base = ring + (((uint32_t)c & (R - 1)) + R);
      T acc = T(0);
      bool have = false;
      if (C.jf > 0) {
        const int fs = (int)(b % kFarSlots);
        t0 = PROF_NOW();
        mbar_wait(&far_full[fs], (unsigned)((b / kFarSlots) & 1));
        PROF_ADD(p_wfar, t0);
        acc = far_part[fs * 32 + lane];
        have = true;
      }
      t0 = PROF_NOW();
      acc = fold_range<OP, T, ASSOC>(acc, have, base, ob, C.jf, C.jn);
      if (kMidLA) {  // the chain warp's look-ahead leaves offsets in [l+33, 63] to mid
        acc = SemiOp<OP, T>::apply(acc, la_ring_group<OP, T>(base, mlm.far));
      }
      const int slot = (int)(b % kMidSlots);
      mid_part[slot * 32 + lane] = acc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&mid_full[slot]);
      PROF_ADD(p_fold, t0);
    }
    PROF_FLUSH(8, p_wfc);
    PROF_FLUSH(9, p_wfar);
    PROF_FLUSH(10, p_fold);
  } else if (role < M + F) {
    // ================================== far =================================
    if (C.jf > 0) {
      // ring slack: the writer may lag the chain; a far read must not reach a
      // ring slot the chain is about to recycle before the writer copied it
      const int64_t slack = ((int64_t)R - S.ring_cover - 64) / 32;
      PROF_DECL(p_ww);
      PROF_DECL(p_wr);
      PROF_DECL(p_fold);
      for (int64_t b = role - M; b < nb; b += F) {
        int64_t need = b + 1 - C.far_look;                       // operands written
        need = max(need, b + 1 - (int64_t)kFarSlots);            // slot consumed
        need = max(need, b + 1 - slack);                         // ring slack
        long long t0 = PROF_NOW();
        wait_batches(written, need);
        PROF_ADD(p_ww, t0);
        const int64_t c = a1 + 32 * b + lane;
        T acc = T(0);
        bool have = false;
        if (REMOTE && C.jr > 0) {
          const int rs = (int)(b % kRemSlots);
          t0 = PROF_NOW();
          spin_eq_gpu(RM.ready + rs, (int)(b + 1), 64);
          PROF_ADD(p_wr, t0);
          acc = ldv_cg<T, int64_t>(reinterpret_cast<const int64_t*>(RM.part) + rs * 32 + lane);
          have = true;
        }
        t0 = PROF_NOW();
        if (GFAR) {
          acc = fold_range<OP, T, ASSOC, int64_t>(acc, have, out + c, obg, C.jr, C.jf);
        } else {
          const T* base = ring + (((uint32_t)c & (R - 1)) + R);
          acc = fold_range<OP, T, ASSOC>(acc, have, base, ob, C.jr, C.jf);
        }
        const int fs = (int)(b % kFarSlots);
        far_part[fs * 32 + lane] = acc;
        __syncwarp();
        if (lane == 0) mbar_arrive(&far_full[fs]);
        PROF_ADD(p_fold, t0);
      }
      PROF_FLUSH(16, p_ww);
      PROF_FLUSH(17, p_wr);
      PROF_FLUSH(18, p_fold);
    }
  } else if (role == M + F) {
    // ================================= writer ===============================
    for (int64_t b = 0; b < nb; ++b) {
      mbar_wait(&batch_done[b % kBatchBars], (unsigned)((b / kBatchBars) & 1));
      const int64_t c = a1 + 32 * b + lane;
      if (c < n) out[c] = (int64_t)ring[(uint32_t)c & (R - 1)];
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&written[b % kBatchBars]);
        // the far warps poll only some phases: observe each phase here, so no
        // phase of the barrier ring is left unobserved (count 1: completes at once)
        mbar_wait(&written[b % kBatchBars], (unsigned)((b / kBatchBars) & 1));
      }
      if (REMOTE && ((b + 1) % kPubEvery == 0 || b + 1 == nb)) {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(reinterpret_cast<long long*>(RM.published), (long long)(b + 1));
      }
    }
  }
}

// A producer warp's fold: 16 independent table loads in flight per chunk
// (two chunks unrolled), so a warp's ~50 L2 reads cost ~2 L2 round trips, not
// one per 4-load group.  Regrouped (associative (x) only).
template <int OP, typename T>
__device__ __forceinline__ T fold_wide(const int64_t* base_elem, const int32_t* __restrict__ ob, int j0, int j1) {
  using O = SemiOp<OP, T>;
  constexpr int W = 16;
  const char* base = reinterpret_cast<const char*>(base_elem);
  T acc = SemiId<OP, T>::value();
  int j = j0;
#pragma unroll 2
  for (; j + W <= j1; j += W) {
    int32_t o[W];
    T v[W];
#pragma unroll
    for (int q = 0; q < W; ++q) o[q] = __ldg(ob + j + q);
#pragma unroll
    for (int q = 0; q < W; ++q) v[q] = at<T, int64_t, true>(base, o[q]);
#pragma unroll
    for (int w = W / 2; w >= 1; w >>= 1)
#pragma unroll
      for (int q = 0; q < w; ++q) v[q] = O::apply(v[q], v[q + w]);
    acc = O::apply(acc, v[0]);
  }
  for (; j < j1; ++j) acc = O::apply(acc, at<T, int64_t, true>(base, __ldg(ob + j)));
  return acc;
}

// The remote operand fold of one batch, split over the CTA's warps in
// contiguous offset ranges and combined in order (requires ASSOC).
template <int OP, typename T>
__device__ __forceinline__ void sdp_producer(const SdpShape& S, const int64_t* __restrict__ offsets,
                                             const int64_t* out, const SdpRemote& RM, int pid, int np) {
  extern __shared__ __align__(16) unsigned char smem[];
  using O = SemiOp<OP, T>;
  // offsets come from the plan's global byte-offset table (RM.obg, read-only,
  // L1-resident): k is unbounded here (the paper's Table I reaches k = 123,928)
  T* red = reinterpret_cast<T*>(smem);  // [warps][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = S.remote_warps;
  const int32_t* obg = RM.obg;
  const int jr = S.j_rem;  // offsets[0, jr) >= a_remote
  if (jr == 0) return;
  const int64_t look = S.rem_look;
  const int per = (jr + W - 1) / W;
  const int lo = min(jr, warp * per), hi = min(jr, lo + per);
  const int64_t nb = (S.n - S.a1 + 31) / 32;
  PROF_DECL(p_wait);
  PROF_DECL(p_fold);
  for (int64_t b = pid; b < nb; b += np) {
    long long t0 = PROF_NOW();
    if (tid == 0) {
      const long long need = (long long)max(b + 1 - look, b + 1 - (int64_t)kRemSlots);
      // every writer's share below `need` (batch y belongs to writer y % writers)
      for (int w = 0; w < S.writers; ++w)
        spin_ge_gpu64(reinterpret_cast<const long long*>(RM.published) + w, need, 128);
    }
    __syncthreads();
    PROF_ADD(p_wait, t0);
    t0 = PROF_NOW();
    const int64_t c = S.a1 + 32 * b + lane;
    if (lo < hi) {
      red[warp * 32 + lane] = fold_wide<OP, T>(out + c, obg, lo, hi);
    }
    __syncthreads();
    if (warp == 0) {
      T acc = red[lane];
      for (int w = 1; w < W; ++w) {
        if (min(jr, w * per) < min(jr, w * per + per)) acc = O::apply(acc, red[w * 32 + lane]);
      }
      const int rs = (int)(b % kRemSlots);
      reinterpret_cast<int64_t*>(RM.part)[rs * 32 + lane] = (int64_t)acc;
      __syncwarp();  // orders the lanes' partial stores before lane 0's (cumulative) release
      if (lane == 0) st_release_gpu_i32(RM.ready + rs, (int)(b + 1));
    }
    PROF_ADD(p_fold, t0);
  }
  if (warp == 0) {
    PROF_FLUSH(24, p_wait);
    PROF_FLUSH(25, p_fold);
  }
}

template <int OP, typename T, bool SMALL, bool ASSOC, bool GFAR>
__global__ void __launch_bounds__(1024, 1)
    sdp_pipeline_cta(const SdpShape S, const int64_t* __restrict__ g_offsets,
                     const int64_t* __restrict__ g_init, int64_t* __restrict__ g_out) {
  const int64_t inst = blockIdx.x;
  sdp_finisher<OP, T, SMALL, ASSOC, GFAR, false>(S, g_offsets + inst * S.k, g_init + inst * S.a1,
                                                 g_out + inst * S.n, SdpRemote{});
}

// Multi-CTA single instance (cooperative launch: all CTAs co-resident).
// Block 0 is the finisher, blocks 1.. are remote producers.
template <int OP, typename T, bool GFAR>
__global__ void __launch_bounds__(1024, 1)
    sdp_pipeline_multi(const SdpShape S, const int64_t* __restrict__ g_offsets,
                       const int64_t* __restrict__ g_init, int64_t* g_out, const SdpRemote RM) {
  if (blockIdx.x == 0) {
    sdp_finisher<OP, T, false, true, GFAR, true>(S, g_offsets, g_init, g_out, RM);
  } else {
    if (threadIdx.x >= 32 * S.remote_warps) return;
    sdp_producer<OP, T>(S, g_offsets, g_out, RM, blockIdx.x - 1, gridDim.x - 1);
  }
}

// -----------------------------------------------------------------------------
// Batched S-DP with a small a_1: one warp per instance runs every stage itself
// -- offsets >= 32 straight from its private mirrored ring, offsets < 32
// through chain_fold.  SMALL: a_1 < 64 (the first operand is assigned inside chain_fold).
template <int OP, typename T, bool SMALL, bool ASSOC>
__global__ void __launch_bounds__(256, 5)
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
                  (size_t)warp * 2 * kpad;
  int32_t* ob = offs + kpad;
  const int64_t gw = (int64_t)blockIdx.x * wpb + warp;
  if (gw >= batch) return;
  // instances grouped by path (dominance-form ones first): a block's warps
  // take the same path and finish together
  const int64_t inst = S.perm ? S.perm[gw] : gw;
  const int64_t a1 = S.a1, n = S.n;
  const int64_t* io = g_offsets + inst * S.k;
  const int64_t* ii = g_init + inst * a1;
  int64_t* o = out + inst * n;
  for (int j = lane; j < S.k; j += 32) {
    offs[j] = (int32_t)io[j];
    ob[j] = offs[j] * (int32_t)sizeof(T);
  }
  for (int64_t i = lane; i < a1; i += 32) {
    const int64_t v = ii[i];
    const uint32_t p = (uint32_t)i & (R - 1);
    ring[p] = (T)v;
    ring[p + R] = (T)v;
    o[i] = v;
  }
  __syncwarp();
  int jn = S.k;  // offsets[0, jn) >= 64 fold from the ring, the rest in chain_fold
  while (jn > 0 && offs[jn - 1] < 64) --jn;
  const ChainMasks cm = chain_masks(offs, S.k, lane);
  constexpr bool kLA = !SMALL && ASSOC && !(OP == kModAdd && sizeof(T) == 8);
  const LaMasks lm = la_masks(offs, S.k, lane);
  const IdemMasks im = idem_masks(offs, S.k, lane);
  // Dominance form (as in the single-instance chain, sdp_v2.cuh): min/max
  // with offset 1 and a_1 <= 128 -- every finished batch is the prefix-(x) of
  // its b vector, so the offsets [l+33, 128) a batch takes from the three
  // batches before it fold to x at one lane each (three shuffles); only
  // offsets >= 128 (a_1 itself) are read from the ring.  From batch 4 on;
  // the first batches take the general path.
  // Second form (dom2): no offset 1 but every d in [2, 127] a sum of offsets
  // (S* >= [2, 127]): then x_l = b_l (x) B(l-2) with B the batch's prefix-(x)
  // of b, the next batch's in-batch terms are B(30) / B(31), and a 32-wide
  // offset range folds to x at its largest position p1 and, when its offset
  // + 1 is an offset too, at p1 - 1 (ST[p] >= ST[p1] for p <= p1 - 2).
  int mode = 0;  // 1: offset 1 (dominance form), 2: dom2, 0: general path
  bool n2 = false, n3 = false, n4 = false;
  if (kLA && IsIdem<OP>::value && a1 <= 128 && S.k >= 2) {
    if (im.scan) {
      mode = 1;
    } else {
      unsigned long long s0 = 0, s1 = 0;  // offsets < 128 as a bit set
      for (int j = lane; j < S.k; j += 32) {
        const int d = offs[j];
        if (d < 64) s0 |= 1ull << d;
        else if (d < 128) s1 |= 1ull << (d - 64);
      }
#pragma unroll
      for (int sh = 16; sh >= 1; sh >>= 1) {
        s0 |= __shfl_xor_sync(0xffffffffu, s0, sh);
        s1 |= __shfl_xor_sync(0xffffffffu, s1, sh);
      }
      unsigned long long r0 = 1ull, r1 = 0;  // S* (with 0) over [0, 127]
      for (int v = 1; v < 128; ++v) {
        bool hit = false;
        for (int j = lane; j < S.k; j += 32) {
          const int u = v - offs[j];
          if (u >= 0) hit = hit || ((u < 64 ? r0 >> u : r1 >> (u - 64)) & 1ull);
        }
        if (__any_sync(0xffffffffu, hit)) {
          if (v < 64) r0 |= 1ull << v;
          else r1 |= 1ull << (v - 64);
        }
      }
      if ((r0 | 3ull) == ~0ull && r1 == ~0ull) mode = 2;
      auto in_s = [&](int d) { return d < 64 ? ((s0 >> d) & 1ull) != 0 : d < 128 && ((s1 >> (d - 64)) & 1ull) != 0; };
      if (mode == 2) {  // per range: is (smallest offset in it) + 1 an offset in it too
        bool seen2 = false, seen3 = false, seen4 = false;
        for (int j = S.k - 1; j >= 0; --j) {  // ascending d
          const int d = offs[j];
          if (d >= 128) break;
          if (!seen2 && d >= lane + 33 && d <= lane + 64) {
            seen2 = true;
            n2 = d + 1 <= min(lane + 64, 127) && in_s(d + 1);
          }
          if (!seen3 && d >= lane + 65 && d <= lane + 96) {
            seen3 = true;
            n3 = d + 1 <= min(lane + 96, 127) && in_s(d + 1);
          }
          if (!seen4 && d >= lane + 97 && d <= lane + 128) {
            seen4 = true;
            n4 = d + 1 <= 127 && in_s(d + 1);
          }
        }
      }
    }
  }
  const bool dom = mode != 0;
  int src2 = -1, src3 = -1, src4 = -1, j128 = 0;
  if (dom) {
    for (int j = S.k - 1; j >= 0; --j) {  // ascending d
      const int d = offs[j];
      if (d >= 128) break;
      if (src2 < 0 && d >= lane + 33 && d <= lane + 64) src2 = lane + 64 - d;
      if (src3 < 0 && d >= lane + 65 && d <= lane + 96) src3 = lane + 96 - d;
      if (src4 < 0 && d >= lane + 97 && d <= lane + 128) src4 = lane + 128 - d;
    }
    while (j128 < S.k && offs[j128] >= 128) ++j128;
  }
  const T idv = SemiId<OP, T>::value();
  T xm1 = idv, xm2 = idv, xm3 = idv, pre_cur = idv;
  T nxt = T(0);
  const int64_t nb = (n - a1 + 31) / 32;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t c = a1 + 32 * b + lane;
    const uint32_t pos = ((uint32_t)c & (R - 1)) + R;
    T acc;
    if (dom && b >= 4) {
      // offsets >= 128 from the ring, [l+33, 128) as pre_cur, [l+1, l+32] as nxt
      acc = SemiOp<OP, T>::apply(fold_range<OP, T, ASSOC>(pre_cur, true, ring + pos, ob, 0, j128), nxt);
      if (mode == 1) {
        idem_closure<OP, T>(acc, nxt, im);
      } else {  // dom2: x_l = b_l (x) B(l-2); next batch's in-batch terms B(30) / B(31)
        T B = acc;
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
          const T o = shfl_up(B, sh);
          if (lane >= sh) B = SemiOp<OP, T>::apply(B, o);
        }
        const T b2 = shfl_up(B, 2);
        const T n30 = shfl_idx(B, 30), n31 = shfl_idx(B, 31);
        if (lane >= 2) acc = SemiOp<OP, T>::apply(acc, b2);
        nxt = lane == 0 ? n30 : n31;
      }
    } else if (kLA) {
      acc = fold_range<OP, T, ASSOC>(T(0), false, ring + pos, ob, 0, jn);
      if (b == 0) {
        bool h = true;
        pre_steps<OP, T, true, ASSOC>(acc, h, ring + pos, cm.hi, cm.lo);
      } else {
        acc = SemiOp<OP, T>::apply(acc, nxt);
      }
      const T nr = la_ring_group<OP, T>(ring + (((uint32_t)(c + 32) & (R - 1)) + R), lm.far);
      if (IsIdem<OP>::value) {
        idem_closure<OP, T>(acc, nxt, im);
        nxt = SemiOp<OP, T>::apply(nxt, nr);
      } else {
        nxt = nr;
        LaSteps<OP, T, 1>::run(acc, nxt, lm);
      }
    } else if (!SMALL) {
      acc = fold_range<OP, T, ASSOC>(T(0), false, ring + pos, ob, 0, jn);
      acc = chain_fold<OP, T, true, ASSOC>(acc, ring, pos, cm);
    } else {
      acc = chain_fold<OP, T, false, ASSOC>(T(0), ring, pos, cm);
    }
    if (dom) {  // batch b+1's [l+33, 128) terms from x of batches b-1, b-2, b-3
      if (b >= 3) {
        const T v2 = shfl_idx(xm1, src2 < 0 ? 0 : src2);
        const T v3 = shfl_idx(xm2, src3 < 0 ? 0 : src3);
        const T v4 = shfl_idx(xm3, src4 < 0 ? 0 : src4);
        pre_cur = SemiOp<OP, T>::apply(SemiOp<OP, T>::apply(src2 < 0 ? idv : v2, src3 < 0 ? idv : v3),
                                       src4 < 0 ? idv : v4);
        if (mode == 2) {  // the positions p1 - 1 (offset + 1 in the same range)
          const T w2 = shfl_idx(xm1, src2 > 0 ? src2 - 1 : 0);
          const T w3 = shfl_idx(xm2, src3 > 0 ? src3 - 1 : 0);
          const T w4 = shfl_idx(xm3, src4 > 0 ? src4 - 1 : 0);
          pre_cur = SemiOp<OP, T>::apply(pre_cur, SemiOp<OP, T>::apply(SemiOp<OP, T>::apply(n2 ? w2 : idv, n3 ? w3 : idv),
                                                                       n4 ? w4 : idv));
        }
      }
      xm3 = xm2;
      xm2 = xm1;
      xm1 = acc;
    }
    __syncwarp();  // every lane's ring reads of this batch before any lane's writes
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
  const uint32_t bits = chain_bits(0xFFFFFFFEu, lane);
  __syncwarp();
  const long long t0 = clock64();
  for (int64_t b = 0; b < batches; ++b) {
#pragma unroll
    for (int t = 1; t < 32; ++t) {
      const T v = shfl_idx(acc, t - 1);
      if ((int32_t)(bits << (t - 1)) < 0) acc = O::apply(acc, v);
    }
    acc = shfl_idx(acc, 31);
  }
  const long long t1 = clock64();
  if (lane == 0) *cycles = t1 - t0;
  sink[lane] = acc;
}

// Hardware floor of the dependency chain: one thread, a loop-carried chain of
// dependent (x) (the empty asm pins x to a register after every op so the
// compiler cannot reassociate the chain).  Whatever the schedule, cell i of
// an instance with a_k = 1 needs at least one (x) that consumes cell i-1, so
// (n - a_1) x this latency bounds every S-DP kernel from below.
template <typename T>
__device__ __forceinline__ void opaque(T& x);
template <>
__device__ __forceinline__ void opaque<int32_t>(int32_t& x) { asm volatile("" : "+r"(x)); }
template <>
__device__ __forceinline__ void opaque<int64_t>(int64_t& x) { asm volatile("" : "+l"(x)); }

template <int OP, typename T>
__global__ void op_latency_probe(int64_t iters, const T* vals, long long* cycles, T* sink) {
  using O = SemiOp<OP, T>;
  T v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = vals[j];
  T x = vals[8];
  const long long t0 = clock64();
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x = O::apply(x, v[j]);
      opaque(x);
    }
  }
  const long long t1 = clock64();
  *cycles = t1 - t0;
  *sink = x;
}

// Isolated chain_fold timing with a real instance's masks (mode 0: full fold,
// 1: shuffle chain only, 2: out-of-batch pre-steps only).  Cycles per batch.
template <int OP, typename T>
__global__ void sdp_chain_fold_probe(int64_t batches, uint32_t hi, uint32_t m32, int mode,
                                     long long* cycles, T* sink) {
  __shared__ T ring[256];
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < 256; i += 32) ring[i] = (T)(i * 7 + 3);
  __syncwarp();
  ChainMasks m{hi, m32 & ~((2u << lane) - 1u), chain_bits(m32, lane)};
  if (mode == 1) m.hi = m.lo = 0;
  if (mode == 2) m.bits = 0;
  T acc = (T)lane;
  const long long t0 = clock64();
  for (int64_t b = 0; b < batches; ++b) {
    acc = chain_fold<OP, T, true, true>(acc, ring, 128 + lane, m);
    ring[128 + lane] = acc;
    __syncwarp();
  }
  const long long t1 = clock64();
  if (lane == 0) *cycles = (t1 - t0) / batches;
  sink[lane] = acc;
}

}  // namespace pipedp_dev

namespace pipedp_dev {

// -----------------------------------------------------------------------------
// Serial chain for tiny offset sets (k <= 8, a_1 < 64; BASELINE config 1 is
// the Fibonacci recurrence, offsets {2, 1}): when a cell has only a handful of
// operands, the warp-wide pipeline's shuffle hand-off costs more than doing
// the recurrence in one thread.  One thread walks the cells in order with the
// reference's exact fold order (sdp.cpp:52-59: assign ST[i-a_1], then fold
// a_2..a_k), keeping the previous cell in a register (offset 1 is the only
// operand that is not already in shared memory when the cell starts) and the
// last 64 cells in a shared ring; lanes 1..31 stream the finished cells to HBM
// in coalesced 32-cell rows.
template <int OP, typename T>
__global__ void __launch_bounds__(32)
    sdp_serial_thread(const int64_t n, const int32_t k, const int64_t* __restrict__ g_offsets,
                      const int64_t* __restrict__ g_init, int64_t* __restrict__ out) {
  using O = SemiOp<OP, T>;
  __shared__ T ring[64];
  __shared__ T row[2][32];
  __shared__ int32_t offs[8];
  const int lane = threadIdx.x;
  if (lane < k) offs[lane] = (int32_t)g_offsets[lane];
  __syncwarp();
  const int a1 = offs[0];
  for (int i = lane; i < a1; i += 32) {
    ring[i & 63] = (T)g_init[i];
    out[i] = g_init[i];
  }
  __syncwarp();
  const bool last_is_1 = offs[k - 1] == 1;
  const int kk = last_is_1 ? k - 1 : k;  // operands read from the ring
  T prev = ring[(a1 - 1) & 63];
  for (int64_t c0 = a1; c0 < n; c0 += 32) {
    const int64_t cend = c0 + 32 < n ? c0 + 32 : n;
    const int rb = (int)((c0 / 32) & 1);
    if (lane == 0) {
      for (int64_t c = c0; c < cend; ++c) {
        T acc = ring[(c - offs[0]) & 63];
        for (int j = 1; j < kk; ++j) acc = O::apply(acc, ring[(c - offs[j]) & 63]);
        if (last_is_1) acc = kk > 0 ? O::apply(acc, prev) : prev;
        ring[c & 63] = acc;
        row[rb][c - c0] = acc;
        prev = acc;
      }
    }
    __syncwarp();
    if (c0 + lane < cend) out[c0 + lane] = (int64_t)row[rb][lane];
  }
}

}  // namespace pipedp_dev

namespace pipedp_dev {

// -----------------------------------------------------------------------------
// The paper's two comparison methods for S-DP, on the GPU,
// behind solve_prefix_parallel / solve_naive_parallel (sdp.cpp:91-111, which
// the reference only models as step counts).  Both walk the cells one at a
// time with the whole CTA on the k operands of the cell; the table lives in
// HBM (operands through L2, ld.global.cg; the finished cell is released with a
// CTA barrier + fence before the next cell reads it).  Associative (x) only --
// the host keeps the strict pipeline for mixed-sign saturating-add.
//
// prefix (tournament): thread t folds a contiguous slice of offsets in j order,
// then a ceil(log2)-level tree combines the slices in order: the levels inside
// a warp are shuffles (no barrier), the levels across the CTA's warps one
// shared-memory exchange and a last warp of shuffles -- two barriers per cell
// instead of one per level: O(n log k) steps, as the method is meant to run.
// RT (int64_t / int32_t for a 32-bit value class; void: none): the last
// R >= a_1 + 1 cells also live in shared memory (when they fit), so a cell's
// operands are shared-memory loads instead of L2 round trips.
template <int OP, typename RT, int NR = 32>  // NR: register-resident slice size (ring path)
__global__ void __launch_bounds__(1024, 1)
    sdp_tournament(int64_t n, int32_t k, const int64_t* __restrict__ g_offsets,
                   const int64_t* __restrict__ g_init, int64_t* out, int32_t R) {
  using O = SemiOp<OP, int64_t>;
  const int64_t id = SemiId<OP, int64_t>::value();
  constexpr bool RING = !std::is_same<RT, void>::value;
  using W = typename std::conditional<RING, RT, int64_t>::type;
  extern __shared__ __align__(16) unsigned char ring_raw[];
  W* ring = reinterpret_cast<W*>(ring_raw);  // [R] (RING)
  __shared__ int64_t red[32];
  const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, warp = t >> 5, nw = nt >> 5;
  const int64_t a1 = g_offsets[0];
  for (int64_t i = t; i < a1; i += nt) {
    out[i] = g_init[i];
    if (RING) ring[i % R] = (W)g_init[i];
  }
  __threadfence();
  __syncthreads();
  const int per = (k + nt - 1) / nt;
  const int lo = min(k, t * per), hi = min(k, lo + per);
  int32_t pos = (int32_t)(a1 % R);  // i mod R
  // a slice of <= 32 offsets stays in registers (ring path): every cell's
  // loads then issue back to back
  constexpr int kRegOffs = NR;
  int32_t roff[kRegOffs];
#pragma unroll
  for (int u = 0; u < kRegOffs; ++u) roff[u] = lo + u < hi ? (int32_t)g_offsets[lo + u] : 0;
  for (int64_t i = a1; i < n; ++i) {
    int64_t acc = id;
    if (RING && hi - lo <= kRegOffs) {
#pragma unroll
      for (int u = 0; u < kRegOffs; ++u) {
        if (lo + u < hi) {
          int32_t q = pos - roff[u];
          q += q < 0 ? R : 0;
          acc = O::apply(acc, (int64_t)ring[q]);
        }
      }
    } else if (RING) {
      for (int j = lo; j < hi; ++j) {
        int32_t q = pos - (int32_t)__ldg(g_offsets + j);
        q += q < 0 ? R : 0;
        acc = O::apply(acc, (int64_t)ring[q]);
      }
    } else {
      // the slice's L2 round trips in flight together: its offsets are
      // loop-invariant (registers, loaded once), sixteen operand loads per trip
      int j = lo;
      for (; j < hi; j += 16) {
        int64_t v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          v[u] = j + u < hi ? (int64_t)__ldcg(reinterpret_cast<const long long*>(out + i - __ldg(g_offsets + j + u)))
                            : id;
#pragma unroll
        for (int u = 0; u < 16; ++u) acc = O::apply(acc, v[u]);
      }
    }
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {  // tournament levels inside the warp: left (x) right
      const int64_t r = (int64_t)__shfl_down_sync(0xffffffffu, (long long)acc, s);
      if ((lane & (2 * s - 1)) == 0) acc = O::apply(acc, r);
    }
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (warp == 0) {  // the levels across warps
      acc = lane < nw ? red[lane] : id;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int64_t r = (int64_t)__shfl_down_sync(0xffffffffu, (long long)acc, s);
        if ((lane & (2 * s - 1)) == 0) acc = O::apply(acc, r);
      }
      if (lane == 0) {
        out[i] = acc;
        if (RING) ring[pos] = (W)acc;
        else __threadfence();
      }
    }
    __syncthreads();
    pos = pos + 1 == R ? 0 : pos + 1;
  }
}

// naive: the first operand is assigned, then k-1 threads fold their operand
// into the one shared accumulator with atomics -- the memory-access conflict
// the paper describes ("using k-1 threads", serialised on ST[i]): O(nk).
__device__ __forceinline__ long long naive_atomic_min(long long* a, long long v) { return atomicMin(a, v); }
__device__ __forceinline__ long long naive_atomic_max(long long* a, long long v) { return atomicMax(a, v); }

template <int OP>
__device__ __forceinline__ void naive_fold(int64_t* acc, int64_t v) {
  if (OP == kMin) {
    atomicMin(reinterpret_cast<long long*>(acc), (long long)v);
  } else if (OP == kMax) {
    atomicMax(reinterpret_cast<long long*>(acc), (long long)v);
  } else {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(acc);
    unsigned long long old = *a, assumed;
    do {
      assumed = old;
      const int64_t nv = SemiOp<OP, int64_t>::apply((int64_t)assumed, v);
      old = atomicCAS(a, assumed, (unsigned long long)nv);
    } while (old != assumed);
  }
}

template <int OP>
__global__ void __launch_bounds__(1024, 1)
    sdp_naive(int64_t n, int32_t k, const int64_t* __restrict__ g_offsets, const int64_t* __restrict__ g_init,
              int64_t* out) {
  __shared__ int64_t acc;
  const int t = threadIdx.x, nt = blockDim.x;
  const int64_t a1 = g_offsets[0];
  for (int64_t i = t; i < a1; i += nt) out[i] = g_init[i];
  __threadfence();
  __syncthreads();
  for (int64_t i = a1; i < n; ++i) {
    if (t == 0) acc = __ldcg(reinterpret_cast<const long long*>(out + i - a1));
    __syncthreads();
    for (int j = 1 + t; j < k; j += nt)
      naive_fold<OP>(&acc, __ldcg(reinterpret_cast<const long long*>(out + i - __ldg(g_offsets + j))));
    __syncthreads();
    if (t == 0) {
      out[i] = acc;
      __threadfence();
    }
    __syncthreads();
  }
}

}  // namespace pipedp_dev

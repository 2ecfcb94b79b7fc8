// sdp_v2.cuh -- single-instance S-DP pipeline, offset-partitioned stages
// (sm_100a).  Used for associative (x) with an identity (min, max, 32-bit
// modular-add, saturating-add without mixed signs); sdp_kernels.cuh keeps the
// strict-order and HBM-ring variants.
//
// Reference semantics: sdp.cpp:48-60 (fill_table), sdp_pipeline.hpp:24-46.
// Regrouping only (never a different set of operands): every cell folds the
// same k operands as the reference; ASSOC lets the fold be split into partial
// folds that are combined later.
//
// Finisher CTA (one per instance), cells in batches of 32 (one per lane):
//   warp 0            chain: folds mid(b) (x) nxt and resolves the in-batch
//                     dependency (idempotent closure for min/max, the 32-step
//                     shuffle hand-off otherwise); owns SM sub-partition 0
//   chain warp also   folds offsets d in [l+33, a_chain) of batch b+1 while
//                     resolving batch b (they only read batches <= b-1)
//   near warps j      each owns a contiguous range of offsets in [a_chain, a_rem),
//                     held in REGISTERS as ring byte offsets; every near warp
//                     folds its range for EVERY batch as soon as the batches
//                     it reads are final (lookahead = its smallest offset / 32)
//   combiner warps    batch b -> warp b % NC: near partials (x) remote partial
//                     -> mid(b) for the chain
//   writer warp       streams finished batches to HBM (coalesced int64) and,
//                     with remote producers, publishes the finished prefix
// Remote producer CTAs (sdp_producer, multi-CTA cooperative launch) fold the
// offsets >= a_rem from the HBM table (long lookahead, gpu-scope flags).
#pragma once

#include "sdp_kernels.cuh"

namespace pipedp_dev {

constexpr int kNearMax = 32;   // offsets per near warp (registers)
constexpr int kNearSlots = 16; // near -> combiner partial slots
constexpr int kNearWarps = 20; // max near warps
constexpr int kFetchSlots = 16; // fetcher -> combiner remote partial slots
constexpr int kMaxWarpsV2 = 24; // 768 threads: the chain warp's register budget
constexpr int kPreMax = 32;     // chain-folded offsets per lane in [l+33, 63] (<= 31)
constexpr int kDomMax = 8;      // dominance form registers (power of two); a_chain <= 256 uses 7
constexpr int kPreUMax = 32;    // chain-folded lane-independent offsets in [64, a_chain)

struct SdpV2Shape {
  int64_t n;
  int32_t k;
  int32_t a1;
  int32_t ring_log2;
  int32_t a_rem;       // offsets >= a_rem come from remote producers (1 << 30: none)
  int32_t a_chain;     // offsets in [l+33, a_chain) are folded by the chain warp itself
  int32_t pub_every;   // writer publishes the finished prefix every pub_every batches
  int32_t fetchers;    // fetcher warps (remote mode): batch b -> fetcher b % fetchers
  int32_t j_rem;       // offsets[0, j_rem) >= a_rem (remote); only [j_rem, k) are staged in smem
  int32_t writers;     // writer warps: batch b -> writer b % writers (each publishes its share)
  int32_t near_warps;  // NW
  int32_t comb_warps;  // NC
  int32_t near_group;  // NG warps per offset range (batch b -> warp b % NG)
  int32_t near_lo[kNearWarps + 1];  // near warp j owns offset indices [near_lo[j], near_lo[j+1])
  int32_t dom;                        // dominance form (min/max with offset 1), a_chain = 32 (M + 1), M <= kDomMax
  int32_t n_pre_u;                    // chain-folded offsets in [64, a_chain), lane-independent:
  int32_t pre_u[kPreUMax];            //   as negative ring byte offsets (uniform-register operands)
};

__host__ __device__ __forceinline__ int sdp2_warps(int NW, int NG, int NC, int NF, int NWR) {
  // chain + NC + NW*NG + NWR writers + NF fetchers, skipping
  // warp ids = 0 mod 4 (SMSP 0 is the chain's)
  return sdp_warps_for_roles(NC + NW * NG + NWR + NF);
}

template <int OP, typename T, bool REMOTE>
__device__ __forceinline__ void sdp_v2_finisher(const SdpV2Shape& S, const int64_t* __restrict__ offsets,
                                                const int64_t* __restrict__ init, int64_t* out,
                                                const SdpRemote& RM) {
  using O = SemiOp<OP, T>;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t R = 1u << S.ring_log2;
  const int kpad = (S.k - S.j_rem + 3) & ~3;
  const int NW = S.near_warps, NC = S.comb_warps, NG = S.near_group;
  T* ring = reinterpret_cast<T*>(smem);                       // 2R, mirrored
  // raw a_j for j >= j_rem only (the offsets below a_rem); offs[j] stays
  // valid for those j (the pointer is shifted; lower j are never read here)
  const int klocal = S.k - S.j_rem;
  int32_t* offs_s = reinterpret_cast<int32_t*>(ring + 2 * R);
  int32_t* offs = offs_s - S.j_rem;
  T* mid_part = reinterpret_cast<T*>(offs_s + kpad);          // [kMidSlots][32]
  T* near_part = mid_part + kMidSlots * 32;                   // [kNearSlots][NW][32]
  T* rem_part = near_part + (size_t)kNearSlots * NW * 32;                  // [kFetchSlots][32]
  int32_t* pre_scratch = reinterpret_cast<int32_t*>(rem_part + kFetchSlots * 32);  // [kPreMax][32]
  int* written_count = reinterpret_cast<int*>(pre_scratch + (size_t)kPreMax * 32);  // [4] (16 B)
  uint64_t* bars = reinterpret_cast<uint64_t*>(written_count + 4);
  uint64_t* batch_done = bars;                   // [kBatchBars] chain -> all
  uint64_t* written = batch_done + kBatchBars;  // [kBatchBars] writer -> chain
  uint64_t* mid_full = written + kBatchBars;    // [kMidSlots] combiner -> chain
  uint64_t* near_full = mid_full + kMidSlots;   // [kNearSlots] near warps -> combiner (count NW)
  uint64_t* rem_full = near_full + kNearSlots;  // [kFetchSlots] fetcher -> combiner

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t a1 = S.a1, n = S.n;
  for (int j = tid; j < klocal; j += blockDim.x) offs_s[j] = (int32_t)offsets[S.j_rem + j];
  const int64_t ring_from = a1 > (int64_t)R ? a1 - (int64_t)R : 0;
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
    for (int w = 0; w < 4; ++w) written_count[w] = 0;
    for (int s = 0; s < 2 * kBatchBars + kMidSlots; ++s) mbar_init(&bars[s], 1);
    for (int s = 0; s < kNearSlots; ++s) mbar_init(&near_full[s], (unsigned)(NW > 0 ? NW : 1));
    for (int s = 0; s < kFetchSlots; ++s) mbar_init(&rem_full[s], 1);
  }
  __syncthreads();
  const int64_t nb = (n - a1 + 31) / 32;
  const int role = sdp_role_of_warp(warp);  // chain, idle SMSP-0 warps: -1
  const T id = SemiId<OP, T>::value();

  if (warp == 0) {
    // ================================= chain ================================
    const LaMasks lm = la_masks(offs, S.k, lane);
    const IdemMasks im = idem_masks(offs, S.k, lane);
    // nxt for batch 0: offsets d in [l+1, l+32] over the preset cells
    T nxt = id;
    {
      const uint32_t pos0 = ((uint32_t)(a1 + lane) & (R - 1)) + R;
      for (int d = lane + 32; d >= lane + 1; --d)
        if ((lm.nbits >> (d - lane - 1)) & 1u) nxt = O::apply(nxt, ring[pos0 - d]);
    }
    // offsets d in [l+33, a_chain): folded here, one batch ahead, interleaved
    // with the closure (they read batches <= b-1 only) -- no hand-off latency
    // on the dependency distance these offsets leave
    // per-lane byte-offset list in shared memory ([i][lane]: conflict-free)
    int32_t* pre = pre_scratch;
    int npre = 0;
    for (int j = S.k - 1; j >= 0; --j) {
      const int d = offs[j];
      if (d >= 64) break;
      if (d >= lane + 33 && npre < kPreMax) pre[(npre++) * 32 + lane] = d * (int32_t)sizeof(T);
    }
    for (int i = npre; i < kPreMax; ++i) pre[i * 32 + lane] = 0;  // own slot; masked below
    __syncwarp();
    int mpre = npre;
#pragma unroll
    for (int sh = 16; sh >= 1; sh >>= 1) mpre = max(mpre, __shfl_xor_sync(0xffffffffu, mpre, sh));
    // the pre-fold is split in a load phase (issued before the closure, so its
    // shared-memory latency overlaps the closure's shuffles) and a tree phase
    // the pre-fold runs 8 offsets per step (all loads issued before any use,
    // branch-free: the padded list entries point at the lane's own slot and are
    // masked to the identity), split in a load phase issued before the closure
    // (its latency overlaps the closure's shuffles) and a combine phase after it
    auto pre_load = [&](const char* base, T* v) {  // v[8]: partial folds
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = id;
      // lane-independent offsets: immediate-free uniform operands, one load each
#pragma unroll
      for (int i0 = 0; i0 < kPreUMax; i0 += 8) {
        if (i0 < S.n_pre_u) {
          T x[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = *reinterpret_cast<const T*>(base + S.pre_u[i0 + j]);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = O::apply(v[j], i0 + j < S.n_pre_u ? x[j] : id);
        }
      }
      // lane-dependent offsets [l+33, 63]
      for (int i0 = 0; i0 < mpre; i0 += 8) {  // warp-uniform trip count <= 4
        int32_t o[8];
        T x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = pre[(i0 + j) * 32 + lane];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = *reinterpret_cast<const T*>(base - o[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = O::apply(v[j], i0 + j < npre ? x[j] : id);
      }
    };
    auto pre_tree = [&](T* v) {
#pragma unroll
      for (int w = 4; w >= 1; w >>= 1) {
#pragma unroll
        for (int i = 0; i < w; ++i) v[i] = O::apply(v[i], v[i + w]);
      }
      return v[0];
    };
    auto pre_fold = [&](const char* base) {
      T v[8];
      pre_load(base, v);
      return pre_tree(v);
    };
    // Dominance form (idempotent (x) with offset 1, S.dom): x of a finished
    // batch is the prefix-(x) of its b vector (see idem_closure), so the terms
    // a later batch takes from it, offsets d in a 32-wide range, fold to x at
    // the single position of the smallest such d.  src[K-2]: that position for
    // the range landing K batches back (d in [l+32(K-1)+1, min(l+32K,
    // a_chain-1)]), -1 when the range holds no offset; K = 2 .. M+1.
    const bool dom = IsIdem<OP>::value && im.scan && S.dom;
    const int M = dom ? S.a_chain / 32 - 1 : 0;  // 3 .. 7
    int src[kDomMax];
#pragma unroll
    for (int q = 0; q < kDomMax; ++q) src[q] = -1;
    if (dom) {
      for (int j = S.k - 1; j >= 0; --j) {  // ascending d
        const int d = offs[j];
        if (d >= S.a_chain) break;
#pragma unroll
        for (int q = 0; q < kDomMax; ++q)
          if (src[q] < 0 && d >= lane + 32 * (q + 1) + 1 && d <= lane + 32 * (q + 2)) src[q] = lane + 32 * (q + 2) - d;
      }
    }
    // the dominance form's first M batches (and batch 0's pre-fold): offsets
    // [l+33, a_chain) of the cell at `cn` straight from the ring
    auto pre_ring = [&](int64_t cn) {
      T v = id;
      for (int j = S.k - 1; j >= 0; --j) {
        const int d = offs[j];
        if (d >= S.a_chain) break;
        if (d >= lane + 33) v = O::apply(v, ring[((uint32_t)(cn - d) & (R - 1)) + R]);
      }
      return v;
    };
    T pre_cur = dom ? pre_ring(a1 + lane)
                    : pre_fold(reinterpret_cast<const char*>(ring + (((uint32_t)(a1 + lane) & (R - 1)) + R)));
    T xm[kDomMax];  // x of batches b-1, b-2, ... (before iteration b's shift)
#pragma unroll
    for (int q = 0; q < kDomMax; ++q) xm[q] = id;
    PROF_DECL(p_wait);
    PROF_DECL(p_fold);
    const long long p_start = PROF_NOW();
    for (int64_t b = 0; b < nb; ++b) {
      if ((b & 15) == 0 && b >= 32) {
        // writer lag <= 48 batches: the ring slots about to be overwritten
        // (R/32 >= 64 batches back) are in HBM, and the writer never trails the
        // 64-entry barrier rings by a full cycle
        // per-writer progress counters (writer w owns batches w, w + NWR, ...):
        // polled here only every 16 batches, so a counter instead of an
        // mbarrier phase per batch that nobody would wait on
        const int64_t X = b - 32;
        for (int w = 0; w < S.writers; ++w) {
          const int need = X > w ? (int)((X - w + S.writers - 1) / S.writers) : 0;
          while (ld_acquire_cta(written_count + w) < need) __nanosleep(32);
        }
      }
      const int64_t c = a1 + 32 * b + lane;
      const uint32_t pos = ((uint32_t)c & (R - 1)) + R;
      const int slot = (int)(b % kMidSlots);
      long long t0 = PROF_NOW();
      mbar_wait(&mid_full[slot], (unsigned)((b / kMidSlots) & 1));
      PROF_ADD(p_wait, t0);
      t0 = PROF_NOW();
      T acc = O::apply(O::apply(mid_part[slot * 32 + lane], pre_cur), nxt);
      if (dom && b >= M) {
        // batch b+1's chain-local offsets from x of batches b-1 .. b-M by the
        // closure's prefix structure: one shuffle per batch range
        idem_closure<OP, T>(acc, nxt, im);
        T pv[kDomMax];
#pragma unroll
        for (int q = 0; q < kDomMax; ++q) {
          const T v = shfl_idx(xm[q], src[q] < 0 ? 0 : src[q]);
          pv[q] = q < M && src[q] >= 0 ? v : id;
        }
#pragma unroll
        for (int w = kDomMax / 2; w >= 1; w >>= 1)
#pragma unroll
          for (int q = 0; q < w; ++q) pv[q] = O::apply(pv[q], pv[q + w]);
        pre_cur = pv[0];
      } else if (dom) {
        idem_closure<OP, T>(acc, nxt, im);
        pre_cur = pre_ring(c + 32);  // reads batches <= b - 1 only
      } else {
        // batch b+1's chain-local offsets: independent of this batch's closure
        T pv[8];
        pre_load(reinterpret_cast<const char*>(ring + (((uint32_t)(c + 32) & (R - 1)) + R)), pv);
        if (IsIdem<OP>::value) {
          idem_closure<OP, T>(acc, nxt, im);
        } else {
          nxt = id;
          LaSteps<OP, T, 1>::run(acc, nxt, lm);
        }
        pre_cur = pre_tree(pv);
      }
#pragma unroll
      for (int q = kDomMax - 1; q >= 1; --q) xm[q] = xm[q - 1];
      xm[0] = acc;
      if (c < n) {
        ring[pos - R] = acc;
        ring[pos] = acc;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&batch_done[b % kBatchBars]);
      PROF_ADD(p_fold, t0);
    }
    PROF_DECL(p_all);
    PROF_ADD(p_all, p_start);
    PROF_FLUSH(0, p_wait);
    PROF_FLUSH(1, p_fold);
    PROF_FLUSH(2, p_all);
    PROF_FLUSH(3, nb);
  } else if (role < 0) {
    // idle: SMSP 0 belongs to the chain warp
  } else if (role < NC) {
    // =============================== combiner ===============================
    PROF_DECL(p_w1);
    PROF_DECL(p_w2);
    PROF_DECL(p_w3);
    PROF_DECL(p_work);
    for (int64_t b = role; b < nb; b += NC) {
      long long t0 = PROF_NOW();
      // mid slot b % kMidSlots was last used by batch b - kMidSlots: the chain
      // must have consumed it (this also keeps every waiter within half a
      // barrier ring of the chain)
      wait_batches(batch_done, b + 1 - kMidSlots / 2);
      PROF_ADD(p_w1, t0);
      t0 = PROF_NOW();
      T acc = id;
      if (NW > 0) {
        const int ns = (int)(b % kNearSlots);
        PROF_ADD(p_work, t0);
        t0 = PROF_NOW();
        mbar_wait(&near_full[ns], (unsigned)((b / kNearSlots) & 1));
        PROF_ADD(p_w2, t0);
        t0 = PROF_NOW();
        for (int j = 0; j < NW; ++j) acc = O::apply(acc, near_part[((size_t)ns * NW + j) * 32 + lane]);
      }
      if (REMOTE) {  // staged into shared memory by the fetcher warp
        const int fs = (int)(b % kFetchSlots);
        PROF_ADD(p_work, t0);
        t0 = PROF_NOW();
        mbar_wait(&rem_full[fs], (unsigned)((b / kFetchSlots) & 1));
        PROF_ADD(p_w3, t0);
        t0 = PROF_NOW();
        acc = O::apply(acc, rem_part[fs * 32 + lane]);
      }
      const int slot = (int)(b % kMidSlots);
      mid_part[slot * 32 + lane] = acc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&mid_full[slot]);
      PROF_ADD(p_work, t0);
    }
    PROF_FLUSH(8, p_w1);
    PROF_FLUSH(9, p_w2);
    PROF_FLUSH(10, p_w3);
    PROF_FLUSH(11, p_work);
  } else if (role < NC + NW * NG) {
    // ================================= near =================================
    const int j = (role - NC) / NG, g = (role - NC) % NG;
    const int j0 = S.near_lo[j], j1 = S.near_lo[j + 1];
    const int cnt = j1 - j0;  // <= kNearMax, warp-uniform
    int32_t ob[kNearMax];  // padded with a valid offset; padded slots fold the identity
#pragma unroll
    for (int i = 0; i < kNearMax; ++i) ob[i] = offs[j0 + (i < cnt ? i : 0)] * (int32_t)sizeof(T);
    const int amin = cnt > 0 ? offs[j1 - 1] : (1 << 30);
    const int64_t look = (amin - 31 + 31) / 32;  // ceil((amin - 31) / 32): batches behind
    PROF_DECL(p_nw);
    PROF_DECL(p_nf);
    for (int64_t b = g; b < nb; b += NG) {
      int64_t need = b + 1 - look;                              // operands final
      need = max(need, b + 1 - (int64_t)kNearSlots + 1);        // slot consumed by the combiner
      long long t0 = PROF_NOW();
      wait_batches(batch_done, need);
      PROF_ADD(p_nw, t0);
      t0 = PROF_NOW();
      const int64_t c = a1 + 32 * b + lane;
      const char* base = reinterpret_cast<const char*>(ring + (((uint32_t)c & (R - 1)) + R));
      T a0 = id, a1v = id, a2 = id, a3 = id;
#pragma unroll
      for (int i = 0; i < kNearMax; i += 4) {
        T v0 = *reinterpret_cast<const T*>(base - ob[i]);
        T v1 = *reinterpret_cast<const T*>(base - ob[i + 1]);
        T v2 = *reinterpret_cast<const T*>(base - ob[i + 2]);
        T v3 = *reinterpret_cast<const T*>(base - ob[i + 3]);
        if (!IsIdem<OP>::value) {  // duplicates are harmless only for idempotent ops
          v0 = i < cnt ? v0 : id;
          v1 = i + 1 < cnt ? v1 : id;
          v2 = i + 2 < cnt ? v2 : id;
          v3 = i + 3 < cnt ? v3 : id;
        }
        a0 = O::apply(a0, v0);
        a1v = O::apply(a1v, v1);
        a2 = O::apply(a2, v2);
        a3 = O::apply(a3, v3);
      }
      const int ns = (int)(b % kNearSlots);
      near_part[((size_t)ns * NW + j) * 32 + lane] = O::apply(O::apply(a0, a1v), O::apply(a2, a3));
      __syncwarp();
      if (lane == 0) mbar_arrive(&near_full[ns]);
      PROF_ADD(p_nf, t0);
    }
    PROF_FLUSH(16 + (j == 0 ? 0 : 2), p_nw);
    PROF_FLUSH(17 + (j == 0 ? 0 : 2), p_nf);
    (void)g;
  } else if (REMOTE && role >= NC + NW * NG + S.writers && role < NC + NW * NG + S.writers + S.fetchers) {
    // ================================ fetchers ==============================
    // copy the remote producers' partials into shared slots ahead of the
    // combiners (batch b -> fetcher b % kFetchers), so no global-memory
    // latency sits on the combine path
    const int f = role - (NC + NW * NG + S.writers);
    for (int64_t b = f; b < nb; b += S.fetchers) {
      const int fs = (int)(b % kFetchSlots);
      wait_batches(batch_done, b + 1 - kFetchSlots);  // slot consumed by the combiner
      if (lane == 0) spin_eq_gpu(RM.ready + (int)(b % kRemSlots), (int)(b + 1), 32);
      __syncwarp();
      fence_acquire_gpu();
      rem_part[fs * 32 + lane] =
          ldv_cg<T, int64_t>(reinterpret_cast<const int64_t*>(RM.part) + (int)(b % kRemSlots) * 32 + lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&rem_full[fs]);
    }
  } else if (role >= NC + NW * NG && role < NC + NW * NG + S.writers) {
    // ================================= writers ==============================
    // batch b -> writer b % writers; each writer's gpu-scope release of its own
    // share overlaps the other writers' stores
    const int w = role - (NC + NW * NG), NWR = S.writers;
    PROF_DECL(p_ww);
    PROF_DECL(p_wp);
    int done = 0;
    for (int64_t b = w; b < nb; b += NWR) {
      long long t0 = PROF_NOW();
      mbar_wait(&batch_done[b % kBatchBars], (unsigned)((b / kBatchBars) & 1));
      PROF_ADD(p_ww, t0);
      const int64_t c = a1 + 32 * b + lane;
      if (c < n) out[c] = (int64_t)ring[(uint32_t)c & (R - 1)];
      __syncwarp();
      ++done;
      if (lane == 0) st_release_cta(written_count + w, done);  // after the warp barrier: all lanes' stores
      if (REMOTE && (done % S.pub_every == 0 || b + NWR >= nb)) {
        t0 = PROF_NOW();
        __syncwarp();
        // the warp barrier orders every lane's table stores before lane 0's
        // gpu-scope release (release is cumulative; the bar.sync + single
        // st.release idiom), so no separate full fence
        if (lane == 0) st_release_gpu(reinterpret_cast<long long*>(RM.published) + w, (long long)(b + 1));
        __syncwarp();
        PROF_ADD(p_wp, t0);
      }
    }
    PROF_FLUSH(28, p_ww);
    PROF_FLUSH(29, p_wp);
    PROF_FLUSH(29, p_wp);
  }
}

template <int OP, typename T>
__global__ void __launch_bounds__(768, 1)
    sdp_v2_cta(const __grid_constant__ SdpV2Shape S, const int64_t* __restrict__ g_offsets, const int64_t* __restrict__ g_init,
               int64_t* __restrict__ g_out) {
  const int64_t inst = blockIdx.x;
  sdp_v2_finisher<OP, T, false>(S, g_offsets + inst * S.k, g_init + inst * S.a1, g_out + inst * S.n,
                                SdpRemote{});
}

// Block 0: finisher; blocks 1..: remote producers (cooperative launch).
template <int OP, typename T>
__global__ void __launch_bounds__(768, 1)
    sdp_v2_multi(const __grid_constant__ SdpV2Shape S, const SdpShape PS, const int64_t* __restrict__ g_offsets,
                 const int64_t* __restrict__ g_init, int64_t* g_out, const SdpRemote RM) {
  if (blockIdx.x == 0) {
    sdp_v2_finisher<OP, T, true>(S, g_offsets, g_init, g_out, RM);
  } else {
    if (threadIdx.x >= 32 * PS.remote_warps) return;
    sdp_producer<OP, T>(PS, g_offsets, g_out, RM, blockIdx.x - 1, gridDim.x - 1);
  }
}

}  // namespace pipedp_dev

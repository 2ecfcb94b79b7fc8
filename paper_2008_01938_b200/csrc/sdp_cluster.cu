// sdp_cluster.cu -- the S-DP pipeline of one instance spread over a
// thread-block cluster (sm_100a: up to 16 CTAs, distributed shared memory).
//
// The paper's k-lane pipeline hands partial (x)-accumulators down the offsets
// (sdp_pipeline.hpp:24-46); here the offsets are split by size:
//   * CTA 0 (finisher): the chain warp (offsets < 32 in-batch, [l+1, l+32]
//     look-ahead: sdp_kernels.cuh), mid warps (offsets [64, a_p) from its
//     ring, the group [l+33, 63], and the producers' partials), and the
//     writer, which stores each finished batch to HBM and PUSHES it into every
//     producer's ring through DSMEM (st.shared::cluster), then arrives on the
//     producer's mbarrier remotely (release.cluster);
//   * CTAs 1..C-1 (producers): each owns a contiguous share of the offsets
//     >= a_p and keeps its own mirrored copy of the last a_1 + 96 cells in
//     shared memory; a batch's fold runs as soon as the batch `look` steps
//     back has arrived, and its 32 partials go back to the finisher through
//     DSMEM with a remote arrive on the finisher's per-slot mbarrier.
// No table operand crosses L2 on the way: every relaxation reads local shared
// memory; the only cluster traffic is 32 values per batch per producer each
// way.  Associative (x) on the 32-bit value class (min, max, normalised
// mod-add), so the producers' partials may be combined in any grouping.
#include "sdp_cluster.hpp"

#include <algorithm>

#include "sdp_kernels.cuh"

namespace pipedp_cluster {

using namespace pipedp_dev;

constexpr int kMid = 32;     // mid -> chain slots
constexpr int kRem = 32;     // producer -> finisher partial slots (batches)
constexpr int kBars = 64;    // batch_done ring
constexpr int kAvail = 256;  // writer -> producer "batch pushed" barriers
constexpr int kMaxCluster = 16;
constexpr int kNearWarps = 4;  // two pairs, each splitting one batch's near fold

struct Params {
  int64_t n;
  int32_t k, a1, a_p, j_p, j_96, j_64, fin_r, prod_r, mid_warps, prod_warps, C, max_share, writers;
  const int64_t* offsets;
  const int64_t* init;
  int64_t* out;
};

// ---- distributed shared memory and cluster-scope mbarriers ----------------
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t raddr, int32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(raddr), "r"(v) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t raddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
// st.async: a store into another CTA's shared memory that completes bytes on
// that CTA's mbarrier (the TMA transaction protocol) -- no fence, no release
// arrive: the consumer's phase completes when every expected byte landed
__device__ __forceinline__ void st_async(uint32_t raddr, int32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
               "r"(rbar)
               : "memory");
}
// arm the next phase of a count-1 barrier: one arrival plus the bytes to expect
__device__ __forceinline__ void arm(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int32_t lds(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// fold the words at byte offsets nob[0, cnt) (nob = -4 a) from base: eight
// independent loads per trip and the < 8 rest issued together (absent slots
// read the base word and fold the identity), so no load waits on the previous
// one's fold -- the [64, 96) group has only ~8 offsets on C2, where a
// one-at-a-time head / tail loop cost ~430 cycles per batch
template <int OP>
__device__ __forceinline__ int32_t fold_smem(int32_t acc, uint32_t base, const int32_t* nob, int cnt) {
  using O = SemiOp<OP, int32_t>;
  const int32_t id = SemiId<OP, int32_t>::value();
  int j = 0;
#pragma unroll 1
  for (; j + 8 <= cnt; j += 8) {
    int32_t v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = lds(base + nob[j + t]);
    acc = O::apply(acc, O::apply(O::apply(O::apply(v[0], v[1]), O::apply(v[2], v[3])),
                                 O::apply(O::apply(v[4], v[5]), O::apply(v[6], v[7]))));
  }
  if (j < cnt) {
    int32_t v[8];
#pragma unroll
    for (int t = 0; t < 7; ++t) {
      const bool live = j + t < cnt;
      const int32_t x = lds(base + (live ? nob[j + t] : 0));
      v[t] = live ? x : id;
    }
    v[7] = id;
    acc = O::apply(acc, O::apply(O::apply(O::apply(v[0], v[1]), O::apply(v[2], v[3])),
                                 O::apply(O::apply(v[4], v[5]), O::apply(v[6], v[7]))));
  }
  return acc;
}

// ---- shared-memory layouts (identical arithmetic in every CTA) ------------
struct FinLayout {
  uint32_t ring, small, nob_mid, mid_part, fm_part, nb_part, cl_part, bars, end;
};
__host__ __device__ inline FinLayout fin_layout(const Params& p) {
  FinLayout L;
  uint32_t o = 0;
  L.ring = o;
  o += 4u * 2 * p.fin_r;
  L.small = o;  // raw offsets < 64 (the chain's masks)
  o += 4u * 64;
  L.nob_mid = o;  // -4 a for offsets [64, a_p)
  o += 4u * (((p.j_p > p.j_64 ? 0 : p.j_64 - p.j_p) + 7) & ~7);
  L.mid_part = o;
  o += 4u * kMid * 32;
  L.fm_part = o;
  o += 4u * kMid * 32;
  L.nb_part = o;  // the second near half's partials
  o += 4u * kMid * 32;
  L.cl_part = o;  // [C-1][kRem][32]
  o += 4u * (p.C - 1) * kRem * 32;
  o = (o + 7) & ~7u;
  L.bars = o;  // batch_done[kBars] | mid_full[kMid] | cl_full[kRem] | fm_full[kMid] | nb_full[kMid]
  o += 8u * (kBars + kMid + kRem + kMid + kMid);
  L.end = o;
  return L;
}
struct ProdLayout {
  uint32_t ring, nob, avail, end;
};
__host__ __device__ inline ProdLayout prod_layout(const Params& p) {
  ProdLayout L;
  uint32_t o = 0;
  L.ring = o;
  o += 4u * 2 * p.prod_r;
  L.nob = o;
  o += 4u * ((p.max_share + 7) & ~7);
  o = (o + 7) & ~7u;
  L.avail = o;
  o += 8u * kAvail;
  L.end = o;
  return L;
}

// producer q's share of the offsets >= a_p: index range [j0, j1)
__host__ __device__ inline void share(const Params& p, int q, int* j0, int* j1) {
  const int P = p.C - 1;
  *j0 = (int)((int64_t)p.j_p * (q - 1) / P);
  *j1 = (int)((int64_t)p.j_p * q / P);
}

template <int OP>
__global__ void __launch_bounds__(32 * 20, 1) sdp_cluster_kernel(const Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  using T = int32_t;
  using O = SemiOp<OP, T>;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int rank = (int)cl_rank();
  const int a1 = p.a1;
  const int64_t n = p.n;
  const int64_t nb = (n - a1 + 31) / 32;
  const uint32_t sbase = smem_u32(smem);
  const FinLayout FL = fin_layout(p);
  const ProdLayout PL = prod_layout(p);
  const T id = SemiId<OP, T>::value();

  if (rank == 0) {
    // ================================ finisher ===============================
    T* ring = reinterpret_cast<T*>(smem + FL.ring);
    int32_t* small = reinterpret_cast<int32_t*>(smem + FL.small);
    int32_t* nob_mid = reinterpret_cast<int32_t*>(smem + FL.nob_mid);
    T* mid_part = reinterpret_cast<T*>(smem + FL.mid_part);
    T* cl_part = reinterpret_cast<T*>(smem + FL.cl_part);
    uint64_t* batch_done = reinterpret_cast<uint64_t*>(smem + FL.bars);
    uint64_t* mid_full = batch_done + kBars;
    uint64_t* cl_full = mid_full + kMid;
    uint64_t* fm_full = cl_full + kRem;
    uint64_t* nb_full = fm_full + kMid;
    T* fm_part = reinterpret_cast<T*>(smem + FL.fm_part);
    T* nb_part = reinterpret_cast<T*>(smem + FL.nb_part);
    const int R = p.fin_r;
    const int nsmall = p.k - p.j_64;
    for (int j = tid; j < nsmall; j += blockDim.x) small[j] = (int32_t)p.offsets[p.j_64 + j];
    for (int j = p.j_p + tid; j < p.j_64; j += blockDim.x) nob_mid[j - p.j_p] = -4 * (int32_t)p.offsets[j];
    for (int i = tid; i < a1; i += blockDim.x) {
      const int64_t v = p.init[i];
      if (i >= a1 - R) {
        ring[i & (R - 1)] = (T)v;
        ring[(i & (R - 1)) + R] = (T)v;
      }
      p.out[i] = v;
    }
    if (tid == 0) {
      for (int s = 0; s < kBars + kMid; ++s) mbar_init(&batch_done[s], 1);
      for (int s = 0; s < kRem; ++s) mbar_init(&cl_full[s], 1);
      for (int s = 0; s < kMid; ++s) mbar_init(&fm_full[s], 1);
      for (int s = 0; s < kMid; ++s) mbar_init(&nb_full[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int s = 0; s < kRem; ++s) arm(&cl_full[s], 128u * (uint32_t)(p.C - 1));
    }
    cluster_sync_all();
    const int M = p.mid_warps;
    // the chain warp keeps SM sub-partition 0 to itself: other roles skip warp
    // ids that are 0 mod 4 (warps map to sub-partitions by id mod 4)
    const int role = sdp_role_of_warp(warp);
    if (warp == 0) {
      // ---------------------------------- chain ------------------------------
      const LaMasks lm = la_masks(small, nsmall, lane);
      const IdemMasks im = idem_masks(small, nsmall, lane);
      T nxt = id;
      {
        const int pos0 = (int)((a1 + lane) & (R - 1)) + R;
        for (int d = lane + 32; d >= lane + 1; --d)
          if ((lm.nbits >> (d - lane - 1)) & 1u) nxt = O::apply(nxt, ring[pos0 - d]);
      }
      PROF_DECL(t_wm);
      PROF_DECL(t_wf);
      PROF_DECL(t_tot);
      const long long t_start = PROF_NOW();
      for (int64_t b = 0; b < nb; ++b) {
        const int64_t c = a1 + 32 * b + lane;
        const int slot = (int)(b % kMid);
        long long t0 = PROF_NOW();
        mbar_wait(&mid_full[slot], (unsigned)((b / kMid) & 1));
        PROF_ADD(t_wm, t0);
        t0 = PROF_NOW();
        mbar_wait(&fm_full[slot], (unsigned)((b / kMid) & 1));
        PROF_ADD(t_wf, t0);
        (void)t0;
        T acc = O::apply(O::apply(mid_part[slot * 32 + lane], fm_part[slot * 32 + lane]), nxt);
        if (IsIdem<OP>::value) {
          idem_closure<OP, T>(acc, nxt, im);
        } else {
          nxt = id;
          LaSteps<OP, T, 1>::run(acc, nxt, lm);
        }
        const int pq = (int)(c & (R - 1));
        ring[pq] = acc;
        ring[pq + R] = acc;
        __syncwarp();
        if (lane == 0) mbar_arrive(&batch_done[b % kBars]);
      }
      PROF_ADD(t_tot, t_start);
      (void)t_start;
      PROF_FLUSH(0, t_wm);
      PROF_FLUSH(1, t_wf);
      PROF_FLUSH(2, t_tot);
      PROF_FLUSH(3, nb);
    } else if (role < 0) {
      // idle: shares sub-partition 0 with the chain
    } else if (role < M) {
      // ----------------------------------- mid -------------------------------
      // split by how far back the operands are, so only a short fold sits on
      // the chain's critical path:
      //   near warps (roles 0..3): [l+33, 63] ring group + [64, 96): batch b-2
      //     final, needed when b-1 finishes -- the pace-setting fold, so each
      //     batch's is split over a PAIR of warps (pairs alternate batches):
      //     half A the ring group, half B [64, 96); B hands its partial to A
      //     (mbarrier), A combines and hands the sum to the chain;
      //   far-mid warps (roles 4..M-1): [96, a_p) + the producers' partials:
      //     batch b-3 final, two batches of slack.
      const LaMasks mlm = la_masks(small, nsmall, lane);
      const int r = role;
      const bool near = r < kNearWarps;
      const int slot_stride = near ? kNearWarps / 2 : M - kNearWarps;
      const int my = near ? r >> 1 : r - kNearWarps;
      const bool half_b = near && (r & 1);
      const int n96 = p.j_96 - p.j_p, nmid = p.j_64 - p.j_p;
      {
        PROF_DECL(t_w1);
        PROF_DECL(t_w2);
        PROF_DECL(t_f);
        long long cntb = 0;
        for (int64_t b = my; b < nb; b += slot_stride) {
          ++cntb;
          const int64_t c = a1 + 32 * b + lane;
          const T* rb = ring + (int)(c & (R - 1)) + R;
          const int slot = (int)(b % kMid);
          T acc;
          long long t0 = PROF_NOW();
          if (near) {
            wait_batches(batch_done, b - 1);  // batches <= b-2 final
            PROF_ADD(t_w1, t0);
            t0 = PROF_NOW();
            if (half_b) {
              acc = fold_smem<OP>(id, smem_u32(rb), nob_mid + n96, nmid - n96);  // [64, 96)
              nb_part[slot * 32 + lane] = acc;
              __syncwarp();
              if (lane == 0) mbar_arrive(&nb_full[slot]);
              PROF_ADD(t_f, t0);
              continue;
            }
            acc = la_ring_group<OP, T>(rb, mlm.far);  // d in [l+33, 63]
            PROF_ADD(t_f, t0);
            t0 = PROF_NOW();
            mbar_wait(&nb_full[slot], (unsigned)((b / kMid) & 1));
            PROF_ADD(t_w2, t0);
            acc = O::apply(acc, nb_part[slot * 32 + lane]);
          } else {
            wait_batches(batch_done, b - 2);  // batches <= b-3 final
            PROF_ADD(t_w1, t0);
            t0 = PROF_NOW();
            acc = fold_smem<OP>(id, smem_u32(rb), nob_mid, n96);
            PROF_ADD(t_f, t0);
            t0 = PROF_NOW();
            const int rs = (int)(b % kRem);
            mbar_wait(&cl_full[rs], (unsigned)((b / kRem) & 1));
            PROF_ADD(t_w2, t0);
            for (int q = 0; q < p.C - 1; ++q) acc = O::apply(acc, cl_part[(q * kRem + rs) * 32 + lane]);
            __syncwarp();
            if (lane == 0) arm(&cl_full[rs], 128u * (uint32_t)(p.C - 1));  // phase of batch b + kRem
          }
          (near ? mid_part : fm_part)[slot * 32 + lane] = acc;
          __syncwarp();
          if (lane == 0) mbar_arrive(&(near ? mid_full : fm_full)[slot]);
        }
        PROF_FLUSH(near ? (half_b ? 16 : 8) : 12, t_w1);
        PROF_FLUSH(near ? (half_b ? 17 : 9) : 13, t_f);
        PROF_FLUSH(near ? (half_b ? 18 : 10) : 14, t_w2);
        PROF_FLUSH(near ? (half_b ? 19 : 11) : 15, cntb);
        (void)cntb;
      }
    } else if (role < M + p.writers) {
      // --------------------------------- writers -----------------------------
      // batch b -> writer (b mod writers): HBM store, push into every
      // producer's ring (DSMEM), then lane q arrives on producer q's barrier
      // (one cluster-scope release per producer, all in parallel)
      const int w = role - M, NW = p.writers;
      const int PR = p.prod_r;
      const uint32_t ring_p = sbase + PL.ring, avail_p = sbase + PL.avail;
      uint32_t rbase[kMaxCluster], rbar[kMaxCluster];  // producer q's ring / barriers, cluster window
#pragma unroll
      for (int q = 1; q < kMaxCluster; ++q) {
        rbase[q] = q < p.C ? mapa(ring_p, (uint32_t)q) : 0u;
        rbar[q] = q < p.C ? mapa(avail_p, (uint32_t)q) : 0u;
      }
      for (int64_t b = w; b < nb; b += NW) {
        mbar_wait(&batch_done[b % kBars], (unsigned)((b / kBars) & 1));
        const int64_t c = a1 + 32 * b + lane;
        const T v = ring[(int)(c & (R - 1))];
        const uint32_t o1 = 4u * (uint32_t)(c % PR), o2 = o1 + 4u * (uint32_t)PR;
        const uint32_t ob = 8u * (uint32_t)(b % kAvail);
#pragma unroll
        for (int q = 1; q < kMaxCluster; ++q) {
          if (q < p.C) {
            st_async(rbase[q] + o1, v, rbar[q] + ob);
            st_async(rbase[q] + o2, v, rbar[q] + ob);
          }
        }
        if (c < n) p.out[c] = (int64_t)v;
      }
    }
  } else {
    // ================================ producer ===============================
    T* ring = reinterpret_cast<T*>(smem + PL.ring);
    int32_t* nob = reinterpret_cast<int32_t*>(smem + PL.nob);
    uint64_t* avail = reinterpret_cast<uint64_t*>(smem + PL.avail);
    const int PR = p.prod_r;
    int j0, j1;
    share(p, rank, &j0, &j1);
    const int cnt = j1 - j0;
    for (int j = tid; j < cnt; j += blockDim.x) nob[j] = -4 * (int32_t)p.offsets[j0 + j];
    for (int i = tid; i < a1; i += blockDim.x) {
      const T v = (T)p.init[i];
      ring[i] = v;  // cell i < a1 <= PR: position i
      ring[i + PR] = v;
    }
    if (tid == 0) {
      for (int s = 0; s < kAvail; ++s) mbar_init(&avail[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int s = 0; s < kAvail; ++s) arm(&avail[s], 256u);  // 32 cells x 2 copies x 4 B
    }
    cluster_sync_all();
    const int a_lo = cnt > 0 ? (int)p.offsets[j1 - 1] : p.a_p;
    const int look = min((a_lo - 31 + 31) / 32, kRem);  // batches between a batch and its newest operand
    const uint32_t part_p = sbase + FL.cl_part + 4u * (uint32_t)(((rank - 1) * kRem) * 32 + lane);
    const uint32_t full_p = sbase + FL.bars + 8u * (uint32_t)(kBars + kMid);
    const int W = p.prod_warps;
    if (warp < W) {
      for (int64_t b = warp; b < nb; b += W) {
        const int64_t X = b - look;
        if (X >= 0) {
          mbar_wait(&avail[X % kAvail], (unsigned)((X / kAvail) & 1));
          __syncwarp();
          if (lane == 0) arm(&avail[X % kAvail], 256u);  // phase of batch X + kAvail
        }
        const int64_t c = a1 + 32 * b + lane;
        const uint32_t base = smem_u32(ring + (int)(c % PR) + PR);
        const T acc = fold_smem<OP>(id, base, nob, cnt);
        const int rs = (int)(b % kRem);
        st_async(mapa(part_p + 4u * (uint32_t)(rs * 32), 0u), acc, mapa(full_p + 8u * (uint32_t)rs, 0u));
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while its shared memory may still be addressed
}

bool plan(const int64_t* offsets, int32_t k, int32_t a1, int64_t n, int op, int device, ClusterPlan* out) {
  if (!(op == kMin || op == kMax || op == kModAdd) || n <= a1) return false;
  int major = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess || major < 9) {
    (void)cudaGetLastError();
    return false;
  }
  ClusterPlan P{};
  P.op = op;
  P.n = n;
  P.k = k;
  P.a1 = a1;
  P.a_p = 256;  // offsets >= 256: producers (measured: 512 and 1024 slower on C2)
  for (int j = 0; j < k; ++j) {
    P.j_p += offsets[j] >= P.a_p;
    P.j_64 += offsets[j] >= 64;
    P.j_96 += offsets[j] >= 96;
  }
  if (P.j_p < 64) return false;  // too little far work for a cluster
  P.cluster = kMaxCluster;
  P.mid_warps = kNearWarps + 3;  // two near pairs + three far-mid warps
  P.writers = 4;
  P.prod_warps = 8;
  P.fin_r = 1;  // >= a_p + 32 (kRem + 4), a power of two
  while (P.fin_r < P.a_p + 32 * (kRem + 4)) P.fin_r <<= 1;
  P.prod_r = (a1 + 96 + 31) & ~31;
  Params q{};
  q.k = k;
  q.j_p = P.j_p;
  q.j_64 = P.j_64;
  q.fin_r = P.fin_r;
  q.prod_r = P.prod_r;
  q.C = P.cluster;
  int ms = 0;
  for (int r = 1; r < q.C; ++r) {
    int j0, j1;
    q.max_share = 0;
    share(q, r, &j0, &j1);
    ms = std::max(ms, j1 - j0);
  }
  q.max_share = ms;
  P.max_prod_offs = ms;
  P.fin_smem = fin_layout(q).end;
  P.prod_smem = prod_layout(q).end;
  P.smem = std::max(P.fin_smem, P.prod_smem);
  if (P.smem > 227 * 1024) return false;
  *out = P;
  return true;
}

cudaError_t launch(const ClusterPlan& P, const int64_t* d_offsets, const int64_t* d_init, int64_t* d_out,
                   cudaStream_t st) {
  Params p{};
  p.n = P.n;
  p.k = P.k;
  p.a1 = P.a1;
  p.a_p = P.a_p;
  p.j_p = P.j_p;
  p.j_64 = P.j_64;
  p.j_96 = P.j_96;
  p.fin_r = P.fin_r;
  p.prod_r = P.prod_r;
  p.mid_warps = P.mid_warps;
  p.prod_warps = P.prod_warps;
  p.C = P.cluster;
  p.max_share = P.max_prod_offs;
  p.writers = P.writers;
  p.offsets = d_offsets;
  p.init = d_init;
  p.out = d_out;
  void (*kern)(Params) = P.op == kMin ? sdp_cluster_kernel<kMin>
                         : P.op == kMax ? sdp_cluster_kernel<kMax>
                                        : sdp_cluster_kernel<kModAdd>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem);
  if (e == cudaSuccess && P.cluster > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)P.cluster);
  cfg.blockDim = dim3((unsigned)(32 * std::max(sdp_warps_for_roles(P.mid_warps + P.writers), P.prod_warps)));
  cfg.dynamicSmemBytes = P.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)P.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

#ifdef PIPEDP_PROFILE
// this translation unit's own role-profiler counters (each TU is its own module)
cudaError_t profile_take(unsigned long long* out128, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out128, pipedp_dev::g_prof, 128 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    static const unsigned long long zero[128] = {};
    e = cudaMemcpyToSymbol(pipedp_dev::g_prof, zero, sizeof zero);
  }
  return e;
}
#endif

}  // namespace pipedp_cluster

// sdp_rank.cu -- the chunk batch of chunked S-DP (min / max) on 16-bit ranks,
// two cells per shared-memory load.
//
// Every value of a min / max table is a copy of an init value (sdp.cpp:52-59
// only ever selects operands), so the table can be computed on the ranks of
// the init values -- rank(v) = lower_bound(sorted init, v) -- and mapped back
// with one lookup per cell: min / max commute with any order-preserving map,
// and the map is injective on the init values, so the result is bit-identical.
// a_1 <= 8192 init values give ranks < 2^13, i.e. 16-bit lanes.  Each cell
// still takes all k of its relaxations; only their representation changes.
//
// Layout (one CTA per chunk, cells [s, s + Lc), preset = chunk entry state):
//  * pair ring: word w holds (rank[w], rank[w + 32]) as u16x2, mirrored
//    (word w and w + R2), R2 >= a_1 + 128 words.  For an offset a >= 96 the
//    operands of cell c (batch b) and of cell c + 32 (batch b + 1) are ONE
//    32-bit word, w = c - a, and one min.u16x2 / max.u16x2 folds both: one
//    LDS per two relaxations (the previous kernel spent two LSU operations --
//    the operand and a reload of the warp-uniform offset -- per relaxation);
//  * the offsets live in the kernel parameter block as byte offsets -4 a_j:
//    read through the uniform datapath (LDCU), they fold into the load as
//    LDS [R + UR]: no per-term address arithmetic;
//  * a scalar rank ring (256 cells) for offsets < 96 and the chain.
// Warp roles (one CTA = one chunk):
//  * chain (warp 0): batch b of 32 cells, in-batch offsets < 32 by the
//    idempotent closure and the look-ahead terms of sdp_kernels.cuh, writes
//    ranks to both rings and the value (sorted[rank]) to the table;
//  * mid warps: batch pair (b, b+1), b even -- offsets in [96, a_mid) paired
//    (needs batches <= b-2 final), then per batch the offsets in [64, 96) and
//    the ring group [l+33, 63] (batch b+1's part once batch b-1 is final);
//  * far warps: offsets >= a_mid paired, far_look batches ahead.
#include "sdp_rank.hpp"

#include "sdp_kernels.cuh"

namespace pipedp_rank {

using pipedp_dev::kMax;
using pipedp_dev::kMin;
using namespace pipedp_dev;

constexpr int kRS = 256;        // scalar rank ring (cells), mirrored
constexpr int kMidS = 32;       // mid -> chain slots (batches)
constexpr int kFarPairs = 16;   // far -> mid slots (pairs)
constexpr int kBars = 64;       // batch_done ring

template <int OP>
struct Pair;
template <>
struct Pair<kMin> {
  static constexpr uint32_t id = 0xFFFFFFFFu;
  __device__ __forceinline__ static uint32_t apply(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
  }
};
template <>
struct Pair<kMax> {
  static constexpr uint32_t id = 0u;
  __device__ __forceinline__ static uint32_t apply(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
  }
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Fold the 32-bit words at byte offsets nob[j0, j1) from the shared-memory
// address base (a 32-bit shared-window address: base + nob[j] becomes one
// LDS [R + UR]).
template <class F, typename W>
__device__ __forceinline__ W fold_words(W acc, uint32_t base, const ChunkRankParams& p, int j0, int j1) {
  int j = j0;
#pragma unroll 1
  for (; j + 8 <= j1; j += 8) {
    W v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = (W)lds_u32(base + (uint32_t)p.nob[j + q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = F::apply(acc, v[q]);
  }
#pragma unroll 1
  for (; j < j1; ++j) acc = F::apply(acc, (W)lds_u32(base + (uint32_t)p.nob[j]));
  return acc;
}

template <int OP>
struct Scal {
  __device__ __forceinline__ static int32_t apply(int32_t a, int32_t b) { return SemiOp<OP, int32_t>::apply(a, b); }
};

__device__ __forceinline__ int32_t rank_of(const int64_t* __restrict__ sorted, int a1, int64_t v) {
  int lo = 0, hi = a1;  // first index with sorted[i] >= v
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(sorted + mid) < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int OP>
__global__ void __launch_bounds__(32 * 16) chunk_rank_kernel(const __grid_constant__ ChunkRankParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  using T = int32_t;
  using O = SemiOp<OP, T>;
  const int R2 = p.r2;
  const int a1 = p.a1;
  uint32_t* ring2 = reinterpret_cast<uint32_t*>(smem);               // [2 R2]
  T* ring = reinterpret_cast<T*>(ring2 + 2 * R2);                     // [2 kRS]
  T* mid_part = ring + 2 * kRS;                                       // [kMidS][32]
  uint32_t* far_part = reinterpret_cast<uint32_t*>(mid_part + kMidS * 32);  // [kFarPairs][32]
  int32_t* offs = reinterpret_cast<int32_t*>(far_part + kFarPairs * 32);   // [k]
  uint64_t* bars = reinterpret_cast<uint64_t*>(offs + ((p.k + 1) & ~1));
  uint64_t* batch_done = bars;
  uint64_t* mid_full = batch_done + kBars;
  uint64_t* far_full = mid_full + kMidS;
  uint16_t* h16 = reinterpret_cast<uint16_t*>(ring2);

  const int tid = threadIdx.x, lane = tid & 31;
  // warp index through a shuffle: the compiler then knows it is warp-uniform,
  // so each role's loop counters and offset reads stay on the uniform
  // datapath (LDCU + LDS [R + UR]) instead of per-lane registers
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int64_t g = p.g0 + blockIdx.x;
  const int64_t s = a1 + g * p.Lc;
  const int64_t e = min(s + p.Lc, p.n);
  const int64_t nb = (e - s + 31) / 32;

  for (int j = tid; j < p.k; j += blockDim.x) offs[j] = (int32_t)p.offsets[j];
  // preset cells [s - a1, s): ranks into both rings
  const int64_t* ci = p.cinit + g * a1;
  for (int i = tid; i < a1; i += blockDim.x) {
    const int64_t q = s - a1 + i;
    const T r = rank_of(p.sorted, a1, ci[i]);
    if (i >= a1 - kRS) {
      const int pq = (int)(q & (kRS - 1));
      ring[pq] = r;
      ring[pq + kRS] = r;
    }
    const int w = (int)(q % R2), w2 = (int)((q - 32 + R2) % R2);
    h16[2 * w] = (uint16_t)r;
    h16[2 * (w + R2)] = (uint16_t)r;
    h16[2 * w2 + 1] = (uint16_t)r;
    h16[2 * (w2 + R2) + 1] = (uint16_t)r;
  }
  if (tid == 0)
    for (int b = 0; b < kBars + kMidS + kFarPairs; ++b) mbar_init(&bars[b], 1);
  __syncthreads();

  const int M = p.mid_warps, F = p.far_warps;
  if (warp == 0) {
    // ================================ chain ================================
    const LaMasks lm = la_masks(offs, p.k, lane);
    const IdemMasks im = idem_masks(offs, p.k, lane);
    T nxt = SemiId<OP, T>::value();
    {  // the previous (virtual) batch's look-ahead over the preset cells
      const int pos0 = (int)((s + lane) & (kRS - 1)) + kRS;
      for (int d = lane + 32; d >= lane + 1; --d)
        if ((lm.nbits >> (d - lane - 1)) & 1u) nxt = O::apply(nxt, ring[pos0 - d]);
    }
    int w = (int)((s + lane) % R2), w2 = (int)((s + lane - 32 + R2) % R2);
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t c = s + 32 * b + lane;
      const int slot = (int)(b % kMidS);
      mbar_wait(&mid_full[slot], (unsigned)((b / kMidS) & 1));
      T acc = O::apply(mid_part[slot * 32 + lane], nxt);
      idem_closure<OP, T>(acc, nxt, im);
      const int pq = (int)(c & (kRS - 1));
      ring[pq] = acc;
      ring[pq + kRS] = acc;
      h16[2 * w] = (uint16_t)acc;
      h16[2 * (w + R2)] = (uint16_t)acc;
      h16[2 * w2 + 1] = (uint16_t)acc;
      h16[2 * (w2 + R2) + 1] = (uint16_t)acc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&batch_done[b % kBars]);
      if (c < e) {
        if (p.out_rank) p.out_rank[c] = (uint16_t)acc;  // 2 B per cell for the trip to the host
        else p.out[c] = __ldg(p.sorted + acc);
      }
      if (p.progress && ((b + 1) % kPublishBatches == 0 || b + 1 == nb)) {
        // this warp's ranks up to batch b are written: order them (system
        // scope -- the reader is the host, then a copy engine) before the count
        __syncwarp();
        if (lane == 0) {
          __threadfence_system();
          const unsigned long long done = (unsigned long long)min(32 * (b + 1), e - s);
          *reinterpret_cast<volatile unsigned long long*>(p.progress + g) = ((unsigned long long)p.epoch << 32) | done;
        }
      }
      w += 32;
      if (w >= R2) w -= R2;
      w2 += 32;
      if (w2 >= R2) w2 -= R2;
    }
  } else if (warp <= M) {
    // ================================= mid =================================
    const LaMasks mlm = la_masks(offs, p.k, lane);
    for (int64_t pr = warp - 1; 2 * pr < nb; pr += M) {
      const int64_t b = 2 * pr;
      const int64_t c = s + 32 * b + lane;
      wait_batches(batch_done, b - 1);  // batches <= b-2 final
      uint32_t P = Pair<OP>::id;
      if (p.j_far > 0) {
        const int fs = (int)(pr % kFarPairs);
        mbar_wait(&far_full[fs], (unsigned)((pr / kFarPairs) & 1));
        P = far_part[fs * 32 + lane];
      }
      const uint32_t base2 = smem_u32(ring2 + (int)(c % R2) + R2);
      P = fold_words<Pair<OP>, uint32_t>(P, base2, p, p.j_far, p.j_pair);
      {  // batch b
        const T* rb = ring + (int)(c & (kRS - 1)) + kRS;
        T lo = fold_words<Scal<OP>, T>((T)(P & 0xFFFFu), smem_u32(rb), p, p.j_pair, p.j_mid);
        lo = O::apply(lo, la_ring_group<OP, T>(rb, mlm.far));
        const int slot = (int)(b % kMidS);
        mid_part[slot * 32 + lane] = lo;
        __syncwarp();
        if (lane == 0) mbar_arrive(&mid_full[slot]);
      }
      if (b + 1 < nb) {  // batch b+1: its [64, 96) and [l+33, 63] operands reach batch b-1
        wait_batches(batch_done, b);
        const T* rb = ring + (int)((c + 32) & (kRS - 1)) + kRS;
        T hi = fold_words<Scal<OP>, T>((T)(P >> 16), smem_u32(rb), p, p.j_pair, p.j_mid);
        hi = O::apply(hi, la_ring_group<OP, T>(rb, mlm.far));
        const int slot = (int)((b + 1) % kMidS);
        mid_part[slot * 32 + lane] = hi;
        __syncwarp();
        if (lane == 0) mbar_arrive(&mid_full[slot]);
      }
    }
  } else if (warp <= M + F) {
    // ================================= far =================================
    for (int64_t pr = warp - 1 - M; 2 * pr < nb; pr += F) {
      const int64_t b = 2 * pr;
      const int64_t c = s + 32 * b + lane;
      int64_t need = b - p.far_look + 1;                        // operands final
      need = max(need, 2 * (pr - kFarPairs) + 1);               // slot consumed
      wait_batches(batch_done, need);
      const uint32_t base2 = smem_u32(ring2 + (int)(c % R2) + R2);
      const uint32_t P = fold_words<Pair<OP>, uint32_t>(Pair<OP>::id, base2, p, 0, p.j_far);
      const int fs = (int)(pr % kFarPairs);
      far_part[fs * 32 + lane] = P;
      __syncwarp();
      if (lane == 0) mbar_arrive(&far_full[fs]);
    }
  }
}

// One CTA: sorted[0, a1) = init ascending (bitonic sort, padded to a power of two).
__global__ void __launch_bounds__(1024) rank_sort_kernel(const int64_t* __restrict__ init, int a1,
                                                         int64_t* __restrict__ sorted) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* v = reinterpret_cast<int64_t*>(smem);
  int N = 1;
  while (N < a1) N <<= 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) v[i] = i < a1 ? init[i] : INT64_MAX;
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const int64_t x = v[i], y = v[l];
          if ((x > y) == up) {
            v[i] = y;
            v[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < a1; i += blockDim.x) sorted[i] = v[i];
}

static size_t smem_bytes(int r2, int k) {
  return sizeof(uint32_t) * 2 * (size_t)r2 + sizeof(int32_t) * 2 * kRS +
         sizeof(int32_t) * kMidS * 32 + sizeof(uint32_t) * kFarPairs * 32 + sizeof(int32_t) * ((k + 1) & ~1) +
         sizeof(uint64_t) * (kBars + kMidS + kFarPairs);
}

bool chunk_rank_plan(const int64_t* offsets, const int64_t* d_offsets, int k, int a1, int64_t n, int64_t Lc,
                     int64_t G, int op, ChunkRankParams* p, int* threads, size_t* smem) {
  if ((op != 0 && op != 1) || k < 1 || k > kMaxK || a1 < 64 || a1 > 8192 || offsets[0] != a1) return false;
  ChunkRankParams q{};
  q.n = n;
  q.Lc = Lc;
  q.G = G;
  q.k = k;
  q.a1 = a1;
  q.op = op;
  q.r2 = (a1 + 128 + 31) & ~31;
  q.a_mid = a1 > 1024 ? 384 : 256;
  for (int j = 0; j < k; ++j) {
    q.nob[j] = -4 * (int32_t)offsets[j];
    q.j_far += offsets[j] >= q.a_mid;
    q.j_pair += offsets[j] >= 96;
    q.j_mid += offsets[j] >= 64;
  }
  q.far_look = (q.a_mid - 63 + 31) / 32;
  q.mid_warps = 1;
  q.far_warps = q.j_far == 0 ? 0 : (int)std::min<int64_t>(6, std::max<int64_t>(1, (q.j_far + 127) / 128));
  q.offsets = d_offsets;
  *p = q;
  *threads = 32 * (1 + q.mid_warps + q.far_warps);
  *smem = smem_bytes(q.r2, k);
  return true;
}

cudaError_t chunk_rank_sort(const int64_t* d_init, int a1, int64_t* d_sorted, cudaStream_t st) {
  int N = 1;
  while (N < a1) N <<= 1;
  const size_t sm = sizeof(int64_t) * N;
  cudaError_t e = cudaFuncSetAttribute(rank_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  rank_sort_kernel<<<1, 1024, sm, st>>>(d_init, a1, d_sorted);
  return cudaGetLastError();
}

cudaError_t chunk_rank_launch(const ChunkRankParams& p, int threads, size_t smem, cudaStream_t st) {
  auto kern = p.op == 0 ? chunk_rank_kernel<kMin> : chunk_rank_kernel<kMax>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)(p.G - p.g0), threads, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace pipedp_rank

// mcm_tournament.cu -- the paper's O(n^2 log n) tournament method for MCM
// as the in-repo GPU comparison kernel, done the way
// the method is meant to run: every cell of a diagonal at once, each cell's D
// terms folded by a group of threads and reduced in a ceil(log2)-level tree
// (shuffle levels inside a warp, shared-memory levels across warps), one grid
// barrier per diagonal (persistent cooperative grid, all SMs).
//
// Same outputs as solve_mcm_sequential (mcm.cpp:85-110): cells and the split
// table (1-based term index, first minimum: (value, j) lexicographic).  The
// table lives in HBM in the reference layout; values are exact int64.  Cells
// written by other SMs are read through L2 (ld.global.cg): L1 is not coherent
// across the grid barrier.
#include "mcm_tournament.hpp"

#include <cstdint>

#include "common.cuh"

namespace pipedp_tour {

using namespace pipedp_dev;

constexpr int kThreads = 256;

__host__ __device__ __forceinline__ int64_t dbase(int64_t d, int64_t n) { return d * n - d * (d - 1) / 2; }

struct Best {
  int64_t v;
  int32_t j;
};
__device__ __forceinline__ void take(Best& b, int64_t v, int32_t j) {
  if (v < b.v || (v == b.v && j < b.j)) {
    b.v = v;
    b.j = j;
  }
}

__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = (unsigned)ld_relaxed_gpu_i32(reinterpret_cast<const int*>(bar + 1));
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while ((unsigned)ld_relaxed_gpu_i32(reinterpret_cast<const int*>(bar + 1)) == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) mcm_tournament_diag(int64_t n, const int64_t* __restrict__ dims,
                                                                int64_t* cells, int64_t* split, unsigned* bar) {
  __shared__ int64_t sv[kThreads / 32];
  __shared__ int32_t sj[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t T = (int64_t)gridDim.x * kThreads;
  const int64_t gt = blockIdx.x * (int64_t)kThreads + tid;
  for (int64_t i = gt; i <= n; i += T) {  // slot 0 and the base cells
    cells[i] = 0;
    split[i] = 0;
  }
  grid_sync(bar);
  for (int64_t D = 1; D < n; ++D) {
    const int64_t m = n - D;  // cells on the diagonal
    // threads per cell: enough to cover the grid, at most D, a power of two, <= a CTA
    int tpc = 1;
    while ((int64_t)tpc * 2 <= D && (int64_t)tpc * 2 * m <= T && tpc * 2 <= kThreads) tpc <<= 1;
    const int64_t db = dbase(D, n);
    if (tpc <= 32) {
      // groups of tpc lanes inside a warp; grid-stride over cells
      const int64_t groups = T / tpc, rounds = (m + groups - 1) / groups;  // uniform trip count
      for (int64_t it = 0; it < rounds; ++it) {
        const int64_t r = gt / tpc + it * groups + 1;
        const bool live = r <= m;
        Best best{INT64_MAX, 0};
        if (live) {
          const int64_t c = r + D;
          const int64_t prc = dims[r - 1] * dims[c];
          for (int64_t j = (gt % tpc) + 1; j <= D; j += tpc)
            take(best, __ldcg(cells + dbase(j - 1, n) + r) + __ldcg(cells + dbase(D - j, n) + r + j) + prc * dims[r + j - 1],
                 (int32_t)j);
        }
        for (int s = tpc >> 1; s > 0; s >>= 1) {  // tournament levels (shuffles)
          const int64_t ov = __shfl_xor_sync(0xffffffffu, best.v, s);
          const int32_t oj = __shfl_xor_sync(0xffffffffu, best.j, s);
          take(best, ov, oj);
        }
        if (live && (gt % tpc) == 0) {
          cells[db + r] = best.v;
          split[db + r] = best.j;
        }
      }
    } else {
      // tpc / 32 warps of one CTA per cell; blocks stride over cells
      const int cpb = kThreads / tpc;  // cells per CTA
      const int wpc = tpc / 32;
      for (int64_t base = (int64_t)blockIdx.x * cpb; base < m; base += (int64_t)gridDim.x * cpb) {
        const int64_t r = base + tid / tpc + 1;
        const bool live = r <= m;
        Best best{INT64_MAX, 0};
        if (live) {
          const int64_t c = r + D;
          const int64_t prc = dims[r - 1] * dims[c];
          for (int64_t j = (tid % tpc) + 1; j <= D; j += tpc)
            take(best, __ldcg(cells + dbase(j - 1, n) + r) + __ldcg(cells + dbase(D - j, n) + r + j) + prc * dims[r + j - 1],
                 (int32_t)j);
        }
        for (int s = 16; s > 0; s >>= 1) {
          const int64_t ov = __shfl_xor_sync(0xffffffffu, best.v, s);
          const int32_t oj = __shfl_xor_sync(0xffffffffu, best.j, s);
          take(best, ov, oj);
        }
        if (lane == 0) {
          sv[warp] = best.v;
          sj[warp] = best.j;
        }
        __syncthreads();
        for (int s = wpc >> 1; s > 0; s >>= 1) {  // levels across the cell's warps
          if (lane == 0 && (warp % wpc) < s) {
            Best a{sv[warp], sj[warp]};
            take(a, sv[warp + s], sj[warp + s]);
            sv[warp] = a.v;
            sj[warp] = a.j;
          }
          __syncthreads();
        }
        if (live && tid % tpc == 0) {
          cells[db + r] = sv[warp];
          split[db + r] = sj[warp];
        }
        __syncthreads();
      }
    }
    grid_sync(bar);
  }
}

cudaError_t launch(int64_t n, const int64_t* d_dims, int64_t* d_cells, int64_t* d_split, unsigned* d_bar,
                   cudaStream_t st) {
  int dev = 0, sms = 0, per = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mcm_tournament_diag, kThreads, 0);
  if (e != cudaSuccess) return e;
  per = per < 1 ? 1 : (per > 4 ? 4 : per);
  e = cudaMemsetAsync(d_bar, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&n, (void*)&d_dims, (void*)&d_cells, (void*)&d_split, (void*)&d_bar};
  return cudaLaunchCooperativeKernel((const void*)mcm_tournament_diag, dim3((unsigned)(sms * per)), dim3(kThreads),
                                     args, 0, st);
}

}  // namespace pipedp_tour

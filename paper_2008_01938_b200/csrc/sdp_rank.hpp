// sdp_rank.hpp -- host interface of the rank-compressed chunk kernel
// (sdp_rank.cu), used by the chunked S-DP mode of capi.cu for min / max.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pipedp_rank {

constexpr int kMaxK = 4096;  // offsets carried in the kernel parameter block
constexpr int kPublishBatches = 128;  // progress granularity: 4096 cells

// Kernel parameters (a __grid_constant__ block: the offsets are read through
// the uniform datapath, LDCU, and fold into the LDS address as [R + UR]).
struct ChunkRankParams {
  int64_t n;       // table size
  int64_t Lc;      // cells per chunk
  int64_t G;       // launch covers chunks [g0, G)
  int64_t g0;
  int32_t k, a1;
  int32_t op;      // 0 min, 1 max
  int32_t r2;      // pair ring: r2 words (>= a_1 + 128), mirrored
  int32_t mid_warps, far_warps;
  int32_t j_far;   // offsets >= a_mid: offs[0, j_far) (far warps, paired)
  int32_t j_pair;  // offsets >= 96:    offs[j_far, j_pair) (mid warps, paired)
  int32_t j_mid;   // offsets >= 64:    offs[j_pair, j_mid) (mid warps, per batch)
  int32_t a_mid;
  int32_t far_look;  // batches between a far pair and the newest cell it reads
  const int64_t* cinit;   // [G][a1] chunk entry states (values)
  const int64_t* sorted;  // [a1] init values ascending: rank -> value
  int64_t* out;           // the table
  uint16_t* out_rank;     // nullable: write each cell's rank here instead (host-bound solves)
  // nullable (out_rank only): per chunk, (epoch << 32) | cells of the chunk
  // final in out_rank, published every kPublish cells into mapped host memory
  // so the host copies and converts the finished part of every chunk while
  // the chunks still run
  unsigned long long* progress;
  uint32_t epoch;
  const int64_t* offsets; // [k] the offsets (device), for the chain's masks
  int32_t nob[kMaxK];     // -4 a_j: byte offset of offset a_j in a ring of 32-bit words
};

// Decide whether the instance takes the rank kernel and fill the shape.
// Returns false (and leaves *p untouched otherwise) when it does not apply.
bool chunk_rank_plan(const int64_t* offsets, const int64_t* d_offsets, int k, int a1, int64_t n, int64_t Lc, int64_t G, int op,
                     ChunkRankParams* p, int* threads, size_t* smem);

// sorted[0, a1) = init ascending (one CTA, bitonic sort in shared memory)
cudaError_t chunk_rank_sort(const int64_t* d_init, int a1, int64_t* d_sorted, cudaStream_t st);

// all G chunks, one CTA each, writing cells [a1, n) of p.out
cudaError_t chunk_rank_launch(const ChunkRankParams& p, int threads, size_t smem, cudaStream_t st);

}  // namespace pipedp_rank

// sdp_cluster.hpp -- host interface of the thread-block-cluster S-DP pipeline
// (sdp_cluster.cu): one instance, associative (x) on 32-bit values, the far
// offsets folded by producer CTAs of the same cluster from their own copies of
// the table's recent past, pushed to them through distributed shared memory.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pipedp_cluster {

struct ClusterPlan {
  int op;          // pipedp_dev::Op (min, max, mod-add: 32-bit value class)
  int cluster;     // CTAs in the cluster (finisher + producers)
  int64_t n;
  int32_t k, a1;
  int32_t a_p;     // offsets >= a_p: producers
  int32_t j_p;     // offsets [0, j_p) are >= a_p
  int32_t j_64;    // offsets [0, j_64) are >= 64
  int32_t j_96;    // offsets [0, j_96) are >= 96
  int32_t fin_r;   // finisher ring (cells, mirrored), power of two
  int32_t prod_r;  // producer ring (cells, mirrored), >= a1 + 96
  int32_t mid_warps, prod_warps, writers;
  int32_t max_prod_offs;  // largest producer share (offsets)
  size_t fin_smem, prod_smem, smem;
};

// Shape for this instance, or false when cluster mode does not apply (ring
// too large for shared memory, too few offsets, no cluster support).
bool plan(const int64_t* offsets, int32_t k, int32_t a1, int64_t n, int op, int device, ClusterPlan* p);

// one cluster solves the instance: out[0, n) (int64), init as int64 [a1]
cudaError_t launch(const ClusterPlan& p, const int64_t* d_offsets, const int64_t* d_init, int64_t* d_out,
                   cudaStream_t st);

#ifdef PIPEDP_PROFILE
cudaError_t profile_take(unsigned long long* out128, bool reset);
#endif

}  // namespace pipedp_cluster

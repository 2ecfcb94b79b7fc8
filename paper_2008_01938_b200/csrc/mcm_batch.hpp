// mcm_batch.hpp -- batched small-n MCM, one warp per instance, packed keys
// (mcm_batch.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pipedp_mcmb {

constexpr int kMaxN = 64;

// n <= kMaxN, every weight p[i] p[k] p[j] < 2^24 (host-checked); overflow bit 2
// set when a cell reaches 2^24 (the host then reruns unpacked)
cudaError_t launch(int32_t n, int64_t batch, const int64_t* d_dims, int64_t* d_cells, int64_t* d_split,
                   int* d_overflow, cudaStream_t st);

}  // namespace pipedp_mcmb

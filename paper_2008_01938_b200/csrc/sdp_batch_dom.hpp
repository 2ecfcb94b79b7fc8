// sdp_batch_dom.hpp -- host interface of the batched S-DP dominance kernel
// (sdp_batch_dom.cu): min / max instances with 64 <= a_1 <= 128 whose offset
// closure covers [g, a_1 - 1] for some g <= 32, one warp per instance, the
// table's recent past in registers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pipedp_bdom {

// Per-instance classification (device-computed): g, F, h, D as in
// sdp_batch_dom.cu; g == 0 means the instance does not qualify.
struct DomInfo {
  uint32_t g, F, h, D;
};

// info[b] for every instance (one thread per instance)
cudaError_t classify(int64_t batch, int32_t k, int32_t a1, const int64_t* d_offsets, DomInfo* d_info,
                     cudaStream_t st);

// the instances perm[0, count) (indices into the batch), op 0 min / 1 max
cudaError_t launch(int op, int64_t count, const int32_t* d_perm, int64_t n, int32_t k, int32_t a1,
                   const int64_t* d_offsets, const int64_t* d_init, int64_t* d_out, const DomInfo* d_info,
                   cudaStream_t st);

}  // namespace pipedp_bdom

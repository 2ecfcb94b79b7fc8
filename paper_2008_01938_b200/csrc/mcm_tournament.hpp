// mcm_tournament.hpp -- the diagonal-parallel tournament comparison kernel
// (mcm_tournament.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pipedp_tour {

// cells / split: cell_count(n) + 1 entries (reference layout); d_bar: two
// zeroed-or-not words of scratch for the grid barrier (reset here)
cudaError_t launch(int64_t n, const int64_t* d_dims, int64_t* d_cells, int64_t* d_split, unsigned* d_bar,
                   cudaStream_t st);

}  // namespace pipedp_tour

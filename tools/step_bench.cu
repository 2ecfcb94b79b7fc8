// step_bench.cu -- microbenchmark of the per-step cost of a CTA-wide wavefront
// step (256 threads, __syncthreads per step), to attribute the tiled MCM
// near-phase time.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_bench tools/step_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void take(uint32_t& bv, uint32_t& bk, uint32_t v, uint32_t k) {
  if (v < bv || (v == bv && k < bk)) { bv = v; bk = k; }
}

template <int MODE>
__global__ void steps(uint32_t* out, long long* cyc, int nsteps) {
  __shared__ uint32_t X[64 * 68];
  for (int i = threadIdx.x; i < 64 * 68; i += 256) X[i] = i * 7 + 1;
  __syncthreads();
  const int tid = threadIdx.x;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int s = 0; s < nsteps; ++s) {
    if (MODE >= 1) {  // runtime G, division
      const int count = 64 - abs(s % 127 - 63);
      int G = 1;
      while (G < 32 && count * G * 2 <= 256) G <<= 1;
      const int ci = tid / G, q = tid % G;
      uint32_t bv = X[(ci * 68 + q) % (64 * 68)], bk = q;
      if (MODE >= 2) {  // reduction over G lanes
        for (int sh = 1; sh < G; sh <<= 1) {
          const uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, sh);
          const uint32_t ok = __shfl_xor_sync(0xffffffffu, bk, sh);
          take(bv, bk, ov, ok);
        }
      }
      if (q == 0 && ci < count) X[(ci * 68 + s) % (64 * 68)] = bv + bk;
      acc += bv;
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (tid == 0) *cyc = (t1 - t0) / nsteps;
  out[tid] = acc;
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 8);
  for (int grid : {1, 148}) {
    long long h;
    steps<0><<<grid, 256>>>(out, cyc, 1270); steps<0><<<grid, 256>>>(out, cyc, 1270);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("grid %d sync only: %lld cyc/step\n", grid, h);
    steps<1><<<grid, 256>>>(out, cyc, 1270); steps<1><<<grid, 256>>>(out, cyc, 1270);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("grid %d + runtime G/div: %lld cyc/step\n", grid, h);
    steps<2><<<grid, 256>>>(out, cyc, 1270); steps<2><<<grid, 256>>>(out, cyc, 1270);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("grid %d + reduce: %lld cyc/step\n", grid, h);
  }
  return 0;
}

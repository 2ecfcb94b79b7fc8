// near_bench.cu -- the tiled MCM near-phase wavefront in isolation (one CTA,
// fake tile data), cycles per step; variants bisect the per-step cost.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2008_01938_b200/csrc -o tools/near_bench tools/near_bench.cu
#include <cstdio>
#include "mcm_tiled.cuh"
using namespace pipedp_dev;

template <int MODE>
__global__ void __launch_bounds__(kTiledThreads, 2) near_bench(long long* cyc, uint32_t* sink) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const TiledSmem sm = tiled_smem(smem_raw);
  const int tid = threadIdx.x;
  for (int e = tid; e < kT * kXP; e += kTiledThreads) {
    sm.A[e] = e * 3 + 1; sm.B[e] = e * 5 + 2; sm.X[e] = e * 7 + 3; sm.KX[e] = e;
  }
  int32_t* pr = sm.P; int32_t* pc = sm.P + (kT + 4); int32_t* pkI = sm.P + 2 * (kT + 4); int32_t* pkJ = sm.P + 3 * (kT + 4);
  if (tid < kT) { pr[tid] = tid + 1; pc[tid] = tid + 2; pkI[tid] = tid + 3; pkJ[tid] = tid + 4; }
  __syncthreads();
  const uint32_t kI = 1, kJ = 65;
  const long long t0 = clock64();
  for (int s = 0; s <= 2 * (kT - 1); ++s) {
    const int ulo = s > kT - 1 ? s - (kT - 1) : 0;
    const int uhi = s < kT - 1 ? s : kT - 1;
    const int lg = step_lanes_log2(uhi - ulo + 1, s), G = 1 << lg;
    const int ci = tid >> lg, q = tid & (G - 1);
    const int ul = ulo + ci;
    const bool live = ul <= uhi;
    TBest b{0xFFFFFFFFu, 0xFFFFFFFFu};
    int rl = 0;
    if (live) {
      rl = (kT - 1) - s + ul;
      if (MODE >= 1) {
        const uint32_t prc = (uint32_t)pr[rl] * (uint32_t)pc[ul];
        const uint32_t* ar = sm.A + rl * kXP;
        const uint32_t* xc = sm.X + kXP + ul;
        const uint32_t* xr = sm.X + rl * kXP;
        const uint32_t* bc = sm.B + kXP + ul;
        if (MODE <= 2) {
          b = fold_terms(rl + q, kT - 1, G, kI, [&](int kl) { return ar[kl] + xc[kl * kXP] + prc * (uint32_t)pkI[kl]; });
          const TBest b2 = fold_terms(q, ul, G, kJ, [&](int kl) { return xr[kl] + bc[kl * kXP] + prc * (uint32_t)pkJ[kl]; });
          tb_take(b, b2.v, b2.k);
        } else if (MODE == 3) {  // row loads only
          b = fold_terms(rl + q, kT - 1, G, kI, [&](int kl) { return ar[kl] + prc * (uint32_t)kl; });
          const TBest b2 = fold_terms(q, ul, G, kJ, [&](int kl) { return xr[kl] + prc * (uint32_t)kl; });
          tb_take(b, b2.v, b2.k);
        } else if (MODE == 4) {  // column loads only
          b = fold_terms(rl + q, kT - 1, G, kI, [&](int kl) { return xc[kl * kXP] + prc * (uint32_t)kl; });
          const TBest b2 = fold_terms(q, ul, G, kJ, [&](int kl) { return bc[kl * kXP] + prc * (uint32_t)kl; });
          tb_take(b, b2.v, b2.k);
        } else {  // no loads
          b = fold_terms(rl + q, kT - 1, G, kI, [&](int kl) { return prc * (uint32_t)kl + (uint32_t)ul; });
          const TBest b2 = fold_terms(q, ul, G, kJ, [&](int kl) { return prc * (uint32_t)kl + (uint32_t)rl; });
          tb_take(b, b2.v, b2.k);
        }
      }
    }
    if (MODE == 2) b = tb_reduce(b, lg);
    if (live && q == 0) {
      TBest cur{sm.X[rl * kXP + ul], sm.KX[rl * kXP + ul]};
      tb_take(cur, b.v, b.k);
      sm.X[rl * kXP + ul] = cur.v;
      sm.KX[rl * kXP + ul] = cur.k;
    }
    __syncthreads();
    if (tid == 0) cyc[2 + s] = clock64() - t0;
    if (tid == 0 && (s == 15 || s == 126)) cyc[s == 15 ? 0 : 1] = clock64() - t0;
  }
  sink[tid] = sm.X[tid];
}

int main() {
  long long* cyc; uint32_t* sink; cudaMalloc(&cyc, 8 * 160); cudaMalloc(&sink, 4096);
  long long h[160];
  auto run = [&](auto kern, const char* nm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTiledSmemBytes);
    kern<<<1, kTiledThreads, kTiledSmemBytes>>>(cyc, sink); kern<<<1, kTiledThreads, kTiledSmemBytes>>>(cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8 * 160, cudaMemcpyDeviceToHost);
    printf("%-28s %s first16 %lld  all127 %lld cyc (%.0f/step)\n   per-step:", nm, cudaGetErrorString(e), h[0], h[1], h[1] / 127.0);
    for (int s = 0; s < 127; s += 8) printf(" %d:%lld", s, h[2 + s] - (s ? h[1 + s] : 0));
    printf("\n");
  };
  run(near_bench<0>, "steps+write only");
  run(near_bench<1>, "+terms");
  run(near_bench<2>, "+reduce (full)");
  run(near_bench<3>, "row loads only");
  run(near_bench<4>, "column loads only");
  run(near_bench<5>, "no loads");
  return 0;
}

// near_pull_test.cu -- standalone check of the pull-mode in-tile pipeline
// (tiled_near_pull) against a host wavefront over the same shared tiles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2008_01938_b200/csrc -o /tmp/npt tools/near_pull_test.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "mcm_tiled.cuh"
using namespace pipedp_dev;

template <int T>
__global__ void run_pull(const uint32_t* gA, const uint32_t* gB, const uint32_t* gX, const int32_t* gP,
                         uint32_t* oX, uint32_t* oK, long long* cyc) {
  extern __shared__ __align__(128) unsigned char raw[];
  constexpr int XP = T + 4;
  auto body = [&](auto sm) {
    for (int e = threadIdx.x; e < T * XP; e += blockDim.x) {
      sm.A[e] = gA[e];
      sm.B[e] = gB[e];
      sm.X[e] = gX[e];
      sm.KX[e] = 1500;  // far/k0 k of the starting value
    }
    for (int e = threadIdx.x; e < 4 * (T + 4); e += blockDim.x) sm.P[e] = gP[e];
    __syncthreads();
    const long long t0 = clock64();
    if constexpr (T == 32)
      t32::tiled_near_pull(sm, sm.P, sm.P + (T + 4), sm.P + 2 * (T + 4), sm.P + 3 * (T + 4));
    else
      t64::tiled_near_pull(sm, sm.P, sm.P + (T + 4), sm.P + 2 * (T + 4), sm.P + 3 * (T + 4));
    __syncthreads();
    if (threadIdx.x == 0) *cyc = clock64() - t0;
    if constexpr (T == 32)
      t32::tiled_near_split(sm, sm.P, sm.P + (T + 4), sm.P + 2 * (T + 4), sm.P + 3 * (T + 4), 1000, 2000);
    else
      t64::tiled_near_split(sm, sm.P, sm.P + (T + 4), sm.P + 2 * (T + 4), sm.P + 3 * (T + 4), 1000, 2000);
    __syncthreads();
    for (int e = threadIdx.x; e < T * XP; e += blockDim.x) {
      oX[e] = sm.X[e];
      oK[e] = sm.KX[e];
    }
  };
  if constexpr (T == 32) body(t32::tiled_smem(raw));
  else body(t64::tiled_smem(raw));
}

template <int T>
int check(bool ties) {
  constexpr int XP = T + 4;
  std::vector<uint32_t> A(T * XP), B(T * XP), X(T * XP), oX(T * XP), oK(T * XP);
  std::vector<int32_t> P(4 * (T + 4));
  srand(T);
  const int m = ties ? 3 : 100000;
  for (auto& v : A) v = rand() % m;
  for (auto& v : B) v = rand() % m;
  for (auto& v : X) v = (ties ? 6 : 200000) + rand() % m;
  for (auto& v : P) v = ties ? 1 : 1 + rand() % 30;
  uint32_t *dA, *dB, *dX, *oXd, *oKd;
  int32_t* dP;
  long long* dc;
  const size_t bytes = sizeof(uint32_t) * T * XP;
  cudaMalloc(&dA, bytes); cudaMalloc(&dB, bytes); cudaMalloc(&dX, bytes);
  cudaMalloc(&oXd, bytes); cudaMalloc(&oKd, bytes); cudaMalloc(&dP, sizeof(int32_t) * P.size()); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), sizeof(int32_t) * P.size(), cudaMemcpyHostToDevice);
  const size_t smem = T == 32 ? t32::kTiledSmemBytes : t64::kTiledSmemBytes;
  cudaFuncSetAttribute(run_pull<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  run_pull<T><<<1, kTiledThreads, smem>>>(dA, dB, dX, dP, oXd, oKd, dc);
  cudaError_t e = cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(oX.data(), oXd, bytes, cudaMemcpyDeviceToHost);
  cudaMemcpy(oK.data(), oKd, bytes, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  // host wavefront: cell (rl, ul) at step T-1-rl+ul
  const int32_t *pr = P.data(), *pc = pr + (T + 4), *pkI = pr + 2 * (T + 4), *pkJ = pr + 3 * (T + 4);
  std::vector<uint32_t> hX = X, hK(T * XP, 1500);
  for (int s = 0; s <= 2 * (T - 1); ++s)
    for (int ul = 0; ul < T; ++ul) {
      const int rl = T - 1 - s + ul;
      if (rl < 0 || rl >= T) continue;
      uint32_t bv = hX[rl * XP + ul], bk = 1500;
      const uint32_t prc = (uint32_t)pr[rl] * (uint32_t)pc[ul];
      auto take = [&](uint32_t v, uint32_t k) { if (v < bv || (v == bv && k < bk)) { bv = v; bk = k; } };
      for (int kl = rl; kl <= T - 2; ++kl) take(A[rl * XP + kl] + hX[(kl + 1) * XP + ul] + prc * (uint32_t)pkI[kl], 1000 + kl);
      for (int kl = 0; kl < ul; ++kl) take(hX[rl * XP + kl] + B[(kl + 1) * XP + ul] + prc * (uint32_t)pkJ[kl], 2000 + kl);
      hX[rl * XP + ul] = bv;
      hK[rl * XP + ul] = bk;
    }
  int bad = 0;
  for (int rl = 0; rl < T; ++rl)
    for (int ul = 0; ul < T; ++ul)
      if (hX[rl * XP + ul] != oX[rl * XP + ul] || hK[rl * XP + ul] != oK[rl * XP + ul]) {
        if (bad < 5) printf("  T=%d (%d,%d): got %u/%u want %u/%u\n", T, rl, ul, oX[rl * XP + ul], oK[rl * XP + ul], hX[rl * XP + ul], hK[rl * XP + ul]);
        ++bad;
      }
  printf("T=%d ties=%d %s mismatches=%d cycles=%lld\n", T, (int)ties, cudaGetErrorString(e), bad, cyc);
  return bad;
}

int main() {
  check<32>(false);
  check<64>(false);
  check<32>(true);
  check<64>(true);
  return 0;
}

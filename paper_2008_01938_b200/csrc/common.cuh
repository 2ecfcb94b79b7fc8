// common.cuh -- device-side building blocks shared by the S-DP and MCM kernels
// (sm_100a only).
//
//  * the semigroup catalog of the reference (semigroup.cpp:12-40) as
//    branch-free device functors, in a 64-bit form that is bit-identical to the
//    reference on every input and a 32-bit form used only when the host has
//    proven that every table value fits (see capi.cu: value-width planning);
//  * acquire/release loads and stores for the cross-warp / cross-CTA flags that
//    sequence the pipelines;
//  * warp helpers.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pipedp_dev {

enum Op : int { kMin = 0, kMax = 1, kSatAdd = 2, kModAdd = 3 };

constexpr int64_t kModulus = 2147483647;  // 2^31 - 1 (semigroup.hpp:15)

// x mod (2^31-1) for x < 2^64 by Mersenne folding.
__device__ __forceinline__ uint64_t mersenne_reduce(uint64_t u) {
  uint64_t x = (u & 0x7FFFFFFFull) + (u >> 31);  // < 2^34
  x = (x & 0x7FFFFFFFull) + (x >> 31);           // <= 2^31 + 6
  return x >= 0x7FFFFFFFull ? x - 0x7FFFFFFFull : x;
}

// normalize_mod (semigroup.cpp:21-24): the mathematical residue in [0, M).
__device__ __forceinline__ int64_t norm_mod64(int64_t a) {
  if (a >= 0) return (int64_t)mersenne_reduce((uint64_t)a);
  const uint64_t mag = (uint64_t)(-(a + 1)) + 1ull;  // |a|, exact for INT64_MIN
  const uint64_t r = mersenne_reduce(mag);
  return r == 0 ? 0 : kModulus - (int64_t)r;
}

template <int OP, typename T>
struct SemiOp;

// ---- 64-bit: the reference's exact semantics ------------------------------
template <>
struct SemiOp<kMin, int64_t> {
  __device__ __forceinline__ static int64_t apply(int64_t a, int64_t b) { return a < b ? a : b; }
};
template <>
struct SemiOp<kMax, int64_t> {
  __device__ __forceinline__ static int64_t apply(int64_t a, int64_t b) { return a > b ? a : b; }
};
template <>
struct SemiOp<kSatAdd, int64_t> {
  // semigroup.cpp:12-19: on overflow clamp to the sign of b.
  __device__ __forceinline__ static int64_t apply(int64_t a, int64_t b) {
    const int64_t s = (int64_t)((uint64_t)a + (uint64_t)b);
    const bool ovf = ((a ^ s) & (b ^ s)) < 0;
    return ovf ? (b > 0 ? INT64_MAX : INT64_MIN) : s;
  }
};
template <>
struct SemiOp<kModAdd, int64_t> {
  // semigroup.cpp:37: (norm(a) + norm(b)) % M
  __device__ __forceinline__ static int64_t apply(int64_t a, int64_t b) {
    const int64_t s = norm_mod64(a) + norm_mod64(b);
    return s >= kModulus ? s - kModulus : s;
  }
};

// ---- 32-bit fast paths (host proves exactness before selecting them) -----
// min/max: every value is a copy of an init value, so int32 init => exact.
template <>
struct SemiOp<kMin, int32_t> {
  __device__ __forceinline__ static int32_t apply(int32_t a, int32_t b) { return min(a, b); }
};
template <>
struct SemiOp<kMax, int32_t> {
  __device__ __forceinline__ static int32_t apply(int32_t a, int32_t b) { return max(a, b); }
};
// mod-add: when every init value is already in [0, M) every table value is a
// residue in [0, M) and norm() is the identity, so (a + b) mod M in uint32.
template <>
struct SemiOp<kModAdd, int32_t> {
  __device__ __forceinline__ static int32_t apply(int32_t a, int32_t b) {
    const uint32_t s = (uint32_t)a + (uint32_t)b;
    return (int32_t)(s >= 0x7FFFFFFFu ? s - 0x7FFFFFFFu : s);
  }
};

// Identity elements, used only where the host proved the fold associative and
// the accumulator already holds a real operand (min/max trivially; mod-add: 0
// since (norm(a) + 0) mod M = norm(a) and the accumulator is normalised once
// two operands were combined; saturating-add on same-signed values: 0).
template <int OP, typename T>
struct SemiId;
template <typename T>
struct SemiId<kMin, T> {
  __device__ __forceinline__ static T value() { return sizeof(T) == 4 ? (T)INT32_MAX : (T)INT64_MAX; }
};
template <typename T>
struct SemiId<kMax, T> {
  __device__ __forceinline__ static T value() { return sizeof(T) == 4 ? (T)INT32_MIN : (T)INT64_MIN; }
};
template <typename T>
struct SemiId<kModAdd, T> {
  __device__ __forceinline__ static T value() { return T(0); }
};
template <typename T>
struct SemiId<kSatAdd, T> {
  __device__ __forceinline__ static T value() { return T(0); }
};

// ---- memory-model helpers --------------------------------------------------
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)),
               "r"(v)
               : "memory");
}
__device__ __forceinline__ long long ld_acquire_gpu(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(long long* p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_i32(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Polling without per-iteration L1 invalidation: an ld.acquire.gpu compiles to
// LDG.STRONG.GPU + CCTL.IVALL, and a CTA spinning on it invalidates its SM's L1
// every iteration -- which stalls the LSU pipe that a co-resident CTA's shared
// memory traffic uses.  Poll with relaxed loads, then one acquire fence.
__device__ __forceinline__ int ld_relaxed_gpu_i32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_relaxed_gpu(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// spin until *p == want / >= want (acquire on exit)
__device__ __forceinline__ void spin_eq_gpu(const int* p, int want, unsigned ns) {
  while (ld_relaxed_gpu_i32(p) != want) __nanosleep(ns);
  fence_acquire_gpu();
}
__device__ __forceinline__ void spin_ge_gpu(const int* p, int want, unsigned ns) {
  while (ld_relaxed_gpu_i32(p) < want) __nanosleep(ns);
  fence_acquire_gpu();
}
__device__ __forceinline__ void spin_ge_gpu64(const long long* p, long long want, unsigned ns) {
  while (ld_relaxed_gpu(p) < want) __nanosleep(ns);
  fence_acquire_gpu();
}

// ---- mbarrier (hardware-suspended waits; no issue slots burnt polling) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// one arrival, release at CTA scope
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// wait for completion of the phase with the given parity, acquire at CTA scope
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

template <typename T>
__device__ __forceinline__ T shfl_idx(T v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}
template <typename T>
__device__ __forceinline__ T shfl_up(T v, int delta) {
  return __shfl_up_sync(0xffffffffu, v, delta);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// ---- opt-in role profiler (build with -DPIPEDP_PROFILE; compiled out otherwise)
// Slots: role * 8 + counter; accumulated in cycles by lane 0 of each warp.
#ifdef PIPEDP_PROFILE
__device__ unsigned long long g_prof[128];
#define PROF_DECL(name) long long name = 0
#define PROF_NOW() clock64()
#define PROF_ADD(acc, t0) (acc) += clock64() - (t0)
#define PROF_FLUSH(slot, v) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&::pipedp_dev::g_prof[(slot)], (unsigned long long)(v))
#else
#define PROF_DECL(name)
#define PROF_NOW() 0
#define PROF_ADD(acc, t0)
#define PROF_FLUSH(slot, v)
#endif

}  // namespace pipedp_dev

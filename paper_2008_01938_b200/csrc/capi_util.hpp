// capi_util.hpp -- shared by the C-ABI translation units (capi.cu, engine.cu):
// error reporting with the reference's errc names, validation with the
// reference's rules, device selection and a per-call stream/buffer scope.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/pipedp_cuda.h"

namespace pipedp_capi {

// ---------------------------------------------------------------- errors ---
inline thread_local std::string g_last_error;

inline const char* errc_name(int code) {  // semigroup.cpp:73-99, indexed by errc + 1
  static const char* names[] = {"",
                                "NonDecreasingOffsets",
                                "NonPositiveOffset",
                                "InitLengthMismatch",
                                "TableTooSmall",
                                "CoordOutOfRange",
                                "AddressOutOfRange",
                                "BaseCellHasNoDeps",
                                "TooLargeForBruteForce",
                                "StallLivelock",
                                "WeightOverflow",
                                "InvalidParams"};
  if (code >= 1 && code <= 11) return names[code];
  switch (code) {
    case PIPEDP_ERR_CUDA: return "CudaError";
    case PIPEDP_ERR_NO_DEVICE: return "NoDevice";
    case PIPEDP_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    case PIPEDP_ERR_UNSUPPORTED: return "Unsupported";
  }
  return "UnknownError";
}

inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = std::string(errc_name(code)) + ": " + buf;
  return code;
}

inline int cuda_fail(cudaError_t e, const char* what) {
  (void)cudaGetLastError();
  return fail(e == cudaErrorMemoryAllocation ? PIPEDP_ERR_OUT_OF_MEMORY : PIPEDP_ERR_CUDA,
              "%s: %s", what, cudaGetErrorString(e));
}

#define CK(expr)                                      \
  do {                                                \
    cudaError_t _e = (expr);                          \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

// ------------------------------------------------------------ validation ---
// sdp.cpp:10-32, in the reference's order.
inline int validate_sdp(const int64_t* offs, int64_t k, int64_t init_len, int64_t n) {
  if (k <= 0 || offs == nullptr) return fail(PIPEDP_E_INVALID_PARAMS, "offset set must be nonempty");
  for (int64_t i = 0; i < k; ++i) {
    if (offs[i] <= 0)
      return fail(PIPEDP_E_NON_POSITIVE_OFFSET, "offset a_%lld is not positive", (long long)(i + 1));
    if (i > 0 && offs[i - 1] <= offs[i])
      return fail(PIPEDP_E_NON_DECREASING_OFFSETS,
                  "offsets must strictly decrease, violated at position %lld", (long long)(i + 1));
  }
  if (init_len != offs[0])
    return fail(PIPEDP_E_INIT_LENGTH_MISMATCH, "expected a_1=%lld initial values, got %lld",
                (long long)offs[0], (long long)init_len);
  if (n <= offs[0])
    return fail(PIPEDP_E_TABLE_TOO_SMALL, "n=%lld leaves nothing to compute past the preset prefix",
                (long long)n);
  return PIPEDP_OK;
}

// mcm.cpp:11-28.  The overflow product is evaluated like the reference's
// signed left-to-right expression compiles on gcc/x86-64 (two's-complement
// wrap), so the accepted set is identical.
inline int validate_mcm(const int64_t* dims, int64_t len) {
  if (len < 2 || dims == nullptr)
    return fail(PIPEDP_E_INVALID_PARAMS, "dimension vector needs at least two entries");
  int64_t max_dim = 1;
  for (int64_t i = 0; i < len; ++i) {
    if (dims[i] < 1) return fail(PIPEDP_E_INVALID_PARAMS, "matrix dimensions must be >= 1");
    max_dim = std::max(max_dim, dims[i]);
  }
  const int64_t n = len - 1;
  uint64_t p = (uint64_t)n * (uint64_t)max_dim;
  p *= (uint64_t)max_dim;
  p *= (uint64_t)max_dim;
  if (max_dim > 1000000 || (int64_t)p > ((int64_t)1 << 61))
    return fail(PIPEDP_E_WEIGHT_OVERFLOW, "dimension products too large for 64-bit cost accumulation");
  return PIPEDP_OK;
}

// ------------------------------------------------------------- devices ---
inline int usable_devices() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  int usable = 0;
  for (int d = 0; d < count; ++d) {
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10) ++usable;
  }
  return usable;
}

inline int select_device(int32_t device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    (void)cudaGetLastError();
    return fail(PIPEDP_ERR_NO_DEVICE, "no CUDA device visible (the solvers have no CPU path)");
  }
  int dev = device;
  if (dev < 0) CK(cudaGetDevice(&dev));
  if (dev >= count) return fail(PIPEDP_ERR_NO_DEVICE, "device %d not present (%d visible)", dev, count);
  int major = 0, minor = 0;  // attribute queries: cudaGetDeviceProperties costs milliseconds
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10)
    return fail(PIPEDP_ERR_NO_DEVICE, "device %d is sm_%d%d; these kernels are built for sm_100a", dev,
                major, minor);
  CK(cudaSetDevice(dev));
  return PIPEDP_OK;
}

// A per-call stream and a tiny RAII set of device buffers.
struct Scope {
  cudaStream_t stream = nullptr;
  std::vector<void*> bufs;
  ~Scope() {
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : bufs) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
  }
  int init() {
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    return PIPEDP_OK;
  }
  template <typename T>
  int alloc(T** p, size_t count) {
    void* q = nullptr;
    CK(cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T)));
    bufs.push_back(q);
    *p = static_cast<T*>(q);
    return PIPEDP_OK;
  }
};

#define TRY(expr)                  \
  do {                             \
    int _rc = (expr);              \
    if (_rc != PIPEDP_OK) return _rc; \
  } while (0)

}  // namespace pipedp_capi

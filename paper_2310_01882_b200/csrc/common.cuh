// common.cuh — shared plumbing of libstencil (error state, launch accounting,
// device load/store helpers). Part of the product; shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "libstencil.h"

namespace st {

// ---------------------------------------------------------------- errors ---
void set_error(const char* fmt, ...);
void clear_error();
const char* g_err_ptr();
std::atomic<uint64_t>& launch_counter();

#define ST_CHECK_CUDA(expr)                                                       \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      ::st::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,               \
                      cudaGetErrorString(e_));                                    \
      return ST_ECUDA;                                                            \
    }                                                                             \
  } while (0)

// After a <<<>>> launch: account for it and surface configuration errors.
#define ST_LAUNCHED()                                                             \
  do {                                                                            \
    ::st::launch_counter().fetch_add(1, std::memory_order_relaxed);               \
    cudaError_t e_ = cudaGetLastError();                                          \
    if (e_ != cudaSuccess) {                                                      \
      ::st::set_error("%s:%d: kernel launch -> %s", __FILE__, __LINE__,           \
                      cudaGetErrorString(e_));                                    \
      return ST_ECUDA;                                                            \
    }                                                                             \
  } while (0)

#define ST_RETURN_IF(cond, code, ...)                                             \
  do {                                                                            \
    if (cond) {                                                                   \
      ::st::set_error(__VA_ARGS__);                                               \
      return code;                                                                \
    }                                                                             \
  } while (0)

#define ST_TRY(expr)                                                              \
  do {                                                                            \
    st_status s_ = (expr);                                                        \
    if (s_ != ST_OK) return s_;                                                   \
  } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline bool overlaps(const void* a, size_t abytes, const void* b, size_t bbytes) {
  auto pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
  return pa < pb + bbytes && pb < pa + abytes;
}

inline int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// --------------------------------------------------------- device helpers ---
// Exact binary64 ops, one rounding each, never contracted into FMA (R11).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Streaming 16-byte load through the non-coherent path (inputs are read-only for
// the duration of a kernel).
__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double ldg1(const double* p) { return __ldg(p); }

__device__ __forceinline__ void stg2(double* p, double2 v) {
  *reinterpret_cast<double2*>(p) = v;
}

}  // namespace st

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

// Correctly rounded x / 6.0 (== __ddiv_rn(x, 6.0), the oracle's `sum / 6.0`) in
// 1 DMUL + 2 DFMA instead of the ~25-instruction generic division:
//   q0 = RN(x * RN(1/6)); r = x - 6*q0 (exact: FMA residual of a faithful
//   quotient); q = RN(q0 + r * RN(1/6)).
// Why it is correctly rounded: x/6 = (x/2)/3 and a 53-bit significand divided
// by 3 is never a rounding midpoint and stays >= ulp/6 away from every
// midpoint, while q0 + r*RN(1/6) differs from x/6 by |r| * |RN(1/6) - 1/6| <=
// 2^-52 ulp. Outside 2^-999 <= |x| < 2^1000 (subnormal results, overflow of
// the residual) and for zero and non-finite x the generic division is used;
// the range test reads the biased exponent (integer ops, not two fp64 compares).
// tests/test_gpu_jacobi3d.py checks it bitwise against __ddiv_rn on random x.
__device__ __forceinline__ double ddiv6(double x) {
  const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;  // 2^-999: 24, 2^1000: 2023
  if (e - 24u > 1998u) return __ddiv_rn(x, 6.0);
  constexpr double kInv6 = 0.16666666666666666;  // RN(1/6) = 0x3FC5555555555555
  const double q0 = __dmul_rn(x, kInv6);
  const double r = __fma_rn(-6.0, q0, x);
  return __fma_rn(r, kInv6, q0);
}

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

// stencil2d.cu — generic linear 2-D stencil.apply executor (reading R23 of
// DESIGN.md; NEXT #4, second half), sm_100a.
//
// The stencil dialect's apply on the offsets the discovery
// pass extracts from a Fortran loop nest, for linear
// right-hand sides:
//     out(y,x) = c_0*a(y+dy_0, x+dx_0) + c_1*a(y+dy_1, x+dx_1) + ...
// evaluated left to right as written, one rounding per product and per sum
// (never contracted). Value semantics (Jacobi ping-pong); the R-wide ring
// (R = max |offset|) is a fixed Dirichlet boundary.
//
// The terms travel by value in the kernel parameters (no device allocation,
// no runtime compilation). HBM-bound like the Listing-1 sweep (16 B per point
// per sweep): a CTA covers 32 columns x 32 rows, a thread 4 rows of one column
// (term-major, so each term's parameters are read once per 4 points), the n
// reads of a point are L1 hits except the tile's halo, and each warp row access
// is a coalesced 256-byte segment.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "common.cuh"
#include "internal.h"

#ifndef ST_STENCIL_RPT
#define ST_STENCIL_RPT 4
#endif
#ifndef ST_STENCIL_TU
#define ST_STENCIL_TU 4
#endif
#ifndef ST_STENCIL_SX
#define ST_STENCIL_SX 64
#endif
#ifndef ST_STENCIL_SY
#define ST_STENCIL_SY 2
#endif

namespace st {

namespace {

struct Terms {
  int32_t n;
  int32_t dy[kStencilMaxTerms];
  int32_t dx[kStencilMaxTerms];
  double c[kStencilMaxTerms];
};

constexpr int kSx = ST_STENCIL_SX, kSy = ST_STENCIL_SY, kRowsPerThread = ST_STENCIL_RPT, kTermUnroll = ST_STENCIL_TU;

__global__ void __launch_bounds__(kSx * kSy)
    stencil2d_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nx, int64_t ny, int64_t ld,
                     int64_t R, const __grid_constant__ Terms t) {
  const int64_t x = R + (int64_t)blockIdx.x * kSx + threadIdx.x;
  if (x >= R + nx) return;
  const int64_t y_base = R + (int64_t)blockIdx.y * (kSy * kRowsPerThread) + threadIdx.y;
  // term-major: each term's offset and coefficient are read once for the thread's
  // rows, which are independent (4-way ILP); per point the terms still combine in
  // the written order
  const double* p[kRowsPerThread];
#pragma unroll
  for (int k = 0; k < kRowsPerThread; ++k) {
    const int64_t y = y_base + k * kSy;
    p[k] = src + (y < R + ny ? y : y_base) * ld + x;  // rows past the grid read (and discard) row y_base
  }
  double acc[kRowsPerThread];
  {
    const int64_t o = (int64_t)t.dy[0] * ld + t.dx[0];
    const double c = t.c[0];
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) acc[k] = dmul(c, __ldg(p[k] + o));
  }
#pragma unroll kTermUnroll
  for (int i = 1; i < t.n; ++i) {
    const int64_t o = (int64_t)t.dy[i] * ld + t.dx[i];
    const double c = t.c[i];
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) acc[k] = dadd(acc[k], dmul(c, __ldg(p[k] + o)));
  }
#pragma unroll
  for (int k = 0; k < kRowsPerThread; ++k) {
    const int64_t y = y_base + k * kSy;
    if (y < R + ny) dst[y * ld + x] = acc[k];
  }
}

}  // namespace

st_status stencil2d_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, stencil2d_kernel));
  return ST_OK;
}

st_status stencil2d_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t R, const int32_t* off,
                        const double* coeffs, int32_t n, int64_t iters, cudaStream_t s) {
  // 16-byte rows: specialise the stencil for its offsets — the terms written as the
  // expression "(c0)*a(dy0,dx0) + (c1)*a(dy1,dx1) + ..." (left to right, one rounding per
  // product and per sum: the same arithmetic as the kernel below; %.17g literals round-trip
  // exactly) go through the NVRTC column-pair generator (§6.8 of DESIGN.md), whose register
  // queues and neighbour shuffles the runtime-term kernel cannot have. Without NVRTC, or with
  // a non-finite coefficient, the runtime-term kernel below runs.
  static const int kJit = env_int("ST_STENCIL_JIT", 1);
  const bool aligned16 = ld % 2 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(b) & 15) == 0;
  if (kJit && aligned16) {
    std::string e;
    bool finite = true;
    for (int i = 0; i < n; ++i) {
      char buf[96];
      finite = finite && std::isfinite(coeffs[i]);
      std::snprintf(buf, sizeof buf, "%s(%.17g)*a(%d,%d)", i ? " + " : "", coeffs[i], off[2 * i], off[2 * i + 1]);
      e += buf;
    }
    std::string cexpr;
    int64_t re = -1;
    int dims = 0;
    if (finite && stencil_expr_translate(e.c_str(), &cexpr, &re, &dims) == ST_OK && re == R && dims == 2) {
      const st_status r = stencil2d_expr_run(a, b, nx, ny, ld, R, cexpr, iters, s);
      if (r != ST_ENOTSUP) return r;  // ST_ENOTSUP: no NVRTC here — the runtime-term kernel instead
      clear_error();
    }
  }
  Terms t{};
  t.n = n;
  for (int i = 0; i < n; ++i) {
    t.dy[i] = off[2 * i];
    t.dx[i] = off[2 * i + 1];
    t.c[i] = coeffs[i];
  }
  // b := copy(a): both buffers carry the ring (value semantics keeps it fixed)
  ST_CHECK_CUDA(cudaMemcpyAsync(b, a, (size_t)(ny + 2 * R) * (size_t)ld * sizeof(double), cudaMemcpyDeviceToDevice, s));
  const dim3 block(kSx, kSy);
  const int64_t gy = (ny + kSy * kRowsPerThread - 1) / (kSy * kRowsPerThread);
  ST_RETURN_IF(gy > 65535, ST_ENOTSUP, "stencil2d: ny = %lld too large for the grid", (long long)ny);
  const dim3 grid((unsigned)((nx + kSx - 1) / kSx), (unsigned)gy);
  const double* src = a;
  double* dst = b;
  for (int64_t it = 0; it < iters; ++it) {
    stencil2d_kernel<<<grid, block, 0, s>>>(src, dst, nx, ny, ld, R, t);
    ST_LAUNCHED();
    const double* nsrc = dst;
    dst = const_cast<double*>(src);
    src = nsrc;
  }
  return ST_OK;
}

}  // namespace st

// jacobi2d.cu — sm_100a kernels for the 2-D Jacobi 5-point sweep.
//
// Operation (Listing 1, under stencil.apply value semantics,
// PAPER.md:126; association order = DESIGN.md R2):
//     dst[y][x] = (((src[y-1][x] + src[y+1][x]) + src[y][x-1]) + src[y][x+1]) * 0.25
//
// The sweep is HBM-bound (4 flop per 16 algorithmic bytes), so the kernels are
// organised around moving each grid value through HBM exactly once per pass:
//
//  * jacobi2d_stream_kernel (T=1): a warp owns a 64-column strip (lane = one
//    16-byte aligned column pair) and streams down a chunk of rows with a
//    3-row register queue (N, C, S) and a U-row software prefetch; the W/E
//    neighbours come from warp shuffles of the adjacent lanes' pairs, the two
//    strip-edge lanes load one extra double. Ring columns are passed through
//    (dst = src) so stores stay 16 bytes wide and the ring stays bit-identical.
//  * jacobi2d_resident_kernel: grids whose two buffers fit in one SM's shared
//    memory (C1, 66x66) run all sweeps inside a single CTA — the C1 case is
//    launch-bound, not HBM-bound.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace st {

namespace {

constexpr int kStreamThreads = 256;
constexpr int kStreamWarps = kStreamThreads / 32;
constexpr int kStripCols = 64;  // doubles per warp strip (32 lanes x 2)

struct RowLoad {
  double2 p;  // the lane's column pair
  double e;   // lane 0: column x-1; lane 31: column x+2 (strip edges)
};

template <int U>
__global__ void __launch_bounds__(kStreamThreads)
    jacobi2d_stream_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nxp2,
                           int64_t ld, int64_t y_lo, int64_t y_hi, int64_t rows_per_chunk,
                           int64_t nstrips) {
  const int lane = threadIdx.x & 31;
  const int64_t strip = (int64_t)blockIdx.x * kStreamWarps + (threadIdx.x >> 5);
  if (strip >= nstrips) return;  // warp-uniform
  const int64_t yc0 = y_lo + (int64_t)blockIdx.y * rows_per_chunk;
  if (yc0 > y_hi) return;  // block-uniform
  const int64_t yc1 = min(y_hi, yc0 + rows_per_chunk - 1);

  const int64_t x = strip * kStripCols + 2 * lane;
  const bool has_pair = x < nxp2;
  const bool has_hi = x + 1 < nxp2;
  const int64_t ext_x = (lane == 0) ? x - 1 : x + 2;
  const bool has_ext = (lane == 0 && x >= 1) || (lane == 31 && x + 2 < nxp2);
  const double* sp = src + x;
  const double* se = src + ext_x;

  auto load = [&](int64_t y) {
    RowLoad r;
    r.p = has_pair ? ldg2(sp + y * ld) : make_double2(0.0, 0.0);
    r.e = has_ext ? ldg1(se + y * ld) : 0.0;
    return r;
  };

  RowLoad qn = load(yc0 - 1);
  RowLoad qc = load(yc0);
  RowLoad pf[U];
#pragma unroll
  for (int k = 0; k < U; ++k)
    if (yc0 + 1 + k <= yc1 + 1) pf[k] = load(yc0 + 1 + k);

  for (int64_t y = yc0; y <= yc1; y += U) {
    RowLoad nx_[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (y + U + 1 + k <= yc1 + 1) nx_[k] = load(y + U + 1 + k);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (y + k <= yc1) {
        const double2 n = qn.p, c = qc.p, s = pf[k].p;
        double w = __shfl_up_sync(0xffffffffu, c.y, 1);
        double e = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (lane == 0) w = qc.e;
        if (lane == 31) e = qc.e;
        double2 o;
        o.x = dmul(dadd(dadd(dadd(n.x, s.x), w), c.y), 0.25);
        o.y = dmul(dadd(dadd(dadd(n.y, s.y), c.x), e), 0.25);
        if (x == 0 || x == nxp2 - 1) o.x = c.x;  // Dirichlet ring columns pass through
        if (x + 1 == nxp2 - 1) o.y = c.y;
        double* dp = dst + (y + k) * ld + x;
        if (has_hi) stg2(dp, o);
        else if (has_pair) *dp = o.x;
        qn = qc;
        qc = pf[k];
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) pf[k] = nx_[k];
  }
}

// All sweeps inside one CTA: both buffers live in shared memory, compact pitch nxp2.
__global__ void __launch_bounds__(1024)
    jacobi2d_resident_kernel(double* __restrict__ a, double* __restrict__ b, int nxp2, int nyp2,
                             int64_t ld, int64_t iters) {
  extern __shared__ double sm[];
  const int n = nxp2 * nyp2;
  double* s0 = sm;
  double* s1 = sm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int y = i / nxp2, x = i - y * nxp2;
    const double v = a[(int64_t)y * ld + x];
    s0[i] = v;
    s1[i] = v;
  }
  __syncthreads();
  const int nx = nxp2 - 2, ny = nyp2 - 2;
  const int ni = nx * ny;
  double* cur = s0;
  double* nxt = s1;
  for (int64_t it = 0; it < iters; ++it) {
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
      const int y = 1 + i / nx, x = 1 + (i - (y - 1) * nx);
      const int c = y * nxp2 + x;
      nxt[c] = dmul(dadd(dadd(dadd(cur[c - nxp2], cur[c + nxp2]), cur[c - 1]), cur[c + 1]), 0.25);
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  double* out = (iters & 1) ? b : a;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int y = i / nxp2, x = i - y * nxp2;
    out[(int64_t)y * ld + x] = cur[i];
  }
}

constexpr size_t kResidentMaxSmem = 200 * 1024;

}  // namespace

st_status jacobi2d_sweep_rows(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo,
                              int64_t y_hi, cudaStream_t s) {
  if (y_hi < y_lo) return ST_OK;
  const int64_t nxp2 = nx + 2;
  const int64_t nstrips = (nxp2 + kStripCols - 1) / kStripCols;
  const int64_t rows = y_hi - y_lo + 1;
  static const int kRows = env_int("ST_JACOBI_ROWS", 128);
  const int64_t rpc = std::max<int64_t>(1, std::min<int64_t>(kRows, rows));
  const int64_t nchunks = (rows + rpc - 1) / rpc;
  ST_RETURN_IF(nchunks > 65535, ST_ENOTSUP, "jacobi2d: %lld row chunks exceed grid.y", (long long)nchunks);
  dim3 grid((unsigned)((nstrips + kStreamWarps - 1) / kStreamWarps), (unsigned)nchunks);
  jacobi2d_stream_kernel<4><<<grid, kStreamThreads, 0, s>>>(src, dst, nxp2, ld, y_lo, y_hi, rpc, nstrips);
  ST_LAUNCHED();
  return ST_OK;
}

bool jacobi2d_resident_fits(int64_t nx, int64_t ny) {
  const int64_t n = (nx + 2) * (ny + 2);
  return n * 2 * (int64_t)sizeof(double) <= (int64_t)kResidentMaxSmem;
}

st_status jacobi2d_resident(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t iters,
                            cudaStream_t s) {
  const size_t smem = (size_t)(nx + 2) * (size_t)(ny + 2) * 2 * sizeof(double);
  ST_CHECK_CUDA(cudaFuncSetAttribute(jacobi2d_resident_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kResidentMaxSmem));
  jacobi2d_resident_kernel<<<1, 1024, smem, s>>>(a, b, (int)(nx + 2), (int)(ny + 2), ld, iters);
  ST_LAUNCHED();
  return ST_OK;
}

namespace {

// Temporal blocking in registers (T sweeps per pass over HBM).
//
// A warp owns a strip of 64 columns (lane = column pair) that overlaps its
// neighbours by 2T columns: after T levels only the centre 64-2T columns are
// exact, so strips advance by 64-2T. Rows stream through a T-level software
// pipeline held entirely in registers: level j keeps its two most recent rows
// (N, C); when level j produces a new row S, level j+1 produces row C. W/E
// neighbours at every level come from warp shuffles. Dirichlet rows/columns are
// passed through unchanged at every level, so every level is exactly one Jacobi
// sweep and the result is bitwise the same as T single sweeps.
template <int T>
__global__ void __launch_bounds__(kStreamThreads)
    jacobi2d_tb_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nxp2, int64_t ld,
                       int64_t y_lo, int64_t y_hi, int64_t rows_per_chunk, int64_t nstrips, int64_t ring_lo,
                       int64_t ring_hi, int64_t nrows_buf) {
  static_assert(T >= 2 && T % 2 == 0 && T <= 16, "even T");
  constexpr int kStride = kStripCols - 2 * T;
  const int lane = threadIdx.x & 31;
  const int64_t strip = (int64_t)blockIdx.x * kStreamWarps + (threadIdx.x >> 5);
  if (strip >= nstrips) return;
  const int64_t yc0 = y_lo + (int64_t)blockIdx.y * rows_per_chunk;
  if (yc0 > y_hi) return;
  const int64_t yc1 = min(y_hi, yc0 + rows_per_chunk - 1);

  const int64_t x = strip * kStride - T + 2 * lane;
  const bool has_pair = x >= 0 && x < nxp2;
  const bool st_lane = lane >= T / 2 && lane <= 31 - T / 2;
  const bool st0 = st_lane && x >= 0 && x < nxp2;
  const bool st1 = st_lane && x + 1 >= 0 && x + 1 < nxp2;
  const bool ring0 = (x == 0) || (x == nxp2 - 1);
  const bool ring1 = (x + 1 == nxp2 - 1);
  const double* sp = src + (has_pair ? x : 0);

  // first/last input rows the pipeline reads; rows beyond are never loaded
  const int64_t r_first = max(max(ring_lo, (int64_t)0), yc0 - T);
  const int64_t r_load_last = min(min(ring_hi, nrows_buf - 1), yc1 + T);
  const int64_t r_end = yc1 + T;  // steps continue past ring_hi (the ring row propagates)

  double2 n_[T], c_[T];  // level j: rows r-j-2 (n_) and r-j-1 (c_) before step r
#pragma unroll
  for (int j = 0; j < T; ++j) n_[j] = c_[j] = make_double2(0.0, 0.0);

  constexpr int U = 4;
  double2 pf[U];
  auto load = [&](int64_t r) -> double2 {
    return (has_pair && r <= r_load_last) ? ldg2(sp + r * ld) : make_double2(0.0, 0.0);
  };
#pragma unroll
  for (int k = 0; k < U; ++k) pf[k] = load(r_first + k);

  for (int64_t r0 = r_first; r0 <= r_end; r0 += U) {
    double2 nx_[U];
#pragma unroll
    for (int k = 0; k < U; ++k) nx_[k] = load(r0 + U + k);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t r = r0 + k;
      if (r <= r_end) {
        double2 s = pf[k];  // level 0, row r
#pragma unroll
        for (int j = 0; j < T; ++j) {
          // level j+1, row r-j-1 from level j rows r-j-2 (n), r-j-1 (c), r-j (s)
          const int64_t row = r - j - 1;
          const double2 c = c_[j];
          double w = __shfl_up_sync(0xffffffffu, c.y, 1);
          double e = __shfl_down_sync(0xffffffffu, c.x, 1);
          double2 o;
          o.x = dmul(dadd(dadd(dadd(n_[j].x, s.x), w), c.y), 0.25);
          o.y = dmul(dadd(dadd(dadd(n_[j].y, s.y), c.x), e), 0.25);
          if (ring0) o.x = c.x;
          if (ring1) o.y = c.y;
          if (row <= ring_lo || row >= ring_hi) o = c;  // Dirichlet rows never change
          n_[j] = c;
          c_[j] = s;
          s = o;
        }
        const int64_t orow = r - T;  // s = level T, row r-T
        if (orow >= yc0 && orow <= yc1) {
          double* dp = dst + orow * ld + x;
          if (st0 && st1) stg2(dp, s);
          else if (st0) dp[0] = s.x;
          else if (st1) dp[1] = s.y;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) pf[k] = nx_[k];
  }
}

template <int T>
st_status launch_tb(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                    int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s) {
  const int64_t nxp2 = nx + 2;
  constexpr int kStride = kStripCols - 2 * T;
  const int64_t nstrips = (nxp2 + kStride - 1) / kStride;
  const int64_t rows = y_hi - y_lo + 1;
  static const int kRows = env_int("ST_JACOBI_TB_ROWS", 512);
  const int64_t rpc = std::max<int64_t>(1, std::min<int64_t>(kRows, rows));
  const int64_t nchunks = (rows + rpc - 1) / rpc;
  ST_RETURN_IF(nchunks > 65535, ST_ENOTSUP, "jacobi2d tb: too many row chunks");
  dim3 grid((unsigned)((nstrips + kStreamWarps - 1) / kStreamWarps), (unsigned)nchunks);
  jacobi2d_tb_kernel<T><<<grid, kStreamThreads, 0, s>>>(src, dst, nxp2, ld, y_lo, y_hi, rpc, nstrips, ring_lo,
                                                        ring_hi, nrows_buf);
  ST_LAUNCHED();
  return ST_OK;
}

}  // namespace

bool jacobi2d_tb_supported(int t) { return t == 2 || t == 4 || t == 6 || t == 8; }

st_status jacobi2d_tb_rows(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                           int t, int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s) {
  if (y_hi < y_lo) return ST_OK;
  switch (t) {
    case 2: return launch_tb<2>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s);
    case 4: return launch_tb<4>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s);
    case 6: return launch_tb<6>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s);
    case 8: return launch_tb<8>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s);
    default: set_error("jacobi2d: tblock=%d not supported (2, 4, 6, 8)", t); return ST_ENOTSUP;
  }
}

}  // namespace st

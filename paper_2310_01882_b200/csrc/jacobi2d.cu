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
                           int64_t nstrips, double* __restrict__ dst2, int64_t delta2) {
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
        if (dst2) {  // fused halo swap: the same row into the neighbour's ghost row
          double* dq = dst2 + (y + k + delta2) * ld + x;
          if (has_hi) stg2(dq, o);
          else if (has_pair) *dq = o.x;
        }
        qn = qc;
        qc = pf[k];
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) pf[k] = nx_[k];
  }
}

// All sweeps inside one CTA: both buffers live in shared memory, compact pitch
// nxp2. 2-D thread block (bx columns x by rows): thread (tx, ty) owns the points
// x = 1+tx+i*bx, y = 1+ty+j*by, so the sweep loop has no integer division.
__global__ void __launch_bounds__(1024)
    jacobi2d_resident_kernel(double* __restrict__ a, double* __restrict__ b, int nxp2, int nyp2,
                             int64_t ld, int64_t iters) {
  extern __shared__ double sm[];
  const int n = nxp2 * nyp2;
  double* s0 = sm;
  double* s1 = sm + n;
  for (int y = threadIdx.y; y < nyp2; y += blockDim.y)
    for (int x = threadIdx.x; x < nxp2; x += blockDim.x) {
      const double v = a[(int64_t)y * ld + x];
      s0[y * nxp2 + x] = v;
      s1[y * nxp2 + x] = v;
    }
  __syncthreads();
  const int nx = nxp2 - 2, ny = nyp2 - 2;
  double* cur = s0;
  double* nxt = s1;
  for (int64_t it = 0; it < iters; ++it) {
    // the two buffers never alias: let the compiler hoist every load of the sweep
    const double* __restrict__ src = cur;
    double* __restrict__ dst = nxt;
#pragma unroll 4
    for (int y = 1 + threadIdx.y; y <= ny; y += blockDim.y) {
      const int row = y * nxp2;
      for (int x = 1 + threadIdx.x; x <= nx; x += blockDim.x) {
        const int c = row + x;
        dst[c] = dmul(dadd(dadd(dadd(src[c - nxp2], src[c + nxp2]), src[c - 1]), src[c + 1]), 0.25);
      }
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  double* out = (iters & 1) ? b : a;
  for (int y = threadIdx.y; y < nyp2; y += blockDim.y)
    for (int x = threadIdx.x; x < nxp2; x += blockDim.x) out[(int64_t)y * ld + x] = cur[y * nxp2 + x];
}

// Register-resident variant for grids up to 64 columns (C1 = 64^2): the state
// lives in registers for all sweeps. Lane l of warp w owns columns 1+2l, 2+2l
// of rows 1+R*w .. R*(w+1); rows beyond ny+1 are idle, the ring row ny+1 (and
// ring column nx+1 when it falls inside a lane) are held but never updated.
// Per sweep: N/S inside a warp's rows come from its own registers, W/E from
// warp shuffles, and the first/last row of every warp goes through shared
// memory (double-buffered by sweep parity, so one barrier per sweep). Shared
// traffic per sweep is 2 rows per warp instead of 4 reads + 1 write per point.
constexpr int kRegResMaxWarps = 22;  // 88 rows with R = 4 (ny <= 87), 66 with R = 3

template <int R>
__global__ void __launch_bounds__(32 * kRegResMaxWarps)
    jacobi2d_regres_kernel(double* __restrict__ a, double* __restrict__ b, int nx, int ny, int64_t ld,
                           int64_t iters) {
  constexpr int kW = 64;  // columns per warp row (32 lanes x 2)
  __shared__ __align__(16) double top_row[2][kRegResMaxWarps][kW];      // first row of each warp, per sweep parity
  __shared__ __align__(16) double bot_row[2][kRegResMaxWarps + 1][kW];  // last row of each warp; [.][0] = ring row 0
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int x0 = 1 + 2 * lane;
  double v[R][2];
  double wr[R], er[R];  // ring column 0 (lane 0) and column 65 (lane 31, when nx == 64)
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int y = 1 + R * w + i;
    const bool row_ok = y <= ny + 1;
    const double* ar = a + (int64_t)(row_ok ? y : 0) * ld;
    v[i][0] = (row_ok && x0 <= nx + 1) ? ar[x0] : 0.0;
    v[i][1] = (row_ok && x0 + 1 <= nx + 1) ? ar[x0 + 1] : 0.0;
    wr[i] = row_ok ? ar[0] : 0.0;
    er[i] = (row_ok && nx + 1 == 2 * 32 + 1) ? ar[nx + 1] : 0.0;
  }
  // ring row 0 as the "last row of warp -1", in both parities
  for (int c = threadIdx.x; c < kW; c += blockDim.x) {
    const double r0 = (c + 1 <= nx + 1) ? a[c + 1] : 0.0;
    bot_row[0][0][c] = r0;
    bot_row[1][0][c] = r0;
  }
  const bool c0_upd = x0 <= nx, c1_upd = x0 + 1 <= nx;
  for (int64_t it = 0; it < iters; ++it) {
    const int p = (int)(it & 1);
    *reinterpret_cast<double2*>(&top_row[p][w][2 * lane]) = make_double2(v[0][0], v[0][1]);
    *reinterpret_cast<double2*>(&bot_row[p][w + 1][2 * lane]) = make_double2(v[R - 1][0], v[R - 1][1]);
    __syncthreads();
    const double2 nrow = *reinterpret_cast<const double2*>(&bot_row[p][w][2 * lane]);
    const double2 srow = (w + 1 < nw) ? *reinterpret_cast<const double2*>(&top_row[p][w + 1][2 * lane])
                                      : make_double2(0.0, 0.0);
    double o[R][2];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int y = 1 + R * w + i;
      const double n0 = i > 0 ? v[i - 1][0] : nrow.x, n1 = i > 0 ? v[i - 1][1] : nrow.y;
      const double s0 = i + 1 < R ? v[i + 1][0] : srow.x, s1 = i + 1 < R ? v[i + 1][1] : srow.y;
      double wv = __shfl_up_sync(0xffffffffu, v[i][1], 1);
      double ev = __shfl_down_sync(0xffffffffu, v[i][0], 1);
      if (lane == 0) wv = wr[i];
      if (lane == 31) ev = er[i];
      const bool row_upd = y <= ny;
      o[i][0] = (row_upd && c0_upd) ? dmul(dadd(dadd(dadd(n0, s0), wv), v[i][1]), 0.25) : v[i][0];
      o[i][1] = (row_upd && c1_upd) ? dmul(dadd(dadd(dadd(n1, s1), v[i][0]), ev), 0.25) : v[i][1];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      v[i][0] = o[i][0];
      v[i][1] = o[i][1];
    }
  }
  double* out = (iters & 1) ? b : a;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int y = 1 + R * w + i;
    if (y > ny + 1) continue;
    double* orow = out + (int64_t)y * ld;
    if (x0 <= nx + 1) orow[x0] = v[i][0];
    if (x0 + 1 <= nx + 1) orow[x0 + 1] = v[i][1];
    if (lane == 0) orow[0] = wr[i];
    if (lane == 31 && nx + 1 == 2 * 32 + 1) orow[nx + 1] = er[i];
  }
  if (iters & 1) {  // the ring row 0 of b
    for (int c = threadIdx.x; c < nx + 2; c += blockDim.x) b[c] = a[c];
  }
}

constexpr int kRegResRows = 3;

constexpr size_t kResidentMaxSmem = 200 * 1024;

}  // namespace

st_status jacobi2d_sweep_rows(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo,
                              int64_t y_hi, cudaStream_t s, Remote rem) {
  if (y_hi < y_lo) return ST_OK;
  const int64_t nxp2 = nx + 2;
  const int64_t nstrips = (nxp2 + kStripCols - 1) / kStripCols;
  const int64_t rows = y_hi - y_lo + 1;
  static const int kRows = env_int("ST_JACOBI_ROWS", 128);
  const int64_t rpc = std::max<int64_t>(1, std::min<int64_t>(kRows, rows));
  const int64_t nchunks = (rows + rpc - 1) / rpc;
  ST_RETURN_IF(nchunks > 65535, ST_ENOTSUP, "jacobi2d: %lld row chunks exceed grid.y", (long long)nchunks);
  dim3 grid((unsigned)((nstrips + kStreamWarps - 1) / kStreamWarps), (unsigned)nchunks);
  jacobi2d_stream_kernel<4><<<grid, kStreamThreads, 0, s>>>(src, dst, nxp2, ld, y_lo, y_hi, rpc, nstrips, rem.base,
                                                             rem.delta);
  ST_LAUNCHED();
  return ST_OK;
}

bool jacobi2d_resident_fits(int64_t nx, int64_t ny) {
  const int64_t n = (nx + 2) * (ny + 2);
  return n * 2 * (int64_t)sizeof(double) <= (int64_t)kResidentMaxSmem;
}

st_status jacobi2d_resident(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t iters,
                            cudaStream_t s) {
  static const int kRegRes = env_int("ST_JACOBI_REGRES", kRegResRows);  // rows per warp (0: shared-memory kernel)
  if (kRegRes && nx <= 64) {
    const int64_t rr = kRegRes == 8 ? 8 : kRegRes == 2 ? 2 : kRegRes == 3 ? 3 : 4;
    const int64_t warps = (ny + 1 + rr - 1) / rr;  // rows 1 .. ny+1 (incl. the ring row)
    if (warps <= kRegResMaxWarps) {
      auto* k = rr == 8   ? jacobi2d_regres_kernel<8>
                : rr == 2 ? jacobi2d_regres_kernel<2>
                : rr == 3 ? jacobi2d_regres_kernel<3>
                          : jacobi2d_regres_kernel<4>;
      k<<<1, (unsigned)(32 * warps), 0, s>>>(a, b, (int)nx, (int)ny, ld, iters);
      ST_LAUNCHED();
      return ST_OK;
    }
  }
  const size_t smem = (size_t)(nx + 2) * (size_t)(ny + 2) * 2 * sizeof(double);
  ST_CHECK_CUDA(cudaFuncSetAttribute(jacobi2d_resident_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kResidentMaxSmem));
  const int bx = (int)std::min<int64_t>(1024, ((nx + 31) / 32) * 32);
  const int by = std::max(1, std::min(1024 / bx, (int)ny));
  jacobi2d_resident_kernel<<<1, dim3(bx, by), smem, s>>>(a, b, (int)(nx + 2), (int)(ny + 2), ld, iters);
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
// (N, C); when level j-1 delivers a new row S, level j produces row C. W/E
// neighbours at every level come from warp shuffles. Dirichlet rows/columns are
// passed through unchanged at every level, so every level is exactly one Jacobi
// sweep and the result is bitwise T single sweeps.
//
// Instruction diet (the kernel is issue-bound once T >= 4): each level keeps two
// row slots; N is slot k%2 and C slot (k+1)%2, and the new row S overwrites the
// N slot once N has been consumed, so with steps unrolled in groups of
// kTbGroup (even) the rotation is register renaming, not moves. The refill
// load of every step is unconditional (its address is clamped to a valid row),
// so no select ever waits on an in-flight load; the per-level Dirichlet-row and
// Dirichlet-column handling is compiled into separate level bodies chosen per
// step by a block-/warp-uniform branch, so steady-state steps carry no checks.
// Load and store addresses advance by one pitch per step.
constexpr int kTbGroup = 4;  // steps per unrolled group (even: the slot rotation period is 2)

template <int T, bool kRows, bool kCols>
__device__ __forceinline__ double2 tb_levels(double2 (&st)[T][2], const int k, double2 s, int64_t r,
                                             bool ring0, bool ring1, int64_t ring_lo, int64_t ring_hi) {
#pragma unroll
  for (int j = 0; j < T; ++j) {
    // level j: N = slot k%2, C = slot (k+1)%2; S (from level j-1) replaces N afterwards
    const double2 n = st[j][k & 1];
    const double2 c = st[j][(k + 1) & 1];
    const double w = __shfl_up_sync(0xffffffffu, c.y, 1);
    const double e = __shfl_down_sync(0xffffffffu, c.x, 1);
    double2 o;
    o.x = dmul(dadd(dadd(dadd(n.x, s.x), w), c.y), 0.25);
    o.y = dmul(dadd(dadd(dadd(n.y, s.y), c.x), e), 0.25);
    if (kCols) {  // Dirichlet columns pass through
      if (ring0) o.x = c.x;
      if (ring1) o.y = c.y;
    }
    if (kRows) {
      const int64_t row = r - j - 1;
      if (row <= ring_lo || row >= ring_hi) o = c;  // Dirichlet rows never change
    }
    st[j][k & 1] = s;
    s = o;
  }
  return s;
}

template <int T, int kMinBlocks>
__global__ void __launch_bounds__(kStreamThreads, kMinBlocks)
    jacobi2d_tb_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nxp2, int64_t ld,
                       int64_t y_lo, int64_t y_hi, int64_t rows_per_chunk, int64_t nstrips, int64_t ring_lo,
                       int64_t ring_hi, int64_t nrows_buf, double* __restrict__ dst2, int64_t delta2) {
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
  const int64_t x_first = strip * kStride - T;
  const bool col_ring = x_first <= 0 || x_first + kStripCols >= nxp2 - 1;  // warp-uniform
  const double* sp = src + (has_pair ? x : 0);  // every lane loads from a valid column

  // input rows the pipeline reads: [r_first, r_load_last]; steps run to r_end
  const int64_t r_first = max(max(ring_lo, (int64_t)0), yc0 - T);
  const int64_t r_load_last = min(min(ring_hi, nrows_buf - 1), yc1 + T);
  const int64_t r_end = yc1 + T;

  double2 st[T][2];
#pragma unroll
  for (int j = 0; j < T; ++j) st[j][0] = st[j][1] = make_double2(0.0, 0.0);
  double2 buf[kTbGroup];  // input rows r0..r0+G-1; slot k is refilled with row r0+k+G after use
  const double* safe = sp + r_first * ld;
#pragma unroll
  for (int k = 0; k < kTbGroup; ++k) buf[k] = ldg2(r_first + k <= r_load_last ? sp + (r_first + k) * ld : safe);
  const double* lp = sp + (r_first + kTbGroup) * ld;  // next row to load
  double* sp_out = dst + x + (r_first - T) * ld;      // row the next step stores
  double* sp_out2 = dst2 ? dst2 + x + (r_first - T + delta2) * ld : nullptr;

  for (int64_t r0 = r_first; r0 <= r_end; r0 += kTbGroup) {
#pragma unroll
    for (int k = 0; k < kTbGroup; ++k) {
      const int64_t r = r0 + k;
      if (r > r_end) break;
      const double2 s0 = buf[k];
      buf[k] = ldg2(r + kTbGroup <= r_load_last ? lp : safe);
      lp += ld;
      // does any level of this step touch a Dirichlet row (rows r-1 .. r-T)?
      const bool rows_chk = (r - T <= ring_lo) || (r - 1 >= ring_hi);
      double2 o;
      if (rows_chk) {
        o = col_ring ? tb_levels<T, true, true>(st, k, s0, r, ring0, ring1, ring_lo, ring_hi)
                     : tb_levels<T, true, false>(st, k, s0, r, ring0, ring1, ring_lo, ring_hi);
      } else {
        o = col_ring ? tb_levels<T, false, true>(st, k, s0, r, ring0, ring1, ring_lo, ring_hi)
                     : tb_levels<T, false, false>(st, k, s0, r, ring0, ring1, ring_lo, ring_hi);
      }
      // o = level T, row r-T
      if (r - T >= yc0 && r - T <= yc1) {
        if (st0 && st1) stg2(sp_out, o);
        else if (st0) sp_out[0] = o.x;
        else if (st1) sp_out[1] = o.y;
        if (sp_out2) {  // fused halo swap
          if (st0 && st1) stg2(sp_out2, o);
          else if (st0) sp_out2[0] = o.x;
          else if (st1) sp_out2[1] = o.y;
        }
      }
      sp_out += ld;
      if (sp_out2) sp_out2 += ld;
    }
  }
}

// ---- 4 columns per lane (two 16-byte pairs): 128-column strips, half the
// shuffles per point and 2T/128 instead of 2T/64 redundant columns.
struct Quad {
  double2 a, b;  // columns x, x+1 | x+2, x+3
};

// G = 3 variant: input rows staged in a per-warp shared-memory ring of kTbRing
// rows by cp.async (each lane copies and later reads only its own 32 bytes, so
// no barrier is needed), read back one step ahead so the LDS latency is off the
// chain; frees the register prefetch for the three-slot level state.
constexpr int kTbRing = 8;
__device__ __forceinline__ void tb_cp16(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(gmem) : "memory");
}
__device__ __forceinline__ void tb_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tb_wait_ring() {
  asm volatile("cp.async.wait_group %0;" ::"n"(kTbRing - 1) : "memory");
}
__device__ __forceinline__ double2 tb_lds2(uint32_t smem) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem) : "memory");
  return v;
}

// State of level j: rows n, c of level j-1's output in slots k % NS, (k+1) % NS; the new
// row s goes to slot (k+2) % NS. NS = 2 overwrites n's slot; NS = 3 writes the free third
// slot, so s and n never need the same registers and a group of G = 3 steps returns every
// value to its register with no copies at the loop edge.
template <int T, int NS, bool kRows, bool kCols>
__device__ __forceinline__ Quad tb4_levels(Quad (&st)[T][NS], const int k, Quad s, int64_t r, const bool (&ring)[4],
                                           int64_t ring_lo, int64_t ring_hi) {
#pragma unroll
  for (int j = 0; j < T; ++j) {
    const Quad n = st[j][k % NS];
    const Quad c = st[j][(k + 1) % NS];
    const double w = __shfl_up_sync(0xffffffffu, c.b.y, 1);
    const double e = __shfl_down_sync(0xffffffffu, c.a.x, 1);
    Quad o;
    o.a.x = dmul(dadd(dadd(dadd(n.a.x, s.a.x), w), c.a.y), 0.25);
    o.a.y = dmul(dadd(dadd(dadd(n.a.y, s.a.y), c.a.x), c.b.x), 0.25);
    o.b.x = dmul(dadd(dadd(dadd(n.b.x, s.b.x), c.a.y), c.b.y), 0.25);
    o.b.y = dmul(dadd(dadd(dadd(n.b.y, s.b.y), c.b.x), e), 0.25);
    if (kCols) {
      if (ring[0]) o.a.x = c.a.x;
      if (ring[1]) o.a.y = c.a.y;
      if (ring[2]) o.b.x = c.b.x;
      if (ring[3]) o.b.y = c.b.y;
    }
    if (kRows) {
      const int64_t row = r - j - 1;
      if (row <= ring_lo || row >= ring_hi) o = c;
    }
    st[j][(k + 2) % NS] = s;
    s = o;
  }
  return s;
}

template <int T, int kMinBlocks, int G>
__global__ void __launch_bounds__(kStreamThreads, kMinBlocks)
    jacobi2d_tb4_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nxp2, int64_t ld,
                        int64_t y_lo, int64_t y_hi, int64_t rows_per_chunk, int64_t nstrips, int64_t ring_lo,
                        int64_t ring_hi, int64_t nrows_buf, double* __restrict__ dst2, int64_t delta2) {
  static_assert(T >= 2 && T % 2 == 0 && T <= 16, "even T");
  constexpr int NS = G % 3 == 0 ? 3 : 2;  // row slots per level (tb4_levels)
  static_assert(G % NS == 0, "row-slot renaming needs a group of whole slot cycles");
  constexpr int P = G == 3 ? 1 : G;  // rows loaded ahead in registers (G = 3: the shared-memory ring instead)
  static_assert(G % P == 0, "prefetch slots renamed within a group");
  constexpr int kCols = 128, kStride = kCols - 2 * T;
  const int lane = threadIdx.x & 31;
  const int64_t strip = (int64_t)blockIdx.x * kStreamWarps + (threadIdx.x >> 5);
  if (strip >= nstrips) return;
  const int64_t yc0 = y_lo + (int64_t)blockIdx.y * rows_per_chunk;
  if (yc0 > y_hi) return;
  const int64_t yc1 = min(y_hi, yc0 + rows_per_chunk - 1);

  const int64_t x = strip * kStride - T + 4 * lane;
  const int64_t x_first = strip * kStride - T;
  const int64_t lo_c = x_first + T, hi_c = x_first + kCols - T;  // exact columns [lo_c, hi_c)
  const bool has_a = x >= 0 && x < nxp2, has_b = x + 2 >= 0 && x + 2 < nxp2;
  const bool sta0 = x >= lo_c && x < hi_c && x >= 0 && x < nxp2;
  const bool sta1 = x + 1 >= lo_c && x + 1 < hi_c && x + 1 >= 0 && x + 1 < nxp2;
  const bool stb0 = x + 2 >= lo_c && x + 2 < hi_c && x + 2 >= 0 && x + 2 < nxp2;
  const bool stb1 = x + 3 >= lo_c && x + 3 < hi_c && x + 3 >= 0 && x + 3 < nxp2;
  bool ring[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) ring[i] = (x + i == 0) || (x + i == nxp2 - 1);
  const bool col_ring = x_first <= 0 || x_first + kCols >= nxp2 - 1;
  const double* spa = src + (has_a ? x : 0);
  const double* spb = src + (has_b ? x + 2 : 0);

  const int64_t r_first = max(max(ring_lo, (int64_t)0), yc0 - T);
  const int64_t r_load_last = min(min(ring_hi, nrows_buf - 1), yc1 + T);
  const int64_t r_end = yc1 + T;

  Quad st[T][NS];
#pragma unroll
  for (int j = 0; j < T; ++j) {
#pragma unroll
    for (int q = 0; q < NS; ++q) st[j][q].a = st[j][q].b = make_double2(0.0, 0.0);
  }
  constexpr bool kRing = G == 3;
  Quad buf[P];
  const int64_t safe_off = r_first * ld;
  // shared-memory row ring (kRing): this lane's 32 bytes of slot q at sring + q * 1024
  extern __shared__ __align__(16) double tb_ring_smem[];
  const uint32_t sring = (uint32_t)__cvta_generic_to_shared(tb_ring_smem) +
                         (uint32_t)((threadIdx.x >> 5) * kTbRing * 1024 + lane * 32);
  int rs = 0;  // ring slot of the current row
  Quad snx;    // the current row, read from the ring one step ahead
  int64_t roff = (r_first + kTbRing) * ld;
  if constexpr (kRing) {
#pragma unroll
    for (int q = 0; q < kTbRing; ++q) {
      const int64_t off = (r_first + q <= r_load_last) ? (r_first + q) * ld : safe_off;
      tb_cp16(sring + q * 1024, spa + off);
      tb_cp16(sring + q * 1024 + 16, spb + off);
      tb_commit();
    }
    tb_wait_ring();
    snx.a = tb_lds2(sring);
    snx.b = tb_lds2(sring + 16);
  } else {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int64_t off = (r_first + k <= r_load_last) ? (r_first + k) * ld : safe_off;
      buf[k].a = ldg2(spa + off);
      buf[k].b = ldg2(spb + off);
    }
  }
  // kRing: the current row; the slot it came from refills with row r + kTbRing, and
  // row r + 1 is read into registers for the next step
  auto ring_row = [&](int64_t r) -> Quad {
    const Quad cur = snx;
    const int64_t off = (r + kTbRing <= r_load_last) ? roff : safe_off;
    roff += ld;
    const uint32_t w = sring + rs * 1024;
    tb_cp16(w, spa + off);
    tb_cp16(w + 16, spb + off);
    tb_commit();
    rs = rs + 1 == kTbRing ? 0 : rs + 1;
    tb_wait_ring();
    snx.a = tb_lds2(sring + rs * 1024);
    snx.b = tb_lds2(sring + rs * 1024 + 16);
    return cur;
  };
  int64_t loff = (r_first + P) * ld;
  double* out = dst + x + (r_first - T) * ld;
  double* out2 = dst2 ? dst2 + x + (r_first - T + delta2) * ld : nullptr;

  auto store_row = [&](double* p, const Quad& o) {
    if (sta0 && sta1) stg2(p, o.a);
    else if (sta0) p[0] = o.a.x;
    else if (sta1) p[1] = o.a.y;
    if (stb0 && stb1) stg2(p + 2, o.b);
    else if (stb0) p[2] = o.b.x;
    else if (stb1) p[3] = o.b.y;
  };

  for (int64_t r0 = r_first; r0 <= r_end; r0 += G) {
    // Steady state: every step of the group stores, touches no ring row and no
    // ring column. The G steps form ONE basic block (no per-step dispatch), so the
    // scheduler can run step k+1's level j beside step k's level j+1 — G times the
    // independent dependency chains of one step (the kernel is latency-bound at
    // 8 warps/SM). A shared-memory cp.async row ring (prefetch 8-16 rows ahead
    // instead of G) measured 16-25 % slower and was dropped.
    if (!col_ring && r0 + G - 1 <= r_end && r0 - T >= yc0 && r0 + G - 1 - T <= yc1 && r0 - T > ring_lo &&
        r0 + G - 2 < ring_hi) {
      Quad o[G];
#pragma unroll
      for (int k = 0; k < G; ++k) {
        Quad s0;
        if constexpr (kRing) {
          s0 = ring_row(r0 + k);
        } else {
          s0 = buf[k % P];
          const int64_t off = (r0 + k + P <= r_load_last) ? loff : safe_off;
          buf[k % P].a = ldg2(spa + off);
          buf[k % P].b = ldg2(spb + off);
          loff += ld;
        }
        o[k] = tb4_levels<T, NS, false, false>(st, k, s0, r0 + k, ring, ring_lo, ring_hi);
      }
#pragma unroll
      for (int k = 0; k < G; ++k) {
        store_row(out + k * ld, o[k]);
        if (out2) store_row(out2 + k * ld, o[k]);
      }
      out += G * ld;
      if (out2) out2 += G * ld;
      continue;
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int64_t r = r0 + k;
      if (r > r_end) break;
      Quad s0;
      if constexpr (kRing) {
        s0 = ring_row(r);
      } else {
        s0 = buf[k % P];
        const int64_t off = (r + P <= r_load_last) ? loff : safe_off;
        buf[k % P].a = ldg2(spa + off);
        buf[k % P].b = ldg2(spb + off);
        loff += ld;
      }
      const bool rows_chk = (r - T <= ring_lo) || (r - 1 >= ring_hi);
      Quad o;
      if (rows_chk) {
        o = col_ring ? tb4_levels<T, NS, true, true>(st, k, s0, r, ring, ring_lo, ring_hi)
                     : tb4_levels<T, NS, true, false>(st, k, s0, r, ring, ring_lo, ring_hi);
      } else {
        o = col_ring ? tb4_levels<T, NS, false, true>(st, k, s0, r, ring, ring_lo, ring_hi)
                     : tb4_levels<T, NS, false, false>(st, k, s0, r, ring, ring_lo, ring_hi);
      }
      if (r - T >= yc0 && r - T <= yc1) {
        store_row(out, o);
        if (out2) store_row(out2, o);  // fused halo swap: the same row into the neighbour's ghost row
      }
      out += ld;
      if (out2) out2 += ld;
    }
  }
}

template <int T>
st_status launch_tb4(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                     int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s, Remote rem) {
  const int64_t nxp2 = nx + 2;
  constexpr int kStride = 128 - 2 * T;
  const int64_t nstrips = (nxp2 + kStride - 1) / kStride;
  const int64_t rows = y_hi - y_lo + 1;
  const int64_t blocks_x = (nstrips + kStreamWarps - 1) / kStreamWarps;
  static const int kOcc = env_int("ST_JACOBI_TB4_OCC", 1);
  // Row chunk: every chunk recomputes 2T warm-up rows, and with one CTA per SM
  // a partly filled last wave idles SMs, so pick the chunk height R that
  // minimises waves(R) x (R + 2T) (C2: R = 357 -> 6 waves of 874 CTAs, +2 %
  // over the fixed 192-row chunks, measured). ST_JACOBI_TB4_ROWS overrides.
  static const int kRows = env_int("ST_JACOBI_TB4_ROWS", 0);
  int64_t rpc = kRows;
  if (rpc <= 0) {
    const int64_t slots = (int64_t)num_sms() * kOcc;
    int64_t best = INT64_MAX;
    rpc = rows;
    for (int64_t r = 160; r <= 448; ++r) {
      const int64_t ctas = blocks_x * ((rows + r - 1) / r);
      const int64_t cost = ((ctas + slots - 1) / slots) * (std::min(r, rows) + 2 * T);
      if (cost < best) { best = cost; rpc = r; }
    }
  }
  rpc = std::max<int64_t>(1, std::min<int64_t>(rpc, rows));
  const int64_t nchunks = (rows + rpc - 1) / rpc;
  ST_RETURN_IF(nchunks > 65535, ST_ENOTSUP, "jacobi2d tb: too many row chunks");
  dim3 grid((unsigned)blocks_x, (unsigned)nchunks);
  // G = steps per group: 2 (default) = two row slots + register prefetch; 3 = three row
  // slots per level (no register copies at the loop edge) with the input rows staged in
  // a shared-memory cp.async ring: 7 % more work per clock, but it runs into the power
  // cap (sw_power_cap, 1833 MHz) and sustains the same 1619 Gpts/s as G=2 at 1965 MHz
  // (DESIGN.md §6.2); 4 spills at T=8
  static const int kG = env_int("ST_JACOBI_TB4_G", 2);
  auto* kern = kG == 3 ? jacobi2d_tb4_kernel<T, 1, 3>
               : kOcc == 1 ? (kG == 4 ? jacobi2d_tb4_kernel<T, 1, 4> : jacobi2d_tb4_kernel<T, 1, 2>)
                           : (kG == 4 ? jacobi2d_tb4_kernel<T, 2, 4> : jacobi2d_tb4_kernel<T, 2, 2>);
  const size_t smem = kG == 3 ? (size_t)kStreamWarps * kTbRing * 1024 : 0;
  if (smem > 0)
    ST_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, kStreamThreads, smem, s>>>(src, dst, nxp2, ld, y_lo, y_hi, rpc, nstrips, ring_lo, ring_hi, nrows_buf,
                                          rem.base, rem.delta);
  ST_LAUNCHED();
  return ST_OK;
}

template <int T>
st_status launch_tb(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                    int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s, Remote rem) {
  const int64_t nxp2 = nx + 2;
  constexpr int kStride = kStripCols - 2 * T;
  const int64_t nstrips = (nxp2 + kStride - 1) / kStride;
  const int64_t rows = y_hi - y_lo + 1;
  static const int kRows = env_int("ST_JACOBI_TB_ROWS", 512);
  const int64_t rpc = std::max<int64_t>(1, std::min<int64_t>(kRows, rows));
  const int64_t nchunks = (rows + rpc - 1) / rpc;
  ST_RETURN_IF(nchunks > 65535, ST_ENOTSUP, "jacobi2d tb: too many row chunks");
  dim3 grid((unsigned)((nstrips + kStreamWarps - 1) / kStreamWarps), (unsigned)nchunks);
  static const int kOcc = env_int("ST_JACOBI_TB_OCC", 2);
  if (kOcc == 3)
    jacobi2d_tb_kernel<T, 3><<<grid, kStreamThreads, 0, s>>>(src, dst, nxp2, ld, y_lo, y_hi, rpc, nstrips, ring_lo,
                                                             ring_hi, nrows_buf, rem.base, rem.delta);
  else if (kOcc == 2)
    jacobi2d_tb_kernel<T, 2><<<grid, kStreamThreads, 0, s>>>(src, dst, nxp2, ld, y_lo, y_hi, rpc, nstrips, ring_lo,
                                                             ring_hi, nrows_buf, rem.base, rem.delta);
  else
    jacobi2d_tb_kernel<T, 1><<<grid, kStreamThreads, 0, s>>>(src, dst, nxp2, ld, y_lo, y_hi, rpc, nstrips, ring_lo,
                                                             ring_hi, nrows_buf, rem.base, rem.delta);
  ST_LAUNCHED();
  return ST_OK;
}

}  // namespace

bool jacobi2d_tb_supported(int t) { return t == 2 || t == 4 || t == 6 || t == 8; }

st_status jacobi2d_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_stream_kernel<4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_resident_kernel));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_regres_kernel<2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_regres_kernel<3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_regres_kernel<4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_regres_kernel<8>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<2, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<2, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<2, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<4, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<4, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<4, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<6, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<6, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<6, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<8, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<8, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb_kernel<8, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<2, 1, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<2, 1, 4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<2, 1, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<2, 2, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<2, 2, 4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<4, 1, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<4, 1, 4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<4, 1, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<4, 2, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<4, 2, 4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<6, 1, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<6, 1, 4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<6, 1, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<6, 2, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<6, 2, 4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<8, 1, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<8, 1, 4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<8, 1, 3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<8, 2, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<8, 2, 4>));
  return ST_OK;
}

st_status jacobi2d_tb_rows(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                           int t, int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s, Remote rem) {
  if (y_hi < y_lo) return ST_OK;
  static const int kColsPerLane = env_int("ST_JACOBI_TB_COLS", 4);
  if (kColsPerLane == 4) {
    switch (t) {
      case 2: return launch_tb4<2>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
      case 4: return launch_tb4<4>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
      case 6: return launch_tb4<6>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
      case 8: return launch_tb4<8>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
      default: break;
    }
  }
  switch (t) {
    case 2: return launch_tb<2>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    case 4: return launch_tb<4>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    case 6: return launch_tb<6>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    case 8: return launch_tb<8>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    default: set_error("jacobi2d: tblock=%d not supported (2, 4, 6, 8)", t); return ST_ENOTSUP;
  }
}

}  // namespace st

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
  static const int kRows = env_int("ST_JACOBI_ROWS", 32);  // 32-row chunks: 402 vs 393 Gpts/s at 128 (C2, round 2)
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
  // register-resident kernel for grids up to 64 columns (C1); shared-memory kernel otherwise
  if (nx <= 64) {
    const int64_t warps = (ny + 1 + kRegResRows - 1) / kRegResRows;  // rows 1 .. ny+1 (incl. the ring row)
    if (warps <= kRegResMaxWarps) {
      jacobi2d_regres_kernel<kRegResRows><<<1, (unsigned)(32 * warps), 0, s>>>(a, b, (int)nx, (int)ny, ld, iters);
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
// A warp owns a strip of 128 columns (lane = two 16-byte column pairs) that
// overlaps its neighbours by 2T columns: after T levels only the centre
// 128-2T columns are exact, so strips advance by 128-2T. Rows stream through a
// T-level software pipeline held entirely in registers: level j keeps its two
// most recent rows (N, C); when level j-1 delivers a new row S, level j
// produces row C. W/E neighbours at every level come from the adjacent lanes:
// warp shuffles in the general path below, a shared-memory exchange in the
// rotated steady state. Dirichlet rows/columns are passed through unchanged at
// every level, so every level is exactly one Jacobi sweep and the result is
// bitwise T single sweeps.
//
// Work decomposition: one warp = one (strip, row chunk) item, items numbered
// chunk-major over a 1-D grid; the chunk height is chosen per grid for whole
// waves of resident warps against the 2T warm-up rows every chunk recomputes
// (tb4_grid: C2 at T = 10 runs 150 interior strips x 15 chunks of 1093 rows plus
// the 2 edge strips in shorter chunks: 2338 warps, two waves of 148 x 8).
//
// Instruction diet: each level keeps two row slots; N is slot k%2 and C slot
// (k+1)%2, and the new row S overwrites the N slot once N has been consumed,
// so with steps unrolled in groups of kTbGroup = 2 the rotation is register
// renaming, not moves. The refill load of every step is unconditional (its
// address is clamped to a valid row), so no select ever waits on an in-flight
// load; the per-level Dirichlet-row and Dirichlet-column handling is compiled
// into separate level bodies chosen per group by a warp-uniform branch.
constexpr int kTbGroup = 2;   // steps per unrolled group (= the row-slot period)
constexpr int kTbCols = 128;  // columns per warp strip (32 lanes x 4)

struct Quad {
  double2 a, b;  // columns x, x+1 | x+2, x+3
};

// 64-bit warp shuffles as two explicit 32-bit shuffles (the generic double
// overload let ptxas swap the halves through three XORs per shuffle).
__device__ __forceinline__ double shfl_up1(double v) {
  const int lo = __shfl_up_sync(0xffffffffu, __double2loint(v), 1);
  const int hi = __shfl_up_sync(0xffffffffu, __double2hiint(v), 1);
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ double shfl_down1(double v) {
  const int lo = __shfl_down_sync(0xffffffffu, __double2loint(v), 1);
  const int hi = __shfl_down_sync(0xffffffffu, __double2hiint(v), 1);
  return __hiloint2double(hi, lo);
}
// Predicated stores (no branch, so the warp provably stays converged for the
// shuffles that follow; a branch here cost a divergence check per step).
__device__ __forceinline__ void stg2_if(bool pred, double* p, double2 v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q st.global.v2.f64 [%0], {%1, %2};\n}" ::"l"(p),
               "d"(v.x), "d"(v.y), "r"((unsigned)pred)
               : "memory");
}
__device__ __forceinline__ void stg1_if(bool pred, double* p, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}" ::"l"(p), "d"(v),
               "r"((unsigned)pred)
               : "memory");
}

template <int T, bool kRows, bool kCols>
__device__ __forceinline__ Quad tb4_levels(Quad (&st)[T][2], const int k, Quad s, int64_t r, const bool (&ring)[4],
                                           int64_t ring_lo, int64_t ring_hi) {
#pragma unroll
  for (int j = 0; j < T; ++j) {
    const Quad n = st[j][k & 1];
    const Quad c = st[j][(k + 1) & 1];
    const double w = shfl_up1(c.b.y);
    const double e = shfl_down1(c.a.x);
    Quad o;
    o.a.x = dadd(dadd(dadd(n.a.x, s.a.x), w), c.a.y);
    o.a.y = dadd(dadd(dadd(n.a.y, s.a.y), c.a.x), c.b.x);
    o.b.x = dadd(dadd(dadd(n.b.x, s.b.x), c.a.y), c.b.y);
    o.b.y = dadd(dadd(dadd(n.b.y, s.b.y), c.b.x), e);
    o.a.x = dmul(o.a.x, 0.25);
    o.a.y = dmul(o.a.y, 0.25);
    o.b.x = dmul(o.b.x, 0.25);
    o.b.y = dmul(o.b.y, 0.25);
    if (kCols) {  // a Dirichlet cell keeps its value
      if (ring[0]) o.a.x = c.a.x;
      if (ring[1]) o.a.y = c.a.y;
      if (ring[2]) o.b.x = c.b.x;
      if (ring[3]) o.b.y = c.b.y;
    }
    if (kRows) {
      const int64_t row = r - j - 1;
      if (row <= ring_lo || row >= ring_hi) o = c;
    }
    st[j][k & 1] = s;
    s = o;
  }
  return s;
}

// Per-warp constants of one (strip, row chunk) item.
struct Tb4Item {
  const double *spa, *spb;  // the lane's two column pairs (clamped to valid columns)
  double *out, *out2;       // stores of the row r_first - T (out2: fused halo swap, or null)
  int64_t ld, yc0, yc1, r_first, r_load_last, r_end, ring_lo, ring_hi;
  bool col_ring;
  bool ring[4], stm[4];  // Dirichlet column / stored column, per lane column
};

// ---- rotated-register steady state ------------------------------------------
// Each level's update is done IN PLACE in the register of its oldest row N:
// P_j = ((N_j + S_j) + W) + E overwrites N_j, and P_j is the next level's S.
// One step later the roles shift: level j's C becomes its N, and the register
// holding P_{j-1} becomes its C. So a physical register climbs one level every
// two steps, and the assignment repeats every M = 2T + 2 steps (the +2: the
// input row of the step and the next one, read from shared memory one step
// ahead). A block of M unrolled steps therefore uses only compile-time register
// indices — no register copies at all (the two-slot rotation of the general
// path spends ~30 % of its instructions on moves). At the start of step k:
//   level j: N = R[(k - 2j) mod M], C = R[(k + 1 - 2j) mod M]
//   input row of step k: R[(k + 2) mod M]
//   free: R[(k + 3) mod M] (it held step k-1's output, already stored).
// Input rows stream through a per-warp shared-memory ring of kTbRing slots by
// cp.async, kTbRing-1 rows ahead: each lane copies and later reads only its own
// 32 bytes, so no barrier is needed, and the registers hold one row in flight
// instead of enough rows to cover the HBM latency. Rows past the item's last
// loaded row are zero-filled (src-size 0), so a block may overrun the item's
// end; its surplus outputs are not stored.
template <int T>
struct TbRot {
  static constexpr int M = 2 * T + 2;
  static constexpr int RS = M / 2 >= 7 ? M / 2 : M;  // ring slots per warp; divides M, so slots are compile-time
  __host__ __device__ static constexpr int at(int i) { return ((i % M) + M) % M; }
};

__device__ __forceinline__ void cp16_zfill(uint32_t smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ double2 lds2(uint32_t smem) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem) : "memory");
  return v;
}

// The warp's shared-memory row ring: slot q holds lane l's column pair a at
// q*1024 + l*16 and b at q*1024 + 512 + l*16 (contiguous 16-byte lanes:
// conflict-free). A run of blocks starting at row r0 keeps row r0 + m in slot
// m mod RS, so every slot offset inside a block is a compile-time constant.
struct TbRing {
  uint32_t lane_base;  // slot 0, column pair a of this lane
  const double* gp;    // this lane's column x in the next row to copy
  int valid;           // rows left before the item's last loaded row (later rows are zero-filled)
  __device__ __forceinline__ void copy(int slot, int64_t ld) {
    const uint32_t s = lane_base + (uint32_t)slot * 1024u;
    cp16_zfill(s, gp, valid > 0);
    cp16_zfill(s + 512, gp + 2, valid > 0);
    cp_commit();
    gp += ld;
    --valid;
  }
  __device__ __forceinline__ Quad read(int slot) const {
    const uint32_t s = lane_base + (uint32_t)slot * 1024u;
    Quad q;
    q.a = lds2(s);
    q.b = lds2(s + 512);
    return q;
  }
};

// Neighbour exchange through shared memory instead of warp shuffles: a 64-bit
// shuffle is two 32-bit SHFLs whose halves ptxas then moves into an aligned
// register pair (~4 extra instructions per level at 255 registers); an LDS.64
// lands in a pair directly. Level j's C at step k+1 is P_{j-1} of step k (the
// input row for j = 0), so each lane publishes those rows' edge columns (a.x,
// b.y) one step ahead into X[(k+1)&1][j], and at step k reads its neighbours'
// from X[k&1][j]; a __syncwarp per step orders the two. Per warp:
// X[parity 2][level T][a.x | b.y][34] doubles, entry l+1 = lane l, so lane l
// reads W at entry l (lane l-1's b.y) and E at entry l+2 (lane l+1's a.x); the
// pad entries only feed the garbage columns of the strip edges.
__device__ __forceinline__ void sts1(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ double lds1(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
template <int T>
struct TbX {
  static constexpr int kBytes = 2 * T * 2 * 34 * 8;  // per warp
  // byte offset of entry idx of (parity, level, which) from the warp's base
  __host__ __device__ static constexpr uint32_t off(int par, int j, int which, int idx) {
    return (uint32_t)((((par * T + j) * 2 + which) * 34 + idx) * 8);
  }
};

// One block of M steps; the run's first row (in slot 0) is a multiple of M rows back.
template <int T>
__device__ __forceinline__ void tb4_rot_block(Quad (&R)[TbRot<T>::M], TbRing& ring, const uint32_t xl, double*& out,
                                              int& i, const int i_lo, const unsigned i_span, const int64_t ld,
                                              const bool sa, const bool sb) {
  using Rot = TbRot<T>;
  constexpr int M = Rot::M, RS = Rot::RS;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    ring.copy((k + RS - 1) % RS, ld);    // row r + RS - 1
    cp_wait<RS - 2>();                   // row r + 1 has landed
    R[Rot::at(k + 3)] = ring.read((k + 1) % RS);  // row r + 1, read one step ahead
    using X = TbX<T>;
    const int par = k & 1, npar = (k + 1) & 1;
    {  // level 0's C of step k+1 is this step's input row
      const Quad& s0 = R[Rot::at(k + 2)];
      sts1(xl + X::off(npar, 0, 0, 1), s0.a.x);
      sts1(xl + X::off(npar, 0, 1, 1), s0.b.y);
    }
    // exchange loads one level ahead of their use (X[par] was written by the previous step)
    double wn = lds1(xl + X::off(par, 0, 1, 0)), en = lds1(xl + X::off(par, 0, 0, 2));
#pragma unroll
    for (int j = 0; j < T; ++j) {
      Quad& n = R[Rot::at(k - 2 * j)];
      const Quad& c = R[Rot::at(k + 1 - 2 * j)];
      const Quad& s = R[Rot::at(j == 0 ? k + 2 : k - 2 * j + 2)];
      const double w = wn;  // lane-1's b.y
      const double e = en;  // lane+1's a.x
      if (j + 1 < T) {
        wn = lds1(xl + X::off(par, j + 1, 1, 0));
        en = lds1(xl + X::off(par, j + 1, 0, 2));
      }
      n.a.x = dadd(dadd(dadd(n.a.x, s.a.x), w), c.a.y);
      n.a.y = dadd(dadd(dadd(n.a.y, s.a.y), c.a.x), c.b.x);
      n.b.x = dadd(dadd(dadd(n.b.x, s.b.x), c.a.y), c.b.y);
      n.b.y = dadd(dadd(dadd(n.b.y, s.b.y), c.b.x), e);
      n.a.x = dmul(n.a.x, 0.25);
      n.a.y = dmul(n.a.y, 0.25);
      n.b.x = dmul(n.b.x, 0.25);
      n.b.y = dmul(n.b.y, 0.25);
      if (j + 1 < T) {  // P_j is level j+1's C at step k+1
        sts1(xl + X::off(npar, j + 1, 0, 1), n.a.x);
        sts1(xl + X::off(npar, j + 1, 1, 1), n.b.y);
      }
    }
    __syncwarp();
    const Quad& o = R[Rot::at(k - 2 * (T - 1))];  // level T-1 output: row r - T
    const bool in = (unsigned)(i - i_lo) <= i_span;
    stg2_if(in && sa, out, o.a);
    stg2_if(in && sb, out + 2, o.b);
    out += ld;
    ++i;
  }
}

// Streams one item.
template <int T>
__device__ __forceinline__ void tb4_item(const Tb4Item& it, const double* __restrict__ src_x, const bool use_rot,
                                        const uint32_t smem_lane, const uint32_t xl) {
  constexpr int G = kTbGroup;
  using Rot = TbRot<T>;
  constexpr int M = Rot::M, RS = Rot::RS;
  const int64_t ld = it.ld;
  Quad st[T][2];
#pragma unroll
  for (int j = 0; j < T; ++j) st[j][0].a = st[j][0].b = st[j][1].a = st[j][1].b = make_double2(0.0, 0.0);
  Quad buf[G];  // input rows r0 .. r0+G-1; slot k is refilled with row r0+k+G once used
  const int64_t safe_off = it.r_first * ld;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int64_t off = (it.r_first + k <= it.r_load_last) ? (it.r_first + k) * ld : safe_off;
    buf[k].a = ldg2(it.spa + off);
    buf[k].b = ldg2(it.spb + off);
  }
  int64_t loff = (it.r_first + G) * ld;
  double* out = it.out;
  double* out2 = it.out2;
  // per-lane stored columns: whole 16-byte pairs where possible (predicated, no branches)
  const bool pa = it.stm[0] && it.stm[1], pb = it.stm[2] && it.stm[3];
  const bool pa0 = it.stm[0] && !it.stm[1], pa1 = !it.stm[0] && it.stm[1];
  const bool pb0 = it.stm[2] && !it.stm[3], pb1 = !it.stm[2] && it.stm[3];
  auto store_row = [&](bool in, double* p, const Quad& o) {
    stg2_if(in && pa, p, o.a);
    stg1_if(in && pa0, p, o.a.x);
    stg1_if(in && pa1, p + 1, o.a.y);
    stg2_if(in && pb, p + 2, o.b);
    stg1_if(in && pb0, p + 2, o.b.x);
    stg1_if(in && pb1, p + 3, o.b.y);
  };
  // the rotated path: no ring column, no Dirichlet row in reach of the block's levels, no
  // fused second store (a block may run past r_end: later rows are zero-filled, outputs
  // past yc1 are not stored)
  auto rot_ok = [&](int64_t r0) { return use_rot && r0 - T > it.ring_lo && r0 + M - 2 < it.ring_hi; };
  int64_t r0 = it.r_first;
  while (r0 <= it.r_end) {
    if (rot_ok(r0)) {
      Quad R[M];
#pragma unroll
      for (int j = 0; j < T; ++j) {
        R[Rot::at(-2 * j)] = st[j][0];
        R[Rot::at(1 - 2 * j)] = st[j][1];
      }
      R[2] = buf[0];  // row r0; rows r0 + 1 .. come through the ring
#pragma unroll
      for (int j = 0; j < T; ++j) {  // the neighbour exchange of step 0: every level's C
        sts1(xl + TbX<T>::off(0, j, 0, 1), st[j][1].a.x);
        sts1(xl + TbX<T>::off(0, j, 1, 1), st[j][1].b.y);
      }
      __syncwarp();
      TbRing ring;
      ring.lane_base = smem_lane;
      ring.gp = src_x + (r0 + 1) * ld;
      ring.valid = (int)min(it.r_load_last - r0, (int64_t)INT32_MAX);
#pragma unroll
      for (int q = 1; q < RS - 1; ++q) ring.copy(q, ld);
      int i = (int)(r0 - it.r_first);
      const int i_lo = (int)(it.yc0 + T - it.r_first);
      const unsigned i_span = (unsigned)(it.yc1 - it.yc0);
      const bool sa = it.stm[0] && it.stm[1], sb = it.stm[2] && it.stm[3];
      do {
        tb4_rot_block<T>(R, ring, xl, out, i, i_lo, i_span, ld, sa, sb);
        r0 += M;
      } while (r0 <= it.r_end && rot_ok(r0));
      cp_wait_all();
      if (r0 > it.r_end) break;
#pragma unroll
      for (int j = 0; j < T; ++j) {
        st[j][0] = R[Rot::at(-2 * j)];
        st[j][1] = R[Rot::at(1 - 2 * j)];
      }
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int64_t off = (r0 + k <= it.r_load_last) ? (r0 + k) * ld : safe_off;
        buf[k].a = ldg2(it.spa + off);
        buf[k].b = ldg2(it.spb + off);
      }
      loff = (r0 + G) * ld;
      continue;
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int64_t r = r0 + k;
      if (r > it.r_end) break;
      const Quad s0 = buf[k];
      const int64_t off = (r + G <= it.r_load_last) ? loff : safe_off;
      buf[k].a = ldg2(it.spa + off);
      buf[k].b = ldg2(it.spb + off);
      loff += ld;
      const bool rows_chk = (r - T <= it.ring_lo) || (r - 1 >= it.ring_hi);
      Quad o;
      if (rows_chk) {
        o = it.col_ring ? tb4_levels<T, true, true>(st, k, s0, r, it.ring, it.ring_lo, it.ring_hi)
                        : tb4_levels<T, true, false>(st, k, s0, r, it.ring, it.ring_lo, it.ring_hi);
      } else {
        o = it.col_ring ? tb4_levels<T, false, true>(st, k, s0, r, it.ring, it.ring_lo, it.ring_hi)
                        : tb4_levels<T, false, false>(st, k, s0, r, it.ring, it.ring_lo, it.ring_hi);
      }
      const bool in = r - T >= it.yc0 && r - T <= it.yc1;
      store_row(in, out, o);
      store_row(in && out2, out2, o);  // fused halo swap: the same row into the neighbour's ghost row
      out += ld;
      if (out2) out2 += ld;
    }
    r0 += G;
  }
}

// Item numbering: items [0, n_int) are the interior strips (no ring column)
// chunk-major, rows_int rows each; items [n_int, n_int + n_edge) the strips that
// hold a ring column (the slower general path), rows_edge rows each.
struct Tb4Grid {
  int64_t s_lo, n_int_strips, rows_int, n_int;  // interior strips s_lo .. s_lo + n_int_strips - 1
  int64_t n_edge_strips, rows_edge, n_edge;     // edge strips: 0 .. s_lo-1 and s_lo + n_int_strips ..
};

template <int T, int W, int kMinBlocks>
__global__ void __launch_bounds__(32 * W, kMinBlocks)
    jacobi2d_tb4_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nxp2, int64_t ld,
                        int64_t y_lo, int64_t y_hi, Tb4Grid g, int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf,
                        double* __restrict__ dst2, int64_t delta2) {
  static_assert(T >= 2 && T % 2 == 0 && T <= 16, "even T");
  constexpr int kStride = kTbCols - 2 * T;
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * W + (threadIdx.x >> 5);
  int64_t strip, chunk, rpc;
  if (item < g.n_int) {
    strip = g.s_lo + item % g.n_int_strips;
    chunk = item / g.n_int_strips;
    rpc = g.rows_int;
  } else if (item < g.n_int + g.n_edge) {
    const int64_t e = item - g.n_int, es = e % g.n_edge_strips;
    strip = es < g.s_lo ? es : es + g.n_int_strips;
    chunk = e / g.n_edge_strips;
    rpc = g.rows_edge;
  } else {
    return;  // warp-uniform
  }
  Tb4Item it;
  it.ld = ld;
  it.yc0 = y_lo + chunk * rpc;
  it.yc1 = min(y_hi, it.yc0 + rpc - 1);
  const int64_t x_first = strip * kStride - T;
  const int64_t x = x_first + 4 * lane;
  const int64_t lo_c = x_first + T, hi_c = x_first + kTbCols - T;  // exact columns [lo_c, hi_c)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    it.ring[i] = (x + i == 0) || (x + i == nxp2 - 1);
    it.stm[i] = x + i >= lo_c && x + i < hi_c && x + i >= 0 && x + i < nxp2;
  }
  it.col_ring = x_first <= 0 || x_first + kTbCols >= nxp2 - 1;
  const bool has_a = x >= 0 && x < nxp2, has_b = x + 2 >= 0 && x + 2 < nxp2;
  it.spa = src + (has_a ? x : 0);
  it.spb = src + (has_b ? x + 2 : 0);
  it.ring_lo = ring_lo;
  it.ring_hi = ring_hi;
  it.r_first = max(max(ring_lo, (int64_t)0), it.yc0 - T);
  it.r_load_last = min(min(ring_hi, nrows_buf - 1), it.yc1 + T);
  it.r_end = it.yc1 + T;
  it.out = dst + x + (it.r_first - T) * ld;
  it.out2 = dst2 ? dst2 + x + (it.r_first - T + delta2) * ld : nullptr;
  // the rotated path needs whole column pairs in every lane and no fused second store
  const bool use_rot = !it.col_ring && !dst2;
  extern __shared__ __align__(16) unsigned char tb_ring_smem[];
  const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(tb_ring_smem);
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t smem_lane = smem0 + warp * TbRot<T>::RS * 1024 + lane * 16;
  const uint32_t xl = smem0 + W * TbRot<T>::RS * 1024 + warp * TbX<T>::kBytes + lane * 8;
  tb4_item<T>(it, src + x, use_rot, smem_lane, xl);
}

// Work decomposition: interior strips run the rotated path at ~R rows per item, the
// (up to 3) strips holding a ring column the general path, which is slower
// (kEdgeCost), so they get shorter chunks. Warps are resident in waves of
// num_sms x 8; the chunk counts minimise waves x the longest item (in rotated-row
// units, warm-up 2T rows included). ST_JACOBI_TB4_ROWS overrides the interior height.
Tb4Grid tb4_grid(int64_t nxp2, int64_t rows, int T, int64_t warps_per_sm) {
  const int64_t stride = kTbCols - 2 * T;
  const int64_t nstrips = (nxp2 + stride - 1) / stride;
  Tb4Grid g{};
  // interior strips: x_first > 0 and x_first + 128 < nxp2 - 1
  int64_t s_hi = -1;
  for (int64_t s = 1; s < nstrips; ++s)
    if (s * stride - T + kTbCols < nxp2 - 1) s_hi = s;
  g.s_lo = 1;
  g.n_int_strips = s_hi >= 1 ? s_hi : 0;
  g.n_edge_strips = nstrips - g.n_int_strips;
  static const int kRows = env_int("ST_JACOBI_TB4_ROWS", 0);
  static const int kEdgeCostPct = env_int("ST_JACOBI_TB4_EDGE_COST", 280);
  const int64_t slots = (int64_t)num_sms() * warps_per_sm;
  auto edge_rows_for = [&](int64_t r_int, int64_t* n_chunks) {  // edge items no longer than interior ones
    const int64_t budget = std::max<int64_t>(1, (r_int + 2 * T) * 100 / kEdgeCostPct - 2 * T);
    const int64_t ne = (rows + budget - 1) / budget;
    *n_chunks = ne;
    return (rows + ne - 1) / ne;
  };
  int64_t best = INT64_MAX, best_r = rows;
  const int64_t max_chunks = std::min<int64_t>(rows, 16 * slots / std::max<int64_t>(1, nstrips) + 1);
  for (int64_t nch = 1; nch <= max_chunks; ++nch) {
    const int64_t r = kRows > 0 ? std::min<int64_t>(kRows, rows) : (rows + nch - 1) / nch;
    const int64_t ni = g.n_int_strips * ((rows + r - 1) / r);
    int64_t ne_chunks = 0;
    edge_rows_for(r, &ne_chunks);
    const int64_t items = ni + g.n_edge_strips * ne_chunks;
    const int64_t cost = ((items + slots - 1) / slots) * (r + 2 * T);
    if (cost < best) {
      best = cost;
      best_r = r;
    }
    if (kRows > 0) break;
  }
  g.rows_int = best_r;
  g.n_int = g.n_int_strips * ((rows + best_r - 1) / best_r);
  int64_t ne_chunks = 0;
  g.rows_edge = edge_rows_for(best_r, &ne_chunks);
  g.n_edge = g.n_edge_strips * ne_chunks;
  return g;
}

// Resident warps per SM of an instantiation: W warps per CTA x kMinBlocks CTAs
// (the register budget is 65536 / (32 W kMinBlocks)). Only 8 x 1 is built: 4 x 3
// (T = 6, 168 registers) and 4 x 4 (T = 4, 128 registers) measured slower — the
// extra warps queue on the shared-memory pipe (row ring + exchange).
template <int T, int W, int kMinBlocks>
st_status launch_tb4_occ(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                         int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s, Remote rem) {
  const int64_t nxp2 = nx + 2;
  const Tb4Grid g = tb4_grid(nxp2, y_hi - y_lo + 1, T, W * kMinBlocks);
  const int64_t blocks = (g.n_int + g.n_edge + W - 1) / W;
  ST_RETURN_IF(blocks > INT32_MAX, ST_ENOTSUP, "jacobi2d tb: grid too large");
  const size_t smem = (size_t)W * (TbRot<T>::RS * 1024 + TbX<T>::kBytes);
  auto kern = jacobi2d_tb4_kernel<T, W, kMinBlocks>;
  ST_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)blocks, 32 * W, smem, s>>>(src, dst, nxp2, ld, y_lo, y_hi, g, ring_lo, ring_hi, nrows_buf,
                                              rem.base, rem.delta);
  ST_LAUNCHED();
  return ST_OK;
}

template <int T>
st_status launch_tb4(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                     int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s, Remote rem) {
  return launch_tb4_occ<T, kStreamWarps, 1>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
}

}  // namespace

bool jacobi2d_tb_supported(int t) { return t == 2 || t == 4 || t == 6 || t == 8 || t == 10; }

st_status jacobi2d_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_stream_kernel<4>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_resident_kernel));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_regres_kernel<kRegResRows>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<2, kStreamWarps, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<4, kStreamWarps, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<6, kStreamWarps, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<8, kStreamWarps, 1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi2d_tb4_kernel<10, kStreamWarps, 1>));
  return ST_OK;
}

st_status jacobi2d_tb_rows(const double* src, double* dst, int64_t nx, int64_t ld, int64_t y_lo, int64_t y_hi,
                           int t, int64_t ring_lo, int64_t ring_hi, int64_t nrows_buf, cudaStream_t s, Remote rem) {
  if (y_hi < y_lo) return ST_OK;
  switch (t) {
    case 2: return launch_tb4<2>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    case 4: return launch_tb4<4>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    case 6: return launch_tb4<6>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    case 8: return launch_tb4<8>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    case 10: return launch_tb4<10>(src, dst, nx, ld, y_lo, y_hi, ring_lo, ring_hi, nrows_buf, s, rem);
    default: set_error("jacobi2d: tblock=%d not supported (2, 4, 6, 8, 10)", t); return ST_ENOTSUP;
  }
}

}  // namespace st

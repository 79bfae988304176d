// jacobi3d.cu — 3-D 7-point Jacobi sweep (the paper's benchmark 1), sm_100a.
//
// Operation ("a 7-point stencil, the orthogonal neighbours in
// three dimensions, and averages values across the six neighbouring cells";
// value semantics PAPER.md:126; readings R20/R21 of DESIGN.md):
//     dst = (((((Zm + Zp) + Ym) + Yp) + Xm) + Xp) / 6.0
// 5 adds + 1 correctly rounded divide = the paper's 6 flops per cell.
//
// HBM-bound (16 algorithmic bytes per point per sweep). Design = the PW
// kernel's 2.5-D z-streaming skeleton with one field: a CTA owns a BX x BY
// interior column (BX = 128 measured best: longer TMA row segments) and a chunk
// of planes; input planes (tile + 1-cell apron)
// stream through an S-slot shared-memory ring filled by TMA
// (cp.async.bulk.tensor.3d, one elected thread, mbarrier completion); a thread
// owns R consecutive rows of one column, keeps its own column at z-1 and z in
// registers, and reads the four in-plane neighbours from shared memory.
// Dirichlet faces are never written by the sweep kernel; the side faces are
// copied a -> b once per call (jacobi3d_copy_faces).
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "tma.cuh"

namespace st {

namespace {

template <int BX, int BY>
struct J3Tile {
  static constexpr int SX = BX + 2;  // smem row: 1-column apron each side
  static constexpr int SY = BY + 2;
  static constexpr int kPlaneBytes = SX * SY * 8;
  static constexpr int kPlaneStride = ((kPlaneBytes + 127) / 128) * 128 / 8;  // doubles, 128-B aligned
  static constexpr uint32_t kTxBytes = kPlaneBytes;
};

template <int BX, int BY, int S, int R>
__global__ void __launch_bounds__((BX / 32) * (BY / R) * 32)
    jacobi3d_kernel(const __grid_constant__ CUtensorMap tm, double* __restrict__ dst, int64_t nx, int64_t ny,
                    int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t y_first, int64_t y_last,
                    int64_t planes_per_chunk, double* __restrict__ dst2, int64_t delta2) {
  using T = J3Tile<BX, BY>;
  constexpr int kSX = T::SX, WX = BX / 32;
  static_assert(S >= 4 && BY % R == 0 && BX % 32 == 0, "ring depth / rows per thread / tile width");
  extern __shared__ __align__(1024) double ring[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * T::kPlaneStride);

  const int lane = threadIdx.x & 31;
  const int wx = (threadIdx.x >> 5) % WX;
  const int wy = (threadIdx.x >> 5) / WX;
  const int64_t x0 = 1 + (int64_t)blockIdx.x * BX;
  const int64_t y0 = y_first + (int64_t)blockIdx.y * BY;  // output rows [y_first, y_last] (a window for pencils)
  const int64_t za = z_lo + (int64_t)blockIdx.z * planes_per_chunk;
  const int64_t zb = min(z_hi, za + planes_per_chunk - 1);
  const int np = (int)(zb - za + 3);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm);
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int32_t cx = (int32_t)(x0 - 1), cy = (int32_t)(y0 - 1);  // even x start (TMA rule)
  auto issue = [&](int p, int slot) {
    mbar_arrive_expect_tx(&full[slot], T::kTxBytes);
    tma_load_3d(ring + slot * T::kPlaneStride, &tm, cx, cy, (int32_t)(za - 1 + p), &full[slot]);
  };
  if (threadIdx.x == 0)
    for (int p = 0; p < S && p < np; ++p) issue(p, p);

  const int oc = (wy * R + 1) * kSX + 1 + wx * 32 + lane;
  const int64_t yb = y0 + (int64_t)wy * R;
  const int64_t x = x0 + wx * 32 + lane;
  bool ok[R];
#pragma unroll
  for (int i = 0; i < R; ++i) ok[i] = (yb + i <= y_last) && (x <= nx);
  const int64_t plane_elems = (ny + 2) * ldx;
  double* out = dst + (za * (ny + 2) + yb) * ldx + x;
  double* out2 = dst2 ? dst2 + ((za + delta2) * (ny + 2) + yb) * ldx + x : nullptr;  // fused halo swap

  int sm_ = 0, sc = 1, sp = 2;
  uint32_t par_p = 0;
  mbar_wait_parity(&full[0], 0);
  mbar_wait_parity(&full[1], 0);
  double m[R], c[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    m[i] = ring[oc + i * kSX];
    c[i] = ring[T::kPlaneStride + oc + i * kSX];
  }
  for (int j = 0; j + 2 < np; ++j) {
    mbar_wait_parity(&full[sp], par_p);
    const double* C = ring + sc * T::kPlaneStride + oc;
    const double* P = ring + sp * T::kPlaneStride + oc;
    double p[R];
#pragma unroll
    for (int i = 0; i < R; ++i) p[i] = P[i * kSX];
    const double n0 = C[-kSX], sR = C[R * kSX];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double ym = i > 0 ? c[i - 1] : n0;
      const double yp = i + 1 < R ? c[i + 1] : sR;
      const double xm = C[i * kSX - 1], xp = C[i * kSX + 1];
      const double sum = dadd(dadd(dadd(dadd(dadd(m[i], p[i]), ym), yp), xm), xp);
      const double v = ddiv6(sum);  // == __ddiv_rn(sum, 6.0), cheaper (common.cuh)
      if (ok[i]) {
        out[i * ldx] = v;
        if (out2) out2[i * ldx] = v;
      }
    }
    out += plane_elems;
    if (out2) out2 += plane_elems;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      m[i] = c[i];
      c[i] = p[i];
    }
    __syncthreads();
    if (threadIdx.x == 0 && j + S < np) {
      fence_proxy_async_smem();
      issue(j + S, sm_);
    }
    const int nsp = (sp + 1 == S) ? 0 : sp + 1;
    if (nsp == 0) par_p ^= 1u;
    sm_ = sc;
    sc = sp;
    sp = nsp;
  }
}

// Self-test of ddiv6 against the generic correctly rounded division.
__global__ void ddiv6_selftest_kernel(const double* __restrict__ x, int64_t n, unsigned long long* mismatches) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = ddiv6(x[i]), b = __ddiv_rn(x[i], 6.0);
    if (__double_as_longlong(a) != __double_as_longlong(b)) atomicAdd(mismatches, 1ull);
  }
}

// dst's side faces (x = 0, nx+1 and y = 0, ny+1) of planes [z_lo, z_hi] <- src
__global__ void jacobi3d_copy_faces_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nx,
                                           int64_t ny, int64_t ldx, int64_t z_lo, int64_t z_hi) {
  const int64_t per_plane = 2 * (nx + 2) + 2 * ny;
  const int64_t total = per_plane * (z_hi - z_lo + 1);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = z_lo + t / per_plane;
    int64_t k = t % per_plane, y, x;
    if (k < nx + 2) { y = 0; x = k; }
    else if (k < 2 * (nx + 2)) { y = ny + 1; x = k - (nx + 2); }
    else { k -= 2 * (nx + 2); y = 1 + (k >> 1); x = (k & 1) ? nx + 1 : 0; }
    const int64_t g = (z * (ny + 2) + y) * ldx + x;
    dst[g] = src[g];
  }
}

template <int BX, int BY, int S, int R>
st_status launch_j3(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf, int64_t ldx,
                    int64_t z_lo, int64_t z_hi, int64_t y_lo, int64_t y_hi, cudaStream_t s, Remote rem) {
  using T = J3Tile<BX, BY>;
  CUtensorMap tm;
  const uint64_t dims[3] = {(uint64_t)(nx + 2), (uint64_t)(ny + 2), (uint64_t)nplanes_buf};
  const uint32_t box[3] = {(uint32_t)T::SX, (uint32_t)T::SY, 1u};
  ST_TRY(make_tmap_3d_f64(&tm, src, dims, (uint64_t)ldx * 8, (uint64_t)ldx * 8 * (uint64_t)(ny + 2), box));
  const size_t smem = (size_t)S * T::kPlaneStride * sizeof(double) + S * sizeof(uint64_t);
  ST_CHECK_CUDA(cudaFuncSetAttribute(jacobi3d_kernel<BX, BY, S, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  const int64_t ntx = (nx + BX - 1) / BX, nty = (y_hi - y_lo + BY) / BY, nz = z_hi - z_lo + 1;
  static const int kPpc = env_int("ST_J3_PLANES", 64);
  const int64_t ppc = std::max<int64_t>(1, std::min<int64_t>(kPpc, nz));
  const int64_t nzc = (nz + ppc - 1) / ppc;
  ST_RETURN_IF(nty > 65535 || nzc > 65535, ST_ENOTSUP, "jacobi3d: grid too large");
  jacobi3d_kernel<BX, BY, S, R><<<dim3((unsigned)ntx, (unsigned)nty, (unsigned)nzc), (BX / 32) * (BY / R) * 32,
                                  smem, s>>>(
      tm, dst, nx, ny, ldx, z_lo, z_hi, y_lo, y_hi, ppc, rem.base, rem.delta);
  ST_LAUNCHED();
  return ST_OK;
}


// ---- Two sweeps per pass (temporal blocking T = 2). A CTA owns a BX x BY
// interior column and a chunk of the output planes [z_lo, z_hi] of a buffer of
// nplanes_buf planes; planes <= ring_lo / >= ring_hi are Dirichlet planes (the
// single domain: 0 and nz+1; a slab: its global boundary plane, or none — then
// the first sweep also runs on the ghost planes z_lo-1 and z_hi+1, which the
// caller's ghost depth >= 2 provides). Input planes (tile +
// 2-cell apron; the box starts at x0-3 so TMA's 16-byte start rule holds) stream
// through an S-slot TMA ring; for every plane L the CTA first computes the
// first-sweep values of the (BX+2) x (BY+2) region around its tile into a 3-plane
// shared-memory ring (Dirichlet points copy their input value), then the second
// sweep of plane L-1 from that ring. Per point and sweep the arithmetic is the
// single-sweep kernel's (sum order z-, z+, y-, y+, x-, x+, then / 6), so two
// passes of this kernel are bitwise two single sweeps.
#ifndef ST_J3T2_UNROLL
#define ST_J3T2_UNROLL 3
#endif
constexpr int kJ3T2Unroll = ST_J3T2_UNROLL;  // plane-loop unroll (3: the z queues rename instead of copying)

template <int BX, int BY>
struct J3T2Tile {
  static constexpr int SX = BX + 6, SY = BY + 4;            // input tile: x0-3 .. x0+BX+2, y0-2 .. y0+BY+1
  static constexpr int kPlaneBytes = SX * SY * 8;
  static constexpr int kPlaneStride = ((kPlaneBytes + 127) / 128) * 128 / 8;
  static constexpr uint32_t kTxBytes = kPlaneBytes;
  static constexpr int LX = BX + 2, LY = BY + 2;             // first-sweep region: x0-1 .. x0+BX, y0-1 .. y0+BY
  static constexpr int kL0 = LX * LY;
};

template <int BX, int BY, int S, int R, bool kRem, bool kWin>
__global__ void __launch_bounds__((BX / 32) * (BY / R) * 32)
    jacobi3d_t2_kernel(const __grid_constant__ CUtensorMap tm, double* __restrict__ dst, int64_t nx, int64_t ny,
                       int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t ring_lo, int64_t ring_hi,
                       int64_t planes_per_chunk, double* __restrict__ dst2, int64_t delta2, int64_t y_lo,
                       int64_t y_hi, int64_t yring_lo, int64_t yring_hi) {
  using T = J3T2Tile<BX, BY>;
  constexpr int NT = (BX / 32) * (BY / R) * 32, WX = BX / 32;
  if (!kWin) {  // the whole y range, Dirichlet rows 0 and ny+1 (a separate instantiation keeps its registers)
    y_lo = 1;
    y_hi = ny;
    yring_lo = 0;
    yring_hi = ny + 1;
  }
  constexpr int kHalo = 2 * T::LX + 2 * BY;  // first-sweep points outside the BX x BY tile
  static_assert(S >= 4 && BY % R == 0 && BX % 32 == 0 && kHalo <= NT, "ring depth / tile shape");
  extern __shared__ __align__(1024) double ring[];  // [S input planes][4 first-sweep planes][S mbarriers]
  double* l0 = ring + S * T::kPlaneStride;
  uint64_t* full = reinterpret_cast<uint64_t*>(l0 + 4 * T::kL0);

  const int lane = threadIdx.x & 31;
  const int wx = (threadIdx.x >> 5) % WX;
  const int wy = (threadIdx.x >> 5) / WX;
  const int64_t x0 = 1 + (int64_t)blockIdx.x * BX;
  const int64_t y0 = y_lo + (int64_t)blockIdx.y * BY;
  const int64_t za = z_lo + (int64_t)blockIdx.z * planes_per_chunk;
  const int64_t zb = min(z_hi, za + planes_per_chunk - 1);
  const int np = (int)(zb - za + 5);  // input planes za-2 .. zb+2

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm);
    for (int q = 0; q < S; ++q) mbar_init(&full[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int32_t cx = (int32_t)(x0 - 3), cy = (int32_t)(y0 - 2);
  auto issue = [&](int p, int slot) {
    mbar_arrive_expect_tx(&full[slot], T::kTxBytes);
    tma_load_3d(ring + slot * T::kPlaneStride, &tm, cx, cy, (int32_t)(za - 2 + p), &full[slot]);
  };
  if (threadIdx.x == 0)
    for (int p = 0; p < S && p < np; ++p) issue(p, p);

  // Own points: column lx = 1 + wx*32 + lane, rows ly0 .. ly0+R-1 of the first-sweep region
  // (= the thread's output points). Their input and first-sweep z columns ride in registers.
  const int lxo = 1 + wx * 32 + lane, ly0 = 1 + wy * R;
  const int qo = ly0 * T::LX + lxo;                 // first-sweep index of row 0
  const int co = (ly0 + 1) * T::SX + lxo + 2;       // input-tile offset of row 0
  const int64_t x = x0 + wx * 32 + lane, yb = y0 + (int64_t)wy * R;
  bool ok[R], oring[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    ok[i] = (yb + i <= y_hi) && (x <= nx);
    oring[i] = (x == nx + 1) || (kWin ? (yb + i <= yring_lo) || (yb + i >= yring_hi) : yb + i == ny + 1);
  }
  // Halo point (threads < kHalo): rows 0 and LY-1 of the region, then columns 0 and LX-1
  const bool has_h = threadIdx.x < kHalo;
  int hq = 0;
  {
    const int t = threadIdx.x;
    int ly, lx;
    if (t < T::LX) { ly = 0; lx = t; }
    else if (t < 2 * T::LX) { ly = T::LY - 1; lx = t - T::LX; }
    else { const int u = t - 2 * T::LX; ly = 1 + (u >> 1); lx = (u & 1) ? T::LX - 1 : 0; }
    hq = has_h ? ly * T::LX + lx : 0;
  }
  const int hly = hq / T::LX, hlx = hq - hly * T::LX;
  const int hc = (hly + 1) * T::SX + hlx + 2;
  const int64_t hgx = x0 - 1 + hlx, hgy = y0 - 1 + hly;
  const bool hring = hgx == 0 || hgx == nx + 1 ||
                     (kWin ? hgy <= yring_lo || hgy >= yring_hi : hgy == 0 || hgy == ny + 1);

  const int64_t plane_elems = (ny + 2) * ldx;
  double* out = dst + (za * (ny + 2) + yb) * ldx + x;
  // fused halo swap (kRem: a separate instantiation, the plain one keeps its registers)
  double* out2 = kRem ? dst2 + ((za + delta2) * (ny + 2) + yb) * ldx + x : nullptr;

  mbar_wait_parity(&full[0], 0);
  mbar_wait_parity(&full[1], 0);
  double im[R], ic[R], ip[R];  // input, own column: planes L-1, L, L+1
  double am[R], ac[R], ap[R];  // first sweep, own column: planes O-1, O, O+1 (O = L-1)
#pragma unroll
  for (int i = 0; i < R; ++i) {
    im[i] = ring[co + i * T::SX];
    ic[i] = ring[T::kPlaneStride + co + i * T::SX];
    am[i] = ac[i] = 0.0;
  }
  double him = ring[hc], hic = ring[T::kPlaneStride + hc];

  // ring slots of input planes j, j+1, j+2 and the fill parity of plane j+2's slot
  // (counters, not j % S and j / S: S = 5 is no power of two)
  int slot_m = 0, s1 = 1, s2 = 2;
  uint32_t par2 = 0;
#pragma unroll kJ3T2Unroll
  for (int j = 0; j < np - 2; ++j) {  // first-sweep planes za-1 .. zb+1
    mbar_wait_parity(&full[s2], par2);
    const int64_t L = za - 1 + j;
    const double* Ic = ring + s1 * T::kPlaneStride;
    const double* Ip = ring + s2 * T::kPlaneStride;
    double* Lout = l0 + (int)(L & 3) * T::kL0;  // 4 slots: a mask, not a 64-bit modulo
    const bool zring = (L <= ring_lo) || (L >= ring_hi);
    // ---- first sweep of plane L: own points (z and own-row y neighbours from registers)
#pragma unroll
    for (int i = 0; i < R; ++i) ip[i] = Ip[co + i * T::SX];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int c = co + i * T::SX;
      const double ym = i > 0 ? ic[i - 1] : Ic[c - T::SX];
      const double yp = i + 1 < R ? ic[i + 1] : Ic[c + T::SX];
      const double sum = dadd(dadd(dadd(dadd(dadd(im[i], ip[i]), ym), yp), Ic[c - 1]), Ic[c + 1]);
      const double v = (zring || oring[i]) ? ic[i] : ddiv6(sum);  // Dirichlet: unchanged by the sweep
      ap[i] = v;
      Lout[qo + i * T::LX] = v;
    }
    // ---- first sweep of plane L: the halo point
    if (has_h) {
      const double hip = Ip[hc];
      const double sum = dadd(dadd(dadd(dadd(dadd(him, hip), Ic[hc - T::SX]), Ic[hc + T::SX]), Ic[hc - 1]), Ic[hc + 1]);
      Lout[hq] = (zring || hring) ? hic : ddiv6(sum);
      him = hic;
      hic = hip;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      im[i] = ic[i];
      ic[i] = ip[i];
    }
    __syncthreads();
    // One barrier per plane: input plane index j (slot slot_m) was last read from shared
    // memory in step j-1, and the first-sweep slot step j+1 writes, (L+1) & 3 = plane L-3,
    // was last read by step j-2's second sweep — both before this barrier; the only
    // shared-memory reads of the first-sweep ring (plane L-1 below) follow step j-1's barrier.
    if (threadIdx.x == 0 && j + S < np) {
      fence_proxy_async_smem();
      issue(j + S, slot_m);
    }
    // ---- second sweep of plane O = L-1: z neighbours from registers, in-plane from the ring
    if (j >= 2) {
      const double* Zc = l0 + (int)((L - 1) & 3) * T::kL0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int q = qo + i * T::LX;
        const double ym = i > 0 ? ac[i - 1] : Zc[q - T::LX];
        const double yp = i + 1 < R ? ac[i + 1] : Zc[q + T::LX];
        const double sum = dadd(dadd(dadd(dadd(dadd(am[i], ap[i]), ym), yp), Zc[q - 1]), Zc[q + 1]);
        if (ok[i]) {
          const double v = ddiv6(sum);
          out[i * ldx] = v;
          if (kRem) out2[i * ldx] = v;
        }
      }
      out += plane_elems;
      if (kRem) out2 += plane_elems;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      am[i] = ac[i];
      ac[i] = ap[i];
    }
    slot_m = s1;
    s1 = s2;
    s2 = s2 + 1 == S ? 0 : s2 + 1;
    par2 ^= s2 == 0 ? 1u : 0u;
  }
}

template <int BX, int BY, int S, int R>
st_status launch_j3t2(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf, int64_t ldx,
                      int64_t z_lo, int64_t z_hi, int64_t ring_lo, int64_t ring_hi, int64_t y_lo, int64_t y_hi,
                      int64_t yring_lo, int64_t yring_hi, cudaStream_t s, Remote rem) {
  using T = J3T2Tile<BX, BY>;
  CUtensorMap tm;
  const uint64_t dims[3] = {(uint64_t)(nx + 2), (uint64_t)(ny + 2), (uint64_t)nplanes_buf};
  const uint32_t box[3] = {(uint32_t)T::SX, (uint32_t)T::SY, 1u};
  ST_TRY(make_tmap_3d_f64(&tm, src, dims, (uint64_t)ldx * 8, (uint64_t)ldx * 8 * (uint64_t)(ny + 2), box));
  const size_t smem = (size_t)S * T::kPlaneStride * sizeof(double) + 4 * T::kL0 * sizeof(double) +
                      S * sizeof(uint64_t);
  const bool win = y_lo != 1 || y_hi != ny || yring_lo != 0 || yring_hi != ny + 1;
  ST_RETURN_IF(win && rem.base, ST_ENOTSUP, "jacobi3d: row windows with the fused swap");
  auto kern = rem.base ? jacobi3d_t2_kernel<BX, BY, S, R, true, false>
                       : (win ? jacobi3d_t2_kernel<BX, BY, S, R, false, true> : jacobi3d_t2_kernel<BX, BY, S, R, false, false>);
  ST_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntx = (nx + BX - 1) / BX, nty = (y_hi - y_lo + BY) / BY, nz = z_hi - z_lo + 1;
  static const int kPpc = env_int("ST_J3T2_PLANES", 96);
  const int64_t ppc = std::max<int64_t>(1, std::min<int64_t>(kPpc, nz));
  const int64_t nzc = (nz + ppc - 1) / ppc;
  ST_RETURN_IF(nty > 65535 || nzc > 65535, ST_ENOTSUP, "jacobi3d: grid too large");
  kern<<<dim3((unsigned)ntx, (unsigned)nty, (unsigned)nzc), (BX / 32) * (BY / R) * 32, smem, s>>>(tm, dst, nx, ny, ldx, z_lo, z_hi, ring_lo, ring_hi, ppc,
                                                rem.base, rem.delta, y_lo, y_hi, yring_lo, yring_hi);
  ST_LAUNCHED();
  return ST_OK;
}
}  // namespace

st_status jacobi3d_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi3d_kernel<128, 8, 8, 2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi3d_copy_faces_kernel));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi3d_t2_kernel<128, 8, 5, 2, false, false>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi3d_t2_kernel<128, 8, 5, 2, true, false>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, jacobi3d_t2_kernel<128, 8, 5, 2, false, true>));
  return ST_OK;
}

st_status jacobi3d_two_sweeps(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                              int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t ring_lo, int64_t ring_hi,
                              cudaStream_t s, Remote rem) {
  return jacobi3d_two_sweeps_block(src, dst, nx, ny, nplanes_buf, ldx, z_lo, z_hi, ring_lo, ring_hi, 1, ny, 0, ny + 1,
                                   s, rem);
}

st_status jacobi3d_two_sweeps_block(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                                    int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t ring_lo, int64_t ring_hi,
                                    int64_t y_lo, int64_t y_hi, int64_t yring_lo, int64_t yring_hi, cudaStream_t s,
                                    Remote rem) {
  if (z_hi < z_lo || y_hi < y_lo) return ST_OK;
  return launch_j3t2<128, 8, 5, 2>(src, dst, nx, ny, nplanes_buf, ldx, z_lo, z_hi, ring_lo, ring_hi, y_lo, y_hi,
                                   yring_lo, yring_hi, s, rem);  // §6.5
}

st_status jacobi3d_sweep_block(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                               int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t y_lo, int64_t y_hi, cudaStream_t s,
                               Remote rem) {
  if (z_hi < z_lo || y_hi < y_lo) return ST_OK;
  return launch_j3<128, 8, 8, 2>(src, dst, nx, ny, nplanes_buf, ldx, z_lo, z_hi, y_lo, y_hi, s, rem);
}

st_status jacobi3d_sweep_planes(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                                int64_t ldx, int64_t z_lo, int64_t z_hi, cudaStream_t s, Remote rem) {
  return jacobi3d_sweep_block(src, dst, nx, ny, nplanes_buf, ldx, z_lo, z_hi, 1, ny, s, rem);
}

st_status ddiv6_selftest(const double* x, int64_t n, unsigned long long* mismatches, cudaStream_t s) {
  ddiv6_selftest_kernel<<<148 * 8, 256, 0, s>>>(x, n, mismatches);
  ST_LAUNCHED();
  return ST_OK;
}

st_status jacobi3d_copy_faces(const double* src, double* dst, int64_t nx, int64_t ny, int64_t ldx, int64_t z_lo,
                              int64_t z_hi, cudaStream_t s) {
  if (z_hi < z_lo) return ST_OK;
  const int64_t total = (2 * (nx + 2) + 2 * ny) * (z_hi - z_lo + 1);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  jacobi3d_copy_faces_kernel<<<blocks, 256, 0, s>>>(src, dst, nx, ny, ldx, z_lo, z_hi);
  ST_LAUNCHED();
  return ST_OK;
}

}  // namespace st

// pw_advect3d.cu — fused Piacsek-Williams advection, 2.5-D z-streaming, sm_100a.
//
// Operation: PAPER.md:216 ("three separate stencil computations across three
// fields which are then fused ... into a single stencil region", 63 flops per
// cell), formula and association trees = DESIGN.md reading R6 (MONC
// pwadvection form); every binary op rounds once.
//
// Design (HBM-bound: 48 algorithmic bytes per point, 63 fp64 flops):
//  * A CTA owns a BX(x) x BY(y) = 128 x 8 tile of the interior and streams a
//    chunk of up to 128 z planes. Each input plane of u, v, w (with a 1-cell
//    x/y apron) is brought into a shared-memory ring of S = 5 plane slots by
//    three TMA tile loads (cp.async.bulk.tensor.3d, issued by one thread,
//    completed on an mbarrier), so S-3 planes are in flight while the CTA computes.
//  * Tiles are aligned to the interior (x0 = 1 + BX*bx): the TMA box then starts
//    at the even coordinate x0-1, which TMA requires (the innermost start
//    coordinate must be a multiple of 16 bytes; odd fp64 coordinates fault).
//  * A thread owns R = 4 consecutive rows of one column; its own column of u, v,
//    w at planes z-1, z rides in registers and neighbours shared by its R points
//    come from registers, the rest are 8-byte shared loads (11 + 10/R per point).
//    Outputs are coalesced 8-byte stores straight to HBM; halo cells of su, sv,
//    sw are never written.
//  * An output row window [y_first, y_last] lets the pencil decomposition
//    advect the ghost-free block while the halo is in flight.
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "tma.cuh"

namespace st {

namespace {

constexpr int kMaxPlanesPerChunk = 256;

#ifndef ST_PW_UNROLL
#define ST_PW_UNROLL 1
#endif
constexpr int kPwUnroll = ST_PW_UNROLL;  // plane-loop unroll of pw_advect3d_kernel

template <int BX, int BY>
struct PwTile {
  static constexpr int SX = BX + 2;  // smem row: 1-column apron each side
  static constexpr int SY = BY + 2;
  static constexpr int kPlaneElems = SX * SY;
  static constexpr int kPlaneBytes = kPlaneElems * 8;
  static constexpr int kPlaneStride = ((kPlaneBytes + 127) / 128) * 128 / 8;  // doubles
  static constexpr int kSlotStride = 3 * kPlaneStride;                        // u, v, w
  static constexpr uint32_t kTxBytes = 3u * kPlaneBytes;
};

// The 27 input values one output point reads (names: field_offset; c = centre,
// w/e = x-1/x+1, n/s = y-1/y+1, m/p = z-1/z+1, combined offsets spelled out).
struct PwPoint {
  double uc, uw, ue, un, us, um, up, u_sw, u_pw;   // u_sw = U(0,+1,-1), u_pw = U(+1,0,-1)
  double vc, vw, ve, vn, vs, vm, vp, v_ne, v_pn;   // v_ne = V(0,-1,+1), v_pn = V(+1,-1,0)
  double wc, ww, we, wn, ws, wm, wp, w_me, w_ms;   // w_me = W(-1,0,+1), w_ms = W(-1,+1,0)
};

struct PwCoef {
  double tcx, tcy, c1, c2, d1, d2;
};

// DESIGN.md R6; operand order mirrors the paper reading, grouping is what matters.
__device__ __forceinline__ void pw_point(const PwPoint& p, const PwCoef& k, double& su, double& sv,
                                         double& sw) {
  double t1, t2, xs, ys, zs;
  t1 = dmul(p.uw, dadd(p.uc, p.uw));
  t2 = dmul(p.ue, dadd(p.uc, p.ue));
  xs = dmul(k.tcx, dsub(t1, t2));
  t1 = dmul(p.un, dadd(p.vn, p.v_ne));
  t2 = dmul(p.us, dadd(p.vc, p.ve));
  ys = dmul(k.tcy, dsub(t1, t2));
  t1 = dmul(dmul(k.c1, p.um), dadd(p.wm, p.w_me));
  t2 = dmul(dmul(k.c2, p.up), dadd(p.wc, p.we));
  zs = dsub(t1, t2);
  su = dadd(dadd(xs, ys), zs);

  t1 = dmul(p.vw, dadd(p.uw, p.u_sw));
  t2 = dmul(p.ve, dadd(p.uc, p.us));
  xs = dmul(k.tcx, dsub(t1, t2));
  t1 = dmul(p.vn, dadd(p.vc, p.vn));
  t2 = dmul(p.vs, dadd(p.vc, p.vs));
  ys = dmul(k.tcy, dsub(t1, t2));
  t1 = dmul(dmul(k.c1, p.vm), dadd(p.wm, p.w_ms));
  t2 = dmul(dmul(k.c2, p.vp), dadd(p.wc, p.ws));
  zs = dsub(t1, t2);
  sv = dadd(dadd(xs, ys), zs);

  t1 = dmul(p.ww, dadd(p.uw, p.u_pw));
  t2 = dmul(p.we, dadd(p.uc, p.up));
  xs = dmul(k.tcx, dsub(t1, t2));
  t1 = dmul(p.wn, dadd(p.vn, p.v_pn));
  t2 = dmul(p.ws, dadd(p.vc, p.vp));
  ys = dmul(k.tcy, dsub(t1, t2));
  t1 = dmul(dmul(k.d1, p.wm), dadd(p.wc, p.wm));
  t2 = dmul(dmul(k.d2, p.wp), dadd(p.wc, p.wp));
  zs = dsub(t1, t2);
  sw = dadd(dadd(xs, ys), zs);
}

// R consecutive rows per thread (BY = R x warps): neighbours shared by the
// thread's own points come from registers, so shared loads per point drop from
// 21 (R=1) to 11 + 10/R, and the R points give the scheduler independent work.
template <int BX, int BY, int S, int R>
__global__ void __launch_bounds__((BX / 32) * (BY / R) * 32)
    pw_advect3d_kernel(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_v,
                       const __grid_constant__ CUtensorMap tm_w, double* __restrict__ su,
                       double* __restrict__ sv, double* __restrict__ sw, int64_t nx, int64_t ny,
                       int64_t ldx, double tcx, double tcy, const double* __restrict__ tzc1,
                       const double* __restrict__ tzc2, const double* __restrict__ tzd1,
                       const double* __restrict__ tzd2, int64_t z_lo, int64_t z_hi, int64_t y_first,
                       int64_t y_last, int64_t planes_per_chunk) {
  using T = PwTile<BX, BY>;
  constexpr int kSX = T::SX, WX = BX / 32;
  static_assert(S >= 4, "ring needs planes z-1, z, z+1 and at least one in flight");
  static_assert(BY % R == 0 && BX % 32 == 0, "BY = R x warp rows, BX = 32 x warp columns");
  // Dynamic smem only (TMA destinations at an aligned base):
  // [ring: S slots x (u, v, w)][coef: (tzc1,tzc2,tzd1,tzd2) per output plane][S mbarriers]
  extern __shared__ __align__(1024) double ring[];
  double4* coef = reinterpret_cast<double4*>(ring + S * T::kSlotStride);
  uint64_t* full = reinterpret_cast<uint64_t*>(coef + kMaxPlanesPerChunk);

  const int lane = threadIdx.x & 31;
  const int wx = (threadIdx.x >> 5) % WX;
  const int wy = (threadIdx.x >> 5) / WX;
  const int64_t x0 = 1 + (int64_t)blockIdx.x * BX;
  const int64_t y0 = y_first + (int64_t)blockIdx.y * BY;  // output rows [y_first, y_last] (pencils: windows)
  const int64_t za = z_lo + (int64_t)blockIdx.z * planes_per_chunk;
  const int64_t zb = min(z_hi, za + planes_per_chunk - 1);
  const int np = (int)(zb - za + 3);  // input planes za-1 .. zb+1

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_u);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_w);
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  for (int j = threadIdx.x; j < np - 2; j += blockDim.x)
    coef[j] = make_double4(__ldg(tzc1 + za + j), __ldg(tzc2 + za + j), __ldg(tzd1 + za + j),
                           __ldg(tzd2 + za + j));
  __syncthreads();

  const int32_t cx = (int32_t)(x0 - 1), cy = (int32_t)(y0 - 1);  // cx even: TMA alignment rule
  auto issue = [&](int p, int slot) {  // input plane za-1+p -> ring slot
    double* dstp = ring + slot * T::kSlotStride;
    uint64_t* bar = &full[slot];
    mbar_arrive_expect_tx(bar, T::kTxBytes);
    const int32_t cz = (int32_t)(za - 1 + p);
    tma_load_3d(dstp, &tm_u, cx, cy, cz, bar);
    tma_load_3d(dstp + T::kPlaneStride, &tm_v, cx, cy, cz, bar);
    tma_load_3d(dstp + 2 * T::kPlaneStride, &tm_w, cx, cy, cz, bar);
  };
  if (threadIdx.x == 0)
    for (int p = 0; p < S && p < np; ++p) issue(p, p);

  constexpr int PS = T::kPlaneStride;
  const int oc = (wy * R + 1) * kSX + 1 + wx * 32 + lane;  // first own cell inside a field plane
  const int64_t yb = y0 + (int64_t)wy * R;
  const int64_t x = x0 + wx * 32 + lane;
  bool ok[R];
#pragma unroll
  for (int i = 0; i < R; ++i) ok[i] = (yb + i <= y_last) && (x <= nx);
  const int64_t plane_elems = (ny + 2) * ldx;
  const int64_t g0 = (za * (ny + 2) + yb) * ldx + x;
  double* pu = su + g0;
  double* pv = sv + g0;
  double* pw = sw + g0;

  // ring slots of input planes j (m), j+1 (c), j+2 (p); parity of slot sp's next phase
  int sm_ = 0, sc = 1, sp = 2;
  uint32_t par_p = 0;
  mbar_wait_parity(&full[0], 0);
  mbar_wait_parity(&full[1], 0);
  double um[R], vm[R], wm[R], uc[R], vc[R], wc[R];  // own column at planes z-1, z
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int o = oc + i * kSX;
    um[i] = ring[o]; vm[i] = ring[PS + o]; wm[i] = ring[2 * PS + o];
    uc[i] = ring[T::kSlotStride + o]; vc[i] = ring[T::kSlotStride + PS + o]; wc[i] = ring[T::kSlotStride + 2 * PS + o];
  }

#pragma unroll kPwUnroll
  for (int j = 0; j + 2 < np; ++j) {  // output plane za+j from input planes j, j+1, j+2
    mbar_wait_parity(&full[sp], par_p);
    const double* U0 = ring + sc * T::kSlotStride + oc;
    const double* V0 = U0 + PS;
    const double* W0 = U0 + 2 * PS;
    const double* Up = ring + sp * T::kSlotStride + oc;
    const double* Vp = Up + PS;
    const double* Wp = Up + 2 * PS;
    const double* Wm = ring + sm_ * T::kSlotStride + 2 * PS + oc;

    double up[R], vp[R], wp[R];
#pragma unroll
    for (int i = 0; i < R; ++i) { up[i] = Up[i * kSX]; vp[i] = Vp[i * kSX]; wp[i] = Wp[i * kSX]; }
    // centre column of plane z at the apron rows -1 and R
    const double u_n0 = U0[-kSX], u_sR = U0[R * kSX];
    const double v_n0 = V0[-kSX], v_sR = V0[R * kSX];
    const double w_n0 = W0[-kSX], w_sR = W0[R * kSX];
    const double vp_n0 = Vp[-kSX];          // V(+1,-1,0) of row 0
    const double u_wR = U0[R * kSX - 1];    // U(0,+1,-1) of row R-1
    const double v_e_1 = V0[-kSX + 1];      // V(0,-1,+1) of row 0
    const double wm_sR = Wm[R * kSX];       // W(-1,+1,0) of row R-1
    const double4 cz = coef[j];
    const PwCoef k = {tcx, tcy, cz.x, cz.y, cz.z, cz.w};
    double uw[R], ue[R], vw[R], ve[R], ww[R], we[R], upw[R], wme[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      uw[i] = U0[i * kSX - 1]; ue[i] = U0[i * kSX + 1];
      vw[i] = V0[i * kSX - 1]; ve[i] = V0[i * kSX + 1];
      ww[i] = W0[i * kSX - 1]; we[i] = W0[i * kSX + 1];
      upw[i] = Up[i * kSX - 1];  // U(+1,0,-1)
      wme[i] = Wm[i * kSX + 1];  // W(-1,0,+1)
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      PwPoint q;
      q.uc = uc[i]; q.vc = vc[i]; q.wc = wc[i];
      q.um = um[i]; q.vm = vm[i]; q.wm = wm[i];
      q.up = up[i]; q.vp = vp[i]; q.wp = wp[i];
      q.uw = uw[i]; q.ue = ue[i]; q.vw = vw[i]; q.ve = ve[i]; q.ww = ww[i]; q.we = we[i];
      q.un = i > 0 ? uc[i - 1] : u_n0;
      q.vn = i > 0 ? vc[i - 1] : v_n0;
      q.wn = i > 0 ? wc[i - 1] : w_n0;
      q.us = i + 1 < R ? uc[i + 1] : u_sR;
      q.vs = i + 1 < R ? vc[i + 1] : v_sR;
      q.ws = i + 1 < R ? wc[i + 1] : w_sR;
      q.u_sw = i + 1 < R ? uw[i + 1] : u_wR;   // U(0,+1,-1)
      q.v_ne = i > 0 ? ve[i - 1] : v_e_1;      // V(0,-1,+1)
      q.u_pw = upw[i];                          // U(+1,0,-1)
      q.v_pn = i > 0 ? vp[i - 1] : vp_n0;      // V(+1,-1,0)
      q.w_me = wme[i];                          // W(-1,0,+1)
      q.w_ms = i + 1 < R ? wm[i + 1] : wm_sR;  // W(-1,+1,0)
      double ou, ov, ow;
      pw_point(q, k, ou, ov, ow);
      if (ok[i]) {
        pu[i * ldx] = ou;
        pv[i * ldx] = ov;
        pw[i * ldx] = ow;
      }
    }
    pu += plane_elems;
    pv += plane_elems;
    pw += plane_elems;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      um[i] = uc[i]; vm[i] = vc[i]; wm[i] = wc[i];
      uc[i] = up[i]; vc[i] = vp[i]; wc[i] = wp[i];
    }

    // every read of input plane j (slot sm_) is done -> refill it with plane j+S
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

template <int BX, int BY, int S, int R>
st_status launch_pw(const PwArgs& a, int64_t z_lo, int64_t z_hi, cudaStream_t s) {
  using T = PwTile<BX, BY>;
  CUtensorMap tm[3];
  const double* f[3] = {a.u, a.v, a.w};
  const uint64_t dims[3] = {(uint64_t)(a.nx + 2), (uint64_t)(a.ny + 2), (uint64_t)(a.nz + 2)};
  const uint32_t box[3] = {(uint32_t)T::SX, (uint32_t)T::SY, 1u};
  for (int i = 0; i < 3; ++i)
    ST_TRY(make_tmap_3d_f64(&tm[i], f[i], dims, (uint64_t)a.ldx * 8,
                            (uint64_t)a.ldx * 8 * (uint64_t)(a.ny + 2), box));
  const size_t smem = (size_t)S * T::kSlotStride * sizeof(double) + kMaxPlanesPerChunk * sizeof(double4) +
                      S * sizeof(uint64_t);
  ST_CHECK_CUDA(cudaFuncSetAttribute(pw_advect3d_kernel<BX, BY, S, R>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntx = (a.nx + BX - 1) / BX;
  const int64_t y_lo = a.y_lo, y_hi = a.y_hi < 0 ? a.ny : a.y_hi;
  if (y_hi < y_lo) return ST_OK;
  const int64_t nty = (y_hi - y_lo + BY) / BY;
  const int64_t nz = z_hi - z_lo + 1;
  static const int kPpc = env_int("ST_PW_PLANES", 128);
  const int64_t ppc = std::max<int64_t>(1, std::min<int64_t>(std::min(kPpc, kMaxPlanesPerChunk), nz));
  const int64_t nzc = (nz + ppc - 1) / ppc;
  ST_RETURN_IF(nty > 65535 || nzc > 65535, ST_ENOTSUP, "pw_advect3d: grid too large");
  dim3 grid((unsigned)ntx, (unsigned)nty, (unsigned)nzc);
  pw_advect3d_kernel<BX, BY, S, R><<<grid, (BX / 32) * (BY / R) * 32, smem, s>>>(tm[0], tm[1], tm[2], a.su, a.sv, a.sw, a.nx,
                                                        a.ny, a.ldx, a.tcx, a.tcy, a.tzc1, a.tzc2,
                                                        a.tzd1, a.tzd2, z_lo, z_hi, y_lo, y_hi, ppc);
  ST_LAUNCHED();
  return ST_OK;
}

}  // namespace

st_status pw_advect3d_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, pw_advect3d_kernel<128, 8, 5, 4>));
  return ST_OK;
}

st_status pw_advect3d_planes(const PwArgs& a, int64_t z_lo, int64_t z_hi, cudaStream_t s) {
  if (z_hi < z_lo) return ST_OK;
  return launch_pw<128, 8, 5, 4>(a, z_lo, z_hi, s);  // tuned on B200
}

}  // namespace st

// gauss_seidel2d_ms.cu — Listing 1 taken literally (in-place lexicographic
// Gauss-Seidel; R22; NEXT #4) with several sweeps
// in flight per warp: temporal blocking of the wavefront.
//
//   data(j,i) = (data(j,i-1)+data(j,i+1)+data(j-1,i)+data(j+1,i)) * 0.25
//
// N (row y-1) and W (column x-1) are this sweep's values, S and E the previous
// sweep's. A point's value after sweep s depends on (y-1, x) and (y, x-1) after
// sweep s and on (y+1, x), (y, x+1) after sweep s-1; every schedule that
// respects these four dependencies and evaluates each point with the same
// association order reproduces the sequential loop nest bit for bit.
//
// Schedule. A warp owns a strip of 32 rows (lane r = row y0 + r) and walks the
// columns with a one-column skew per lane, as the single-sweep kernel does, but
// it runs KC sweeps ("chains") at once: at step k, lane r computes column
// x_j = k + 1 - r - 2j of sweep s + j for j = 0..KC-1. Chain j trails chain
// j-1 by two columns, so every input of chain j is a register holding a result
// of the PREVIOUS step:
//   E_j = lane r's chain j-1 result (column x_j + 1, sweep s+j-1),
//   S_j = lane r+1's chain j-1 result (shuffle),
//   N_j = lane r-1's chain j result (shuffle),
//   W_j = the lane's own chain j result;
// chain 0 reads E and S (sweep s-1 values) from a shared-memory tile ring. The
// KC updates of a step are therefore independent of each other — a warp keeps
// KC shuffle->4-op chains in flight where the single-sweep kernel kept one (with
// a one-column lag the chains of a step would depend on each other and issue
// one after another).
//
// Ghost rows. Chain j at lane 31 would need row y0+32 after sweep s+j-1, which
// the strip below computes. Instead the strip below's first KC-1 rows are
// recomputed here as ghost rows: a strip owns R = 33 - K rows (lanes 0..R-1)
// and lanes R..31 hold the next K-1 rows, whose chain j is exact for lanes
// r <= 31 - j (their S comes from the lane below, exact one chain earlier; lane
// 31's chain 0 reads row y0+32 from the tile). Ghost results are never written
// back. The last strip has no strip below: it owns up to 32 rows, and its last
// real lane takes S_j from the Dirichlet row (the tile value, delayed j steps).
//
// Strip-to-strip data. Lane 0's N_j is row y0-1 after sweep s+j: the strip
// above's last real row, which that strip publishes as "edge entries"
// (v_0[c], v_1[c-2], ..., v_{KC-1}[c-2KC+2]) — exactly what its lane R-1
// computes in one step — into a global edge buffer. The ghost rows read the
// strip below's rows as of the previous pass, which that strip writes back.
//
// Warp roles. A CTA holds 4 strips, each served by three warps: compute (warp
// ids 8..11), loader (4..7) and storer (0..3), so SMSP w % 4 runs one of each.
// The loader streams 16-column tiles of the strip's 33 rows and the above
// entries into a 10-tile shared-memory ring (16-byte cp.async, completion on an
// mbarrier) once the neighbours' progress words allow; the storer writes
// finished tiles back, copies edge entries out and publishes progress (release
// store): the compute warp never waits on global memory or a fence. Helpers
// sleep between tests of their waits. Tile rows are stored rotated (column
// c of row rho at ring position c + rho + 2KC - 4) so every shared-memory access
// of the compute warp is lane-independent: one base register per group plus an
// immediate offset (a mirrored tail absorbs the ring wrap inside a group).
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "tma.cuh"

namespace st {

namespace {

constexpr int kMsStrips = 4;          // strips per CTA (compute warps 8..11, loaders 4..7, storers 0..3)
constexpr int kMsTW = 16;             // tile width (columns) = steps per compute group
constexpr int kMsSlots = 10;          // tiles in the ring per strip
constexpr int kMsNP = kMsTW * kMsSlots;  // ring positions per row
#ifndef ST_GS_MS_P
#define ST_GS_MS_P 2
#endif
constexpr int kMsP = ST_GS_MS_P;      // shared-memory prefetch distance (steps)
constexpr int kMsProgStride = 16;     // u64 per progress word (one 128-byte line each)
constexpr int kMsMinTiles = 24;       // narrower grids take the single-sweep kernel (helper/compute coupling)
// helper wait loops sleep between tests (ns): a spinning helper takes issue slots and
// shared-memory / L1TEX bandwidth from the compute warp on its SMSP
#ifndef ST_GS_MS_SSLEEP
#define ST_GS_MS_SSLEEP 2000  // storer: a tile is finished every ~2 us
#endif
#ifndef ST_GS_MS_LSLEEP
#define ST_GS_MS_LSLEEP 500   // loader, slot wait (it runs several tiles ahead)
#endif
#ifndef ST_GS_MS_PSLEEP
#define ST_GS_MS_PSLEEP 200   // loader, neighbour progress polls
#endif
constexpr int kMsEdgePad = 8;         // edge entries per strip: columns 0 .. nx + 2K - 2 (< nx + 8)

template <int KC>
struct MsGeo {
  static constexpr int kEntD = KC == 1 ? 2 : KC == 3 ? 4 : KC;  // doubles per edge entry (a 16-byte multiple)
  static constexpr int EB = 8 * kEntD;
  static constexpr int MIR = kMsP + 2 * KC + 1;    // mirrored tail of a tile row (reads reach base+TW-1+P+2KC-2)
  static constexpr int L = (kMsNP + MIR + 1) | 1;  // row length in doubles, odd: conflict-free column access
  static constexpr int ROWB = 8 * L;
  static constexpr int TILE_B = 33 * ROWB;
  static constexpr int MIRA = kMsP + 2;            // mirrored tail of the above-entry ring
  static constexpr int ABOVE_OFF = (TILE_B + 15) / 16 * 16;
  static constexpr int ABOVE_B = (kMsNP + MIRA) * EB;
  static constexpr int STAGE_OFF = ABOVE_OFF + ABOVE_B;
  static constexpr int STAGE_B = kMsNP * EB;
  static constexpr int BAR_OFF = STAGE_OFF + STAGE_B;
  static constexpr int STRIP_B = (BAR_OFF + 3 * kMsSlots * 8 + 127) / 128 * 128;
  static constexpr int CTA_B = kMsStrips * STRIP_B;
  // a tile is finished (results of its columns final, its edge entries staged)
  // kLagT groups after its own: stores of step k reach back to column k - 28 - 2KC
  static constexpr int kLagT = (27 + 2 * KC) / kMsTW + 1;
  static constexpr int SH = 2 * KC;                // S history ring (the sd lane's S_j = S_0 of step k - 2j)
  static constexpr int DR = 2 * KC - 2;            // ring offset of chain 0's reads (E, S) from the step
};

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
__device__ __forceinline__ double lds1(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void lds1_if(bool p, uint32_t a, double& v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}"
               : "+d"(v)
               : "r"(a), "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ double2 lds2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts1_if(bool p, uint32_t a, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}" ::"r"(a), "d"(v),
               "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ void sts2_if(bool p, uint32_t a, double x, double y) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(a),
               "d"(x), "d"(y), "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ void cp8(uint32_t s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
// Helper-warp waits test and then __nanosleep: a spinning helper takes issue slots
// and L1TEX bandwidth from the compute warp on its SMSP (measured: a try_wait loop
// with a suspend hint ran every ~20 ns in this kernel; sleeping 2 us in the storer
// and 0.2-0.5 us in the loader gave +4 %).
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct MsArgs {
  double* a;
  int nx;
  int64_t ny, ld;
  int64_t passes;  // KC-sweep passes of this launch
  int R;           // rows owned by every strip but the last (= 33 - K of the run)
  int nstrips, ntiles;
  unsigned long long* prog;  // prog[I * kMsProgStride] = tiles of strip I written back and edge-published
  char* edge;                // edge[I] = nx + kMsEdgePad entries of EB bytes
  int64_t edge_stride;       // bytes per strip
};

// Per-lane constants of the compute warp.
struct MsLane {
  bool top;    // lane 0: N from the above entries
  bool sd;     // last strip's last real lane: S of chains >= 1 from the Dirichlet row
  bool stage;  // lane R-1 of a strip with a strip below: writes the edge entries
  double w0, eD;
  int lane, nx, R;
};

template <int KC>
struct MsState {
  double res[KC];           // chain results of the previous step
  double pe[kMsP], ps[kMsP];  // prefetched E and S of chain 0
  double pa[kMsP][KC];      // prefetched above entries (lane 0)
  double sh[2 * KC];        // chain 0's S of the last 2KC steps (sh[k % 2KC] = step k)
};

// Loads step k's chain-0 inputs (E, S: tile rows r and r+1 at ring position
// base + d + 2KC - 2; the above entry at base + d + 1) into prefetch slot d % P.
template <int KC, bool kChk>
__device__ __forceinline__ void ms_prefetch(MsState<KC>& S, const uint32_t gt, const uint32_t ga, const int d,
                                            const int k, const MsLane& L) {
  using G = MsGeo<KC>;
  const int q = d % kMsP;
  const uint32_t ot = (uint32_t)(d + G::DR) * 8u;
  if (kChk) {  // never read a position of a column before this pass (the helper may be refilling it)
    const bool ok = k + 1 - L.lane >= 0;
    lds1_if(ok, gt + ot, S.pe[q]);
    lds1_if(ok, gt + G::ROWB + ot, S.ps[q]);
  } else {
    S.pe[q] = lds1(gt + ot);
    S.ps[q] = lds1(gt + G::ROWB + ot);
  }
  const uint32_t oa = ga + (uint32_t)(d + 1) * G::EB;
  if (KC == 1) {
    S.pa[q][0] = lds1(oa);
  } else {
#pragma unroll
    for (int j = 0; j < KC; j += 2) {
      const double2 v = lds2(oa + 8 * j);
      S.pa[q][j] = v.x;
      if (j + 1 < KC) S.pa[q][j + 1] = v.y;
    }
  }
}

// One group of 32 steps (k = k0 .. k0+31); gt/ga/gs = this lane's tile row, the
// above ring and the staging ring at the group's base position.
// One group of kMsTW steps (k = k0 .. k0+TW-1); gt/ga/gs = this lane's tile
// row, the above ring and the staging ring at the group's base position. Chain
// KC-1's result of step d goes to ring position base + d - 1; gst0 = the address
// for d = 0 (the last position of the previous group's slot).
#ifndef ST_GS_MS_UNROLL
#define ST_GS_MS_UNROLL 16
#endif
constexpr int kMsHalf = ST_GS_MS_UNROLL;  // steps per unrolled body (a group runs TW / kMsHalf bodies):
                                          // small bodies keep the compute loop in the instruction cache
static_assert(kMsTW % kMsHalf == 0, "whole bodies per group");
template <int KC, bool kChk>
__device__ __forceinline__ void ms_group(MsState<KC>& S, const uint32_t gt, const uint32_t gst0, const uint32_t ga,
                                         const uint32_t gs, const int k0, const MsLane& L) {
  using G = MsGeo<KC>;
  static_assert(kMsHalf % kMsP == 0, "prefetch slots must line up across halves");
#pragma unroll
  for (int d = 0; d < kMsHalf; ++d) {
    const int k = k0 + d;
    const int q = d % kMsP;
    const double e0 = S.pe[q], s0 = S.ps[q];
    double ab[KC];
#pragma unroll
    for (int j = 0; j < KC; ++j) ab[j] = S.pa[q][j];
    ms_prefetch<KC, kChk>(S, gt, ga, d + kMsP, k + kMsP, L);
    double v[KC];
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      double n = shfl_up1(S.res[j]);
      n = L.top ? ab[j] : n;
      double s, e;
      if (j == 0) {
        s = s0;
        e = e0;
      } else {
        s = shfl_down1(S.res[j - 1]);
        s = L.sd ? S.sh[((d - 2 * j) % G::SH + G::SH) % G::SH] : s;
        e = S.res[j - 1];
      }
      double r = dmul(dadd(dadd(dadd(n, s), S.res[j]), e), 0.25);
      if (kChk) {  // outside the interior a chain carries the Dirichlet column values
        const int x = k + 1 - L.lane - 2 * j;
        r = x < 1 ? L.w0 : (x > L.nx ? L.eD : r);
      }
      v[j] = r;
    }
#pragma unroll
    for (int j = 0; j < KC; ++j) S.res[j] = v[j];
    S.sh[d % G::SH] = s0;
    // chain KC-1's result -> the tile (row lane, column x_{KC-1}, ring position base + d - 1)
    bool pst = true, pstg = L.stage;
    if (kChk) {
      const int x = k + 3 - L.lane - 2 * KC;
      pst = x >= 0 && x <= L.nx + 1;
      const int c = k + 2 - L.R;
      pstg = pstg && c >= 0 && c <= L.nx + 2 * KC - 2;
    }
    sts1_if(pst, d == 0 ? gst0 : gt + (uint32_t)(d - 1) * 8u, v[KC - 1]);
    // edge entry (v_0[c], v_1[c-2], ...) of column c = k + 2 - R (lane R-1 only)
    const uint32_t os = gs + (uint32_t)d * G::EB;
    if (KC == 1) {
      sts1_if(pstg, os, v[0]);
    } else {
#pragma unroll
      for (int j = 0; j < KC; j += 2) sts2_if(pstg, os + 8 * j, v[j], j + 1 < KC ? v[j + 1] : 0.0);
    }
  }
  if (kMsHalf % G::SH != 0) {  // re-align the S history ring to the next half's step numbering
    double t[G::SH];
#pragma unroll
    for (int i = 0; i < G::SH; ++i) t[i] = S.sh[(i + kMsHalf) % G::SH];
#pragma unroll
    for (int i = 0; i < G::SH; ++i) S.sh[i] = t[i];
  }
}

template <int KC>
__device__ __forceinline__ void ms_compute(const MsArgs& A, unsigned char* sm, const int I, const int lane) {
  using G = MsGeo<KC>;
  uint64_t* loaded = reinterpret_cast<uint64_t*>(sm + G::BAR_OFF);
  uint64_t* consumed = loaded + kMsSlots;
  const uint32_t tbase = smem_u32(sm) + (uint32_t)lane * G::ROWB;
  const uint32_t abase = smem_u32(sm) + G::ABOVE_OFF;
  const uint32_t sbase = smem_u32(sm) + G::STAGE_OFF;
  const int64_t y0 = 1 + (int64_t)I * A.R;
  const bool last = I == A.nstrips - 1;
  const int nreal = last ? (int)(A.ny - y0 + 1) : A.R;
  const int64_t y = y0 + lane;
  MsLane L;
  L.lane = lane;
  L.nx = A.nx;
  L.R = A.R;
  L.top = lane == 0;
  L.sd = last && lane == nreal - 1;
  L.stage = !last && lane == A.R - 1;
  L.w0 = y <= A.ny + 1 ? A.a[y * A.ld] : 0.0;
  L.eD = y <= A.ny + 1 ? A.a[y * A.ld + A.nx + 1] : 0.0;
  MsState<KC> S;
#pragma unroll
  for (int j = 0; j < KC; ++j) S.res[j] = 0.0;
#pragma unroll
  for (int j = 0; j < G::SH; ++j) S.sh[j] = 0.0;
#pragma unroll
  for (int q = 0; q < kMsP; ++q) {
    S.pe[q] = S.ps[q] = 0.0;
#pragma unroll
    for (int j = 0; j < KC; ++j) S.pa[q][j] = 0.0;
  }
  const int ntiles = A.ntiles;
  const int ngroups = (A.nx + 2 * KC + 29 + kMsTW - 1) / kMsTW;  // steps 0 .. nx + 2KC + 28
  const int64_t Ttot = A.passes * ntiles;
  for (int64_t p = 0; p < A.passes; ++p) {
    const int64_t T0 = p * ntiles;
    mbar_wait_parity(&loaded[T0 % kMsSlots], (uint32_t)((T0 / kMsSlots) & 1));
    // W of the first column is the Dirichlet column (lane 0's chain 0 is at x = 1 in step 0;
    // every other chain passes x = 0 first, where the checked group selects w0 anyway)
#pragma unroll
    for (int j = 0; j < KC; ++j) S.res[j] = L.w0;
    {  // prologue: steps 0 .. P-1 from the group-0 base
      const uint32_t b = (uint32_t)(T0 % kMsSlots) * kMsTW;
#pragma unroll
      for (int i = 0; i < kMsP; ++i) ms_prefetch<KC, true>(S, tbase + b * 8u, abase + b * G::EB, i, i, L);
    }
    for (int g = 0; g < ngroups; ++g) {
      const int64_t Gi = T0 + g;
      if (Gi + 1 < Ttot) mbar_wait_parity(&loaded[(Gi + 1) % kMsSlots], (uint32_t)(((Gi + 1) / kMsSlots) & 1));
      const uint32_t b = (uint32_t)(Gi % kMsSlots) * kMsTW;
      const uint32_t bp = (uint32_t)((Gi + kMsSlots - 1) % kMsSlots) * kMsTW;
      // unchecked when every lane and chain stays inside columns 1..nx for the whole group
      const bool chk = kMsTW * g < 2 * KC + 29 || kMsTW * (g + 1) > A.nx;
#pragma unroll 1
      for (int h = 0; h < kMsTW; h += kMsHalf) {
        const uint32_t gt = tbase + (b + h) * 8u, ga = abase + (b + h) * G::EB, gs = sbase + (b + h) * G::EB;
        const uint32_t gst0 = h == 0 ? tbase + (bp + kMsTW - 1) * 8u : gt - 8u;
        if (chk)
          ms_group<KC, true>(S, gt, gst0, ga, gs, kMsTW * g + h, L);
        else
          ms_group<KC, false>(S, gt, gst0, ga, gs, kMsTW * g + h, L);
      }
      const int td = g - G::kLagT;
      if (td >= 0 && td < ntiles) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&consumed[(T0 + td) % kMsSlots]);
      }
    }
    for (int td = max(0, ngroups - G::kLagT); td < ntiles; ++td) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&consumed[(T0 + td) % kMsSlots]);
    }
  }
}

// Ring position of column c of tile t in tile row rho (helper warps).
__device__ __forceinline__ int ms_mod(int64_t v) { return (int)(((v % kMsNP) + kMsNP) % kMsNP); }

// Loader: tile t's 33 rows and above entries into the ring (cp.async; the last
// lane-op arrives on loaded[t % slots] when this lane's copies have landed).
// wide = 16-byte pair copies (even KC, even pitch, aligned base: every pair is
// 16-byte aligned on both sides and never straddles the ring wrap).
template <int KC>
__device__ __forceinline__ void ms_load_tile(const MsArgs& A, unsigned char* sm, const int I, const int lane,
                                             const int64_t t, const bool wide) {
  using G = MsGeo<KC>;
  const uint32_t s0 = smem_u32(sm);
  const int m = (int)(t % A.ntiles);
  const int64_t y0 = 1 + (int64_t)I * A.R;
  const int rows = (int)min((int64_t)33, A.ny + 2 - y0);
  constexpr int kPairs = kMsTW / 2, kRowsW = 32 / kPairs;  // wide: lanes per row, rows per warp op
  if (wide) {  // lane: column pair 2 * (lane % kPairs) of row lane / kPairs (+ kRowsW per op)
    const int cc = 2 * (lane % kPairs), c = kMsTW * m + cc;
    if (c <= A.nx + 1) {
      for (int rho = lane / kPairs; rho < rows; rho += kRowsW) {
        const int pos = ms_mod(kMsTW * t + cc + rho + 2 * KC - 4);
        const uint32_t dst = s0 + (uint32_t)rho * G::ROWB + (uint32_t)pos * 8u;
        const double* gp = A.a + (y0 + rho) * A.ld + c;
        cp16(dst, gp);  // at pos = NP-1 the second value lands on the mirror of position 0 ...
        if (pos < G::MIR) cp16(dst + kMsNP * 8, gp);
        if (pos == kMsNP - 1) cp8(s0 + (uint32_t)rho * G::ROWB, gp + 1);  // ... and position 0 itself
      }
    }
  } else {  // lane: column lane % TW of row lane / TW (+ 32 / TW per op)
    const int cc = lane % kMsTW, c = kMsTW * m + cc;
    if (c <= A.nx + 1) {
      for (int rho = lane / kMsTW; rho < rows; rho += 32 / kMsTW) {
        const int pos = ms_mod(kMsTW * t + cc + rho + 2 * KC - 4);
        const uint32_t dst = s0 + (uint32_t)rho * G::ROWB + (uint32_t)pos * 8u;
        const double* gp = A.a + (y0 + rho) * A.ld + c;
        cp8(dst, gp);
        if (pos < G::MIR) cp8(dst + kMsNP * 8, gp);
      }
    }
  }
  // above entries of column c (lane 0's chain j reads entry x_j + 2j <= nx + 2KC - 2): row 0
  // for the first strip, else the strip above's edge
  const int c = kMsTW * m + lane;
  if (lane < kMsTW && c <= A.nx + 2 * KC - 2) {
    const int pa = ms_mod(kMsTW * t + lane);
    const uint32_t dst = s0 + G::ABOVE_OFF + (uint32_t)pa * G::EB;
    if (I == 0) {
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        if (c - 2 * j >= 0 && c - 2 * j <= A.nx + 1) {  // entry c = (a0[c], a0[c-2], ...)
          cp8(dst + 8 * j, A.a + (c - 2 * j));
          if (pa < G::MIRA) cp8(dst + kMsNP * G::EB + 8 * j, A.a + (c - 2 * j));
        }
      }
    } else {
      const char* src = A.edge + (int64_t)(I - 1) * A.edge_stride + (int64_t)c * G::EB;
#pragma unroll
      for (int j = 0; j < G::EB; j += 16) {  // 16-byte copies bypass L1: never a stale line
        cp16(dst + j, src + j);
        if (pa < G::MIRA) cp16(dst + kMsNP * G::EB + j, src + j);
      }
    }
  }
  cp_arrive_noinc(reinterpret_cast<uint64_t*>(sm + G::BAR_OFF) + (t % kMsSlots));
}

// Storer: tile t's real rows back to the grid and its edge entries out.
template <int KC>
__device__ __forceinline__ void ms_writeback_tile(const MsArgs& A, unsigned char* sm, const int I, const int lane,
                                                  const int64_t t, const bool wide) {
  using G = MsGeo<KC>;
  const uint32_t s0 = smem_u32(sm);
  const int m = (int)(t % A.ntiles);
  const int64_t y0 = 1 + (int64_t)I * A.R;
  const bool last = I == A.nstrips - 1;
  const int nreal = last ? (int)(A.ny - y0 + 1) : A.R;
  constexpr int kPairs = kMsTW / 2, kRowsW = 32 / kPairs;
  if (wide) {  // pairs (c, c+1), c even: column 0 / nx+1 in a pair are written back unchanged (Dirichlet)
    const int cc = 2 * (lane % kPairs), c = kMsTW * m + cc;
    if (c <= A.nx) {
      for (int rho = lane / kPairs; rho < nreal; rho += kRowsW) {
        const int pos = ms_mod(kMsTW * t + cc + rho + 2 * KC - 4);
        const uint32_t row = s0 + (uint32_t)rho * G::ROWB;
        double2 v;
        if (pos == kMsNP - 1) {  // the pair wraps: results live at the canonical positions NP-1 and 0
          v.x = lds1(row + (uint32_t)pos * 8u);
          v.y = lds1(row);
        } else {
          v = lds2(row + (uint32_t)pos * 8u);
        }
        *reinterpret_cast<double2*>(A.a + (y0 + rho) * A.ld + c) = v;
      }
    }
  } else {
    const int cc = lane % kMsTW, c = kMsTW * m + cc;
    if (c >= 1 && c <= A.nx) {
      for (int rho = lane / kMsTW; rho < nreal; rho += 32 / kMsTW) {
        const int pos = ms_mod(kMsTW * t + cc + rho + 2 * KC - 4);
        A.a[(y0 + rho) * A.ld + c] = lds1(s0 + (uint32_t)rho * G::ROWB + (uint32_t)pos * 8u);
      }
    }
  }
  const int c = kMsTW * m + lane;
  if (!last && lane < kMsTW && c >= 1 && c <= A.nx + 2 * KC - 2) {  // edge entries of column c for the strip below
    const uint32_t src = s0 + G::STAGE_OFF + (uint32_t)ms_mod(kMsTW * t + lane + A.R - 2) * G::EB;
    char* dst = A.edge + (int64_t)I * A.edge_stride + (int64_t)c * G::EB;
#pragma unroll
    for (int j = 0; j < G::EB; j += 16) *reinterpret_cast<double2*>(dst + j) = lds2(src + j);
  }
}

// Loader warp: tiles in order, each once its slot is free (the storer has read
// the tile before it), the strip above has published the tile's edge entries
// and the strip below has written back the same columns of the previous pass.
template <int KC>
__device__ __forceinline__ void ms_loader(const MsArgs& A, unsigned char* sm, const int I, const int lane,
                                          const bool wide) {
  using G = MsGeo<KC>;
  uint64_t* freed = reinterpret_cast<uint64_t*>(sm + G::BAR_OFF) + 2 * kMsSlots;
  const int64_t Ttot = A.passes * A.ntiles;
  const unsigned long long* up = I > 0 ? A.prog + (int64_t)(I - 1) * kMsProgStride : nullptr;
  const unsigned long long* dn = I + 1 < A.nstrips ? A.prog + (int64_t)(I + 1) * kMsProgStride : nullptr;
  const int64_t y0 = 1 + (int64_t)I * A.R;
  unsigned long long acq_up = 0, acq_dn = 0;
  for (int64_t t = 0; t < Ttot; ++t) {
    const unsigned long long need_up = (unsigned long long)(t + 1);
    const int64_t need_dn = t - A.ntiles + 1;
    const bool wu = up != nullptr, wd = dn != nullptr && need_dn > 0;
    // Wait for the neighbours' progress words. With 16-byte copies (cp.async.cg) every
    // read of another strip's data goes to L2, the coherence point, and is issued only
    // after the poll has returned a value published by a release store that followed
    // the data: a relaxed poll suffices, and no acquire is taken — an ld.acquire.gpu is
    // LDG.STRONG + CCTL.IVALL, and the L1 invalidation stalls the SM's L1TEX pipeline,
    // shared memory included (measured: it and L2 prefetch hints cost the compute warps
    // ~8 %). 8-byte copies (odd pitch) go through L1: they acquire per tile.
    const bool have = wide && (!wu || acq_up >= need_up) && (!wd || acq_dn >= (unsigned long long)need_dn);
    if (!have) {
      unsigned long long vu = wu ? ld_relaxed(up) : 0, vd = wd ? ld_relaxed(dn) : 0;
      bool ok = (!wu || vu >= need_up) && (!wd || vd >= (unsigned long long)need_dn);
      while (!__all_sync(0xffffffffu, ok)) {
        __nanosleep(ST_GS_MS_PSLEEP);
        vu = wu ? ld_relaxed(up) : 0;
        vd = wd ? ld_relaxed(dn) : 0;
        ok = (!wu || vu >= need_up) && (!wd || vd >= (unsigned long long)need_dn);
      }
      if (wide) {
        acq_up = vu;
        acq_dn = vd;
      } else {
        if (wu) (void)ld_acquire(up);
        if (wd) (void)ld_acquire(dn);
        if (!wu && !wd) (void)ld_acquire(A.prog + (int64_t)I * kMsProgStride);
      }
    }
    if (t >= kMsSlots)
      while (!mbar_test(&freed[t % kMsSlots], (uint32_t)((t / kMsSlots - 1) & 1))) __nanosleep(ST_GS_MS_LSLEEP);
    ms_load_tile<KC>(A, sm, I, lane, t, wide);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Storer warp: writes finished tiles back, frees their slots, and publishes
// progress (a release store of its progress word every kMsPub tiles and at the end).
#ifndef ST_GS_MS_PUB
#define ST_GS_MS_PUB 4
#endif
constexpr int kMsPub = ST_GS_MS_PUB;
template <int KC>
__device__ __forceinline__ void ms_storer(const MsArgs& A, unsigned char* sm, const int I, const int lane,
                                          const bool wide) {
  using G = MsGeo<KC>;
  uint64_t* consumed = reinterpret_cast<uint64_t*>(sm + G::BAR_OFF) + kMsSlots;
  uint64_t* freed = consumed + kMsSlots;
  const int64_t Ttot = A.passes * A.ntiles;
  unsigned long long* mine = A.prog + (int64_t)I * kMsProgStride;
  for (int64_t t = 0; t < Ttot; ++t) {
    while (!mbar_test(&consumed[t % kMsSlots], (uint32_t)((t / kMsSlots) & 1))) __nanosleep(ST_GS_MS_SSLEEP);
    ms_writeback_tile<KC>(A, sm, I, lane, t, wide);
    __syncwarp();  // every lane's shared reads of the tile are done (their values are in the stores)
    if (lane == 0) mbar_arrive(&freed[t % kMsSlots]);
    if ((t + 1) % kMsPub == 0 || t + 1 == Ttot) {
      // publish: the warp's write-back and edge stores, then the progress word. A
      // release store by lane 0 after the warp barrier (which orders the other lanes'
      // stores before it) instead of a full __threadfence on every lane.
      __syncwarp();
      if (lane == 0) st_release(mine, (unsigned long long)(t + 1));
    }
  }
}

template <int KC>
__global__ void __launch_bounds__(96 * kMsStrips, 1) gauss_seidel2d_ms_kernel(const MsArgs A) {
  using G = MsGeo<KC>;
  extern __shared__ __align__(128) unsigned char ms_smem[];
  // the role is warp-uniform; broadcasting it lets the compiler see that, so the
  // shuffles of the compute loop stay plain SHFL (no collective emulation)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // the SMSP arbiter favours the highest warp id among eligible warps, so the compute
  // warps take the top ids (8..11) and win every cycle they are eligible against a
  // helper polling on the same SMSP (warps 0..3 load, 4..7 store)
  const int s = warp % kMsStrips, role = (2 - warp / kMsStrips + 3) % 3;  // 0 compute, 1 loader, 2 storer
  const int I = blockIdx.x * kMsStrips + s;
  unsigned char* sm = ms_smem + s * G::STRIP_B;
  if (role == 1 && lane == 0 && I < A.nstrips) {
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + G::BAR_OFF);
    for (int q = 0; q < kMsSlots; ++q) {
      mbar_init(&bars[q], 32);                // loaded: one noinc arrive per loader lane
      mbar_init(&bars[kMsSlots + q], 1);      // consumed: the compute warp's lane 0
      mbar_init(&bars[2 * kMsSlots + q], 1);  // freed: the storer's lane 0
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (I >= A.nstrips) return;
  // 16-byte tile copies: even pitch, aligned base (with the rotation c + rho + 2KC - 4, an even
  // column c lands on a 16-byte aligned ring address in every row, for every KC)
  const bool wide = (A.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(A.a) & 15) == 0);
  if (role == 0)
    ms_compute<KC>(A, sm, I, lane);
  else if (role == 1)
    ms_loader<KC>(A, sm, I, lane, wide);
  else
    ms_storer<KC>(A, sm, I, lane, wide);
}

template <int KC>
st_status launch_ms(const MsArgs& A, cudaStream_t s) {
  using G = MsGeo<KC>;
  auto* k = gauss_seidel2d_ms_kernel<KC>;
  ST_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, G::CTA_B));
  const unsigned blocks = (unsigned)((A.nstrips + kMsStrips - 1) / kMsStrips);
  int per_sm = 0;
  ST_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 96 * kMsStrips, G::CTA_B));
  ST_RETURN_IF((int64_t)blocks > (int64_t)per_sm * num_sms(), ST_ENOTSUP,
               "gauss_seidel2d: %d strips exceed the resident capacity", A.nstrips);
  MsArgs a = A;
  void* args[] = {&a};
  // cooperative: every strip's CTA is co-resident (the strips wait on each other)
  ST_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(blocks), dim3(96 * kMsStrips), args, G::CTA_B, s));
  ST_LAUNCHED();
  return ST_OK;
}

int ms_strips(int64_t ny, int R) { return ny <= 32 ? 1 : (int)(1 + (ny - 32 + R - 1) / R); }

}  // namespace

int gauss_seidel2d_ms_depth() {
  static const int k = env_int("ST_GS_MS_K", 4);
  return k >= 1 && k <= 4 ? k : 4;
}

bool gauss_seidel2d_ms_supported(int64_t nx, int64_t ny) {
  const int K = gauss_seidel2d_ms_depth();
  const int64_t ntiles = (nx + 2 + kMsTW - 1) / kMsTW;
  return env_int("ST_GS_MS", 1) != 0 && ntiles >= kMsMinTiles && nx <= (1 << 28) &&
         (int64_t)ms_strips(ny, 33 - K) <= (int64_t)kMsStrips * num_sms();
}

int64_t gauss_seidel2d_ms_workspace_bytes(int64_t nx, int64_t ny) {
  const int K = gauss_seidel2d_ms_depth();
  const int64_t n = ms_strips(ny, 33 - K);
  return n * kMsProgStride * 8 + n * (nx + kMsEdgePad) * 32;
}

// `iters` sweeps: passes of K sweeps, then one pass of iters % K sweeps (same strips).
st_status gauss_seidel2d_ms_run(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters, void* workspace,
                                cudaStream_t s) {
  const int K = gauss_seidel2d_ms_depth();
  MsArgs A{};
  A.a = a;
  A.nx = (int)nx;
  A.ny = ny;
  A.ld = ld;
  A.R = 33 - K;
  A.nstrips = ms_strips(ny, A.R);
  A.prog = static_cast<unsigned long long*>(workspace);
  A.edge = static_cast<char*>(workspace) + (int64_t)A.nstrips * kMsProgStride * 8;
  A.edge_stride = (nx + kMsEdgePad) * 32;

  const int64_t full = iters / K;
  const int rem = (int)(iters % K);
  for (int part = 0; part < 2; ++part) {
    const int kc = part == 0 ? K : rem;
    A.passes = part == 0 ? full : 1;
    if (kc == 0 || A.passes == 0) continue;
    A.ntiles = (int)((std::max(nx + 2, nx + 2 * kc - 1) + kMsTW - 1) / kMsTW);  // columns 0..nx+1, edge entries
    ST_CHECK_CUDA(cudaMemsetAsync(A.prog, 0, (size_t)A.nstrips * kMsProgStride * 8, s));
    switch (kc) {
      case 1: ST_TRY(launch_ms<1>(A, s)); break;
      case 2: ST_TRY(launch_ms<2>(A, s)); break;
      case 3: ST_TRY(launch_ms<3>(A, s)); break;
      default: ST_TRY(launch_ms<4>(A, s)); break;
    }
  }
  return ST_OK;
}

st_status gauss_seidel2d_ms_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, gauss_seidel2d_ms_kernel<1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, gauss_seidel2d_ms_kernel<2>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, gauss_seidel2d_ms_kernel<3>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, gauss_seidel2d_ms_kernel<4>));
  return ST_OK;
}

}  // namespace st

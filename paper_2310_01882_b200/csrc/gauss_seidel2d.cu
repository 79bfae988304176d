// gauss_seidel2d.cu — Listing 1 taken literally: in-place lexicographic
// Gauss-Seidel (reading R22 of DESIGN.md; NEXT #4), sm_100a.
//
//   do i = 2, 255 ; do j = 2, 255
//     data(j,i) = (data(j,i-1)+data(j,i+1)+data(j-1,i)+data(j+1,i)) * 0.25
//
// N (row y-1) and W (column x-1) are this sweep's values, S and E the previous
// sweep's. The result is bitwise the sequential loop nest because every point
// is computed with the same association order from exactly the values the
// sequential order gives it — the parallel schedule only respects dependencies:
//
//  * A warp owns a strip of 32 rows (lane = row) and walks the columns with a
//    one-column skew per lane (lane r computes column k-r+1 at step k). Then N
//    is lane r-1's result of the previous step (warp shuffle), W the lane's own
//    previous result, S the old value lane r+1 is about to overwrite (its E,
//    shuffled down), E the lane's own old value one column ahead (prefetched).
//  * Strips are chained through progress words in global memory: a strip's top
//    row needs the strip above's bottom row of THIS sweep (wait until the strip
//    above has published that column), and its bottom row needs the strip
//    below's top row of the PREVIOUS sweep (wait until the strip below has
//    published it for sweep s-1; the strip below cannot overwrite it for sweep
//    s before this strip publishes the column, so no extra guard is needed).
//    Waits and publications happen between groups of kPf columns
//    (relaxed polling + ld.acquire / st.release at GPU scope; cross-strip data via L2).
//  * All sweeps run in ONE launch; strips drift into a diagonal pipeline across
//    sweeps. Every strip's warp must be resident (checked at launch), so the
//    spin-waits cannot deadlock.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace st {

namespace {

constexpr int kGsWarps = 4;  // strips per CTA
constexpr int kPf = 32;      // steps per group = prefetch distance (own row E; N for lane 0, S for lane 31)
static_assert(kPf >= 32, "refill columns must stay >= 1 without a check");

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// prog[2*I] = columns of strip I's bottom row finished (sweep-major: s*nx + x);
// prog[2*I+1] = the same for its top row. Zeroed before the launch.
//
// A step is one dependent chain (a shuffle and 4 fp64 ops), so everything else
// is kept off it: every value a step reads is loaded kPf steps ahead into
// registers (the lane's own row; the row above for lane 0, the row below for
// lane 31 — one array, the two lanes are distinct), the steps of a group are
// straight-line code (no per-step branches, so the shuffles stay plain SHFL),
// and progress waits/publications happen between groups, every kPub groups.
// A wait polls with relaxed loads under a warp vote, then takes one acquire
// load: an ld.acquire.gpu invalidates the SM's whole L1 (CCTL.IVALL), which
// measured ruinous as a polling loop.
template <int kPub>
__global__ void __launch_bounds__(32 * kGsWarps)
    gauss_seidel2d_kernel(double* __restrict__ a, int nx, int64_t ny, int64_t ld, int64_t iters,
                          unsigned long long* __restrict__ prog, int64_t nstrips) {
  const int lane = threadIdx.x & 31;
  const int64_t I = (int64_t)blockIdx.x * kGsWarps + (threadIdx.x >> 5);
  if (I >= nstrips) return;
  const int64_t y = 32 * I + 1 + lane;
  const bool real = y <= ny;        // rows this warp updates
  const bool ring = y == ny + 1;    // the bottom Dirichlet row: supplies S, never changes
  const bool live = real || ring;   // lanes beyond ny+1 only take part in the shuffles
  const bool top_lane = lane == 0, bottom_lane = lane == 31;
  const bool has_above = I > 0;              // row 0 is the Dirichlet ring otherwise
  const bool has_below = I + 1 < nstrips;    // lane 31's S row belongs to strip I+1
  const bool need_below = bottom_lane && real;
  const bool pub_bot = real && (bottom_lane || y == ny);  // the strip's last real row
  double* const row = a + (live ? y : 0) * ld;
  const double* const above = a + (32 * I) * ld;       // row y-1 of lane 0
  const double* const below = a + (32 * I + 33) * ld;   // row y+1 of lane 31
  unsigned long long* const my_bot = prog + 2 * I;
  unsigned long long* const my_top = prog + 2 * I + 1;
  const unsigned long long* const up_bot = prog + 2 * (I - 1);     // strip above, bottom row
  const unsigned long long* const dn_top = prog + 2 * (I + 1) + 1;  // strip below, top row
  const int nsteps = nx + 31;
  const int ngroups = (nsteps + kPf - 1) / kPf;
  const int x0 = 1 - lane;  // this lane's column at step 0 (x = k + x0)
  // refill at step k: own row column k + x0 + 1 + kPf (valid while <= nx + 1);
  // lane 0: row above, column k + 1 + kPf; lane 31: row below, column k - 30 + kPf (valid while <= nx)
  const int k_pf_max = live ? nx - x0 - kPf : -1;
  const double* const nbr = top_lane ? above + 1 + kPf : below + kPf - 30;
  const int k_nb_max = top_lane ? nx - 1 - kPf : need_below ? nx + 30 - kPf : -1;

  for (int64_t s = 0; s < iters; ++s) {
    const unsigned long long base = (unsigned long long)(s * nx);
    // Before group g (g % kPub == 0): the steps of groups g .. g+kPub-1 load the
    // row above up to column (g+kPub+1)*kPf (this sweep) and the row below up to
    // (g+kPub+1)*kPf - 31 (previous sweep; sweep 0 reads the initial values).
    auto wait = [&](int g) {
      const int lim = (g + kPub + 1) * kPf;
      const unsigned long long need_t = base + (unsigned long long)min(nx, lim);
      const int cb = min(nx, lim - 31);
      const bool wt = top_lane && has_above;
      const bool wb = need_below && has_below && s > 0 && cb >= 1;
      const unsigned long long need_b = base - (unsigned long long)nx + (unsigned long long)cb;
      bool ok = (!wt || ld_relaxed(up_bot) >= need_t) && (!wb || ld_relaxed(dn_top) >= need_b);
      while (!__all_sync(0xffffffffu, ok)) {
        __nanosleep(32);
        ok = (!wt || ld_relaxed(up_bot) >= need_t) && (!wb || ld_relaxed(dn_top) >= need_b);
      }
      if (wt) (void)ld_acquire(up_bot);  // synchronizes with the release that published it
      if (wb) (void)ld_acquire(dn_top);
    };
    wait(0);
    double res = row[0];  // W of column 1 = the Dirichlet column
    double e_prev = res;  // the lane's old value at column x-1 (the ring row's "result")
    double pf[kPf], pn[kPf];  // slot d <-> steps k == d (mod kPf)
#pragma unroll
    for (int d = 0; d < kPf; ++d) {
      const int c = x0 + 1 + d;  // E of this lane at step d
      pf[d] = (live && c >= 1 && c <= nx + 1) ? row[c] : 0.0;
      const int cn = top_lane ? 1 + d : d - 30;  // N of lane 0 / S of lane 31 at step d
      pn[d] = ((top_lane || need_below) && cn >= 1 && cn <= nx) ? __ldcg((top_lane ? above : below) + cn) : 0.0;
    }
    for (int g = 0; g < ngroups; ++g) {
      const int k0 = g * kPf;
      if (g > 0 && g % kPub == 0) wait(g);
      double* const rp = row + (k0 + x0);  // this lane's column at step k0 (dereferenced only in range)
#pragma unroll
      for (int d = 0; d < kPf; ++d) {
        const int k = k0 + d;
        const int x = k + x0;
        const bool act = (unsigned)(x - 1) < (unsigned)nx;
        const double e = pf[d];
        const double n_sh = __shfl_up_sync(0xffffffffu, res, 1);   // lane r-1's result of step k-1
        const double s_sh = __shfl_down_sync(0xffffffffu, e, 1);  // lane r+1's old value at this x
        const double nn = top_lane ? pn[d] : n_sh;
        const double ss = bottom_lane ? pn[d] : s_sh;
        const double v = dmul(dadd(dadd(dadd(nn, ss), res), e), 0.25);
        const bool upd = act && real;
        if (upd) rp[d] = v;
        res = upd ? v : ((act && ring) ? e_prev : res);  // Dirichlet row: its "result" is its value
        e_prev = e;
        // out-of-range slots keep stale values: only lanes past the grid edge read them
        if (k <= k_pf_max) pf[d] = rp[d + 1 + kPf];
        if (k <= k_nb_max) pn[d] = __ldcg(nbr + k);
      }
      if ((g + 1) % kPub == 0 || g + 1 == ngroups) {  // publish the finished columns
        const int k_last = k0 + kPf - 1;
        if (top_lane) st_release(my_top, base + (unsigned long long)min(nx, k_last + 1));
        const int cb = min(nx, k_last + x0);
        if (pub_bot && cb >= 1) st_release(my_bot, base + (unsigned long long)cb);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Tiled variant: the strip's rows are staged through shared memory in 32x32
// tiles, so global traffic is whole 256-byte row segments (cp.async loads,
// 16-byte stores) instead of one 8-byte access per lane and step to 32
// different rows (which saturated the LSU / L2 request rate with 512 strips).
// Lane r at step k still works on column x = k + 1 - r; it reads E (old value
// at x+1) from the tile and writes its result at x into the tile — a diagonal
// of the tile, conflict-free for a 32-double row pitch ((32r + c) mod 16 =
// c mod 16 = (k - r) mod 16 distinct over 16 lanes).
//
// Tile m = columns [32m, 32m+32) of the strip's 32 rows (even start column:
// 16-byte aligned for ld even). A warp keeps 4 tiles in flight: at the start of
// group g (steps 32g..32g+31) tile g-2 is complete (lane 31 finished column
// 32g-33 at step 32g-3): it is written back, its slot reloaded with tile g+2;
// tiles g-1, g are being written, g+1 is read (E). Progress words count
// columns written back to global memory (fence, then a relaxed flag store).
constexpr int kTile = 32;
constexpr int kRingTiles = 4;
constexpr int kEpf = 8;  // steps of E prefetch from the tile (kTile % kEpf == 0)
constexpr size_t kTiledSmem = (size_t)kRingTiles * kTile * kTile * sizeof(double);  // 32 KB per warp

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One CTA = one warp = one strip (the strips spin on each other: all must be resident).
// The CTA is a single warp, so its barrier is a warp barrier (racecheck-clean:
// cp.async.wait_group + bar.warp.sync order the tile writes against the reads).
__device__ __forceinline__ void cta_sync() { __syncwarp(); }

// kPubT: tiles written back per progress publication (one GPU-scope fence each).
template <int kPubT>
__global__ void __launch_bounds__(32)
    gauss_seidel2d_tiled_kernel(double* __restrict__ a, int nx, int64_t ny, int64_t ld, int64_t iters,
                                unsigned long long* __restrict__ prog, int64_t nstrips) {
  extern __shared__ __align__(16) double tiles[];  // [kRingTiles][32 rows][32 cols]
  const int lane = threadIdx.x;
  const int64_t I = blockIdx.x;
  const int64_t y0 = 32 * I + 1;  // the strip's first row
  const int64_t y = y0 + lane;
  const bool real = y <= ny;
  const bool ring = y == ny + 1;
  const bool live = real || ring;
  const bool top_lane = lane == 0, bottom_lane = lane == 31;
  const bool has_above = I > 0;
  const bool has_below = I + 1 < nstrips;
  const bool need_below = bottom_lane && real;
  const bool pub_bot = real && (bottom_lane || y == ny);
  const double* const above = a + (y0 - 1) * ld;
  const double* const below = a + (y0 + 32) * ld;
  unsigned long long* const my_bot = prog + 2 * I;
  unsigned long long* const my_top = prog + 2 * I + 1;
  const unsigned long long* const up_bot = prog + 2 * (I - 1);
  const unsigned long long* const dn_top = prog + 2 * (I + 1) + 1;
  const int nsteps = nx + 31;
  const int ngroups = (nsteps + kTile - 1) / kTile;
  const int ntiles = (nx + 2 + kTile - 1) / kTile;
  const int x0 = 1 - lane;
  const int k_nb_max = top_lane ? nx - 1 - kPf : need_below ? nx + 30 - kPf : -1;
  const double* const nbr = top_lane ? above + 1 + kPf : below + kPf - 30;
  // tile copies: lane l moves the 16-byte chunk (l & 15) of tile rows 2i + (l >> 4), i = 0..15
  const int cr = lane >> 4, cc = 2 * (lane & 15);
  double* const my_tile_row = tiles + lane * kTile;  // this lane's row inside tile slot 0

  auto tile_load = [&](int m) {  // tile m -> slot m % 4 (cp.async, one commit group)
    double* slot = tiles + (m & (kRingTiles - 1)) * (kTile * kTile);
    const int col = m * kTile + cc;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = 2 * i + cr;
      if (col <= nx + 1 && y0 + r <= ny + 1) cp_async16_cg(slot + r * kTile + cc, a + (y0 + r) * ld + col);
    }
  };
  auto tile_store = [&](int m) {  // rows 1..ny of tile m back to global (16-byte stores)
    const double* slot = tiles + (m & (kRingTiles - 1)) * (kTile * kTile);
    const int col = m * kTile + cc;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = 2 * i + cr;
      if (col <= nx + 1 && y0 + r <= ny)
        *reinterpret_cast<double2*>(a + (y0 + r) * ld + col) = *reinterpret_cast<const double2*>(slot + r * kTile + cc);
    }
  };
  auto publish = [&](unsigned long long base, int col_done) {  // columns 1..col_done of both edge rows are in global
    __threadfence();
    cta_sync();
    if (col_done >= 1) {
      if (top_lane) st_relaxed(my_top, base + (unsigned long long)min(nx, col_done));
      if (pub_bot) st_relaxed(my_bot, base + (unsigned long long)min(nx, col_done));
    }
  };

  for (int64_t s = 0; s < iters; ++s) {
    const unsigned long long base = (unsigned long long)(s * nx);
    // before group g (every kPubT groups): groups g .. g+kPubT-1 read the row above up
    // to column (g+kPubT+1)*32 (this sweep) and the row below up to that - 31 (previous sweep)
    auto wait = [&](int g) {
      const int lim = (g + kPubT + 1) * kPf;
      const unsigned long long need_t = base + (unsigned long long)min(nx, lim);
      const int cb = min(nx, lim - 31);
      const bool wt = top_lane && has_above;
      const bool wb = need_below && has_below && s > 0 && cb >= 1;
      const unsigned long long need_b = base - (unsigned long long)nx + (unsigned long long)cb;
      bool ok = (!wt || ld_relaxed(up_bot) >= need_t) && (!wb || ld_relaxed(dn_top) >= need_b);
      while (!__all_sync(0xffffffffu, ok)) {
        __nanosleep(32);
        ok = (!wt || ld_relaxed(up_bot) >= need_t) && (!wb || ld_relaxed(dn_top) >= need_b);
      }
      if (wt) (void)ld_acquire(up_bot);
      if (wb) (void)ld_acquire(dn_top);
    };
    tile_load(0);
    cp_async_commit_group();
    if (ntiles > 1) tile_load(1);
    cp_async_commit_group();
    wait(0);
    double pn[kPf];
#pragma unroll
    for (int d = 0; d < kPf; ++d) {
      const int cn = top_lane ? 1 + d : d - 30;
      pn[d] = ((top_lane || need_below) && cn >= 1 && cn <= nx) ? __ldcg((top_lane ? above : below) + cn) : 0.0;
    }
    cp_async_wait_group<1>();  // tile 0
    cta_sync();
    // res = the lane's result of the previous step, taken unconditionally (no
    // select on the chain): before a lane starts and after it ends it computes
    // garbage that nobody reads — N of lane r+1 at column x is lane r's result
    // at x, which is real whenever lane r+1 is active, the ring row's result is
    // never used (only its old values, as S), and W of column 1 is the
    // Dirichlet column w0, selected off the chain (W enters at the second add).
    const double w0 = my_tile_row[0];
    double res = w0;
    // E values are read kEpf steps ahead from the tile: the compiler cannot prove
    // that the read of column x+1 does not alias the store to column x of the
    // step before, so an in-step read would put LDS latency on the chain
    auto toff = [&](int c) { return lane * kTile + ((c >> 5) & (kRingTiles - 1)) * (kTile * kTile) + (c & 31); };
    double ep[kEpf];
#pragma unroll
    for (int d = 0; d < kEpf; ++d) ep[d] = tiles[toff(x0 + 1 + d)];
    for (int g = 0; g < ngroups; ++g) {
      if (g >= 2) {  // tile g-2 is complete: write it back (and publish every kPubT tiles)
        cta_sync();
        tile_store(g - 2);
        cta_sync();
        if ((g - 2) % kPubT == kPubT - 1) publish(base, (g - 2) * kTile + kTile - 1);
      }
      // lanes that have not reached column 0 yet read stale slots (negative columns
      // wrap to slot 3): order those reads before the slot's refill
      if (g < 2) cta_sync();
      if (g + 2 < ntiles) tile_load(g + 2);
      cp_async_commit_group();
      cp_async_wait_group<1>();  // tiles <= g+1 have landed
      cta_sync();
      if (g > 0 && g % kPubT == 0) wait(g);
      const int k0 = g * kTile;
#pragma unroll
      for (int d = 0; d < kTile; ++d) {
        const int k = k0 + d;
        const int x = k + x0;
        const bool act = (unsigned)(x - 1) < (unsigned)nx;
        const double e = ep[d % kEpf];
        ep[d % kEpf] = tiles[toff(x + 1 + kEpf)];
        const double n_sh = __shfl_up_sync(0xffffffffu, res, 1);
        const double s_sh = __shfl_down_sync(0xffffffffu, e, 1);
        const double nn = top_lane ? pn[d] : n_sh;
        const double ss = bottom_lane ? pn[d] : s_sh;
        const double ww = x == 1 ? w0 : res;
        const double v = dmul(dadd(dadd(dadd(nn, ss), ww), e), 0.25);
        if (act && real) tiles[toff(x)] = v;
        res = v;
        if (k <= k_nb_max) pn[d] = __ldcg(nbr + k);
      }
    }
    // flush the tiles not yet written back, then publish the whole row
    cta_sync();
    for (int m = max(0, ngroups - 2); m < ntiles; ++m) tile_store(m);
    cta_sync();
    publish(base, nx);
    cp_async_wait_group<0>();
    cta_sync();
  }
}

}  // namespace

st_status gauss_seidel2d_run(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters, void* workspace,
                             cudaStream_t s) {
  ST_RETURN_IF(nx > (1 << 30), ST_ENOTSUP, "gauss_seidel2d: nx = %lld > 2^30", (long long)nx);
  if (gauss_seidel2d_ms_supported(nx, ny)) return gauss_seidel2d_ms_run(a, nx, ny, ld, iters, workspace, s);
  unsigned long long* progress = static_cast<unsigned long long*>(workspace);
  const int64_t nstrips = (ny + 31) / 32;
  // the tiled kernel moves 16-byte row chunks: even pitch, 16-byte aligned base
  static const int kVariant = env_int("ST_GS_TILED", 1);
  const bool tiled = kVariant != 0 && (ld % 2) == 0 && aligned16(a);
  ST_CHECK_CUDA(cudaMemsetAsync(progress, 0, (size_t)(2 * nstrips) * sizeof(unsigned long long), s));
  int per_sm = 0;
  if (tiled) {
    auto* tk = gauss_seidel2d_tiled_kernel<4>;  // a fence per 4 written-back tiles
    ST_CHECK_CUDA(cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTiledSmem));
    ST_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tk, 32, kTiledSmem));
    // every strip's warp must be resident at once (the strips spin on each other)
    ST_RETURN_IF(nstrips > (int64_t)per_sm * num_sms(), ST_ENOTSUP,
                 "gauss_seidel2d: %lld strips exceed the resident capacity (%d CTAs/SM)", (long long)nstrips, per_sm);
    // cooperative launch: the driver guarantees every strip's CTA is co-resident
    // (or refuses the launch) — the strips spin on each other's progress words
    int nx_i = (int)nx;
    void* args[] = {&a, &nx_i, &ny, &ld, &iters, &progress, (void*)&nstrips};
    ST_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)tk, dim3((unsigned)nstrips), dim3(32), args, kTiledSmem, s));
    ST_LAUNCHED();
    return ST_OK;
  }
  auto* kern = gauss_seidel2d_kernel<1>;  // a publication per group of kPf columns
  ST_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kGsWarps, 0));
  const int64_t blocks = (nstrips + kGsWarps - 1) / kGsWarps;
  ST_RETURN_IF(blocks > (int64_t)per_sm * num_sms(), ST_ENOTSUP,
               "gauss_seidel2d: %lld strips exceed the resident capacity (%d CTAs/SM)", (long long)nstrips, per_sm);
  int nx_i = (int)nx;
  void* args[] = {&a, &nx_i, &ny, &ld, &iters, &progress, (void*)&nstrips};
  ST_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)blocks), dim3(32 * kGsWarps), args, 0, s));
  ST_LAUNCHED();
  return ST_OK;
}

int64_t gauss_seidel2d_workspace_bytes(int64_t nx, int64_t ny) {
  const int64_t single = 2 * ((ny + 31) / 32) * 8;
  return gauss_seidel2d_ms_supported(nx, ny) ? std::max(single, gauss_seidel2d_ms_workspace_bytes(nx, ny)) : single;
}

st_status gauss_seidel2d_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, gauss_seidel2d_kernel<1>));
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, gauss_seidel2d_tiled_kernel<4>));
  return gauss_seidel2d_ms_preload();
}

}  // namespace st

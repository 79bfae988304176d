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
//    Waits and publications happen once per chunk of kChunk columns
//    (ld.acquire / st.release at GPU scope; cross-strip data via L2).
//  * All sweeps run in ONE launch; strips drift into a diagonal pipeline across
//    sweeps. Every strip's warp must be resident (checked at launch), so the
//    spin-waits cannot deadlock.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace st {

namespace {

constexpr int kGsWarps = 4;    // strips per CTA
constexpr int kChunk = 64;     // columns per progress publication / wait
constexpr int kPrefetch = 8;   // own-row E values loaded this many steps ahead

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void spin_until(const unsigned long long* p, unsigned long long need) {
  while (ld_acquire(p) < need) __nanosleep(64);
}

// prog[2*I] = columns of strip I's bottom row finished (sweep-major: s*nx + x);
// prog[2*I+1] = the same for its top row. Zeroed before the launch.
__global__ void __launch_bounds__(32 * kGsWarps)
    gauss_seidel2d_kernel(double* __restrict__ a, int64_t nx, int64_t ny, int64_t ld, int64_t iters,
                          unsigned long long* __restrict__ prog, int64_t nstrips) {
  const int lane = threadIdx.x & 31;
  const int64_t I = (int64_t)blockIdx.x * kGsWarps + (threadIdx.x >> 5);
  if (I >= nstrips) return;
  const int64_t y = 32 * I + 1 + lane;
  const bool real = y <= ny;        // rows this warp updates
  const bool ring = y == ny + 1;    // the bottom Dirichlet row: supplies S, never changes
  const bool live = real || ring;   // lanes beyond ny+1 only take part in the shuffles
  const bool top_lane = lane == 0, bottom_lane = lane == 31;
  const bool has_above = I > 0;                          // row 0 is the Dirichlet ring otherwise
  const bool has_below = I + 1 < nstrips;                // lane 31's S comes from strip I+1
  double* row = a + (live ? y : 0) * ld;
  const double* above = a + (32 * I) * ld;               // row y-1 of lane 0
  const double* below = a + (32 * I + 33) * ld;          // row y+1 of lane 31
  unsigned long long* my_bot = prog + 2 * I;
  unsigned long long* my_top = prog + 2 * I + 1;
  const unsigned long long* up_bot = prog + 2 * (I - 1);   // strip above, bottom row
  const unsigned long long* dn_top = prog + 2 * (I + 1) + 1;  // strip below, top row
  const int64_t nsteps = nx + 31;

  for (int64_t s = 0; s < iters; ++s) {
    double res = row[0];  // W of column 1 = the Dirichlet column
    double pf[kPrefetch];  // E values: old row entries at columns x+1 .. x+kPrefetch
#pragma unroll
    for (int d = 0; d < kPrefetch; ++d) {
      const int64_t c = 1 - lane + 1 + d;  // column x_r(step 0) + 1 + d
      pf[d] = (live && c >= 1 && c <= nx + 1) ? row[c] : 0.0;
    }
    for (int64_t k0 = 0; k0 < nsteps; k0 += kPrefetch) {
#pragma unroll
      for (int d = 0; d < kPrefetch; ++d) {
        const int64_t k = k0 + d;
        if (k >= nsteps) break;  // warp-uniform
        const int64_t x = k - lane + 1;
        const bool act = x >= 1 && x <= nx;
        // chunk boundaries: wait for the neighbours' progress (the whole warp waits)
        if (((k) % kChunk) == 0) {
          if (top_lane && has_above) {  // strip above's bottom row, this sweep, columns x .. x+kChunk-1
            const int64_t need_x = min(nx, k + (int64_t)kChunk);
            spin_until(up_bot, (unsigned long long)(s * nx + need_x));
          }
        }
        if (((k - 31) % kChunk) == 0 && k >= 31) {
          if (bottom_lane && has_below && real) {  // strip below's top row, previous sweep
            const int64_t need_x = min(nx, k - 31 + (int64_t)kChunk);
            if (s > 0) spin_until(dn_top, (unsigned long long)((s - 1) * nx + need_x));
          }
        }
        __syncwarp();
        const double e = pf[d];
        const double n_sh = __shfl_up_sync(0xffffffffu, res, 1);   // lane r-1's result of step k-1
        const double s_sh = __shfl_down_sync(0xffffffffu, e, 1);  // lane r+1's old value at this x
        if (act && real) {
          const double nn = top_lane ? (has_above ? __ldcg(above + x) : above[x]) : n_sh;
          const double ss = bottom_lane ? __ldcg(below + x) : s_sh;
          const double v = dmul(dadd(dadd(dadd(nn, ss), res), e), 0.25);
          row[x] = v;
          res = v;
        } else if (act && ring) {
          res = row[x];  // Dirichlet row: its "result" is its value
        }
        // refill the slot with the old value kPrefetch columns ahead
        const int64_t c = x + 1 + kPrefetch;
        pf[d] = (live && c >= 1 && c <= nx + 1) ? row[c] : 0.0;
        // publish progress at chunk ends and at the end of the row
        if (act && real && (x % kChunk == 0 || x == nx)) {
          if (bottom_lane || y == ny) st_release(my_bot, (unsigned long long)(s * nx + x));
          if (top_lane) st_release(my_top, (unsigned long long)(s * nx + x));
        }
      }
    }
  }
}

}  // namespace

st_status gauss_seidel2d_run(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters,
                             unsigned long long* progress, cudaStream_t s) {
  const int64_t nstrips = (ny + 31) / 32;
  // every strip's warp must be resident at once (the strips spin on each other)
  int per_sm = 0, dev = 0;
  ST_CHECK_CUDA(cudaGetDevice(&dev));
  ST_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gauss_seidel2d_kernel, 32 * kGsWarps, 0));
  const int64_t blocks = (nstrips + kGsWarps - 1) / kGsWarps;
  ST_RETURN_IF(blocks > (int64_t)per_sm * num_sms(), ST_ENOTSUP,
               "gauss_seidel2d: %lld strips exceed the resident capacity (%d CTAs/SM)", (long long)nstrips, per_sm);
  ST_CHECK_CUDA(cudaMemsetAsync(progress, 0, (size_t)(2 * nstrips) * sizeof(unsigned long long), s));
  gauss_seidel2d_kernel<<<(unsigned)blocks, 32 * kGsWarps, 0, s>>>(a, nx, ny, ld, iters, progress, nstrips);
  ST_LAUNCHED();
  return ST_OK;
}

int64_t gauss_seidel2d_workspace_bytes(int64_t ny) { return 2 * ((ny + 31) / 32) * 8; }

st_status gauss_seidel2d_preload() {
  cudaFuncAttributes fa;
  ST_CHECK_CUDA(cudaFuncGetAttributes(&fa, gauss_seidel2d_kernel));
  return ST_OK;
}

}  // namespace st

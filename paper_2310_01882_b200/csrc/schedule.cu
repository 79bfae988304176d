// schedule.cu — the per-rank step schedule of st_jacobi2d_run (host code).
//
// One schedule covers the single-domain run (nranks == 1: the ghost rows are
// the Dirichlet rows) and the slab decomposition (PAPER.md:268
// "halo swap between iterations"; PAPER.md:277 decomposed domain): it decides
// how the sweeps are grouped into passes (temporal blocking), when the ghost
// rows must be swapped (every `halo` sweeps at the latest), which rows each
// pass writes (redundant ghost-row recomputation between swaps) and how a
// pass whose results are swapped right away is split into boundary rows ->
// async swap -> interior rows -> join (SURVEY.md §8(e) overlap schedule).
// It is exported (st_jacobi2d_schedule) so this logic is tested on CPU.
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace st {

namespace {
constexpr int kAutoTblock = 10;  // tblock=0 (tuned on B200 under the board power cap)
constexpr int64_t kAutoMinExtent = 128;  // ... on grids at least this large in x and y

void push(std::vector<st_op>& v, int32_t kind, int32_t buf, int32_t sweeps, int32_t flag, int64_t lo = 0,
          int64_t hi = -1, int64_t rlo = -1, int64_t rhi = -1) {
  st_op o;
  o.kind = kind;
  o.buf = buf;
  o.sweeps = sweeps;
  o.flag = flag;
  o.y_lo = lo;
  o.y_hi = hi;
  o.ring_lo = rlo;
  o.ring_hi = rhi;
  v.push_back(o);
}
}  // namespace

int choose_tblock(int32_t nranks, int64_t nx, int64_t n, int32_t h, int32_t tblock) {
  if (tblock > 0) return tblock;
  const int want = env_int("ST_JACOBI_T", kAutoTblock);
  if (nx < kAutoMinExtent || n < kAutoMinExtent) return 1;
  if (nranks == 1) return jacobi2d_tb_supported(want) ? want : 1;
  int t = want < h ? want : h;  // ghosts must cover a whole pass
  t &= ~1;
  while (t >= 2 && !jacobi2d_tb_supported(t)) t -= 2;
  return t >= 2 ? t : 1;
}

// dims=3: two sweeps per pass (jacobi3d_t2_kernel) whenever the ghosts cover them
int choose_tblock3d(int32_t nranks, int32_t h, int32_t tblock) {
  if (tblock > 0) return tblock;
  static const int kT2 = env_int("ST_J3_T2", 1);
  return kT2 && (nranks == 1 || h >= 2) ? 2 : 1;
}

st_status build_jacobi_schedule(int32_t rank, int32_t nranks, int64_t nx, int64_t n, int32_t h,
                                int64_t iters, int32_t tblock, std::vector<st_op>& ops, int dims) {
  ST_RETURN_IF(nranks < 1 || rank < 0 || rank >= nranks, ST_EINVAL, "schedule: rank %d of %d", rank, nranks);
  ST_RETURN_IF(nx < 1 || n < 1 || h < 1 || iters < 0 || tblock < 0, ST_EINVAL, "schedule: bad extents/counts");
  ST_RETURN_IF(nranks > 1 && n < h, ST_EINVAL, "schedule: slab of %lld rows < halo %d", (long long)n, h);
  ST_RETURN_IF(dims == 3 && tblock > 2, ST_ENOTSUP, "jacobi3d: tblock=%d not supported (0, 1, 2)", tblock);
  const int T = dims == 3 ? choose_tblock3d(nranks, h, tblock) : choose_tblock(nranks, nx, n, h, tblock);
  ST_RETURN_IF(dims == 2 && T > 1 && !jacobi2d_tb_supported(T), ST_ENOTSUP,
               "jacobi2d: tblock=%d not supported (1, 2, 4, 6, 8, 10)", T);
  ST_RETURN_IF(nranks > 1 && T > h, ST_EINVAL, "jacobi%dd: tblock=%d needs halo >= %d", dims, T, T);

  // passes: T-sweep (temporally blocked) passes, a remainder, and the parity
  // fix-up of plan_passes so the result lands in b iff iters is odd
  std::vector<int64_t> passes;
  if (T == 1) {
    passes.assign((size_t)iters, 1);
  } else {
    int64_t left = iters;
    while (left >= T) { passes.push_back(T); left -= T; }
    if (left >= 2) { passes.push_back(left & ~int64_t(1)); left &= 1; }
    if (left == 1) passes.push_back(1);
    if ((int64_t)(passes.size() & 1) != (iters & 1)) {
      for (size_t i = 0; i < passes.size(); ++i) {
        if (passes[i] >= 4) { passes[i] -= 2; passes.insert(passes.begin() + i + 1, 2); break; }
        if (passes[i] == 2) { passes[i] = 1; passes.insert(passes.begin() + i + 1, 1); break; }
      }
    }
  }

  const bool multi = nranks > 1;
  const bool lo_edge = rank == 0, hi_edge = rank == nranks - 1;
  const int64_t nrows = n + 2 * (int64_t)h;
  const int64_t ring_lo = lo_edge ? h - 1 : -1;
  const int64_t ring_hi = hi_edge ? h + n : nrows;
  int32_t cur = 0;
  int64_t fresh = multi ? 0 : INT64_MAX / 2;  // sweeps the current ghosts still support
  int64_t sw = 0;                            // sweeps since the last swap
  ops.clear();
  for (size_t i = 0; i < passes.size(); ++i) {
    const int64_t b = passes[i];
    if (multi && fresh < b) {
      push(ops, ST_OP_EXCHANGE, cur, h, 0);
      fresh = h;
      sw = 0;
    }
    const int64_t next_b = i + 1 < passes.size() ? passes[i + 1] : 0;
    const bool swap_after = multi && next_b > 0 && fresh - b < next_b;
    if (swap_after) {
      // only the owned rows are needed: boundary rows, async swap, interior rows, join
      if (n >= 2 * (int64_t)h) {
        push(ops, ST_OP_SWEEP, cur, (int32_t)b, 0, h, 2 * (int64_t)h - 1, ring_lo, ring_hi);
        push(ops, ST_OP_SWEEP, cur, (int32_t)b, 0, n, n + h - 1, ring_lo, ring_hi);
        push(ops, ST_OP_EXCHANGE, 1 - cur, h, 1);
        if (2 * (int64_t)h <= n - 1) push(ops, ST_OP_SWEEP, cur, (int32_t)b, 0, 2 * (int64_t)h, n - 1, ring_lo, ring_hi);
        push(ops, ST_OP_JOIN, 1 - cur, h, 0);
      } else {
        push(ops, ST_OP_SWEEP, cur, (int32_t)b, 0, h, h + n - 1, ring_lo, ring_hi);
        push(ops, ST_OP_EXCHANGE, 1 - cur, h, 0);
      }
      push(ops, ST_OP_SWAP, cur, 0, 0);
      cur = 1 - cur;
      fresh = h;
      sw = 0;
    } else {
      const int64_t lo = lo_edge ? h : sw + b;
      const int64_t hi = hi_edge ? h + n - 1 : nrows - 1 - sw - b;
      push(ops, ST_OP_SWEEP, cur, (int32_t)b, 0, lo, hi, ring_lo, ring_hi);
      push(ops, ST_OP_SWAP, cur, 0, 0);
      cur = 1 - cur;
      fresh -= b;
      sw += b;
    }
  }
  return ST_OK;
}

}  // namespace st

extern "C" st_status st_jacobi3d_schedule(int32_t rank, int32_t nranks, int64_t nx, int64_t nz_local,
                                          int32_t halo, int64_t iters, int32_t tblock, st_op* ops, int64_t cap,
                                          int64_t* nops) {
  st::clear_error();
  ST_RETURN_IF(!nops || (cap > 0 && !ops), ST_EINVAL, "st_jacobi3d_schedule: null output");
  std::vector<st_op> v;
  ST_TRY(st::build_jacobi_schedule(rank, nranks, nx, nz_local, halo, iters, tblock, v, 3));
  *nops = (int64_t)v.size();
  for (int64_t i = 0; i < cap && i < (int64_t)v.size(); ++i) ops[i] = v[(size_t)i];
  return ST_OK;
}

extern "C" st_status st_jacobi2d_schedule(int32_t rank, int32_t nranks, int64_t nx, int64_t ny_local,
                                          int32_t halo, int64_t iters, int32_t tblock, st_op* ops, int64_t cap,
                                          int64_t* nops) {
  st::clear_error();
  ST_RETURN_IF(!nops || (cap > 0 && !ops), ST_EINVAL, "st_jacobi2d_schedule: null output");
  std::vector<st_op> v;
  ST_TRY(st::build_jacobi_schedule(rank, nranks, nx, ny_local, halo, iters, tblock, v));
  *nops = (int64_t)v.size();
  for (int64_t i = 0; i < cap && i < (int64_t)v.size(); ++i) ops[i] = v[(size_t)i];
  return ST_OK;
}

/* oracle/oracle.c — plain, slow, obviously-correct CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2310_01882_b200/) never links, imports or calls it, and this file
 * shares no code, header, constant or helper with the CUDA path.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp (IEEE binary64,
 * round-to-nearest-even, no contraction, no FTZ/DAZ) — SURVEY.md §8(c4) A11/A13.
 *
 * Layout ("arrays index precedence is from
 * left to right in Fortran", i.e. the first Fortran index is contiguous):
 *   2-D field: row-major a[y*ld + x], 0 <= y <= ny+1, 0 <= x <= nx+1, ld >= nx+2.
 *              Row/col 0 and ny+1/nx+1 are the 1-cell Dirichlet ring
 *              (PAPER.md:99-100 loops 2..255; PAPER.md:122 bounds [-1,255] -> [0,254]).
 *   3-D field: f[(z*(ny+2) + y)*ldx + x], x fastest, z slowest.
 *
 * Functions and the passages they follow:
 *   or_jacobi2d        PAPER.md:98-104 (Listing 1) under the value semantics of
 *                      stencil.apply, PAPER.md:126 ("executing lines 3 to 12 for
 *                      every grid cell") => Jacobi double buffering; reading A1/A2
 *                      of DESIGN.md: sum order ((N+S)+W)+E, then *0.25.
 *   or_pw_advect3d     PAPER.md:216 (Piacsek-Williams advection, three stencils
 *                      over three fields fused into one region, 63 flop/cell);
 *                      formula = DESIGN.md reading R6 (MONC pwadvection form,
 *                      SURVEY.md §8(c2)). Overwrites su,sv,sw interior (R8).
 *   or_jacobi2d_slabs  PAPER.md:268/277 (halo swap between iterations over a
 *                      decomposed domain); SPEC.md:399 block split, remainder to
 *                      high ranks. Ghost depth H, exchange every H sweeps.
 *   or_pw_slabs        PAPER.md:268 (PW halo swapped before the time step).
 *   or_jacobi3d        PAPER.md:214 (benchmark 1: Laplace by a 7-point stencil,
 *                      "averages values across the six neighbouring cells", six
 *                      flops per cell) under the value semantics of PAPER.md:126;
 *                      readings R20/R21 of DESIGN.md: sum order z-,z+,y-,y+,x-,x+
 *                      (slowest index first, as Listing 1 orders i before j),
 *                      then / 6.0 (5 adds + 1 divide = 6 flops).
 *   or_jacobi3d_slabs  z-slab decomposition of or_jacobi3d (1 ghost plane).
 *   or_gauss_seidel2d  PAPER.md:98-104 Listing 1 taken literally: the Fortran loop
 *                      nest updates `data` IN PLACE, i (= y) outer, j (= x)
 *                      inner, so (y-1, x) and (y, x-1) are this sweep's values
 *                      and (y+1, x), (y, x+1) the previous sweep's
 *                      (lexicographic Gauss-Seidel).
 *   or_stencil2d       generic linear stencil.apply (PAPER.md:107-126 apply/access,
 *                      offsets from the discovery pass PAPER.md:149-191, 185):
 *                      out = c_0*a(off_0) + c_1*a(off_1) + ... left to right;
 *                      value semantics; R-wide Dirichlet ring (R = max |offset|,
 *                      SPEC.md:197-205). Reading R23 of DESIGN.md.
 *   or_pencils_jacobi3d / or_pencils_pw
 *                      2-D (y, z) process grid ("decompose the 3D space into
 *                      two dimensions"): Py x Pz blocks with one
 *                      ghost layer in y and z, swapped before every sweep /
 *                      application (y rows of all planes first, then whole z
 *                      planes, so the (y, z) corner ghosts PW reads are filled).
 *
 * Pins (tests/test_oracle_*.py): J1-J10, P1-P9, D1 of SURVEY.md §8(c5).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IDX2(y, x, ld) ((int64_t)(y) * (int64_t)(ld) + (int64_t)(x))
#define IDX3(z, y, x, ny2, ldx) ((((int64_t)(z) * (int64_t)(ny2)) + (int64_t)(y)) * (int64_t)(ldx) + (int64_t)(x))

/* ------------------------------------------------------------------------- */
/* 2-D Jacobi                                                                 */
/* ------------------------------------------------------------------------- */

/* One Jacobi sweep over rows [ylo, yhi] (inclusive) and columns 1..nx:
 * dst[y][x] = (((src[y-1][x] + src[y+1][x]) + src[y][x-1]) + src[y][x+1]) * 0.25
 * Listing 1: data(j,i) = (data(j,i-1)+data(j,i+1)+data(j-1,i)+data(j+1,i)) * 0.25,
 * j contiguous (= x), i = y; Fortran evaluates + left to right. */
static void jacobi_sweep_rows(const double* src, double* dst, int64_t nx, int64_t ld,
                              int64_t ylo, int64_t yhi, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t y = ylo; y <= yhi; ++y) {
    for (int64_t x = 1; x <= nx; ++x) {
      double n = src[IDX2(y - 1, x, ld)];
      double s = src[IDX2(y + 1, x, ld)];
      double w = src[IDX2(y, x - 1, ld)];
      double e = src[IDX2(y, x + 1, ld)];
      double sum = n + s;
      sum = sum + w;
      sum = sum + e;
      dst[IDX2(y, x, ld)] = sum * 0.25;
    }
  }
}

/* B := copy(A) (ring included); repeat iters: B = sweep(A); swap(A, B).
 * Returns 1 if the result is in b (iters odd), 0 if in a, -1 on bad args. */
int or_jacobi2d(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t iters,
                int nthreads) {
  if (!a || !b || nx < 1 || ny < 1 || ld < nx + 2 || iters < 0) return -1;
  if (nthreads < 1) nthreads = 1;
  memcpy(b, a, sizeof(double) * (size_t)((ny + 2) * ld));
  double* src = a;
  double* dst = b;
  for (int64_t it = 0; it < iters; ++it) {
    jacobi_sweep_rows(src, dst, nx, ld, 1, ny, nthreads);
    double* t = src; src = dst; dst = t;
  }
  return (int)(iters & 1);
}

/* Block split of n items over P ranks, remainder to the HIGH ranks. */
static void block_split(int64_t n, int p, int r, int64_t* start, int64_t* count) {
  int64_t base = n / p, rem = n % p;
  int64_t lo_ranks = p - rem; /* ranks [0, p-rem) get base, the rest base+1 */
  if (r < lo_ranks) { *count = base; *start = (int64_t)r * base; }
  else { *count = base + 1; *start = lo_ranks * base + (int64_t)(r - lo_ranks) * (base + 1); }
}

/* Decomposed Jacobi: rows 1..ny are split into P slabs of
 * n_r rows; each slab holds H ghost rows per side (local rows 0..H-1 and
 * H+n_r..2H+n_r-1). Every H sweeps the H ghost rows are refreshed from the
 * neighbouring slabs' owned rows (the halo swap); between swaps slab r sweeps
 * a shrinking row range (redundant ghost-row recomputation). On the first/last
 * slab the ghost row adjacent to the owned rows is the global Dirichlet row and
 * is never updated. Result (after `iters` sweeps) is gathered into `out`
 * (rows 0..ny+1 x ld). Must be bitwise equal to or_jacobi2d (pin D1).
 * Returns 0, or -1 on bad args / empty slab / allocation failure. */
int or_jacobi2d_slabs(const double* a, double* out, int64_t nx, int64_t ny, int64_t ld,
                      int64_t iters, int p, int h) {
  if (!a || !out || nx < 1 || ny < 1 || ld < nx + 2 || iters < 0 || p < 1 || h < 1) return -1;
  if (ny / p < 1 || ny / p < h) return -1; /* every slab must own >= H rows */
  double** A = calloc((size_t)p, sizeof(double*));
  double** B = calloc((size_t)p, sizeof(double*));
  int64_t* st = calloc((size_t)p, sizeof(int64_t));
  int64_t* nr = calloc((size_t)p, sizeof(int64_t));
  int ok = A && B && st && nr;
  for (int r = 0; ok && r < p; ++r) {
    block_split(ny, p, r, &st[r], &nr[r]);
    int64_t rows = nr[r] + 2 * h;
    A[r] = calloc((size_t)(rows * ld), sizeof(double));
    B[r] = calloc((size_t)(rows * ld), sizeof(double));
    ok = A[r] && B[r];
    if (!ok) break;
    /* local row l <-> global padded row g = st + 1 + (l - h); fill what exists */
    for (int64_t l = 0; l < rows; ++l) {
      int64_t g = st[r] + 1 + (l - h);
      if (g < 0 || g > ny + 1) continue;
      memcpy(&A[r][IDX2(l, 0, ld)], &a[IDX2(g, 0, ld)], sizeof(double) * (size_t)ld);
    }
    memcpy(B[r], A[r], sizeof(double) * (size_t)(rows * ld));
  }
  if (ok) {
    for (int64_t it = 0; it < iters; ++it) {
      int64_t k = it % h;
      if (k == 0 && p > 1) {
        /* halo swap on the current source buffers A[r]: ghost rows <- neighbour owned rows */
        for (int r = 0; r < p; ++r) {
          if (r > 0) /* lower ghosts 0..h-1 <- rank r-1 owned rows n-h..n-1 (local h+n-h..) */
            memcpy(&A[r][IDX2(0, 0, ld)], &A[r - 1][IDX2(nr[r - 1], 0, ld)],
                   sizeof(double) * (size_t)(h * ld));
          if (r < p - 1) /* upper ghosts h+n..2h+n-1 <- rank r+1 owned rows h..2h-1 */
            memcpy(&A[r][IDX2(h + nr[r], 0, ld)], &A[r + 1][IDX2(h, 0, ld)],
                   sizeof(double) * (size_t)(h * ld));
        }
      }
      for (int r = 0; r < p; ++r) {
        int64_t lo = (r == 0) ? h : k + 1;
        int64_t hi = (r == p - 1) ? h + nr[r] - 1 : 2 * h + nr[r] - 2 - k;
        jacobi_sweep_rows(A[r], B[r], nx, ld, lo, hi, 1);
        double* t = A[r]; A[r] = B[r]; B[r] = t;
      }
    }
    /* gather: owned rows, plus the global Dirichlet rows from the edge slabs */
    for (int r = 0; r < p; ++r) {
      memcpy(&out[IDX2(st[r] + 1, 0, ld)], &A[r][IDX2(h, 0, ld)],
             sizeof(double) * (size_t)(nr[r] * ld));
    }
    memcpy(&out[IDX2(0, 0, ld)], &A[0][IDX2(h - 1, 0, ld)], sizeof(double) * (size_t)ld);
    memcpy(&out[IDX2(ny + 1, 0, ld)], &A[p - 1][IDX2(h + nr[p - 1], 0, ld)],
           sizeof(double) * (size_t)ld);
  }
  for (int r = 0; r < p && A && B; ++r) { free(A[r]); free(B[r]); }
  free(A); free(B); free(st); free(nr);
  return ok ? 0 : -1;
}

/* ------------------------------------------------------------------------- */
/* 3-D Piacsek-Williams advection                                             */
/* ------------------------------------------------------------------------- */

typedef struct {
  const double *u, *v, *w;
  int64_t ny2, ldx;
  double tcx, tcy;
  const double *tzc1, *tzc2, *tzd1, *tzd2;
} pw_in;

/* U(dz,dy,dx) == u[z+dz][y+dy][x+dx] */
#define U(dz, dy, dx) p->u[IDX3(z + (dz), y + (dy), x + (dx), p->ny2, p->ldx)]
#define V(dz, dy, dx) p->v[IDX3(z + (dz), y + (dy), x + (dx), p->ny2, p->ldx)]
#define W(dz, dy, dx) p->w[IDX3(z + (dz), y + (dy), x + (dx), p->ny2, p->ldx)]

/* One grid point, the association trees of DESIGN.md R6;
 * every binary op rounds once; 21 flops per output, 63 per point. */
static void pw_point(const pw_in* p, int64_t z, int64_t y, int64_t x, double out[3]) {
  double t1, t2, xs, ys, zs;
  /* su */
  t1 = U(0, 0, -1) * (U(0, 0, 0) + U(0, 0, -1));
  t2 = U(0, 0, +1) * (U(0, 0, 0) + U(0, 0, +1));
  xs = p->tcx * (t1 - t2);
  t1 = U(0, -1, 0) * (V(0, -1, 0) + V(0, -1, +1));
  t2 = U(0, +1, 0) * (V(0, 0, 0) + V(0, 0, +1));
  ys = p->tcy * (t1 - t2);
  t1 = (p->tzc1[z] * U(-1, 0, 0)) * (W(-1, 0, 0) + W(-1, 0, +1));
  t2 = (p->tzc2[z] * U(+1, 0, 0)) * (W(0, 0, 0) + W(0, 0, +1));
  zs = t1 - t2;
  out[0] = (xs + ys) + zs;
  /* sv */
  t1 = V(0, 0, -1) * (U(0, 0, -1) + U(0, +1, -1));
  t2 = V(0, 0, +1) * (U(0, 0, 0) + U(0, +1, 0));
  xs = p->tcx * (t1 - t2);
  t1 = V(0, -1, 0) * (V(0, 0, 0) + V(0, -1, 0));
  t2 = V(0, +1, 0) * (V(0, 0, 0) + V(0, +1, 0));
  ys = p->tcy * (t1 - t2);
  t1 = (p->tzc1[z] * V(-1, 0, 0)) * (W(-1, 0, 0) + W(-1, +1, 0));
  t2 = (p->tzc2[z] * V(+1, 0, 0)) * (W(0, 0, 0) + W(0, +1, 0));
  zs = t1 - t2;
  out[1] = (xs + ys) + zs;
  /* sw */
  t1 = W(0, 0, -1) * (U(0, 0, -1) + U(+1, 0, -1));
  t2 = W(0, 0, +1) * (U(0, 0, 0) + U(+1, 0, 0));
  xs = p->tcx * (t1 - t2);
  t1 = W(0, -1, 0) * (V(0, -1, 0) + V(+1, -1, 0));
  t2 = W(0, +1, 0) * (V(0, 0, 0) + V(+1, 0, 0));
  ys = p->tcy * (t1 - t2);
  t1 = (p->tzd1[z] * W(-1, 0, 0)) * (W(0, 0, 0) + W(-1, 0, 0));
  t2 = (p->tzd2[z] * W(+1, 0, 0)) * (W(0, 0, 0) + W(+1, 0, 0));
  zs = t1 - t2;
  out[2] = (xs + ys) + zs;
}
#undef U
#undef V
#undef W

/* Overwrites the interior (1..nz, 1..ny, 1..nx) of su, sv, sw; never touches
 * their halos. tz*: nz+2 doubles indexed by plane. Returns 0 or -1. */
int or_pw_advect3d(const double* u, const double* v, const double* w, double* su, double* sv,
                   double* sw, int64_t nx, int64_t ny, int64_t nz, int64_t ldx, double tcx,
                   double tcy, const double* tzc1, const double* tzc2, const double* tzd1,
                   const double* tzd2, int nthreads) {
  if (!u || !v || !w || !su || !sv || !sw || !tzc1 || !tzc2 || !tzd1 || !tzd2) return -1;
  if (nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2) return -1;
  if (nthreads < 1) nthreads = 1;
  pw_in p = {u, v, w, ny + 2, ldx, tcx, tcy, tzc1, tzc2, tzd1, tzd2};
#pragma omp parallel for schedule(static) num_threads(nthreads) collapse(2)
  for (int64_t z = 1; z <= nz; ++z) {
    for (int64_t y = 1; y <= ny; ++y) {
      for (int64_t x = 1; x <= nx; ++x) {
        double o[3];
        pw_point(&p, z, y, x, o);
        int64_t i = IDX3(z, y, x, ny + 2, ldx);
        su[i] = o[0]; sv[i] = o[1]; sw[i] = o[2];
      }
    }
  }
  return 0;
}

/* Sampled evaluation for full-size parity: out[3*k + c] = s_c at point k
 * (zyx[3k], zyx[3k+1], zyx[3k+2]), each an interior point. Returns 0 or -1. */
int or_pw_points(const double* u, const double* v, const double* w, int64_t nx, int64_t ny,
                 int64_t nz, int64_t ldx, double tcx, double tcy, const double* tzc1,
                 const double* tzc2, const double* tzd1, const double* tzd2,
                 const int64_t* zyx, int64_t npts, double* out) {
  if (!u || !v || !w || !zyx || !out || ldx < nx + 2) return -1;
  pw_in p = {u, v, w, ny + 2, ldx, tcx, tcy, tzc1, tzc2, tzd1, tzd2};
  for (int64_t k = 0; k < npts; ++k) {
    int64_t z = zyx[3 * k], y = zyx[3 * k + 1], x = zyx[3 * k + 2];
    if (z < 1 || z > nz || y < 1 || y > ny || x < 1 || x > nx) return -1;
    pw_point(&p, z, y, x, &out[3 * k]);
  }
  return 0;
}

/* Decomposed PW: planes 1..nz split into P z-slabs, each
 * with one ghost plane per side for u, v, w. The halo swap copies the
 * neighbour slab's first/last owned plane into the ghost planes (edge slabs
 * keep the global halo planes); each slab then advects its owned planes with
 * its slice of the tz* coefficients; outputs are gathered into su,sv,sw
 * (interior only). Must be bitwise equal to or_pw_advect3d (pin D1). */
int or_pw_slabs(const double* u, const double* v, const double* w, double* su, double* sv,
                double* sw, int64_t nx, int64_t ny, int64_t nz, int64_t ldx, double tcx,
                double tcy, const double* tzc1, const double* tzc2, const double* tzd1,
                const double* tzd2, int p) {
  if (!u || !v || !w || !su || !sv || !sw || nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2 ||
      p < 1 || nz / p < 1)
    return -1;
  const int64_t plane = (ny + 2) * ldx;
  const double* gin[3] = {u, v, w};
  double* gout[3] = {su, sv, sw};
  int rc = 0;
  double** f = calloc((size_t)(6 * p), sizeof(double*)); /* [r*6 + field], fields 0-2 in, 3-5 out */
  int64_t* st = calloc((size_t)p, sizeof(int64_t));
  int64_t* nr = calloc((size_t)p, sizeof(int64_t));
  if (!f || !st || !nr) rc = -1;
  for (int r = 0; !rc && r < p; ++r) {
    block_split(nz, p, r, &st[r], &nr[r]);
    for (int c = 0; c < 6; ++c) {
      f[r * 6 + c] = calloc((size_t)((nr[r] + 2) * plane), sizeof(double));
      if (!f[r * 6 + c]) { rc = -1; break; }
    }
    if (rc) break;
    for (int c = 0; c < 3; ++c) /* owned planes local 1..n <- global st+1..st+n */
      memcpy(f[r * 6 + c] + plane, gin[c] + (st[r] + 1) * plane,
             sizeof(double) * (size_t)(nr[r] * plane));
  }
  for (int r = 0; !rc && r < p; ++r) {
    for (int c = 0; c < 3; ++c) {
      double* loc = f[r * 6 + c];
      if (r == 0) memcpy(loc, gin[c], sizeof(double) * (size_t)plane);
      else memcpy(loc, f[(r - 1) * 6 + c] + nr[r - 1] * plane, sizeof(double) * (size_t)plane);
      if (r == p - 1)
        memcpy(loc + (nr[r] + 1) * plane, gin[c] + (nz + 1) * plane, sizeof(double) * (size_t)plane);
      else
        memcpy(loc + (nr[r] + 1) * plane, f[(r + 1) * 6 + c] + plane, sizeof(double) * (size_t)plane);
    }
  }
  for (int r = 0; !rc && r < p; ++r) {
    const int64_t o = st[r]; /* local plane k <-> global plane st + k */
    rc = or_pw_advect3d(f[r * 6 + 0], f[r * 6 + 1], f[r * 6 + 2], f[r * 6 + 3], f[r * 6 + 4],
                        f[r * 6 + 5], nx, ny, nr[r], ldx, tcx, tcy, tzc1 + o, tzc2 + o, tzd1 + o,
                        tzd2 + o, 1);
    for (int c = 0; !rc && c < 3; ++c)
      for (int64_t k = 1; k <= nr[r]; ++k)
        for (int64_t y = 1; y <= ny; ++y)
          memcpy(gout[c] + IDX3(st[r] + k, y, 1, ny + 2, ldx),
                 f[r * 6 + 3 + c] + IDX3(k, y, 1, ny + 2, ldx), sizeof(double) * (size_t)nx);
  }
  for (int i = 0; f && i < 6 * p; ++i) free(f[i]);
  free(f); free(st); free(nr);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* 3-D 7-point Jacobi (the paper's benchmark 1)       */
/* ------------------------------------------------------------------------- */

/* One sweep over planes [zlo, zhi] (inclusive), all interior rows/columns:
 * dst = (((((Zm + Zp) + Ym) + Yp) + Xm) + Xp) / 6.0 */
static void jacobi3d_sweep_planes(const double* src, double* dst, int64_t nx, int64_t ny, int64_t ldx,
                                  int64_t zlo, int64_t zhi, int nthreads) {
  const int64_t ny2 = ny + 2;
#pragma omp parallel for schedule(static) num_threads(nthreads) collapse(2)
  for (int64_t z = zlo; z <= zhi; ++z) {
    for (int64_t y = 1; y <= ny; ++y) {
      for (int64_t x = 1; x <= nx; ++x) {
        double sum = src[IDX3(z - 1, y, x, ny2, ldx)] + src[IDX3(z + 1, y, x, ny2, ldx)];
        sum = sum + src[IDX3(z, y - 1, x, ny2, ldx)];
        sum = sum + src[IDX3(z, y + 1, x, ny2, ldx)];
        sum = sum + src[IDX3(z, y, x - 1, ny2, ldx)];
        sum = sum + src[IDX3(z, y, x + 1, ny2, ldx)];
        dst[IDX3(z, y, x, ny2, ldx)] = sum / 6.0;
      }
    }
  }
}

/* B := copy(A); repeat iters: B = sweep(A); swap. Returns 1 if the result is in b. */
int or_jacobi3d(double* a, double* b, int64_t nx, int64_t ny, int64_t nz, int64_t ldx, int64_t iters,
                int nthreads) {
  if (!a || !b || nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2 || iters < 0) return -1;
  if (nthreads < 1) nthreads = 1;
  memcpy(b, a, sizeof(double) * (size_t)((nz + 2) * (ny + 2) * ldx));
  double* src = a;
  double* dst = b;
  for (int64_t it = 0; it < iters; ++it) {
    jacobi3d_sweep_planes(src, dst, nx, ny, ldx, 1, nz, nthreads);
    double* t = src; src = dst; dst = t;
  }
  return (int)(iters & 1);
}

/* z-slab decomposition with one ghost plane per side, swapped before every
 * sweep; gathered into `out`. Must equal or_jacobi3d bitwise. */
int or_jacobi3d_slabs(const double* a, double* out, int64_t nx, int64_t ny, int64_t nz, int64_t ldx,
                      int64_t iters, int p) {
  if (!a || !out || nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2 || iters < 0 || p < 1 || nz / p < 1) return -1;
  const int64_t plane = (ny + 2) * ldx;
  double** A = calloc((size_t)p, sizeof(double*));
  double** B = calloc((size_t)p, sizeof(double*));
  int64_t* st = calloc((size_t)p, sizeof(int64_t));
  int64_t* nr = calloc((size_t)p, sizeof(int64_t));
  int ok = A && B && st && nr;
  for (int r = 0; ok && r < p; ++r) {
    block_split(nz, p, r, &st[r], &nr[r]);
    A[r] = malloc(sizeof(double) * (size_t)((nr[r] + 2) * plane));
    B[r] = malloc(sizeof(double) * (size_t)((nr[r] + 2) * plane));
    ok = A[r] && B[r];
    if (!ok) break;
    /* local plane k <-> global plane st + k, k = 0..n+1 */
    memcpy(A[r], a + st[r] * plane, sizeof(double) * (size_t)((nr[r] + 2) * plane));
    memcpy(B[r], A[r], sizeof(double) * (size_t)((nr[r] + 2) * plane));
  }
  for (int64_t it = 0; ok && it < iters; ++it) {
    for (int r = 0; r < p; ++r) {
      if (r > 0) memcpy(A[r], A[r - 1] + nr[r - 1] * plane, sizeof(double) * (size_t)plane);
      if (r < p - 1) memcpy(A[r] + (nr[r] + 1) * plane, A[r + 1] + plane, sizeof(double) * (size_t)plane);
    }
    for (int r = 0; r < p; ++r) {
      jacobi3d_sweep_planes(A[r], B[r], nx, ny, ldx, 1, nr[r], 1);
      double* t = A[r]; A[r] = B[r]; B[r] = t;
    }
  }
  if (ok) {
    for (int r = 0; r < p; ++r)
      memcpy(out + (st[r] + 1) * plane, A[r] + plane, sizeof(double) * (size_t)(nr[r] * plane));
    memcpy(out, A[0], sizeof(double) * (size_t)plane);
    memcpy(out + (nz + 1) * plane, A[p - 1] + (nr[p - 1] + 1) * plane, sizeof(double) * (size_t)plane);
  }
  for (int r = 0; r < p && A && B; ++r) { free(A[r]); free(B[r]); }
  free(A); free(B); free(st); free(nr);
  return ok ? 0 : -1;
}

/* ------------------------------------------------------------------------- */
/* Pencil (2-D y-z) decomposition of the 3-D stencils                          */
/* ------------------------------------------------------------------------- */

typedef struct {
  int64_t y0, ny, z0, nz; /* owned global interior rows y0+1..y0+ny, planes z0+1..z0+nz */
  double* f[6];           /* local (nz+2) x (ny+2) x ldx buffers */
} pencil;

/* local (z, y) <-> global (z0+z, y0+y); copy whole local block from a global field */
static void pencil_fill(pencil* b, int c, const double* g, int64_t gny, int64_t ldx) {
  for (int64_t z = 0; z < b->nz + 2; ++z)
    for (int64_t y = 0; y < b->ny + 2; ++y)
      memcpy(b->f[c] + IDX3(z, y, 0, b->ny + 2, ldx), g + IDX3(b->z0 + z, b->y0 + y, 0, gny + 2, ldx),
             sizeof(double) * (size_t)ldx);
}

/* halo swap of field c over the Py x Pz grid: y rows of every plane 0..nz+1
 * first (the z-halo planes of the edge ranks carry global boundary values that
 * the diagonal PW offsets read), then whole z planes (rows 0..ny+1, incl. the
 * fresh y ghosts -> the (y, z) corner ghosts) */
static void pencil_swap(pencil* B, int py, int pz, int c, int64_t ldx) {
  for (int iz = 0; iz < pz; ++iz)
    for (int iy = 0; iy < py; ++iy) {
      pencil* b = &B[iz * py + iy];
      const int64_t ny2 = b->ny + 2;
      if (iy > 0) {
        pencil* n = &B[iz * py + iy - 1];
        for (int64_t z = 0; z <= b->nz + 1; ++z) /* my ghost row 0 <- lower neighbour's last owned row */
          memcpy(b->f[c] + IDX3(z, 0, 0, ny2, ldx), n->f[c] + IDX3(z, n->ny, 0, n->ny + 2, ldx),
                 sizeof(double) * (size_t)ldx);
      }
      if (iy < py - 1) {
        pencil* n = &B[iz * py + iy + 1];
        for (int64_t z = 0; z <= b->nz + 1; ++z)
          memcpy(b->f[c] + IDX3(z, b->ny + 1, 0, ny2, ldx), n->f[c] + IDX3(z, 1, 0, n->ny + 2, ldx),
                 sizeof(double) * (size_t)ldx);
      }
    }
  for (int iz = 0; iz < pz; ++iz)
    for (int iy = 0; iy < py; ++iy) {
      pencil* b = &B[iz * py + iy];
      const int64_t plane = (b->ny + 2) * ldx;
      if (iz > 0) {
        pencil* n = &B[(iz - 1) * py + iy];
        memcpy(b->f[c], n->f[c] + n->nz * plane, sizeof(double) * (size_t)plane);
      }
      if (iz < pz - 1) {
        pencil* n = &B[(iz + 1) * py + iy];
        memcpy(b->f[c] + (b->nz + 1) * plane, n->f[c] + plane, sizeof(double) * (size_t)plane);
      }
    }
}

static pencil* pencils_make(int64_t ny, int64_t nz, int py, int pz, int64_t ldx, int nf) {
  pencil* B = calloc((size_t)(py * pz), sizeof(pencil));
  if (!B) return NULL;
  for (int iz = 0; iz < pz; ++iz)
    for (int iy = 0; iy < py; ++iy) {
      pencil* b = &B[iz * py + iy];
      block_split(ny, py, iy, &b->y0, &b->ny);
      block_split(nz, pz, iz, &b->z0, &b->nz);
      for (int c = 0; c < nf; ++c) {
        b->f[c] = calloc((size_t)((b->nz + 2) * (b->ny + 2) * ldx), sizeof(double));
        if (!b->f[c]) return NULL;
      }
    }
  return B;
}

static void pencils_free(pencil* B, int n) {
  for (int i = 0; B && i < n; ++i)
    for (int c = 0; c < 6; ++c) free(B[i].f[c]);
  free(B);
}

/* gather the owned interior of field c into the global field g */
static void pencil_gather(pencil* B, int py, int pz, int c, double* g, int64_t gny, int64_t nx, int64_t ldx) {
  for (int i = 0; i < py * pz; ++i) {
    pencil* b = &B[i];
    for (int64_t z = 1; z <= b->nz; ++z)
      for (int64_t y = 1; y <= b->ny; ++y)
        memcpy(g + IDX3(b->z0 + z, b->y0 + y, 1, gny + 2, ldx), b->f[c] + IDX3(z, y, 1, b->ny + 2, ldx),
               sizeof(double) * (size_t)nx);
  }
}

int or_pencils_jacobi3d(const double* a, double* out, int64_t nx, int64_t ny, int64_t nz, int64_t ldx,
                        int64_t iters, int py, int pz) {
  if (!a || !out || nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2 || iters < 0 || py < 1 || pz < 1 || ny / py < 1 ||
      nz / pz < 1)
    return -1;
  pencil* B = pencils_make(ny, nz, py, pz, ldx, 2);
  if (!B) return -1;
  for (int i = 0; i < py * pz; ++i) {
    pencil_fill(&B[i], 0, a, ny, ldx);
    pencil_fill(&B[i], 1, a, ny, ldx);
  }
  int cur = 0;
  for (int64_t it = 0; it < iters; ++it) {
    pencil_swap(B, py, pz, cur, ldx);
    for (int i = 0; i < py * pz; ++i)
      jacobi3d_sweep_planes(B[i].f[cur], B[i].f[1 - cur], nx, B[i].ny, ldx, 1, B[i].nz, 1);
    cur = 1 - cur;
  }
  memcpy(out, a, sizeof(double) * (size_t)((nz + 2) * (ny + 2) * ldx));
  pencil_gather(B, py, pz, cur, out, ny, nx, ldx);
  pencils_free(B, py * pz);
  return 0;
}

int or_pencils_pw(const double* u, const double* v, const double* w, double* su, double* sv, double* sw,
                  int64_t nx, int64_t ny, int64_t nz, int64_t ldx, double tcx, double tcy, const double* tzc1,
                  const double* tzc2, const double* tzd1, const double* tzd2, int py, int pz) {
  if (!u || !v || !w || !su || !sv || !sw || nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2 || py < 1 || pz < 1 ||
      ny / py < 1 || nz / pz < 1)
    return -1;
  pencil* B = pencils_make(ny, nz, py, pz, ldx, 6);
  if (!B) return -1;
  const double* gin[3] = {u, v, w};
  for (int i = 0; i < py * pz; ++i)
    for (int c = 0; c < 3; ++c) pencil_fill(&B[i], c, gin[c], ny, ldx);
  /* the ghosts of u, v, w come from the neighbours (poisoned first so a missed cell shows) */
  for (int i = 0; i < py * pz; ++i) {
    pencil* b = &B[i];
    const int iy = i % py, iz = i / py;
    for (int c = 0; c < 3; ++c)
      for (int64_t z = 0; z < b->nz + 2; ++z)
        for (int64_t y = 0; y < b->ny + 2; ++y) {
          const int ghost_y = (y == 0 && iy > 0) || (y == b->ny + 1 && iy < py - 1);
          const int ghost_z = (z == 0 && iz > 0) || (z == b->nz + 1 && iz < pz - 1);
          if (ghost_y || ghost_z)
            for (int64_t x = 0; x < nx + 2; ++x) b->f[c][IDX3(z, y, x, b->ny + 2, ldx)] = 1e300;
        }
  }
  for (int c = 0; c < 3; ++c) pencil_swap(B, py, pz, c, ldx);
  for (int i = 0; i < py * pz; ++i) {
    pencil* b = &B[i];
    const int64_t o = b->z0;
    if (or_pw_advect3d(b->f[0], b->f[1], b->f[2], b->f[3], b->f[4], b->f[5], nx, b->ny, b->nz, ldx, tcx, tcy,
                       tzc1 + o, tzc2 + o, tzd1 + o, tzd2 + o, 1) != 0) {
      pencils_free(B, py * pz);
      return -1;
    }
  }
  double* gout[3] = {su, sv, sw};
  for (int c = 0; c < 3; ++c) pencil_gather(B, py, pz, 3 + c, gout[c], ny, nx, ldx);
  pencils_free(B, py * pz);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Lexicographic in-place Gauss-Seidel (Listing 1 literally, NEXT #4)          */
/* ------------------------------------------------------------------------- */

/* `iters` in-place sweeps of a (rows 0..ny+1) x ld field; ring untouched. */
int or_gauss_seidel2d(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters) {
  if (!a || nx < 1 || ny < 1 || ld < nx + 2 || iters < 0) return -1;
  for (int64_t it = 0; it < iters; ++it)
    for (int64_t y = 1; y <= ny; ++y)     /* do i = 2, 255 */
      for (int64_t x = 1; x <= nx; ++x) { /* do j = 2, 255 */
        double sum = a[IDX2(y - 1, x, ld)] + a[IDX2(y + 1, x, ld)];
        sum = sum + a[IDX2(y, x - 1, ld)];
        sum = sum + a[IDX2(y, x + 1, ld)];
        a[IDX2(y, x, ld)] = sum * 0.25;
      }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Generic linear 2-D stencil.apply (reading R23 of DESIGN.md)                 */
/* ------------------------------------------------------------------------- */

/* The stencil dialect's apply (stencil.access at constant
 * offsets inside an apply region) for the loop nests the discovery pass
 * extracts (Listing 3; RHS offsets PAPER.md:185), restricted
 * to linear right-hand sides:
 *   out(y,x) = c_0*a(y+dy_0, x+dx_0) + c_1*a(y+dy_1, x+dx_1) + ...
 * evaluated left to right as written (Fortran order, one rounding per product
 * and per sum, no contraction). Value semantics: Jacobi double
 * buffering. Halo width R = max |offset| (input bounds = output bounds widened
 * by the offsets); the R-wide ring is never written.
 * a, b: (ny + 2R) rows x ld, interior rows R..R+ny-1, columns R..R+nx-1.
 * off = [dy_0, dx_0, dy_1, dx_1, ...]. Returns 1 if the result is in b, 0 if in a. */
int or_stencil2d(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, const int32_t* off,
                 const double* c, int32_t n, int64_t iters, int nthreads) {
  if (!a || !b || !off || !c || n < 1 || nx < 1 || ny < 1 || iters < 0) return -1;
  int64_t R = 0;
  for (int32_t i = 0; i < 2 * n; ++i) {
    int64_t m = off[i] < 0 ? -off[i] : off[i];
    if (m > R) R = m;
  }
  if (ld < nx + 2 * R) return -1;
  if (nthreads < 1) nthreads = 1;
  memcpy(b, a, sizeof(double) * (size_t)((ny + 2 * R) * ld));
  double* src = a;
  double* dst = b;
  for (int64_t it = 0; it < iters; ++it) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t y = R; y < R + ny; ++y)
      for (int64_t x = R; x < R + nx; ++x) {
        double acc = c[0] * src[IDX2(y + off[0], x + off[1], ld)];
        for (int32_t i = 1; i < n; ++i) {
          double t = c[i] * src[IDX2(y + off[2 * i], x + off[2 * i + 1], ld)];
          acc = acc + t;
        }
        dst[IDX2(y, x, ld)] = acc;
      }
    double* t = src; src = dst; dst = t;
  }
  return (int)(iters & 1);
}

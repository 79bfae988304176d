// internal.h — launchers shared between the C-ABI layer (api.cu, comm.cu) and
// the kernel translation units. Not part of the public ABI.
#pragma once

#include <string>

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"
#include "libstencil.h"

namespace st {

// Optional second destination of a sweep (fused halo swap, NEXT #3): every row
// r the sweep writes to dst is also written to base[(r + delta) * ld ...] —
// the neighbour rank's ghost rows — so boundary rows travel to the neighbour
// in the same kernel that computes them (peer memory / NVLink when the
// neighbour lives on another GPU). base == nullptr: no second destination.
struct Remote {
  double* base = nullptr;
  int64_t delta = 0;
};

// ------------------------------------------------ generic 2-D stencil ---
constexpr int kStencilMaxTerms = 32;
constexpr int kStencilMaxOffset = 8;
st_status stencil2d_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t R, const int32_t* off,
                        const double* coeffs, int32_t n, int64_t iters, cudaStream_t s);

st_status stencil_expr_translate(const char* expr, std::string* cexpr, int64_t* R, int* dims);
st_status stencil2d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int64_t R,
                             const std::string& cexpr, int64_t iters, cudaStream_t s);
st_status stencil3d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t nz, int64_t ldx, int64_t R,
                             const std::string& cexpr, int64_t iters, cudaStream_t s);
st_status stencil3d_fused_run(const double* const* in, int32_t nin, double* const* out, int32_t nout,
                              const char* const* exprs, const double* const* coefs, int32_t ncoef, int64_t nx,
                              int64_t ny, int64_t nz, int64_t ldx, int64_t* R_out, bool validate_only,
                              cudaStream_t s);

// ----------------------------------------------------------- Jacobi 2-D ---
// One sweep dst = J(src) over buffer rows [y_lo, y_hi] (buffer row indices,
// inclusive) and interior columns 1..nx; columns 0 and nx+1 are passed through
// (dst = src) so the Dirichlet ring is preserved bit for bit. Rows outside the
// range are neither read (except y_lo-1 and y_hi+1) nor written.
st_status jacobi2d_sweep_rows(const double* src, double* dst, int64_t nx, int64_t ld,
                              int64_t y_lo, int64_t y_hi, cudaStream_t s, Remote rem = Remote());

// `iters` sweeps entirely inside one CTA's shared memory (small grids: both
// buffers fit in SMEM). Writes the final state (whole (ny+2) x (nx+2) window)
// into a (iters even) or b (iters odd).
bool jacobi2d_resident_fits(int64_t nx, int64_t ny);
st_status jacobi2d_resident(double* a, double* b, int64_t nx, int64_t ny, int64_t ld,
                            int64_t iters, cudaStream_t s);

// Temporal blocking: T sweeps in one pass over HBM; writes rows [y_lo, y_hi]
// of dst with the state after T sweeps (src rows y_lo-T .. y_hi+T are read
// where they exist; intermediate levels are recomputed redundantly on a
// shrinking halo and never stored). Buffer rows <= ring_lo and >= ring_hi are
// Dirichlet (identical at every level); pass ring_lo = -1 / ring_hi = nrows_buf
// for none. T must be even (2, 4, 6, 8).
bool jacobi2d_tb_supported(int t);
st_status jacobi2d_tb_rows(const double* src, double* dst, int64_t nx, int64_t ld,
                           int64_t y_lo, int64_t y_hi, int t, int64_t ring_lo,
                           int64_t ring_hi, int64_t nrows_buf, cudaStream_t s, Remote rem = Remote());

// ------------------------------------------------------------ Jacobi 3-D ---
// One 7-point sweep dst = J(src) over planes [z_lo, z_hi] (buffer plane indices)
// and the interior rows/columns; reads planes z_lo-1 .. z_hi+1. nplanes_buf =
// planes in the buffer (TMA extent).
st_status jacobi3d_sweep_planes(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                                int64_t ldx, int64_t z_lo, int64_t z_hi, cudaStream_t s, Remote rem = Remote());
// The same over output rows [y_lo, y_hi] only (pencils: the interior block while the halo is in flight).
st_status jacobi3d_sweep_block(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                               int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t y_lo, int64_t y_hi, cudaStream_t s,
                               Remote rem = Remote());
st_status ddiv6_selftest(const double* x, int64_t n, unsigned long long* mismatches, cudaStream_t s);
// dst's side faces (x = 0, nx+1; y = 0, ny+1) of planes [z_lo, z_hi] <- src.
st_status jacobi3d_copy_faces(const double* src, double* dst, int64_t nx, int64_t ny, int64_t ldx, int64_t z_lo,
                              int64_t z_hi, cudaStream_t s);

// ------------------------------------------------------------ Gauss-Seidel 2-D ---
// `iters` in-place lexicographic sweeps (Listing 1 literally); `workspace` =
// gauss_seidel2d_workspace_bytes(nx, ny) of device scratch.
st_status gauss_seidel2d_run(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters, void* workspace,
                             cudaStream_t s);
int64_t gauss_seidel2d_workspace_bytes(int64_t nx, int64_t ny);
st_status gauss_seidel2d_preload();
// multi-sweep wavefront (gauss_seidel2d_ms.cu): K sweeps in flight per warp
int gauss_seidel2d_ms_depth();
bool gauss_seidel2d_ms_supported(int64_t nx, int64_t ny);
int64_t gauss_seidel2d_ms_workspace_bytes(int64_t nx, int64_t ny);
st_status gauss_seidel2d_ms_run(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters, void* workspace,
                                cudaStream_t s);
st_status gauss_seidel2d_ms_preload();

// ------------------------------------------------------------ PW 3-D ---
struct PwArgs {
  const double *u, *v, *w;
  double *su, *sv, *sw;
  int64_t nx, ny, nz, ldx;
  double tcx, tcy;
  const double *tzc1, *tzc2, *tzd1, *tzd2;
  int64_t y_lo = 1, y_hi = -1;  // output rows [y_lo, y_hi] (-1: ny); pencils sweep windows
};
// Computes output planes [z_lo, z_hi] (local plane indices, 1-based interior).
st_status pw_advect3d_planes(const PwArgs& a, int64_t z_lo, int64_t z_hi, cudaStream_t s);

// ------------------------------------------------------------ schedule ---
// dims = 2: rows of a 2-D grid (temporal blocking T in {1,2,4,6,8});
// dims = 3: planes of a 3-D grid (T = 1).
int choose_tblock(int32_t nranks, int64_t nx, int64_t n, int32_t h, int32_t tblock);
st_status build_jacobi_schedule(int32_t rank, int32_t nranks, int64_t nx, int64_t n, int32_t h,
                                int64_t iters, int32_t tblock, std::vector<st_op>& ops, int dims = 2);

// Eagerly loads every kernel of the library on the current device. Under CUDA's
// lazy module loading, the first launch of a kernel may wait for the device to
// drain; if another rank's stream is parked on a device-side wait (NCCL, or the
// LOCAL transport's flag waits) that wait never ends. Communicators therefore
// preload all kernels at creation.
st_status jacobi2d_preload();
st_status jacobi3d_preload();
// two sweeps per launch (T = 2) of output planes [z_lo, z_hi]; planes <= ring_lo / >= ring_hi are Dirichlet
st_status jacobi3d_two_sweeps(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                              int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t ring_lo, int64_t ring_hi,
                              cudaStream_t s, Remote rem = Remote());
// the same for the output rows [y_lo, y_hi] only (a pencil block: the buffer has ny+2 rows per
// plane; rows <= yring_lo / >= yring_hi are Dirichlet, the others of the first sweep's region
// are swept — ghost rows included)
st_status jacobi3d_two_sweeps_block(const double* src, double* dst, int64_t nx, int64_t ny, int64_t nplanes_buf,
                                    int64_t ldx, int64_t z_lo, int64_t z_hi, int64_t ring_lo, int64_t ring_hi,
                                    int64_t y_lo, int64_t y_hi, int64_t yring_lo, int64_t yring_hi, cudaStream_t s,
                                    Remote rem = Remote());
st_status stencil2d_preload();
st_status pw_advect3d_preload();
inline st_status preload_kernels() {
  ST_TRY(jacobi2d_preload());
  ST_TRY(gauss_seidel2d_preload());
  ST_TRY(jacobi3d_preload());
  ST_TRY(stencil2d_preload());
  return pw_advect3d_preload();
}

// --------------------------------------------------------------- misc ---
int env_int(const char* name, int dflt);

}  // namespace st

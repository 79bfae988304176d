// api.cu — the C ABI of libstencil (include/libstencil.h): argument validation,
// launch orchestration and error state. Every compute step runs in this
// library's own kernels (jacobi2d.cu, pw_advect3d.cu); there is no CPU path.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "internal.h"
#include "tma.cuh"

namespace st {

namespace {
thread_local char g_err[512] = {0};
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = 0; }
const char* g_err_ptr() { return g_err; }
std::atomic<uint64_t>& launch_counter() { return g_launches; }

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoi(v);
}

// ------------------------------------------------------------- TMA host ---
st_status get_encode_tiled(PFN_encodeTiled* fn) {
  static PFN_encodeTiled cached = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  static cudaDriverEntryPointQueryResult qres = cudaDriverEntryPointSuccess;
  std::call_once(once, [] {
    void* p = nullptr;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qres);
    cached = reinterpret_cast<PFN_encodeTiled>(p);
  });
  ST_RETURN_IF(err != cudaSuccess || qres != cudaDriverEntryPointSuccess || !cached, ST_ECUDA,
               "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(err));
  *fn = cached;
  return ST_OK;
}

st_status make_tmap_3d_f64(CUtensorMap* map, const double* base, const uint64_t dims[3],
                           uint64_t pitch_y_bytes, uint64_t pitch_z_bytes, const uint32_t box[3]) {
  PFN_encodeTiled enc;
  ST_TRY(get_encode_tiled(&enc));
  const cuuint64_t gdim[3] = {dims[0], dims[1], dims[2]};
  const cuuint64_t gstride[2] = {pitch_y_bytes, pitch_z_bytes};
  const cuuint32_t bx[3] = {box[0], box[1], box[2]};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), gdim, gstride,
                   bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ST_RETURN_IF(r != CUDA_SUCCESS, ST_ECUDA, "cuTensorMapEncodeTiled(3d) failed: %d", (int)r);
  return ST_OK;
}

// ------------------------------------------------------- Jacobi driver ---
namespace {

st_status check_device_ptr(const void* p, const char* what) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("%s: cudaPointerGetAttributes -> %s", what, cudaGetErrorString(e));
    return ST_EINVAL;
  }
  ST_RETURN_IF(at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged, ST_EINVAL,
               "%s is not a device pointer", what);
  return ST_OK;
}

// Executes a schedule of build_jacobi_schedule (schedule.cu) on the GPU.
// `sweep(src, dst, op, remote)` runs one SWEEP op. With a LOCAL communicator the
// pattern [boundary sweep lo, boundary sweep hi, async EXCHANGE of their
// destination, (interior sweep), JOIN] is executed fused: the boundary sweeps
// store their rows straight into the neighbours' ghost rows (NEXT #3) and the
// exchange becomes device-side flag signalling; otherwise the exchange is the
// transport's swap (NCCL p2p or copy engine).
template <typename Sweep>
st_status run_schedule_generic(const std::vector<st_op>& ops, st_comm* comm, double* a, double* b, int64_t n,
                               int64_t pitch, cudaStream_t s, Sweep sweep) {
  double* buf[2] = {a, b};
  const bool fuse = fused_halo_available(comm);
  bool pending_fused = false;  // the exchange the next JOIN completes was fused
  for (size_t i = 0; i < ops.size(); ++i) {
    const st_op& o = ops[i];
    if (fuse && o.kind == ST_OP_SWEEP && i + 2 < ops.size() && ops[i + 1].kind == ST_OP_SWEEP &&
        ops[i + 2].kind == ST_OP_EXCHANGE && ops[i + 2].flag == 1 && ops[i + 2].buf == 1 - o.buf) {
      Remote lo, hi;
      cudaEvent_t p0 = prof_mark(comm, s);
      ST_TRY(fused_halo_begin(comm, buf[1 - o.buf], n, s, &lo, &hi));
      cudaEvent_t p1 = prof_mark(comm, s);
      prof_add(comm, ST_PHASE_READY_WAIT, p0, p1);
      ST_TRY(sweep(buf[o.buf], buf[1 - o.buf], o, lo));               // first owned slabs -> rank-1
      ST_TRY(sweep(buf[o.buf], buf[1 - o.buf], ops[i + 1], hi));      // last owned slabs  -> rank+1
      prof_add(comm, ST_PHASE_BOUNDARY, p1, prof_mark(comm, s));
      ST_TRY(fused_halo_signal(comm, s));
      pending_fused = true;
      i += 2;  // the exchange op is replaced by the fused stores + flags
      continue;
    }
    switch (o.kind) {
      case ST_OP_SWEEP: {
        // a sweep right before an asynchronous exchange computes boundary slabs; others the interior
        const bool boundary = i + 1 < ops.size() && (ops[i + 1].kind == ST_OP_EXCHANGE ||
                                                     (ops[i + 1].kind == ST_OP_SWEEP && i + 2 < ops.size() &&
                                                      ops[i + 2].kind == ST_OP_EXCHANGE && ops[i + 2].flag == 1));
        cudaEvent_t p0 = prof_mark(comm, s);
        ST_TRY(sweep(buf[o.buf], buf[1 - o.buf], o, Remote()));
        prof_add(comm, boundary ? ST_PHASE_BOUNDARY : ST_PHASE_INTERIOR, p0, prof_mark(comm, s));
        break;
      }
      case ST_OP_EXCHANGE:
        ST_TRY(halo_exchange_async(comm, &buf[o.buf], 1, n, pitch, o.sweeps, s, o.flag == 0));
        break;
      case ST_OP_JOIN:
        if (comm && comm->nranks > 1) {
          cudaEvent_t p0 = prof_mark(comm, s);
          if (pending_fused) ST_TRY(fused_halo_join(comm, s));
          else ST_CHECK_CUDA(cudaStreamWaitEvent(s, comm->ev_done, 0));
          prof_add(comm, ST_PHASE_JOIN_WAIT, p0, prof_mark(comm, s));
        }
        pending_fused = false;
        break;
      case ST_OP_SWAP:
        break;
      default:
        ST_RETURN_IF(true, ST_EINTERNAL, "jacobi: bad schedule op %d", o.kind);
    }
  }
  return ST_OK;
}

st_status run_schedule(const std::vector<st_op>& ops, st_comm* comm, double* a, double* b, int64_t nx, int64_t n,
                       int64_t ld, int32_t h, cudaStream_t s) {
  const int64_t nrows = n + 2 * (int64_t)h;
  return run_schedule_generic(ops, comm, a, b, n, ld, s,
                              [&](const double* src, double* dst, const st_op& o, Remote rem) -> st_status {
                                if (o.sweeps == 1)
                                  return jacobi2d_sweep_rows(src, dst, nx, ld, o.y_lo, o.y_hi, s, rem);
                                return jacobi2d_tb_rows(src, dst, nx, ld, o.y_lo, o.y_hi, o.sweeps, o.ring_lo,
                                                        o.ring_hi, nrows, s, rem);
                              });
}

// dims=3 schedule: sweeps of planes, swaps of whole planes.
st_status run_schedule3d(const std::vector<st_op>& ops, st_comm* comm, double* a, double* b, int64_t nx,
                         int64_t ny, int64_t n, int64_t ldx, int32_t h, cudaStream_t s) {
  const int64_t nplanes = n + 2 * (int64_t)h;
  return run_schedule_generic(ops, comm, a, b, n, (ny + 2) * ldx, s,
                              [&](const double* src, double* dst, const st_op& o, Remote rem) -> st_status {
                                ST_RETURN_IF(o.sweeps != 1 && o.sweeps != 2, ST_EINTERNAL,
                                             "jacobi3d: pass of %d sweeps", o.sweeps);
                                if (o.sweeps == 2)
                                  return jacobi3d_two_sweeps(src, dst, nx, ny, nplanes, ldx, o.y_lo, o.y_hi,
                                                             o.ring_lo, o.ring_hi, s, rem);
                                return jacobi3d_sweep_planes(src, dst, nx, ny, nplanes, ldx, o.y_lo, o.y_hi, s, rem);
                              });
}

}  // namespace
}  // namespace st

using namespace st;

extern "C" {

int32_t st_abi_version(void) { return ST_ABI_VERSION; }

const char* st_last_error(void) { return g_err_ptr(); }

uint64_t st_launch_count(void) { return launch_counter().load(); }

st_status st_jacobi2d_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, int32_t halo,
                          int64_t iters, int32_t tblock, st_comm* comm, void* cuda_stream,
                          int32_t* result_in_b) {
  clear_error();
  ST_RETURN_IF(!a || !b, ST_EINVAL, "st_jacobi2d_run: null field pointer");
  ST_RETURN_IF(nx < 1 || ny < 1, ST_EINVAL, "st_jacobi2d_run: empty interior (nx=%lld, ny=%lld)",
               (long long)nx, (long long)ny);
  ST_RETURN_IF(ld < nx + 2 || (ld & 1), ST_EINVAL, "st_jacobi2d_run: ld=%lld must be even and >= nx+2",
               (long long)ld);
  ST_RETURN_IF(!aligned16(a) || !aligned16(b), ST_EINVAL, "st_jacobi2d_run: fields must be 16-byte aligned");
  ST_RETURN_IF(iters < 0 || tblock < 0 || halo < 1, ST_EINVAL,
               "st_jacobi2d_run: iters=%lld tblock=%d halo=%d", (long long)iters, tblock, halo);
  ST_RETURN_IF(!comm && halo != 1, ST_EINVAL, "st_jacobi2d_run: halo must be 1 without a comm");
  ST_RETURN_IF(comm && ny < halo, ST_EINVAL, "st_jacobi2d_run: slab of %lld rows < halo %d",
               (long long)ny, halo);
  const size_t bytes = (size_t)(ny + 2 * halo) * (size_t)ld * sizeof(double);
  ST_RETURN_IF(overlaps(a, bytes, b, bytes), ST_EINVAL, "st_jacobi2d_run: a and b overlap");
  ST_TRY(check_device_ptr(a, "a"));
  ST_TRY(check_device_ptr(b, "b"));
  if (result_in_b) *result_in_b = (int32_t)(iters & 1);
  if (iters == 0) return ST_OK;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  const int32_t nranks = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
  if (comm) ST_RETURN_IF(comm->broken, ST_ENCCL, "st_comm is unusable after an earlier NCCL error");
  // launch-bound small grids: every sweep inside one CTA's shared memory
  if (nranks == 1 && tblock == 0 && halo == 1 && jacobi2d_resident_fits(nx, ny))
    return jacobi2d_resident(a, b, nx, ny, ld, iters, s);
  std::vector<st_op> ops;
  ST_TRY(build_jacobi_schedule(rank, nranks, nx, ny, halo, iters, tblock, ops));
  // ghost / Dirichlet rows a -> b (ring columns are passed through by every sweep); pitch padding untouched
  const size_t pitch = (size_t)ld * sizeof(double), width = (size_t)(nx + 2) * sizeof(double);
  ST_CHECK_CUDA(cudaMemcpy2DAsync(b, pitch, a, pitch, width, (size_t)halo, cudaMemcpyDeviceToDevice, s));
  ST_CHECK_CUDA(cudaMemcpy2DAsync(b + (halo + ny) * ld, pitch, a + (halo + ny) * ld, pitch, width, (size_t)halo,
                                  cudaMemcpyDeviceToDevice, s));
  return run_schedule(ops, comm, a, b, nx, ny, ld, halo, s);
}

st_status st_stencil2d_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, const int32_t* offsets,
                           const double* coeffs, int32_t nterms, int64_t iters, void* cuda_stream,
                           int32_t* result_in_b) {
  clear_error();
  ST_RETURN_IF(!a || !b || !offsets || !coeffs, ST_EINVAL, "st_stencil2d_run: null pointer");
  ST_RETURN_IF(nterms < 1 || nterms > kStencilMaxTerms, ST_EINVAL, "st_stencil2d_run: %d terms (1..%d)", nterms,
               kStencilMaxTerms);
  int64_t R = 0;
  for (int i = 0; i < 2 * nterms; ++i) {
    const int64_t m = offsets[i] < 0 ? -(int64_t)offsets[i] : offsets[i];
    ST_RETURN_IF(m > kStencilMaxOffset, ST_EINVAL, "st_stencil2d_run: |offset| %lld > %d", (long long)m,
                 kStencilMaxOffset);
    R = std::max(R, m);
  }
  ST_RETURN_IF(nx < 1 || ny < 1 || ld < nx + 2 * R || iters < 0, ST_EINVAL,
               "st_stencil2d_run: bad extents (nx %lld, ny %lld, ld %lld, halo %lld)", (long long)nx, (long long)ny,
               (long long)ld, (long long)R);
  const size_t bytes = (size_t)(ny + 2 * R) * (size_t)ld * sizeof(double);
  ST_RETURN_IF(overlaps(a, bytes, b, bytes), ST_EINVAL, "st_stencil2d_run: a and b overlap");
  ST_TRY(check_device_ptr(a, "a"));
  ST_TRY(check_device_ptr(b, "b"));
  if (result_in_b) *result_in_b = (int32_t)(iters & 1);
  if (iters == 0) return ST_OK;
  return stencil2d_run(a, b, nx, ny, ld, R, offsets, coeffs, nterms, iters, static_cast<cudaStream_t>(cuda_stream));
}

st_status st_stencil_expr_info(const char* expr, int32_t* halo, int32_t* dims) {
  clear_error();
  ST_RETURN_IF(!expr || !halo || !dims, ST_EINVAL, "st_stencil_expr_info: null pointer");
  std::string cexpr;
  int64_t R = 0;
  int d = 0;
  ST_TRY(stencil_expr_translate(expr, &cexpr, &R, &d));
  *halo = (int32_t)R;
  *dims = d;
  return ST_OK;
}

st_status st_stencil2d_expr_halo(const char* expr, int32_t* halo) {
  int32_t dims = 0;
  ST_TRY(st_stencil_expr_info(expr, halo, &dims));
  ST_RETURN_IF(dims != 2, ST_EINVAL, "expression: 2-D accesses a(dy, dx) expected");
  return ST_OK;
}

st_status st_stencil3d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t nz, int64_t ldx,
                                const char* expr, int64_t iters, void* cuda_stream, int32_t* result_in_b) {
  clear_error();
  ST_RETURN_IF(!a || !b || !expr, ST_EINVAL, "st_stencil3d_expr_run: null pointer");
  std::string cexpr;
  int64_t R = 0;
  int dims = 0;
  ST_TRY(stencil_expr_translate(expr, &cexpr, &R, &dims));
  ST_RETURN_IF(dims != 3, ST_EINVAL, "st_stencil3d_expr_run: 3-D accesses a(dz, dy, dx) expected");
  ST_RETURN_IF(nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2 * R || iters < 0, ST_EINVAL,
               "st_stencil3d_expr_run: bad extents (nx %lld, ny %lld, nz %lld, ldx %lld, halo %lld)", (long long)nx,
               (long long)ny, (long long)nz, (long long)ldx, (long long)R);
  const size_t bytes = (size_t)(nz + 2 * R) * (size_t)(ny + 2 * R) * (size_t)ldx * sizeof(double);
  ST_RETURN_IF(overlaps(a, bytes, b, bytes), ST_EINVAL, "st_stencil3d_expr_run: a and b overlap");
  ST_TRY(check_device_ptr(a, "a"));
  ST_TRY(check_device_ptr(b, "b"));
  if (result_in_b) *result_in_b = (int32_t)(iters & 1);
  if (iters == 0) return ST_OK;
  return stencil3d_expr_run(a, b, nx, ny, nz, ldx, R, cexpr, iters, static_cast<cudaStream_t>(cuda_stream));
}

st_status st_stencil2d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, const char* expr,
                                int64_t iters, void* cuda_stream, int32_t* result_in_b) {
  clear_error();
  ST_RETURN_IF(!a || !b || !expr, ST_EINVAL, "st_stencil2d_expr_run: null pointer");
  std::string cexpr;
  int64_t R = 0;
  int dims = 0;
  ST_TRY(stencil_expr_translate(expr, &cexpr, &R, &dims));
  ST_RETURN_IF(dims != 2, ST_EINVAL, "st_stencil2d_expr_run: 2-D accesses a(dy, dx) expected");
  ST_RETURN_IF(nx < 1 || ny < 1 || ld < nx + 2 * R || iters < 0, ST_EINVAL,
               "st_stencil2d_expr_run: bad extents (nx %lld, ny %lld, ld %lld, halo %lld)", (long long)nx,
               (long long)ny, (long long)ld, (long long)R);
  const size_t bytes = (size_t)(ny + 2 * R) * (size_t)ld * sizeof(double);
  ST_RETURN_IF(overlaps(a, bytes, b, bytes), ST_EINVAL, "st_stencil2d_expr_run: a and b overlap");
  ST_TRY(check_device_ptr(a, "a"));
  ST_TRY(check_device_ptr(b, "b"));
  if (result_in_b) *result_in_b = (int32_t)(iters & 1);
  if (iters == 0) return ST_OK;
  return stencil2d_expr_run(a, b, nx, ny, ld, R, cexpr, iters, static_cast<cudaStream_t>(cuda_stream));
}

st_status st_stencil3d_fused_run(const double* const* inputs, int32_t nin, double* const* outputs, int32_t nout,
                                 const char* const* exprs, const double* const* plane_coefs, int32_t ncoef,
                                 int64_t nx, int64_t ny, int64_t nz, int64_t ldx, void* cuda_stream) {
  clear_error();
  ST_RETURN_IF(!inputs || !outputs || !exprs || (ncoef > 0 && !plane_coefs), ST_EINVAL,
               "st_stencil3d_fused_run: null pointer");
  int64_t R = 0;
  ST_TRY(stencil3d_fused_run(inputs, nin, outputs, nout, exprs, plane_coefs, ncoef, nx, ny, nz, ldx, &R, true,
                             nullptr));
  ST_RETURN_IF(nx < 1 || ny < 1 || nz < 1 || ldx < nx + 2 * R, ST_EINVAL,
               "st_stencil3d_fused_run: bad extents (nx %lld, ny %lld, nz %lld, ldx %lld, halo %lld)", (long long)nx,
               (long long)ny, (long long)nz, (long long)ldx, (long long)R);
  const size_t bytes = (size_t)(nz + 2 * R) * (size_t)(ny + 2 * R) * (size_t)ldx * sizeof(double);
  for (int i = 0; i < nin; ++i) {
    ST_RETURN_IF(!inputs[i], ST_EINVAL, "st_stencil3d_fused_run: null input %d", i);
    ST_TRY(check_device_ptr(inputs[i], "input"));
  }
  for (int j = 0; j < nout; ++j) {
    ST_RETURN_IF(!outputs[j], ST_EINVAL, "st_stencil3d_fused_run: null output %d", j);
    ST_TRY(check_device_ptr(outputs[j], "output"));
    for (int i = 0; i < nin; ++i)  // outputs never overlap inputs or each other (inputs may alias)
      ST_RETURN_IF(overlaps(outputs[j], bytes, inputs[i], bytes), ST_EINVAL, "output %d overlaps input %d", j, i);
    for (int q = 0; q < j; ++q)
      ST_RETURN_IF(overlaps(outputs[j], bytes, outputs[q], bytes), ST_EINVAL, "outputs %d and %d overlap", q, j);
  }
  for (int j = 0; j < ncoef; ++j) {
    ST_RETURN_IF(!plane_coefs[j], ST_EINVAL, "st_stencil3d_fused_run: null coefficient array %d", j);
    ST_TRY(check_device_ptr(plane_coefs[j], "plane coefficients"));
  }
  return stencil3d_fused_run(inputs, nin, outputs, nout, exprs, plane_coefs, ncoef, nx, ny, nz, ldx, &R, false,
                             static_cast<cudaStream_t>(cuda_stream));
}

int64_t st_gauss_seidel2d_workspace_bytes(int64_t nx, int64_t ny) {
  return nx < 1 || ny < 1 ? 0 : gauss_seidel2d_workspace_bytes(nx, ny);
}

st_status st_gauss_seidel2d_run(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters, void* workspace,
                                int64_t workspace_bytes, void* cuda_stream) {
  clear_error();
  ST_RETURN_IF(!a || !workspace, ST_EINVAL, "st_gauss_seidel2d_run: null pointer");
  ST_RETURN_IF(nx < 1 || ny < 1 || ld < nx + 2 || iters < 0, ST_EINVAL, "st_gauss_seidel2d_run: bad extents");
  ST_RETURN_IF(workspace_bytes < gauss_seidel2d_workspace_bytes(nx, ny), ST_EINVAL,
               "st_gauss_seidel2d_run: workspace of %lld bytes < %lld", (long long)workspace_bytes,
               (long long)gauss_seidel2d_workspace_bytes(nx, ny));
  ST_RETURN_IF(overlaps(a, (size_t)(ny + 2) * (size_t)ld * sizeof(double), workspace, (size_t)workspace_bytes),
               ST_EINVAL, "st_gauss_seidel2d_run: workspace overlaps the field");
  ST_TRY(check_device_ptr(a, "a"));
  ST_TRY(check_device_ptr(workspace, "workspace"));
  if (iters == 0) return ST_OK;
  return gauss_seidel2d_run(a, nx, ny, ld, iters, workspace, static_cast<cudaStream_t>(cuda_stream));
}

st_status st_selftest_div6(const double* x, int64_t n, unsigned long long* mismatches, void* cuda_stream) {
  clear_error();
  ST_RETURN_IF(!x || !mismatches || n < 0, ST_EINVAL, "st_selftest_div6: bad arguments");
  return ddiv6_selftest(x, n, mismatches, static_cast<cudaStream_t>(cuda_stream));
}

st_status st_jacobi3d_run(double* a, double* b, int64_t nx, int64_t ny, int64_t nz, int64_t ldx, int32_t halo,
                          int64_t iters, int32_t tblock, st_comm* comm, void* cuda_stream, int32_t* result_in_b) {
  clear_error();
  ST_RETURN_IF(!a || !b, ST_EINVAL, "st_jacobi3d_run: null field pointer");
  ST_RETURN_IF(nx < 1 || ny < 1 || nz < 1, ST_EINVAL, "st_jacobi3d_run: empty interior");
  ST_RETURN_IF(ldx < nx + 2 || (ldx & 1), ST_EINVAL, "st_jacobi3d_run: ldx=%lld must be even and >= nx+2",
               (long long)ldx);
  ST_RETURN_IF(!aligned16(a) || !aligned16(b), ST_EINVAL, "st_jacobi3d_run: fields must be 16-byte aligned");
  ST_RETURN_IF(iters < 0 || tblock < 0 || halo < 1, ST_EINVAL, "st_jacobi3d_run: iters=%lld tblock=%d halo=%d",
               (long long)iters, tblock, halo);
  ST_RETURN_IF(tblock > 2, ST_ENOTSUP, "st_jacobi3d_run: tblock=%d not supported (0, 1, 2)", tblock);
  ST_RETURN_IF(tblock == 2 && comm && comm->nranks > 1 && halo < 2, ST_EINVAL,
               "st_jacobi3d_run: tblock=2 across ranks needs halo >= 2");
  ST_RETURN_IF(!comm && halo != 1, ST_EINVAL, "st_jacobi3d_run: halo must be 1 without a comm");
  ST_RETURN_IF(comm && nz < halo, ST_EINVAL, "st_jacobi3d_run: slab of %lld planes < halo %d", (long long)nz, halo);
  ST_RETURN_IF(nx + 2 > (int64_t)INT32_MAX || ny + 2 > (int64_t)INT32_MAX || nz + 2 * halo > (int64_t)INT32_MAX,
               ST_EINVAL, "st_jacobi3d_run: extents exceed TMA coordinate range");
  const size_t bytes = (size_t)(nz + 2 * halo) * (size_t)(ny + 2) * (size_t)ldx * sizeof(double);
  ST_RETURN_IF(overlaps(a, bytes, b, bytes), ST_EINVAL, "st_jacobi3d_run: a and b overlap");
  ST_TRY(check_device_ptr(a, "a"));
  ST_TRY(check_device_ptr(b, "b"));
  if (result_in_b) *result_in_b = (int32_t)(iters & 1);
  if (iters == 0) return ST_OK;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  const int32_t nranks = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
  if (comm) ST_RETURN_IF(comm->broken, ST_ENCCL, "st_comm is unusable after an earlier NCCL error");
  std::vector<st_op> ops;
  ST_TRY(build_jacobi_schedule(rank, nranks, nx, nz, halo, iters, tblock, ops, 3));
  // ghost / Dirichlet planes and the side faces of the owned planes a -> b (pitch padding untouched)
  const size_t pitch = (size_t)ldx * sizeof(double), width = (size_t)(nx + 2) * sizeof(double);
  const int64_t plane = (ny + 2) * ldx;
  ST_CHECK_CUDA(cudaMemcpy2DAsync(b, pitch, a, pitch, width, (size_t)halo * (size_t)(ny + 2),
                                  cudaMemcpyDeviceToDevice, s));
  ST_CHECK_CUDA(cudaMemcpy2DAsync(b + (halo + nz) * plane, pitch, a + (halo + nz) * plane, pitch, width,
                                  (size_t)halo * (size_t)(ny + 2), cudaMemcpyDeviceToDevice, s));
  ST_TRY(jacobi3d_copy_faces(a, b, nx, ny, ldx, halo, halo + nz - 1, s));
  // Two-sweep passes across ranks also sweep the ghost planes once, which reads their side
  // faces; the fused swap stores only the interior of a plane, so b's ghost planes get their
  // (constant) side faces from a after one whole-plane swap into a.
  bool t2_ranks = false;
  for (const st_op& o : ops) t2_ranks |= nranks > 1 && o.kind == ST_OP_SWEEP && o.sweeps == 2;
  if (t2_ranks) {
    ST_TRY(halo_exchange_async(comm, &a, 1, nz, plane, halo, s, true));
    ST_TRY(jacobi3d_copy_faces(a, b, nx, ny, ldx, 0, halo - 1, s));
    ST_TRY(jacobi3d_copy_faces(a, b, nx, ny, ldx, halo + nz, nz + 2 * halo - 1, s));
    // that swap already refreshed a's ghost planes: the schedule's leading swap of a is redundant
    if (!ops.empty() && ops[0].kind == ST_OP_EXCHANGE && ops[0].buf == 0 && ops[0].flag == 0) ops.erase(ops.begin());
  }
  // two sweeps per pass (temporal blocking T = 2) where the ghosts allow it: the single domain
  // and slabs with halo >= 2 (schedule.cu choose_tblock3d); the schedule keeps the parity so
  // the result lands in b iff iters is odd
  return run_schedule3d(ops, comm, a, b, nx, ny, nz, ldx, halo, s);
}

st_status st_jacobi3d_run_pencils(double* a, double* b, int64_t nx, int64_t nyl, int64_t nzl, int64_t ldx,
                                  int32_t halo, int64_t iters, int32_t tblock, st_comm* comm, void* cuda_stream,
                                  int32_t* result_in_b) {
  clear_error();
  if (!comm || comm->nranks == 1) {
    ST_RETURN_IF(halo != 1, ST_EINVAL, "st_jacobi3d_run_pencils: halo must be 1 without a comm");
    return st_jacobi3d_run(a, b, nx, nyl, nzl, ldx, 1, iters, tblock, nullptr, cuda_stream, result_in_b);
  }
  ST_RETURN_IF(!a || !b || nx < 1 || nyl < 1 || nzl < 1 || iters < 0, ST_EINVAL,
               "st_jacobi3d_run_pencils: bad arguments");
  ST_RETURN_IF(halo < 1 || halo > 2 || nyl < halo || nzl < halo, ST_EINVAL,
               "st_jacobi3d_run_pencils: halo %d (1 or 2, <= the block's %lld rows and %lld planes)", halo,
               (long long)nyl, (long long)nzl);
  ST_RETURN_IF(tblock < 0 || tblock > 2, ST_ENOTSUP, "st_jacobi3d_run_pencils: tblock=%d not supported (0, 1, 2)",
               tblock);
  ST_RETURN_IF(tblock == 2 && halo < 2, ST_EINVAL, "st_jacobi3d_run_pencils: tblock=2 needs halo >= 2");
  ST_RETURN_IF(ldx < nx + 2 || (ldx & 1) || !aligned16(a) || !aligned16(b), ST_EINVAL,
               "st_jacobi3d_run_pencils: ldx even >= nx+2, 16-byte aligned fields");
  const int64_t H = halo, nyb = nyl + 2 * H, nb = nzl + 2 * H;
  ST_RETURN_IF(nx + 2 > (int64_t)INT32_MAX || nyb > (int64_t)INT32_MAX || nb > (int64_t)INT32_MAX, ST_EINVAL,
               "st_jacobi3d_run_pencils: extents exceed TMA coordinate range");
  const size_t bytes = (size_t)nb * (size_t)nyb * (size_t)ldx * sizeof(double);
  ST_RETURN_IF(overlaps(a, bytes, b, bytes), ST_EINVAL, "st_jacobi3d_run_pencils: a and b overlap");
  ST_TRY(check_device_ptr(a, "a"));
  ST_TRY(check_device_ptr(b, "b"));
  ST_RETURN_IF(comm->broken, ST_ENCCL, "st_comm is unusable after an earlier error");
  if (result_in_b) *result_in_b = (int32_t)(iters & 1);
  if (iters == 0) return ST_OK;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  // passes: the single-domain schedule's (two sweeps per pass where tblock allows; parity
  // kept so the result lands in b iff iters is odd)
  const int32_t T = tblock == 0 ? (halo >= 2 ? 2 : 1) : tblock;
  std::vector<st_op> ops;
  ST_TRY(build_jacobi_schedule(0, 1, nx, nzl, 1, iters, T, ops, 3));
  // ghost / Dirichlet shell a -> b (the global boundary faces of an edge block live in its
  // ghost layer; interior ghosts are refreshed before every pass)
  const size_t pitch = (size_t)ldx * sizeof(double), width = (size_t)(nx + 2) * sizeof(double);
  const int64_t plane = nyb * ldx;
  if (H == 1) {
    ST_CHECK_CUDA(cudaMemcpy2DAsync(b, pitch, a, pitch, width, (size_t)nyb, cudaMemcpyDeviceToDevice, s));
    ST_CHECK_CUDA(cudaMemcpy2DAsync(b + (nzl + 1) * plane, pitch, a + (nzl + 1) * plane, pitch, width, (size_t)nyb,
                                    cudaMemcpyDeviceToDevice, s));
    ST_TRY(jacobi3d_copy_faces(a, b, nx, nyl, ldx, 1, nzl, s));
  } else {
    ST_CHECK_CUDA(cudaMemcpy2DAsync(b, pitch, a, pitch, width, (size_t)(nb * nyb), cudaMemcpyDeviceToDevice, s));
  }
  // Dirichlet rows / planes of the first sweep of a two-sweep pass: the global boundary (in
  // the ghost layer next to the block) on the grid's edges; none elsewhere (ghosts are swept)
  const int32_t py = comm->grid_py, iy = comm->rank % py, iz = comm->rank / py, pz = comm->nranks / py;
  const int64_t yr_lo = iy == 0 ? H - 1 : -1, yr_hi = iy == py - 1 ? H + nyl : nyb;
  const int64_t zr_lo = iz == 0 ? H - 1 : -1, zr_hi = iz == pz - 1 ? H + nzl : nb;
  const int64_t ny_k = nyb - 2;  // the kernels address ny_k + 2 rows per plane
  // one pass over the output block [z0, z1] x [y0, y1] (buffer coordinates)
  auto pass = [&](const double* src, double* dst, int sweeps, int64_t z0, int64_t z1, int64_t y0,
                  int64_t y1) -> st_status {
    if (z1 < z0 || y1 < y0) return ST_OK;
    if (sweeps == 2)
      return jacobi3d_two_sweeps_block(src, dst, nx, ny_k, nb, ldx, z0, z1, zr_lo, zr_hi, y0, y1, yr_lo, yr_hi, s);
    return jacobi3d_sweep_block(src, dst, nx, ny_k, nb, ldx, z0, z1, y0, y1, s);
  };
  double* src = a;
  double* dst = b;
  for (const st_op& o : ops) {
    if (o.kind != ST_OP_SWEEP) continue;
    const int64_t d = o.sweeps;  // the ghost depth one pass reads
    // the y/z ghost swap runs on the comm stream while the block that reads no ghost
    // (d layers in from every side) is swept; then the shell
    ST_TRY(pencil_exchange_async(comm, &src, 1, nx, nyl, nzl, ldx, halo, s, false));
    const int64_t zi0 = H + d, zi1 = H + nzl - 1 - d, yi0 = H + d, yi1 = H + nyl - 1 - d;
    cudaEvent_t p0 = prof_mark(comm, s);
    const bool split = zi1 >= zi0 && yi1 >= yi0;
    if (split) ST_TRY(pass(src, dst, (int)d, zi0, zi1, yi0, yi1));
    cudaEvent_t p1 = prof_mark(comm, s);
    prof_add(comm, ST_PHASE_INTERIOR, p0, p1);
    ST_CHECK_CUDA(cudaStreamWaitEvent(s, comm->ev_done, 0));
    cudaEvent_t p2 = prof_mark(comm, s);
    prof_add(comm, ST_PHASE_JOIN_WAIT, p1, p2);
    if (split) {
      ST_TRY(pass(src, dst, (int)d, H, zi0 - 1, H, H + nyl - 1));              // low z band
      ST_TRY(pass(src, dst, (int)d, zi1 + 1, H + nzl - 1, H, H + nyl - 1));    // high z band
      ST_TRY(pass(src, dst, (int)d, zi0, zi1, H, yi0 - 1));                    // low y band
      ST_TRY(pass(src, dst, (int)d, zi0, zi1, yi1 + 1, H + nyl - 1));          // high y band
    } else {
      ST_TRY(pass(src, dst, (int)d, H, H + nzl - 1, H, H + nyl - 1));
    }
    prof_add(comm, ST_PHASE_BOUNDARY, p2, prof_mark(comm, s));
    double* t = src;
    src = dst;
    dst = t;
  }
  return ST_OK;
}

static st_status pw_validate(double* u, double* v, double* w, double* su, double* sv, double* sw, int64_t nx,
                             int64_t ny, int64_t nz, int64_t ldx, const double* tzc1, const double* tzc2,
                             const double* tzd1, const double* tzd2, bool distinct);

st_status st_pw_advect3d_pencils(double* u, double* v, double* w, double* su, double* sv, double* sw, int64_t nx,
                                 int64_t nyl, int64_t nzl, int64_t ldx, double tcx, double tcy, const double* tzc1,
                                 const double* tzc2, const double* tzd1, const double* tzd2, st_comm* comm,
                                 void* cuda_stream) {
  clear_error();
  if (!comm || comm->nranks == 1)
    return st_pw_advect3d(u, v, w, su, sv, sw, nx, nyl, nzl, ldx, tcx, tcy, tzc1, tzc2, tzd1, tzd2, nullptr,
                          cuda_stream);
  ST_TRY(pw_validate(u, v, w, su, sv, sw, nx, nyl, nzl, ldx, tzc1, tzc2, tzd1, tzd2, true));
  ST_RETURN_IF(comm->broken, ST_ENCCL, "st_comm is unusable after an earlier error");
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  // y/z ghosts (incl. the corners the diagonal offsets read) in flight on the comm stream
  // while the block that reads none (planes 2..nzl-1 x rows 2..nyl-1) is advected; then
  // the shell
  double* f[3] = {u, v, w};
  ST_TRY(pencil_exchange_async(comm, f, 3, nx, nyl, nzl, ldx, 1, s, false));
  PwArgs args{u, v, w, su, sv, sw, nx, nyl, nzl, ldx, tcx, tcy, tzc1, tzc2, tzd1, tzd2};
  auto window = [&](int64_t z0, int64_t z1, int64_t y0, int64_t y1) {
    PwArgs a = args;
    a.y_lo = y0;
    a.y_hi = y1;
    return pw_advect3d_planes(a, z0, z1, s);
  };
  cudaEvent_t p0 = prof_mark(comm, s);
  ST_TRY(window(2, nzl - 1, 2, nyl - 1));
  cudaEvent_t p1 = prof_mark(comm, s);
  prof_add(comm, ST_PHASE_INTERIOR, p0, p1);
  ST_CHECK_CUDA(cudaStreamWaitEvent(s, comm->ev_done, 0));
  cudaEvent_t p2 = prof_mark(comm, s);
  prof_add(comm, ST_PHASE_JOIN_WAIT, p1, p2);
  ST_TRY(window(1, 1, 1, nyl));
  if (nzl > 1) ST_TRY(window(nzl, nzl, 1, nyl));
  if (nzl > 2) {
    ST_TRY(window(2, nzl - 1, 1, 1));
    if (nyl > 1) ST_TRY(window(2, nzl - 1, nyl, nyl));
  }
  prof_add(comm, ST_PHASE_BOUNDARY, p2, prof_mark(comm, s));
  return ST_OK;
}

static st_status pw_validate(double* u, double* v, double* w, double* su, double* sv, double* sw, int64_t nx,
                             int64_t ny, int64_t nz, int64_t ldx, const double* tzc1, const double* tzc2,
                             const double* tzd1, const double* tzd2, bool distinct) {
  const double* f[6] = {u, v, w, su, sv, sw};
  for (int i = 0; i < 6; ++i) {
    ST_RETURN_IF(!f[i], ST_EINVAL, "st_pw_advect3d: null field %d", i);
    ST_RETURN_IF(!aligned16(f[i]), ST_EINVAL, "st_pw_advect3d: field %d not 16-byte aligned", i);
  }
  ST_RETURN_IF(!tzc1 || !tzc2 || !tzd1 || !tzd2, ST_EINVAL, "st_pw_advect3d: null coefficient array");
  ST_RETURN_IF(nx < 1 || ny < 1 || nz < 1, ST_EINVAL, "st_pw_advect3d: empty interior");
  ST_RETURN_IF(ldx < nx + 2 || (ldx & 1), ST_EINVAL, "st_pw_advect3d: ldx=%lld must be even and >= nx+2",
               (long long)ldx);
  ST_RETURN_IF(nx + 2 > (int64_t)INT32_MAX || ny + 2 > (int64_t)INT32_MAX || nz + 2 > (int64_t)INT32_MAX,
               ST_EINVAL, "st_pw_advect3d: extents exceed TMA coordinate range");
  const size_t bytes = (size_t)(nz + 2) * (size_t)(ny + 2) * (size_t)ldx * sizeof(double);
  for (int o = 3; o < 6; ++o)
    for (int i = 0; i < 6; ++i)
      if (i != o)
        ST_RETURN_IF(overlaps(f[o], bytes, f[i], bytes), ST_EINVAL,
                     "st_pw_advect3d: output %d overlaps field %d", o, i);
  if (distinct)
    ST_RETURN_IF(overlaps(u, bytes, v, bytes) || overlaps(u, bytes, w, bytes) || overlaps(v, bytes, w, bytes),
                 ST_EINVAL, "st_pw_advect3d: u, v, w must be distinct with a comm");
  for (int i = 0; i < 6; ++i) ST_TRY(check_device_ptr(f[i], "st_pw_advect3d field"));
  return ST_OK;
}

st_status st_pw_advect3d(double* u, double* v, double* w, double* su, double* sv, double* sw,
                         int64_t nx, int64_t ny, int64_t nz, int64_t ldx, double tcx, double tcy,
                         const double* tzc1, const double* tzc2, const double* tzd1,
                         const double* tzd2, st_comm* comm, void* cuda_stream) {
  clear_error();
  ST_TRY(pw_validate(u, v, w, su, sv, sw, nx, ny, nz, ldx, tzc1, tzc2, tzd1, tzd2, comm != nullptr));
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  PwArgs args{u, v, w, su, sv, sw, nx, ny, nz, ldx, tcx, tcy, tzc1, tzc2, tzd1, tzd2};
  if (!comm || comm->nranks == 1) return pw_advect3d_planes(args, 1, nz, s);
  ST_RETURN_IF(comm->broken, ST_ENCCL, "st_comm is unusable after an earlier NCCL error");
  // ghost planes of u, v, w in flight while the planes that do not read them are computed
  double* fields[3] = {u, v, w};
  const int64_t plane = (ny + 2) * ldx;
  ST_TRY(halo_exchange_async(comm, fields, 3, nz, plane, 1, s, false));
  cudaEvent_t p0 = prof_mark(comm, s);
  ST_TRY(pw_advect3d_planes(args, 2, nz - 1, s));
  cudaEvent_t p1 = prof_mark(comm, s);
  prof_add(comm, ST_PHASE_INTERIOR, p0, p1);
  ST_CHECK_CUDA(cudaStreamWaitEvent(s, comm->ev_done, 0));
  cudaEvent_t p2 = prof_mark(comm, s);
  prof_add(comm, ST_PHASE_JOIN_WAIT, p1, p2);
  ST_TRY(pw_advect3d_planes(args, 1, 1, s));
  if (nz >= 2) ST_TRY(pw_advect3d_planes(args, nz, nz, s));
  prof_add(comm, ST_PHASE_BOUNDARY, p2, prof_mark(comm, s));
  return ST_OK;
}

}  // extern "C"

/* libstencil.h — C ABI of the B200-native stencil hot path (ABI version 1).
 *
 * The library implements the data-parallel hot path that the paper's
 * Flang -> stencil-dialect flow accelerates (arXiv 2310.01882): repeated
 * application of the stencils extracted from Fortran loop nests, on fields
 * that stay resident in device memory ("optimised" data
 * approach: allocation and copies hoisted out of the iteration loop, device
 * references held by the host as pointers), with a halo swap between
 * iterations when the grid is decomposed.
 *
 * Conventions (all entry points)
 *   - Field and coefficient pointers are CUDA DEVICE pointers to IEEE binary64.
 *     The caller allocates and owns every buffer and keeps it alive until the
 *     stream work completes; the library never allocates per call. `st_comm`
 *     is the only library-owned object.
 *   - Layout (the first Fortran index is contiguous):
 *       2-D: row-major a[y*ld + x]; rows 0..ny+1, columns 0..nx+1; ld >= nx+2,
 *            ld EVEN (16-byte rows); base 16-byte aligned.
 *       3-D: f[(z*(ny+2) + y)*ldx + x]; x fastest, z slowest; ldx >= nx+2, even.
 *     The outermost cell layer is the 1-cell halo ("ring"): Listing 2's input
 *     temp is one cell wider than its output, [-1,255]^2 -> [0,254]^2
 *     (PAPER.md:122).
 *   - Work is enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default
 *     stream) after all prior work on it; calls return without a host sync.
 *   - Errors: argument validation is synchronous, returns ST_EINVAL and
 *     enqueues nothing. CUDA launch/API failures return ST_ECUDA, NCCL failures
 *     ST_ENCCL (the st_comm is unusable afterwards). Asynchronous device faults
 *     surface at the caller's next synchronisation (CUDA semantics). No
 *     exceptions cross the ABI, nothing aborts or prints. st_last_error()
 *     describes the most recent failure on the calling thread.
 *   - Threads: calls without a comm are reentrant. An st_comm is used by one
 *     thread, and all ranks issue the same sequence of comm calls (NCCL rule).
 *   - Arithmetic: every kernel evaluates the association trees of DESIGN.md
 *     R2/R6 with one rounding per operation (no FMA contraction), so results
 *     are bitwise identical to the CPU oracle, for every tiling, temporal
 *     blocking depth and decomposition.
 */
#ifndef LIBSTENCIL_H
#define LIBSTENCIL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ST_OK = 0,
  ST_EINVAL = 1,    /* bad argument; nothing was enqueued */
  ST_ECUDA = 2,     /* CUDA runtime/driver error */
  ST_ENCCL = 3,     /* NCCL error; the communicator is unusable */
  ST_ENOTSUP = 4,   /* valid request this build does not support */
  ST_EINTERNAL = 5, /* library bug */
  ST_ETIMEDOUT = 6  /* st_comm_wait: queued work did not finish in time (e.g. a rank never joined a swap) */
} st_status;

#define ST_ABI_VERSION 1

/* Returns ST_ABI_VERSION of the loaded library. */
int32_t st_abi_version(void);

/* Thread-local description of the last failing call on this thread ("" if none).
 * Valid until the next st_* call on the same thread. */
const char* st_last_error(void);

/* Number of kernel launches this library has issued in this process (all
 * devices, all threads). Diagnostic counter used by the benchmark's
 * `gpu_launches` report; never reset. */
uint64_t st_launch_count(void);

/* ------------------------------------------------------------------------ */
/* Communicator (slab decomposition across ranks; one process per GPU)       */
/* ------------------------------------------------------------------------ */

typedef struct st_comm st_comm; /* opaque, library-owned */

#define ST_UNIQUE_ID_BYTES 128 /* == sizeof(ncclUniqueId) */

/* Rank 0 creates the id; the caller broadcasts it (e.g. over torch.distributed). */
st_status st_comm_unique_id(uint8_t id[ST_UNIQUE_ID_BYTES]);

/* Collective over `nranks` processes: creates the NCCL communicator, an
 * internal comm stream and events on `cuda_device`. Rank r owns slab r of the
 * slowest axis (block split, remainder to the high ranks: st_block_split). */
st_status st_comm_init(st_comm** out, int32_t nranks, int32_t rank,
                       const uint8_t id[ST_UNIQUE_ID_BYTES], int32_t cuda_device);

/* Borrow an existing NCCL communicator (e.g. torch's ProcessGroupNCCL
 * `_comm_ptr()` for the group's device): `nccl_comm` is an ncclComm_t living on
 * `cuda_device`; rank and size are taken from it. The library adds its own comm
 * stream and events but never destroys the borrowed communicator — the owner
 * keeps it alive until st_comm_destroy returns. ST_ENCCL if `nccl_comm` is not a
 * valid communicator of the NCCL the library is linked against (one NCCL per
 * process: the torch wheel's), ST_EINVAL if it lives on another device.
 * SURVEY.md §8(b); NCCL p2p halo swaps over NVLink. */
st_status st_comm_from_nccl(st_comm** out, void* nccl_comm, int32_t cuda_device);

/* Failure detection: blocks until all work queued so far on
 * `cuda_stream` (and the comm's own stream) has completed, polling every
 * ~100 us instead of a blocking synchronize. NCCL communicators are also
 * polled with ncclCommGetAsyncError. Returns ST_OK; ST_ENCCL on an asynchronous
 * NCCL error (the communicator is aborted and unusable); ST_ECUDA on a device
 * fault; ST_ETIMEDOUT if `timeout_ms` > 0 elapsed with work still pending —
 * typically a neighbour that never joined a halo swap. On timeout an NCCL
 * communicator is aborted (ncclCommAbort) so its kernels drain; a LOCAL/IPC
 * flag wait cannot be cancelled: the work completes if the late rank joins,
 * otherwise the caller must tear the process down. After a timeout the comm is
 * marked broken (any transport): later calls on it fail with ST_ENCCL instead of
 * queueing behind the stuck wait. timeout_ms <= 0: no limit. */
st_status st_comm_wait(st_comm* comm, void* cuda_stream, int32_t timeout_ms);

/* Phase profiler (SURVEY.md §5 "overlap evidence"; PAPER.md:268 halo swap
 * overlapped with interior compute). With profiling enabled, every st_* call on
 * `comm` records CUDA timing events around its phases:
 *   ST_PHASE_BOUNDARY    boundary rows/planes (their fused neighbour stores included)
 *   ST_PHASE_INTERIOR    rows/planes computed while the swap is in flight (and
 *                        whole-slab sweeps that overlap nothing)
 *   ST_PHASE_JOIN_WAIT   time the caller's stream is blocked waiting for the
 *                        neighbours' ghosts (0 when the swap is fully hidden)
 *   ST_PHASE_SWAP        the swap on the comm stream (copy-engine / NCCL transports)
 *   ST_PHASE_READY_WAIT  fused transport: waiting until the neighbours' ghost rows
 *                        may be overwritten
 * st_comm_profile_read waits for the recorded events, writes per-phase totals in
 * milliseconds and interval counts, and clears them. Profiling adds event records
 * to the streams; leave it off for timed runs. enable = 0 stops recording. */
enum { ST_PHASE_BOUNDARY = 0, ST_PHASE_INTERIOR = 1, ST_PHASE_JOIN_WAIT = 2, ST_PHASE_SWAP = 3,
       ST_PHASE_READY_WAIT = 4, ST_PHASES = 5 };
st_status st_comm_profile(st_comm* comm, int32_t enable);
st_status st_comm_profile_read(st_comm* comm, double ms[ST_PHASES], int64_t counts[ST_PHASES]);

/* Single-process group of `nranks` ranks (LOCAL transport): comms[r] is rank r,
 * on CUDA device devices[r] (devices may repeat; distinct devices get peer
 * access enabled). The halo swap copies boundary slabs straight into the
 * neighbour's ghost slabs with the copy engines, ordered by device-side flags
 * (stream memory operations), so no SM and no host synchronisation is used and
 * the ranks' st_* calls may be issued sequentially from one host thread.
 * Every rank must st_comm_bind the buffers it will swap. Ranks that share a device
 * order each other with stream waits, which deadlock if two of their streams share a
 * hardware queue: with k > 1 ranks on one device CUDA_DEVICE_MAX_CONNECTIONS must be
 * >= 2k+1 (set before CUDA initialises), else ST_ENOTSUP. */
st_status st_comm_init_local(st_comm** comms, int32_t nranks, const int32_t* devices);

/* One rank of a multi-process group using the IPC transport: the LOCAL
 * protocol (copy-engine or fused swaps ordered by device-side flags) on
 * CUDA-IPC mappings of the neighbour processes' buffers and flags. Works across
 * GPUs of one node (NVLink peer access) and for several ranks on one GPU.
 * Follow with st_comm_export on every rank, an all-gather of the blobs by the
 * caller (e.g. torch.distributed), and st_comm_import of the neighbours. */
st_status st_comm_init_ipc(st_comm** out, int32_t nranks, int32_t rank, int32_t cuda_device);

/* Binds `buffers` (as st_comm_bind) and writes this rank's IPC description
 * (flags + buffers: handles, offsets, slab count) into blob[0..cap); *used =
 * bytes written (call with cap = 0 to size it). IPC comms only. */
st_status st_comm_export(st_comm* comm, double* const* buffers, int32_t nbuffers, int64_t n_slow_local,
                         uint8_t* blob, int64_t cap, int64_t* used);

/* Maps the blob exported by rank `peer` if it is a neighbour (rank -/+ 1);
 * other ranks' blobs are ignored. IPC comms only. Re-importing a peer replaces its
 * mappings; the library synchronises the device before unmapping the old ones, so
 * work still queued against them completes first. */
st_status st_comm_import(st_comm* comm, int32_t peer, const uint8_t* blob, int64_t bytes);

/* Pencils (2-D (y, z) process grid, "decompose the 3D space into two
 * dimensions"; IPC/LOCAL transports): py ranks along y,
 * nranks/py along z, rank = iz*py + iy; ny_local = this rank's owned rows.
 * Call before st_comm_export / the pencil entry points. */
st_status st_comm_set_grid(st_comm* comm, int32_t py, int64_t ny_local);

/* Block of `rank` in a py x pz grid over ny rows and nz planes (remainder to
 * the high ranks in each dimension). Host-only. */
st_status st_pencil_split(int64_t ny, int64_t nz, int32_t py, int32_t pz, int32_t rank, int64_t* y0, int64_t* ny_local,
                          int64_t* z0, int64_t* nz_local);

/* Registers the buffers this rank swaps (LOCAL transport; no-op for NCCL): all
 * ranks bind the same number of buffers in the same order (buffer i of rank r
 * exchanges with buffer i of its neighbours), each holding n_slow_local owned
 * slabs. Re-binding replaces the previous set. */
st_status st_comm_bind(st_comm* comm, double* const* buffers, int32_t nbuffers, int64_t n_slow_local);

/* Frees the communicator's NCCL comm or group slot, stream, events and flags
 * (waits for pending comm work). */
st_status st_comm_destroy(st_comm* comm);

st_status st_comm_query(const st_comm* comm, int32_t* rank, int32_t* nranks, int32_t* cuda_device);

/* Block split of n items over nranks (remainder to the high
 * ranks). Host-only; no device needed. */
st_status st_block_split(int64_t n, int32_t nranks, int32_t rank, int64_t* start, int64_t* count);

/* One transfer of a halo swap: `count` doubles starting at element `offset`
 * of a field, to/from rank `peer`. */
typedef struct {
  int32_t peer;
  int64_t offset;
  int64_t count;
} st_xfer;

/* The halo-swap plan of st_halo_exchange for one rank (host-only; no device
 * needed, so the decomposition logic is testable on CPU): a field holds
 * n_slow_local + 2*width slabs of slab_pitch doubles, slabs 0..width-1 and
 * width+n_slow_local.. are ghosts. Sends the first/last `width` owned slabs to
 * rank-1/rank+1 and receives into the ghost slabs; the edge ranks skip the
 * missing side (non-periodic). Fills up to two sends and two
 * receives, ordered by direction (low neighbour first). */
st_status st_halo_plan(int32_t rank, int32_t nranks, int64_t n_slow_local, int64_t slab_pitch,
                       int32_t width, st_xfer sends[2], int32_t* nsend, st_xfer recvs[2],
                       int32_t* nrecv);

/* Slowest-axis halo swap of `nfields` fields (device pointers), all in one
 * NCCL group, ordered on `cuda_stream` (the comm stream joins back with an
 * event). Requires n_slow_local >= width >= 1. nranks == 1: no-op. */
st_status st_halo_exchange(st_comm* comm, double* const* fields, int32_t nfields,
                           int64_t n_slow_local, int64_t slab_pitch, int32_t width,
                           void* cuda_stream);

/* ------------------------------------------------------------------------ */
/* 2-D Jacobi 5-point sweep (Listing 1)                      */
/* ------------------------------------------------------------------------ */

/* One step of the per-rank schedule st_jacobi2d_run executes (host-only, so
 * the decomposition / halo-swap / temporal-blocking logic is testable without
 * a GPU). Buffers: 0 = a, 1 = b.
 *   ST_OP_SWEEP     dst = buffer 1-buf gets rows [y_lo, y_hi] (buffer rows) of
 *                   the state `sweeps` Jacobi sweeps after buffer `buf`; rows
 *                   <= ring_lo and >= ring_hi are Dirichlet (unchanged at every
 *                   level). sweeps == 1: one sweep; sweeps >= 2 (even): one
 *                   temporally blocked pass.
 *   ST_OP_EXCHANGE  halo swap (st_halo_plan, width `sweeps`) of buffer `buf`;
 *                   flag = 1: asynchronous (overlaps the following sweeps and
 *                   must be joined by ST_OP_JOIN), 0: joined immediately.
 *   ST_OP_JOIN      the main stream waits for the pending exchange.
 *   ST_OP_SWAP      the roles of the buffers swap (the next state lives in 1-buf). */
enum { ST_OP_SWEEP = 1, ST_OP_EXCHANGE = 2, ST_OP_JOIN = 3, ST_OP_SWAP = 4 };

typedef struct {
  int32_t kind;
  int32_t buf;
  int32_t sweeps;
  int32_t flag;
  int64_t y_lo, y_hi;
  int64_t ring_lo, ring_hi;
} st_op;

/* Builds the schedule of st_jacobi2d_run for one rank: `iters` sweeps of a
 * slab of ny_local owned rows with `halo` ghost rows per side (nranks == 1:
 * halo must be 1 and the ghost rows are the Dirichlet rows), temporal
 * blocking depth `tblock` (1, or even T <= halo; 0 = auto). Writes up to `cap`
 * ops and the total count to *nops (call with cap = 0 to size the buffer).
 * Host-only; no device needed. */
st_status st_jacobi2d_schedule(int32_t rank, int32_t nranks, int64_t nx, int64_t ny_local,
                               int32_t halo, int64_t iters, int32_t tblock, st_op* ops,
                               int64_t cap, int64_t* nops);

/* The schedule of st_jacobi3d_run for one rank, as st_jacobi2d_schedule with
 * planes for rows: nz_local owned planes, `halo` ghost planes per side,
 * tblock 0 (auto), 1 or 2 (sweeps per pass; y_lo/y_hi/ring_lo/ring_hi are
 * plane indices of the slab buffer). Host-only; no device needed. */
st_status st_jacobi3d_schedule(int32_t rank, int32_t nranks, int64_t nx, int64_t nz_local,
                               int32_t halo, int64_t iters, int32_t tblock, st_op* ops,
                               int64_t cap, int64_t* nops);

/* `iters` sweeps of
 *     B[y][x] = (((A[y-1][x] + A[y+1][x]) + A[y][x-1]) + A[y][x+1]) * 0.25
 * over the interior 1 <= y <= ny_local, 1 <= x <= nx, with value semantics
 * (stencil.apply evaluates over every cell of a snapshot), i.e.
 * Jacobi double buffering: roles of a and b swap after every sweep.
 *
 *   a, b      (ny_local + 2*halo) rows x ld doubles each, non-overlapping.
 *             `a` holds the initial state including the halo; the library
 *             copies the halo rows a -> b. Columns 0 and nx+1 are the
 *             Dirichlet ring and are never changed.
 *   comm NULL halo must be 1; rows 0 and ny_local+1 are the Dirichlet ring.
 *   comm set  rank-local row slab of a global grid; halo = ghost depth
 *             (>= max(1, tblock)); ghost rows are refreshed from the
 *             neighbouring ranks whenever the sweeps since the last swap
 *             would exceed `halo`, and the swap of a pass's boundary rows
 *             overlaps that pass's interior rows. On the first/last rank the
 *             ghost row adjacent to the owned rows holds the global Dirichlet
 *             row. Requires ny_local >= halo. The exact step sequence is
 *             st_jacobi2d_schedule's.
 *   iters     >= 0; 0 is a no-op.
 *   tblock    0 = auto (10 on grids >= 128^2, capped by the ghost depth across
 *             ranks); 1 = one sweep per pass over HBM; T in {2, 4, 6, 8, 10} =
 *             temporal blocking (T sweeps per pass); other T: ST_ENOTSUP. Any
 *             choice gives bitwise the same result.
 *   *result_in_b (may be NULL) set to 1 if the result is in b (iters odd),
 *             else 0. The other buffer's interior is unspecified afterwards.
 */
st_status st_jacobi2d_run(double* a, double* b, int64_t nx, int64_t ny_local, int64_t ld,
                          int32_t halo, int64_t iters, int32_t tblock, st_comm* comm,
                          void* cuda_stream, int32_t* result_in_b);

/* Generic linear 2-D stencil.apply (reading R23 of DESIGN.md; NEXT #4): the
 * stencil dialect's apply over constant-offset accesses of a
 * loop nest the discovery pass extracts (RHS offsets
 * PAPER.md:185), for linear right-hand sides:
 *     out(y,x) = c_0*a(y+dy_0, x+dx_0) + c_1*a(y+dy_1, x+dx_1) + ...
 * evaluated left to right, one rounding per product and per sum (no FMA).
 * `offsets` (HOST, nterms x {dy, dx}, |offset| <= 8) and `coeffs` (HOST,
 * nterms <= 32) are copied at the call. Halo R = max |offset|:
 * a, b are (ny + 2R) rows x ld (ld >= nx + 2R), interior rows R..R+ny-1 and
 * columns R..R+nx-1; the R-wide ring is a fixed Dirichlet boundary. Value
 * semantics (Jacobi ping-pong): the library copies a -> b first; after `iters`
 * sweeps the result is in b iff (*result_in_b = iters & 1). Errors as
 * st_jacobi2d_run (ST_EINVAL before anything is enqueued). */
st_status st_stencil2d_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, const int32_t* offsets,
                           const double* coeffs, int32_t nterms, int64_t iters, void* cuda_stream,
                           int32_t* result_in_b);

/* Expression stencil (reading R24 of DESIGN.md; NEXT #4 "offset list +
 * expression -> NVRTC-compiled kernel"): `expr` is the loop body's right-hand
 * side over accesses a(dy, dx) (|offset| <= 8), numeric literals, + - * /,
 * unary signs and parentheses, e.g. Listing 1:
 *     "(a(-1,0) + a(1,0) + a(0,-1) + a(0,1)) * 0.25"
 * C/Fortran precedence, left associative; literals are binary64 (never integer
 * arithmetic); every operation rounds once, none is contracted. The text is
 * validated and translated token by token, compiled once per (expression,
 * device) with NVRTC for sm_100a (--fmad=false; loaded with dlopen:
 * ST_ENOTSUP without libnvrtc) and cached for the process. Layout, halo
 * R = max |offset|, ring, value semantics and result_in_b as st_stencil2d_run.
 * st_stencil2d_expr_halo validates `expr` on the host only and returns R
 * (ST_EINVAL with the reason in st_last_error for anything outside the grammar). */
st_status st_stencil2d_expr_halo(const char* expr, int32_t* halo);
/* The same for 3-D fields (x fastest, z slowest; R5): accesses
 * a(dz, dy, dx); arrays (nz + 2R) planes x (ny + 2R) rows x ldx, interior
 * planes/rows/columns R .. R+n-1. The paper's benchmark 1 is
 * "(a(-1,0,0)+a(1,0,0)+a(0,-1,0)+a(0,1,0)+a(0,0,-1)+a(0,0,1))/6" (R20/R21).
 * st_stencil_expr_info returns the halo and the access arity (2 or 3). */
st_status st_stencil_expr_info(const char* expr, int32_t* halo, int32_t* dims);
st_status st_stencil3d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t nz, int64_t ldx,
                                const char* expr, int64_t iters, void* cuda_stream, int32_t* result_in_b);

/* Fused region ("three separate stencil computations across three
 * fields which are then fused ... into a single stencil region"): one pass over
 * the interior computes nout (<= 8) outputs from nin (<= 8) input fields. Each
 * exprs[j] (HOST string) uses f<i>(dz, dy, dx) for input field i, k<c> for the
 * value of per-plane coefficient array c (device, nz + 2R doubles) at the output
 * point's plane, literals, + - * /, unary signs and parentheses (grammar and
 * rounding as st_stencil2d_expr_run; compiled once per region with NVRTC). All
 * fields are (nz + 2R) x (ny + 2R) x ldx, x fastest, R = max |offset|; only
 * interior points of the outputs are written. Inputs may alias each other,
 * outputs may not overlap anything. One application per call (not iterated).
 * The Piacsek-Williams advection as such a region: st_pw_fused_expression. */
st_status st_stencil3d_fused_run(const double* const* inputs, int32_t nin, double* const* outputs, int32_t nout,
                                 const char* const* exprs, const double* const* plane_coefs, int32_t ncoef,
                                 int64_t nx, int64_t ny, int64_t nz, int64_t ldx, void* cuda_stream);
st_status st_stencil2d_expr_run(double* a, double* b, int64_t nx, int64_t ny, int64_t ld, const char* expr,
                                int64_t iters, void* cuda_stream, int32_t* result_in_b);

/* The Piacsek-Williams advection (association trees of DESIGN.md
 * reading R6) as the expression `which` (0 = su, 1 = sv, 2 = sw) of a fused region
 * over f0 = u, f1 = v, f2 = w and per-plane coefficients k0 = tzc1, k1 = tzc2,
 * k2 = tzd1, k3 = tzd2, with tcx and tcy written as 17-significant-digit literals
 * (they round-trip binary64). Writes the NUL-terminated text into out[0..cap) and
 * its size incl. the NUL into *used (cap = 0: size only). Host-only. */
st_status st_pw_fused_expression(double tcx, double tcy, int32_t which, char* out, int64_t cap, int64_t* used);

/* Listing 1 taken literally (R22; NEXT #4): `iters`
 * IN-PLACE lexicographic Gauss-Seidel sweeps of `a` ((ny+2) rows x ld, ring =
 * Dirichlet): rows in increasing y, columns in increasing x, each point
 *     a[y][x] = (((a[y-1][x] + a[y+1][x]) + a[y][x-1]) + a[y][x+1]) * 0.25
 * with the values the sequential loop sees (N, W already updated). Bitwise the
 * sequential loop nest. `workspace` = st_gauss_seidel2d_workspace_bytes(nx, ny)
 * bytes of caller-owned device memory (progress words of the wavefront and, for
 * the multi-sweep schedule, one edge row per strip: ~32 B x (nx+2) x ny/29).
 * Grids at least 224 columns wide run K = 4 sweeps per pass over the grid
 * (strips of 29 rows; ST_GS_MS_K = 1..4 overrides K, ST_GS_MS=0 disables it),
 * narrower ones one sweep per pass (strips of 32 rows). ST_ENOTSUP if the
 * strips cannot all be resident on the device; the launch is cooperative
 * (co-residency guaranteed by the driver, or ST_ECUDA). */
int64_t st_gauss_seidel2d_workspace_bytes(int64_t nx, int64_t ny);
st_status st_gauss_seidel2d_run(double* a, int64_t nx, int64_t ny, int64_t ld, int64_t iters, void* workspace,
                                int64_t workspace_bytes, void* cuda_stream);

/* ------------------------------------------------------------------------ */
/* 3-D 7-point Jacobi (the paper's benchmark 1)                 */
/* ------------------------------------------------------------------------ */

/* `iters` sweeps of the 7-point average
 *     B = (((((A[z-1] + A[z+1]) + A[y-1]) + A[y+1]) + A[x-1]) + A[x+1]) / 6.0
 * ("averages values across the six neighbouring cells", six flops per cell,
 * PAPER.md:214; R20/R21) over the interior with value semantics
 * (Jacobi double buffering, as st_jacobi2d_run).
 *
 *   a, b      (nz_local + 2*halo) planes x (ny+2) rows x ldx doubles, x fastest,
 *             ldx even >= nx+2, 16-byte aligned, non-overlapping. `a` holds the
 *             initial state including every Dirichlet face; the library copies
 *             the faces and ghost planes a -> b. The side faces (x = 0, nx+1;
 *             y = 0, ny+1) and, without a comm, planes 0 and nz_local+1 are
 *             Dirichlet and never change.
 *   comm      NULL: halo must be 1. Set: rank-local z-slab, halo = ghost-plane
 *             depth; planes are swapped with rank -/+ 1 every `halo` sweeps
 *             (boundary planes first, swap overlapped with the interior
 *             planes); edge ranks keep the global Dirichlet plane next to their
 *             owned planes. Requires nz_local >= halo. The exact step
 *             sequence is st_jacobi3d_schedule's.
 *   tblock    1 = one sweep per pass over HBM; 2 = two sweeps per pass
 *             (temporal blocking; across ranks it needs halo >= 2, else
 *             ST_EINVAL); 0 = auto: 2 on a single domain and on slabs with
 *             halo >= 2, else 1; others -> ST_ENOTSUP. Any choice gives
 *             bitwise the same result.
 *   *result_in_b (may be NULL) = iters & 1. */
st_status st_jacobi3d_run(double* a, double* b, int64_t nx, int64_t ny, int64_t nz_local, int64_t ldx,
                          int32_t halo, int64_t iters, int32_t tblock, st_comm* comm,
                          void* cuda_stream, int32_t* result_in_b);

/* The 3-D 7-point Jacobi on a pencil block (the paper's "decompose the 3D
 * space into two dimensions"): a, b hold (nz_local+2*halo)
 * planes x (ny_local+2*halo) rows x ldx (halo ghost layers in y and z; on the
 * grid's edges the ghost layer next to the block holds the global Dirichlet
 * face). Before every pass the halo y ghost rows and then the halo z ghost
 * planes are swapped with the 4 grid neighbours (comm set up with
 * st_comm_set_grid; IPC or LOCAL transport; NCCL -> ST_ENOTSUP), overlapped
 * with the part of the block that reads no ghost.
 *   halo     1 or 2 (<= ny_local, nz_local); 1 without a comm.
 *   tblock   1 = one sweep per pass; 2 = two sweeps per pass (needs halo 2:
 *            the first sweep also runs on the first ghost layer); 0 = auto
 *            (2 if halo >= 2). Bitwise the same result either way.
 *   comm NULL: single block (st_jacobi3d_run).
 *   *result_in_b (may be NULL) = iters & 1. */
st_status st_jacobi3d_run_pencils(double* a, double* b, int64_t nx, int64_t ny_local, int64_t nz_local, int64_t ldx,
                                  int32_t halo, int64_t iters, int32_t tblock, st_comm* comm, void* cuda_stream,
                                  int32_t* result_in_b);

/* Diagnostic: counts into *mismatches (device, uint64, caller-zeroed) the x[i]
 * (device, n doubles) for which the kernels' fast correctly rounded x/6 differs
 * bitwise from the generic IEEE division. Used by the tests. */
st_status st_selftest_div6(const double* x, int64_t n, unsigned long long* mismatches, void* cuda_stream);

/* ------------------------------------------------------------------------ */
/* 3-D Piacsek-Williams advection                              */
/* ------------------------------------------------------------------------ */

/* One fused application of the three PW advection stencils (su from u, v, w;
 * sv; sw — "three separate stencil computations across three fields ... fused
 * into a single stencil region", 63 flops per cell), formula =
 * DESIGN.md reading R6 (MONC pwadvection form). Overwrites the interior
 * (1..nz_local, 1..ny, 1..nx) of su, sv, sw; never touches their halos.
 *
 *   u,v,w,su,sv,sw  (nz_local+2) planes x (ny+2) rows x ldx doubles each.
 *                   su, sv, sw must not overlap each other or the inputs.
 *                   Without comm u, v, w are read only and may alias each
 *                   other; with comm their z-ghost planes are written and they
 *                   must be distinct.
 *   tcx, tcy        x/y coefficients (scalars).
 *   tzc1..tzd2      nz_local+2 doubles each (device), indexed by local plane.
 *   comm NULL       the halos of u, v, w are inputs.
 *   comm set        rank-local z-slab; the z-ghost planes of u, v, w are first
 *                   swapped with rank -/+ 1 (the PW halo swap "before the next
 *                   timestep"), overlapped with interior planes.
 */
st_status st_pw_advect3d(double* u, double* v, double* w, double* su,
                         double* sv, double* sw, int64_t nx, int64_t ny, int64_t nz_local,
                         int64_t ldx, double tcx, double tcy, const double* tzc1,
                         const double* tzc2, const double* tzd1, const double* tzd2,
                         st_comm* comm, void* cuda_stream);

/* PW advection on a pencil block (layout as st_jacobi3d_run_pencils; u, v, w
 * ghosts — including the (y, z) corners the diagonal offsets read — are first
 * swapped y-then-z with the grid neighbours). tz*: nz_local+2 doubles. */
st_status st_pw_advect3d_pencils(double* u, double* v, double* w, double* su, double* sv, double* sw, int64_t nx,
                                 int64_t ny_local, int64_t nz_local, int64_t ldx, double tcx, double tcy,
                                 const double* tzc1, const double* tzc2, const double* tzd1, const double* tzd2,
                                 st_comm* comm, void* cuda_stream);

#ifdef __cplusplus
}
#endif

#endif /* LIBSTENCIL_H */

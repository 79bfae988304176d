// comm.h — st_comm: a rank of a slab decomposition plus the streams/events that
// let the halo swap of one sweep run concurrently with the interior rows.
//
// Two transports:
//  * NCCL  — one process per GPU, ncclSend/ncclRecv on a comm stream.
//  * IPC   — one process per rank (torchrun), same protocol as LOCAL on
//            CUDA-IPC-mapped buffers and flags of the neighbour processes
//            (so it also runs with several ranks on ONE GPU, which NCCL refuses).
//  * LOCAL — a group of ranks inside one process (same or different GPUs):
//            the swap is a copy-engine cudaMemcpyAsync into the neighbour's
//            ghost slabs, ordered by device-side flags written/waited with
//            stream memory operations (cuStreamWriteValue32/WaitValue32), so
//            no SM and no host synchronisation is involved and the ranks'
//            calls may be issued one after another from one host thread.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <vector>

#include "libstencil.h"

struct st_local_group;

// A neighbour rank's swap targets as seen from this process: its flags and its
// bound buffers (direct pointers for LOCAL; IPC-mapped pointers for IPC).
struct st_peer {
  bool valid = false;
  uint32_t* flags = nullptr;
  std::vector<double*> bound;
  int64_t n_slow = 0;
  int64_t n_mid = 0;  // pencils: owned rows (y) of the peer's blocks
  int32_t device = 0;
  std::vector<void*> opened;  // IPC mappings to close
};

struct st_comm {
  enum Kind { NCCL = 0, LOCAL = 1, IPC = 2 };
  Kind kind = NCCL;
  ncclComm_t nccl = nullptr;
  int32_t rank = 0;
  int32_t nranks = 1;
  int32_t device = 0;
  cudaStream_t comm_stream = nullptr;  // swap work runs here
  cudaEvent_t ev_ready = nullptr;      // main -> comm: boundary rows are written
  cudaEvent_t ev_done = nullptr;       // comm -> main: ghost rows have arrived
  bool broken = false;                 // set after an NCCL error
  bool borrowed = false;               // nccl came from st_comm_from_nccl: not destroyed here
  // LOCAL transport
  st_local_group* group = nullptr;
  uint32_t* flags = nullptr;  // device: [0] ready, [1]/[2] done from the low/high slab (or z) neighbour,
                              // [3]/[4] done from the low/high y neighbour (pencils)
  uint32_t seq = 0;           // swaps issued so far (all ranks issue the same sequence)
  std::vector<double*> bound;  // buffers registered with st_comm_bind (same order on every rank)
  int64_t bound_n_slow = 0;    // owned slabs of this rank's bound buffers
  // IPC transport: the neighbour ranks imported from their blobs (rank, view)
  std::vector<std::pair<int32_t, st_peer>> ipc_peers;
  // pencil grid (st_comm_set_grid): grid_py ranks along y, nranks/grid_py along z,
  // rank = iz * grid_py + iy; n_mid = this rank's owned rows. grid_py == 0: slabs.
  int32_t grid_py = 0;
  int64_t n_mid = 0;
  // phase profiler (st_comm_profile): CUDA-event pairs per phase, summed and reset by
  // st_comm_profile_read; events come from a pool owned by the comm
  bool prof = false;
  std::vector<cudaEvent_t> prof_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[ST_PHASES];
};

struct st_local_group {
  int32_t nranks = 0;
  int32_t alive = 0;
  std::vector<st_comm*> ranks;
};

namespace st {

// Posts the plan of st_halo_plan for `nfields` fields as one NCCL group on
// comm->comm_stream (which first waits for all prior work on `main`), then
// records comm->ev_done. If `join` is true, `main` waits for ev_done.
st_status halo_exchange_async(st_comm* comm, double* const* fields, int32_t nfields,
                              int64_t n_slow_local, int64_t slab_pitch, int32_t width,
                              cudaStream_t main, bool join);

// Fused halo swap (LOCAL transport, NEXT #3): the boundary-row kernels of a
// pass store their rows into the neighbours' ghost rows themselves.
//   begin: main stream publishes "my ghost rows of `dst` are free" and waits
//          until both neighbours published the same; returns the second
//          destinations of the low/high boundary sweeps (base == nullptr if
//          there is no neighbour on that side).
//   signal: after the boundary sweeps, tell the neighbours their ghosts landed.
//   join:  before the next pass, wait until the neighbours' rows landed here.
// `n` = owned slabs; deltas are in slabs (rows for 2-D, planes for 3-D).
bool fused_halo_available(const st_comm* comm);
st_status fused_halo_begin(st_comm* comm, double* dst, int64_t n, cudaStream_t main, void* rem_lo, void* rem_hi);
st_status fused_halo_signal(st_comm* comm, cudaStream_t main);
st_status fused_halo_join(st_comm* comm, cudaStream_t main);

// Pencil halo swap (LOCAL/IPC), ghost depth h (block of (nzl+2h) planes x (nyl+2h)
// rows): h boundary rows of every plane with the y neighbours, then h whole planes
// with the z neighbours (corner ghosts included).
st_status pencil_exchange_async(st_comm* comm, double* const* fields, int32_t nfields, int64_t nx, int64_t nyl,
                                int64_t nzl, int64_t ldx, int32_t h, cudaStream_t main, bool join);

// Phase profiler: prof_mark records a timing event on `s` (nullptr when profiling is
// off); prof_add files the interval [a, b] under `phase`.
cudaEvent_t prof_mark(st_comm* comm, cudaStream_t s);
void prof_add(st_comm* comm, int phase, cudaEvent_t a, cudaEvent_t b);

st_status halo_plan(int32_t rank, int32_t nranks, int64_t n_slow_local, int64_t slab_pitch,
                    int32_t width, st_xfer sends[2], int32_t* nsend, st_xfer recvs[2],
                    int32_t* nrecv);

}  // namespace st

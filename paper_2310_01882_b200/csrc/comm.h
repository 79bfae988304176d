// comm.h — st_comm: an NCCL communicator plus the streams/events that let the
// halo swap of one sweep run concurrently with the interior rows of that sweep.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include "libstencil.h"

struct st_comm {
  ncclComm_t nccl = nullptr;
  int32_t rank = 0;
  int32_t nranks = 1;
  int32_t device = 0;
  cudaStream_t comm_stream = nullptr;  // NCCL work runs here
  cudaEvent_t ev_ready = nullptr;      // main -> comm: boundary rows are written
  cudaEvent_t ev_done = nullptr;       // comm -> main: ghost rows have arrived
  bool broken = false;                 // set after an NCCL error
};

namespace st {

// Posts the plan of st_halo_plan for `nfields` fields as one NCCL group on
// comm->comm_stream (which first waits for all prior work on `main`), then
// records comm->ev_done. If `join` is true, `main` waits for ev_done.
st_status halo_exchange_async(st_comm* comm, double* const* fields, int32_t nfields,
                              int64_t n_slow_local, int64_t slab_pitch, int32_t width,
                              cudaStream_t main, bool join);

st_status halo_plan(int32_t rank, int32_t nranks, int64_t n_slow_local, int64_t slab_pitch,
                    int32_t width, st_xfer sends[2], int32_t* nsend, st_xfer recvs[2],
                    int32_t* nrecv);

}  // namespace st

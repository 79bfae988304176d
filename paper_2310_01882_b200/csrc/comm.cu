// comm.cu — st_comm (NCCL point-to-point over NVLink/NVSwitch) and the
// slowest-axis halo swap of a slab decomposition.
//
// The paper swaps halos between iterations through xDSL's DMP -> MPI lowering
// on a 2-D process grid. Here one
// process drives one B200; the slabs are contiguous along the slowest axis so
// every message is one contiguous run of doubles (no pack kernels), sent with
// ncclSend/ncclRecv inside one group on a dedicated comm stream so the swap of
// sweep t overlaps the interior rows of sweep t.
#include <cstring>

#include "comm.h"
#include "common.cuh"
#include "internal.h"

#define ST_CHECK_NCCL(comm, expr)                                                  \
  do {                                                                             \
    ncclResult_t r_ = (expr);                                                      \
    if (r_ != ncclSuccess) {                                                       \
      if (comm) (comm)->broken = true;                                             \
      ::st::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,                \
                      ncclGetErrorString(r_));                                     \
      return ST_ENCCL;                                                             \
    }                                                                              \
  } while (0)

namespace st {

st_status halo_plan(int32_t rank, int32_t nranks, int64_t n_slow_local, int64_t slab_pitch,
                    int32_t width, st_xfer sends[2], int32_t* nsend, st_xfer recvs[2],
                    int32_t* nrecv) {
  ST_RETURN_IF(nranks < 1 || rank < 0 || rank >= nranks, ST_EINVAL, "halo_plan: rank %d of %d",
               rank, nranks);
  ST_RETURN_IF(width < 1 || slab_pitch < 1 || n_slow_local < width, ST_EINVAL,
               "halo_plan: need n_slow_local (%lld) >= width (%d) >= 1, slab_pitch >= 1",
               (long long)n_slow_local, width, (long long)slab_pitch);
  ST_RETURN_IF(!sends || !recvs || !nsend || !nrecv, ST_EINVAL, "halo_plan: null output");
  const int64_t cnt = (int64_t)width * slab_pitch;
  int ns = 0, nr = 0;
  if (rank > 0) {  // low neighbour first (by dimension, then direction)
    sends[ns++] = {rank - 1, (int64_t)width * slab_pitch, cnt};  // first owned slabs
    recvs[nr++] = {rank - 1, 0, cnt};                           // low ghost slabs
  }
  if (rank < nranks - 1) {
    sends[ns++] = {rank + 1, n_slow_local * slab_pitch, cnt};                  // last owned
    recvs[nr++] = {rank + 1, (int64_t)(width + n_slow_local) * slab_pitch, cnt};  // high ghosts
  }
  *nsend = ns;
  *nrecv = nr;
  return ST_OK;
}

st_status halo_exchange_async(st_comm* comm, double* const* fields, int32_t nfields,
                              int64_t n_slow_local, int64_t slab_pitch, int32_t width,
                              cudaStream_t main, bool join) {
  st_xfer sends[2], recvs[2];
  int32_t ns = 0, nr = 0;
  ST_TRY(halo_plan(comm->rank, comm->nranks, n_slow_local, slab_pitch, width, sends, &ns, recvs, &nr));
  if (comm->nranks == 1) return ST_OK;
  ST_RETURN_IF(comm->broken, ST_ENCCL, "st_comm is unusable after an earlier NCCL error");
  ST_CHECK_CUDA(cudaEventRecord(comm->ev_ready, main));
  ST_CHECK_CUDA(cudaStreamWaitEvent(comm->comm_stream, comm->ev_ready, 0));
  ST_CHECK_NCCL(comm, ncclGroupStart());
  for (int f = 0; f < nfields; ++f) {
    for (int i = 0; i < ns; ++i)
      ST_CHECK_NCCL(comm, ncclSend(fields[f] + sends[i].offset, (size_t)sends[i].count, ncclFloat64,
                                   sends[i].peer, comm->nccl, comm->comm_stream));
    for (int i = 0; i < nr; ++i)
      ST_CHECK_NCCL(comm, ncclRecv(fields[f] + recvs[i].offset, (size_t)recvs[i].count, ncclFloat64,
                                   recvs[i].peer, comm->nccl, comm->comm_stream));
  }
  ST_CHECK_NCCL(comm, ncclGroupEnd());
  ST_CHECK_CUDA(cudaEventRecord(comm->ev_done, comm->comm_stream));
  if (join) ST_CHECK_CUDA(cudaStreamWaitEvent(main, comm->ev_done, 0));
  return ST_OK;
}

}  // namespace st

using namespace st;

extern "C" {

st_status st_comm_unique_id(uint8_t id[ST_UNIQUE_ID_BYTES]) {
  clear_error();
  static_assert(sizeof(ncclUniqueId) == ST_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ST_RETURN_IF(!id, ST_EINVAL, "st_comm_unique_id: null id");
  ncclUniqueId uid;
  ST_CHECK_NCCL((st_comm*)nullptr, ncclGetUniqueId(&uid));
  std::memcpy(id, &uid, sizeof(uid));
  return ST_OK;
}

st_status st_comm_init(st_comm** out, int32_t nranks, int32_t rank,
                       const uint8_t id[ST_UNIQUE_ID_BYTES], int32_t cuda_device) {
  clear_error();
  ST_RETURN_IF(!out || !id, ST_EINVAL, "st_comm_init: null argument");
  ST_RETURN_IF(nranks < 1 || rank < 0 || rank >= nranks, ST_EINVAL, "st_comm_init: rank %d of %d",
               rank, nranks);
  ST_CHECK_CUDA(cudaSetDevice(cuda_device));
  st_comm* c = new st_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = cuda_device;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank -> %s", ncclGetErrorString(r));
    delete c;
    return ST_ENCCL;
  }
  if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess) {
    set_error("st_comm_init: stream/event creation failed");
    ncclCommDestroy(c->nccl);
    delete c;
    return ST_ECUDA;
  }
  *out = c;
  return ST_OK;
}

st_status st_comm_destroy(st_comm* c) {
  clear_error();
  if (!c) return ST_OK;
  cudaSetDevice(c->device);
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  st_status s = ST_OK;
  if (c->nccl && ncclCommDestroy(c->nccl) != ncclSuccess) s = ST_ENCCL;
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  delete c;
  return s;
}

st_status st_comm_query(const st_comm* c, int32_t* rank, int32_t* nranks, int32_t* dev) {
  clear_error();
  ST_RETURN_IF(!c, ST_EINVAL, "st_comm_query: null comm");
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  if (dev) *dev = c->device;
  return ST_OK;
}

st_status st_block_split(int64_t n, int32_t nranks, int32_t rank, int64_t* start, int64_t* count) {
  clear_error();
  ST_RETURN_IF(n < 0 || nranks < 1 || rank < 0 || rank >= nranks || !start || !count, ST_EINVAL,
               "st_block_split: bad arguments");
  const int64_t base = n / nranks, rem = n % nranks, lo = nranks - rem;
  if (rank < lo) {
    *count = base;
    *start = (int64_t)rank * base;
  } else {
    *count = base + 1;
    *start = lo * base + (int64_t)(rank - lo) * (base + 1);
  }
  return ST_OK;
}

st_status st_halo_plan(int32_t rank, int32_t nranks, int64_t n_slow_local, int64_t slab_pitch,
                       int32_t width, st_xfer sends[2], int32_t* nsend, st_xfer recvs[2],
                       int32_t* nrecv) {
  clear_error();
  return halo_plan(rank, nranks, n_slow_local, slab_pitch, width, sends, nsend, recvs, nrecv);
}

st_status st_halo_exchange(st_comm* comm, double* const* fields, int32_t nfields, int64_t n_slow_local,
                           int64_t slab_pitch, int32_t width, void* cuda_stream) {
  clear_error();
  ST_RETURN_IF(!comm || (!fields && nfields > 0) || nfields < 0, ST_EINVAL,
               "st_halo_exchange: bad arguments");
  for (int f = 0; f < nfields; ++f) ST_RETURN_IF(!fields[f], ST_EINVAL, "st_halo_exchange: null field %d", f);
  return halo_exchange_async(comm, fields, nfields, n_slow_local, slab_pitch, width,
                             static_cast<cudaStream_t>(cuda_stream), true);
}

}  // extern "C"

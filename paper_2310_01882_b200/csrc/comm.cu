// comm.cu — st_comm (NCCL point-to-point over NVLink/NVSwitch) and the
// slowest-axis halo swap of a slab decomposition.
//
// The paper swaps halos between iterations through xDSL's DMP -> MPI lowering
// on a 2-D process grid. Here one
// process drives one B200; the slabs are contiguous along the slowest axis so
// every message is one contiguous run of doubles (no pack kernels), sent with
// ncclSend/ncclRecv inside one group on a dedicated comm stream so the swap of
// sweep t overlaps the interior rows of sweep t.
#include <cuda.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <thread>

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

// ------------------------------------------------------------ profiler ---
cudaEvent_t prof_mark(st_comm* c, cudaStream_t s) {
  if (!c || !c->prof) return nullptr;
  cudaEvent_t e = nullptr;
  if (!c->prof_pool.empty()) {
    e = c->prof_pool.back();
    c->prof_pool.pop_back();
  } else if (cudaEventCreate(&e) != cudaSuccess) {
    return nullptr;
  }
  if (cudaEventRecord(e, s) != cudaSuccess) {
    c->prof_pool.push_back(e);
    return nullptr;
  }
  return e;
}

void prof_add(st_comm* c, int phase, cudaEvent_t a, cudaEvent_t b) {
  if (!c || !a || !b || phase < 0 || phase >= ST_PHASES) return;
  c->prof_ev[phase].emplace_back(a, b);
}

// ------------------------------------------------ stream memory operations ---
namespace {
using PFN_waitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_writeValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitValue32 g_wait32 = nullptr;
PFN_writeValue32 g_write32 = nullptr;
// CU_STREAM_WAIT_VALUE_FLUSH where the device supports it: the flag a wait sees
// was written by a peer after its data stores (the default write carries a
// system-scope fence); the flush makes those remote data writes visible to the
// work queued behind the wait on platforms that could otherwise hold them back.
// (The B200s of this pool report no support: there the writer's fence, and NVLink
// peer stores landing in the owner's L2 in order, are what order data and flag.)
unsigned g_wait_flush = 0;

st_status load_stream_memops() {
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    void* pw = nullptr;
    void* pr = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &pw, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &pr, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && pw && pr) {
      g_wait32 = reinterpret_cast<PFN_waitValue32>(pw);
      g_write32 = reinterpret_cast<PFN_writeValue32>(pr);
      ok = true;
      using PFN_attr = CUresult (*)(int*, CUdevice_attribute, CUdevice);
      void* pa = nullptr;
      cudaDriverEntryPointQueryResult q3;
      int dev = 0, can = 0;
      if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &pa, cudaEnableDefault, &q3) == cudaSuccess &&
          q3 == cudaDriverEntryPointSuccess && pa && cudaGetDevice(&dev) == cudaSuccess &&
          reinterpret_cast<PFN_attr>(pa)(&can, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, (CUdevice)dev) ==
              CUDA_SUCCESS &&
          can)
        g_wait_flush = CU_STREAM_WAIT_VALUE_FLUSH;
    }
  });
  ST_RETURN_IF(!ok, ST_ECUDA, "stream memory operations (cuStreamWaitValue32) unavailable");
  return ST_OK;
}

st_status stream_write(cudaStream_t s, uint32_t* addr, uint32_t v) {
  CUresult r = g_write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v, 0);
  ST_RETURN_IF(r != CUDA_SUCCESS, ST_ECUDA, "cuStreamWriteValue32 failed: %d", (int)r);
  return ST_OK;
}

st_status stream_wait_geq(cudaStream_t s, uint32_t* addr, uint32_t v) {
  CUresult r = g_wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                        CU_STREAM_WAIT_VALUE_GEQ | g_wait_flush);
  ST_RETURN_IF(r != CUDA_SUCCESS, ST_ECUDA, "cuStreamWaitValue32 failed: %d", (int)r);
  return ST_OK;
}

// Flag words of a rank, all WRITTEN BY ITS NEIGHBOURS (remote stream writes) and
// awaited only by the rank itself (local stream waits — no polling of peer
// memory across NVLink): DoneFromX = the X neighbour has delivered my ghosts,
// ReadyFromX = the X neighbour's ghosts facing me are free, so I may send.
constexpr int kFlagDoneFromLo = 1, kFlagDoneFromHi = 2, kFlagDoneFromYLo = 3, kFlagDoneFromYHi = 4;
constexpr int kFlagReadyFromLo = 5, kFlagReadyFromHi = 6, kFlagReadyFromYLo = 7, kFlagReadyFromYHi = 8;
constexpr int kFlagWords = 16;

// View of rank `peer` of a LOCAL/IPC comm (direct for LOCAL, IPC-mapped for IPC).
st_status peer_of(st_comm* c, int32_t peer, st_peer* out) {
  out->valid = false;
  if (peer < 0 || peer >= c->nranks) return ST_OK;
  if (c->kind == st_comm::LOCAL) {
    st_comm* pc = c->group->ranks[(size_t)peer];
    ST_RETURN_IF(!pc, ST_EINVAL, "LOCAL comm: rank %d was destroyed", peer);
    out->valid = true;
    out->flags = pc->flags;
    out->bound = pc->bound;
    out->n_slow = pc->bound_n_slow;
    out->n_mid = pc->n_mid;
    out->device = pc->device;
  } else {
    const st_peer* p = nullptr;
    for (const auto& kv : c->ipc_peers)
      if (kv.first == peer) p = &kv.second;
    ST_RETURN_IF(!p || !p->valid, ST_EINVAL, "IPC comm: rank %d's blob was not imported", peer);
    *out = *p;
    out->opened.clear();
  }
  ST_RETURN_IF(out->bound.size() != c->bound.size(), ST_EINVAL, "rank %d has not bound the same buffers", peer);
  return ST_OK;
}

// Slab neighbour on `side` (0 = rank-1, 1 = rank+1); valid=false if none.
st_status peer_view(st_comm* c, int side, st_peer* out) {
  return peer_of(c, side == 0 ? c->rank - 1 : c->rank + 1, out);
}

// LOCAL transport: push my boundary slabs into the neighbours' ghost slabs.
st_status local_exchange(st_comm* c, double* const* fields, int32_t nfields, int64_t n, int64_t pitch,
                         int32_t width, cudaStream_t main, bool join) {
  ST_RETURN_IF(c->bound.empty(), ST_EINVAL, "LOCAL comm: st_comm_bind the swapped buffers first");
  ST_RETURN_IF(n != c->bound_n_slow, ST_EINVAL, "LOCAL comm: %lld owned slabs, bound with %lld",
               (long long)n, (long long)c->bound_n_slow);
  int idx[8];
  ST_RETURN_IF(nfields > 8, ST_EINVAL, "LOCAL comm: at most 8 fields per swap");
  for (int f = 0; f < nfields; ++f) {
    idx[f] = -1;
    for (size_t i = 0; i < c->bound.size(); ++i)
      if (c->bound[i] == fields[f]) idx[f] = (int)i;
    ST_RETURN_IF(idx[f] < 0, ST_EINVAL, "LOCAL comm: field %d was not bound", f);
  }
  const uint32_t k = ++c->seq;
  cudaStream_t cs = c->comm_stream;
  ST_CHECK_CUDA(cudaEventRecord(c->ev_ready, main));
  ST_CHECK_CUDA(cudaStreamWaitEvent(cs, c->ev_ready, 0));
  cudaEvent_t p0 = prof_mark(c, cs);
  // my ghost slabs may now be overwritten: tell both neighbours (I am rank-1's high, rank+1's low neighbour)
  for (int side = 0; side < 2; ++side) {
    st_peer pc;
    ST_TRY(peer_view(c, side, &pc));
    if (pc.valid) ST_TRY(stream_write(cs, pc.flags + (side == 0 ? kFlagReadyFromHi : kFlagReadyFromLo), k));
  }
  const size_t bytes = (size_t)width * (size_t)pitch * sizeof(double);
  for (int side = 0; side < 2; ++side) {
    st_peer pc;
    ST_TRY(peer_view(c, side, &pc));
    if (!pc.valid) continue;
    ST_TRY(stream_wait_geq(cs, c->flags + (side == 0 ? kFlagReadyFromLo : kFlagReadyFromHi), k));
    for (int f = 0; f < nfields; ++f) {
      double* src = fields[f];
      double* dst = pc.bound[(size_t)idx[f]];
      // to rank-1: my first owned slabs -> its high ghosts; to rank+1: my last owned -> its low ghosts
      const int64_t soff = side == 0 ? (int64_t)width * pitch : n * pitch;
      const int64_t doff = side == 0 ? ((int64_t)width + pc.n_slow) * pitch : 0;
      // unified addressing: same-device, peer (NVLink) and IPC-mapped destinations alike
      ST_CHECK_CUDA(cudaMemcpyAsync(dst + doff, src + soff, bytes, cudaMemcpyDefault, cs));
    }
    ST_TRY(stream_write(cs, pc.flags + (side == 0 ? kFlagDoneFromHi : kFlagDoneFromLo), k));
  }
  if (c->rank > 0) ST_TRY(stream_wait_geq(cs, c->flags + kFlagDoneFromLo, k));
  if (c->rank < c->nranks - 1) ST_TRY(stream_wait_geq(cs, c->flags + kFlagDoneFromHi, k));
  prof_add(c, ST_PHASE_SWAP, p0, prof_mark(c, cs));
  ST_CHECK_CUDA(cudaEventRecord(c->ev_done, cs));
  if (join) ST_CHECK_CUDA(cudaStreamWaitEvent(main, c->ev_done, 0));
  return ST_OK;
}
}  // namespace

st_status pencil_exchange_async(st_comm* c, double* const* fields, int32_t nfields, int64_t nx, int64_t nyl,
                                int64_t nzl, int64_t ldx, int32_t h, cudaStream_t main, bool join) {
  ST_RETURN_IF(c->kind == st_comm::NCCL, ST_ENOTSUP, "pencil decomposition needs the IPC or LOCAL transport");
  ST_RETURN_IF(c->broken, ST_ENCCL, "st_comm is unusable after an earlier error or timeout");
  ST_RETURN_IF(c->grid_py < 1 || c->nranks % c->grid_py != 0, ST_EINVAL, "pencils: st_comm_set_grid first");
  ST_RETURN_IF(c->bound.empty(), ST_EINVAL, "pencils: st_comm_bind/st_comm_export the swapped buffers first");
  ST_RETURN_IF(nyl != c->n_mid || nzl != c->bound_n_slow, ST_EINVAL, "pencils: block %lldx%lld, bound %lldx%lld",
               (long long)nyl, (long long)nzl, (long long)c->n_mid, (long long)c->bound_n_slow);
  ST_RETURN_IF(nfields > 8, ST_EINVAL, "pencils: at most 8 fields per swap");
  ST_RETURN_IF(h < 1 || h > nyl || h > nzl, ST_EINVAL, "pencils: ghost depth %d vs a %lldx%lld block", h,
               (long long)nyl, (long long)nzl);
  int idx[8];
  for (int f = 0; f < nfields; ++f) {
    idx[f] = -1;
    for (size_t i = 0; i < c->bound.size(); ++i)
      if (c->bound[i] == fields[f]) idx[f] = (int)i;
    ST_RETURN_IF(idx[f] < 0, ST_EINVAL, "pencils: field %d was not bound", f);
  }
  const int32_t py = c->grid_py, iy = c->rank % py, iz = c->rank / py, pz = c->nranks / py;
  const uint32_t k = ++c->seq;
  cudaStream_t cs = c->comm_stream;
  // h rows of a plane: one span from the first row's column 0 to the last row's column nx+1
  const size_t rows_bytes = (size_t)((h - 1) * ldx + nx + 2) * sizeof(double);
  const int64_t my_plane = (nyl + 2 * (int64_t)h) * ldx;
  ST_CHECK_CUDA(cudaEventRecord(c->ev_ready, main));
  ST_CHECK_CUDA(cudaStreamWaitEvent(cs, c->ev_ready, 0));
  cudaEvent_t p0 = prof_mark(c, cs);
  // my ghosts may now be overwritten: tell the y and z neighbours
  for (int side = 0; side < 2; ++side) {
    if (!((side == 0 && iy == 0) || (side == 1 && iy == py - 1))) {
      st_peer pc;
      ST_TRY(peer_of(c, side == 0 ? c->rank - 1 : c->rank + 1, &pc));
      ST_TRY(stream_write(cs, pc.flags + (side == 0 ? kFlagReadyFromYHi : kFlagReadyFromYLo), k));
    }
    if (!((side == 0 && iz == 0) || (side == 1 && iz == pz - 1))) {
      st_peer pc;
      ST_TRY(peer_of(c, side == 0 ? c->rank - py : c->rank + py, &pc));
      ST_TRY(stream_write(cs, pc.flags + (side == 0 ? kFlagReadyFromHi : kFlagReadyFromLo), k));
    }
  }
  // phase y: h boundary rows per plane into the y neighbours' ghost rows. The
  // planes that are z ghosts (filled whole by phase z, possibly concurrently)
  // are skipped; the z-halo planes of the grid's z edges are global boundary
  // planes and are included (the diagonal PW offsets read their corners).
  // y neighbours share this rank's z range, so they skip the same planes.
  const int64_t zlo = iz > 0 ? h : 0, zhi = iz < pz - 1 ? h + nzl - 1 : nzl + 2 * (int64_t)h - 1;
  for (int side = 0; side < 2; ++side) {
    if ((side == 0 && iy == 0) || (side == 1 && iy == py - 1)) continue;
    st_peer pc;
    ST_TRY(peer_of(c, side == 0 ? c->rank - 1 : c->rank + 1, &pc));
    ST_TRY(stream_wait_geq(cs, c->flags + (side == 0 ? kFlagReadyFromYLo : kFlagReadyFromYHi), k));
    const int64_t peer_plane = (pc.n_mid + 2 * (int64_t)h) * ldx;
    const int64_t src_row = side == 0 ? h : nyl, dst_row = side == 0 ? pc.n_mid + h : 0;
    for (int f = 0; f < nfields; ++f)
      ST_CHECK_CUDA(cudaMemcpy2DAsync(pc.bound[(size_t)idx[f]] + zlo * peer_plane + dst_row * ldx,
                                      (size_t)peer_plane * sizeof(double), fields[f] + zlo * my_plane + src_row * ldx,
                                      (size_t)my_plane * sizeof(double), rows_bytes, (size_t)(zhi - zlo + 1),
                                      cudaMemcpyDefault, cs));
    ST_TRY(stream_write(cs, pc.flags + (side == 0 ? kFlagDoneFromYHi : kFlagDoneFromYLo), k));
  }
  if (iy > 0) ST_TRY(stream_wait_geq(cs, c->flags + kFlagDoneFromYLo, k));
  if (iy < py - 1) ST_TRY(stream_wait_geq(cs, c->flags + kFlagDoneFromYHi, k));
  // phase z: h whole boundary planes (all rows, i.e. with the fresh y ghosts)
  for (int side = 0; side < 2; ++side) {
    if ((side == 0 && iz == 0) || (side == 1 && iz == pz - 1)) continue;
    st_peer pc;
    ST_TRY(peer_of(c, side == 0 ? c->rank - py : c->rank + py, &pc));
    ST_TRY(stream_wait_geq(cs, c->flags + (side == 0 ? kFlagReadyFromLo : kFlagReadyFromHi), k));
    const int64_t src_plane = side == 0 ? h : nzl, dst_plane = side == 0 ? pc.n_slow + h : 0;
    for (int f = 0; f < nfields; ++f)
      ST_CHECK_CUDA(cudaMemcpyAsync(pc.bound[(size_t)idx[f]] + dst_plane * my_plane, fields[f] + src_plane * my_plane,
                                    (size_t)h * (size_t)my_plane * sizeof(double), cudaMemcpyDefault, cs));
    ST_TRY(stream_write(cs, pc.flags + (side == 0 ? kFlagDoneFromHi : kFlagDoneFromLo), k));
  }
  if (iz > 0) ST_TRY(stream_wait_geq(cs, c->flags + kFlagDoneFromLo, k));
  if (iz < pz - 1) ST_TRY(stream_wait_geq(cs, c->flags + kFlagDoneFromHi, k));
  prof_add(c, ST_PHASE_SWAP, p0, prof_mark(c, cs));
  ST_CHECK_CUDA(cudaEventRecord(c->ev_done, cs));
  if (join) ST_CHECK_CUDA(cudaStreamWaitEvent(main, c->ev_done, 0));
  return ST_OK;
}

bool fused_halo_available(const st_comm* comm) {
  static const int kFused = env_int("ST_FUSED_HALO", 1);
  return comm && comm->kind != st_comm::NCCL && comm->nranks > 1 && kFused != 0;
}

st_status fused_halo_begin(st_comm* c, double* dst, int64_t n, cudaStream_t main, void* rem_lo_v, void* rem_hi_v) {
  Remote* rem_lo = static_cast<Remote*>(rem_lo_v);
  Remote* rem_hi = static_cast<Remote*>(rem_hi_v);
  *rem_lo = Remote();
  *rem_hi = Remote();
  ST_RETURN_IF(c->bound.empty(), ST_EINVAL, "LOCAL comm: st_comm_bind the swapped buffers first");
  ST_RETURN_IF(n != c->bound_n_slow, ST_EINVAL, "LOCAL comm: %lld owned slabs, bound with %lld", (long long)n,
               (long long)c->bound_n_slow);
  int idx = -1;
  for (size_t i = 0; i < c->bound.size(); ++i)
    if (c->bound[i] == dst) idx = (int)i;
  ST_RETURN_IF(idx < 0, ST_EINVAL, "LOCAL comm: destination buffer was not bound");
  const uint32_t k = ++c->seq;
  for (int side = 0; side < 2; ++side) {  // my ghost slabs of dst are free: tell the neighbours
    st_peer pc;
    ST_TRY(peer_view(c, side, &pc));
    if (pc.valid) ST_TRY(stream_write(main, pc.flags + (side == 0 ? kFlagReadyFromHi : kFlagReadyFromLo), k));
  }
  for (int side = 0; side < 2; ++side) {
    st_peer pc;
    ST_TRY(peer_view(c, side, &pc));
    if (!pc.valid) continue;
    ST_TRY(stream_wait_geq(main, c->flags + (side == 0 ? kFlagReadyFromLo : kFlagReadyFromHi), k));
    Remote& r = side == 0 ? *rem_lo : *rem_hi;
    r.base = pc.bound[(size_t)idx];
    // my first owned slabs -> rank-1's high ghosts (+n_{r-1}); my last owned -> rank+1's low ghosts (-n)
    r.delta = side == 0 ? pc.n_slow : -n;
  }
  return ST_OK;
}

st_status fused_halo_signal(st_comm* c, cudaStream_t main) {
  const uint32_t k = c->seq;
  for (int side = 0; side < 2; ++side) {
    st_peer pc;
    ST_TRY(peer_view(c, side, &pc));
    if (pc.valid) ST_TRY(stream_write(main, pc.flags + (side == 0 ? kFlagDoneFromHi : kFlagDoneFromLo), k));
  }
  return ST_OK;
}

st_status fused_halo_join(st_comm* c, cudaStream_t main) {
  const uint32_t k = c->seq;
  if (c->rank > 0) ST_TRY(stream_wait_geq(main, c->flags + kFlagDoneFromLo, k));
  if (c->rank < c->nranks - 1) ST_TRY(stream_wait_geq(main, c->flags + kFlagDoneFromHi, k));
  return ST_OK;
}

st_status halo_exchange_async(st_comm* comm, double* const* fields, int32_t nfields,
                              int64_t n_slow_local, int64_t slab_pitch, int32_t width,
                              cudaStream_t main, bool join) {
  st_xfer sends[2], recvs[2];
  int32_t ns = 0, nr = 0;
  ST_TRY(halo_plan(comm->rank, comm->nranks, n_slow_local, slab_pitch, width, sends, &ns, recvs, &nr));
  if (comm->nranks == 1) return ST_OK;
  ST_RETURN_IF(comm->broken, ST_ENCCL, "st_comm is unusable after an earlier error or timeout");
  if (comm->kind != st_comm::NCCL)
    return local_exchange(comm, fields, nfields, n_slow_local, slab_pitch, width, main, join);
  ST_CHECK_CUDA(cudaEventRecord(comm->ev_ready, main));
  ST_CHECK_CUDA(cudaStreamWaitEvent(comm->comm_stream, comm->ev_ready, 0));
  cudaEvent_t p0 = prof_mark(comm, comm->comm_stream);
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
  prof_add(comm, ST_PHASE_SWAP, p0, prof_mark(comm, comm->comm_stream));
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
  ST_TRY(preload_kernels());
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

st_status st_comm_from_nccl(st_comm** out, void* nccl_comm, int32_t cuda_device) {
  clear_error();
  ST_RETURN_IF(!out || !nccl_comm, ST_EINVAL, "st_comm_from_nccl: null argument");
  ST_CHECK_CUDA(cudaSetDevice(cuda_device));
  ncclComm_t nc = static_cast<ncclComm_t>(nccl_comm);
  int nranks = 0, rank = 0, dev = -1;
  ST_RETURN_IF(ncclCommCount(nc, &nranks) != ncclSuccess || ncclCommUserRank(nc, &rank) != ncclSuccess ||
                   ncclCommCuDevice(nc, &dev) != ncclSuccess,
               ST_ENCCL, "st_comm_from_nccl: not a valid NCCL communicator");
  ST_RETURN_IF(dev != cuda_device, ST_EINVAL, "st_comm_from_nccl: communicator is on device %d, not %d", dev,
               cuda_device);
  ST_TRY(preload_kernels());
  st_comm* c = new st_comm();
  c->nccl = nc;
  c->borrowed = true;
  c->rank = rank;
  c->nranks = nranks;
  c->device = cuda_device;
  if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess) {
    set_error("st_comm_from_nccl: stream/event creation failed");
    delete c;
    return ST_ECUDA;
  }
  *out = c;
  return ST_OK;
}

st_status st_comm_wait(st_comm* c, void* cuda_stream, int32_t timeout_ms) {
  clear_error();
  ST_RETURN_IF(!c, ST_EINVAL, "st_comm_wait: null comm");
  ST_CHECK_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    bool pending = false;
    for (cudaStream_t q : {s, c->comm_stream}) {
      if (!q && q != s) continue;
      const cudaError_t e = cudaStreamQuery(q);
      if (e == cudaErrorNotReady) pending = true;
      else ST_CHECK_CUDA(e);
    }
    if (c->nccl && !c->broken) {
      ncclResult_t ar = ncclSuccess;
      if (ncclCommGetAsyncError(c->nccl, &ar) != ncclSuccess || ar != ncclSuccess) {
        c->broken = true;
        if (!c->borrowed) ncclCommAbort(c->nccl), c->nccl = nullptr;
        set_error("st_comm_wait: asynchronous NCCL error: %s", ncclGetErrorString(ar));
        return ST_ENCCL;
      }
    }
    if (!pending) return ST_OK;
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
    if (timeout_ms > 0 && ms.count() >= timeout_ms) {
      if (c->nccl && !c->borrowed) {
        ncclCommAbort(c->nccl);
        c->nccl = nullptr;
      }
      c->broken = true;  // later calls fail fast instead of queueing behind a wait that may never end
      set_error("st_comm_wait: rank %d: work still pending after %d ms (a neighbour did not join the swap?)",
                c->rank, timeout_ms);
      return ST_ETIMEDOUT;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
}

st_status st_comm_init_local(st_comm** comms, int32_t nranks, const int32_t* devices) {
  clear_error();
  ST_RETURN_IF(!comms || !devices || nranks < 1, ST_EINVAL, "st_comm_init_local: bad arguments");
  ST_TRY(load_stream_memops());
  int ndev = 0;
  ST_CHECK_CUDA(cudaGetDeviceCount(&ndev));
  for (int r = 0; r < nranks; ++r)
    ST_RETURN_IF(devices[r] < 0 || devices[r] >= ndev, ST_EINVAL, "st_comm_init_local: device %d", devices[r]);
  // Ranks sharing a device order each other with stream waits (cuStreamWaitValue32). If two
  // of their streams share a hardware queue, a waiting stream blocks the one that would
  // release it, so every stream of the group on a device needs its own connection:
  // 2 per rank (main + comm) plus the legacy default stream.
  {
    const char* cv = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    const int conns = (cv && *cv) ? std::atoi(cv) : 8;
    for (int r = 0; r < nranks; ++r) {
      int same = 0;
      for (int q = 0; q < nranks; ++q) same += devices[q] == devices[r];
      ST_RETURN_IF(same > 1 && conns < 2 * same + 1, ST_ENOTSUP,
                   "st_comm_init_local: %d ranks share device %d; set CUDA_DEVICE_MAX_CONNECTIONS >= %d before "
                   "CUDA initialises (now %d)", same, devices[r], 2 * same + 1, conns);
    }
  }
  int prev = 0;
  cudaGetDevice(&prev);
  // peer access between the distinct devices of the group (copies and flag writes go device to device)
  for (int i = 0; i < nranks; ++i)
    for (int j = 0; j < nranks; ++j)
      if (devices[i] != devices[j]) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices[i], devices[j]);
        ST_RETURN_IF(!can, ST_ENOTSUP, "st_comm_init_local: no peer access %d -> %d", devices[i], devices[j]);
        cudaSetDevice(devices[i]);
        cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else ST_CHECK_CUDA(e);
      }
  for (int r = 0; r < nranks; ++r) {
    cudaSetDevice(devices[r]);
    ST_TRY(preload_kernels());
  }
  st_local_group* g = new st_local_group();
  g->nranks = nranks;
  g->ranks.assign((size_t)nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    st_comm* c = new st_comm();
    c->kind = st_comm::LOCAL;
    c->rank = r;
    c->nranks = nranks;
    c->device = devices[r];
    c->group = g;
    cudaSetDevice(c->device);
    if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&c->flags, kFlagWords * sizeof(uint32_t)) != cudaSuccess ||
        cudaMemset(c->flags, 0, kFlagWords * sizeof(uint32_t)) != cudaSuccess) {
      set_error("st_comm_init_local: stream/event/flag allocation failed");
      delete c;
      for (int q = 0; q < r; ++q) st_comm_destroy(comms[q]);
      cudaSetDevice(prev);
      return ST_ECUDA;
    }
    g->ranks[(size_t)r] = c;
    g->alive++;
    comms[r] = c;
  }
  ST_CHECK_CUDA(cudaDeviceSynchronize());  // flags are zero before any stream uses them
  cudaSetDevice(prev);
  return ST_OK;
}

// ------------------------------------------------------------------ IPC ---
namespace {
constexpr uint32_t kBlobMagic = 0x53544950u;  // "STIP"
struct BlobHeader {
  uint32_t magic, version;
  int32_t rank, device, nbuf, pad;
  int64_t n_slow, n_mid;
};
struct BlobEntry {
  cudaIpcMemHandle_t handle;
  int64_t offset;  // pointer - allocation base
};
using PFN_getRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

st_status ipc_entry(const void* ptr, BlobEntry* e) {
  static PFN_getRange get_range = nullptr;
  if (!get_range) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ST_CHECK_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q));
    ST_RETURN_IF(!p || q != cudaDriverEntryPointSuccess, ST_ECUDA, "cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<PFN_getRange>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  ST_RETURN_IF(get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS, ST_EINVAL,
               "IPC export: pointer is not device memory");
  ST_CHECK_CUDA(cudaIpcGetMemHandle(&e->handle, reinterpret_cast<void*>(base)));
  e->offset = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - (uintptr_t)base);
  return ST_OK;
}
}  // namespace

st_status st_comm_init_ipc(st_comm** out, int32_t nranks, int32_t rank, int32_t cuda_device) {
  clear_error();
  ST_RETURN_IF(!out || nranks < 1 || rank < 0 || rank >= nranks, ST_EINVAL, "st_comm_init_ipc: bad arguments");
  ST_TRY(load_stream_memops());
  ST_CHECK_CUDA(cudaSetDevice(cuda_device));
  ST_TRY(preload_kernels());
  st_comm* c = new st_comm();
  c->kind = st_comm::IPC;
  c->rank = rank;
  c->nranks = nranks;
  c->device = cuda_device;
  if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&c->flags, kFlagWords * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(c->flags, 0, kFlagWords * sizeof(uint32_t)) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    set_error("st_comm_init_ipc: stream/event/flag allocation failed");
    st_comm_destroy(c);
    return ST_ECUDA;
  }
  *out = c;
  return ST_OK;
}

st_status st_comm_export(st_comm* c, double* const* buffers, int32_t nbuf, int64_t n_slow, uint8_t* blob, int64_t cap,
                         int64_t* used) {
  clear_error();
  ST_RETURN_IF(!c || c->kind != st_comm::IPC, ST_EINVAL, "st_comm_export: needs an IPC comm");
  ST_RETURN_IF(!used || nbuf < 0 || (nbuf > 0 && !buffers) || n_slow < 1, ST_EINVAL, "st_comm_export: bad arguments");
  const int64_t need = (int64_t)sizeof(BlobHeader) + (int64_t)(nbuf + 1) * (int64_t)sizeof(BlobEntry);
  *used = need;
  if (cap == 0) return ST_OK;
  ST_RETURN_IF(!blob || cap < need, ST_EINVAL, "st_comm_export: blob of %lld bytes < %lld", (long long)cap,
               (long long)need);
  c->bound.assign(buffers, buffers + nbuf);
  c->bound_n_slow = n_slow;
  BlobHeader h{kBlobMagic, 2u, c->rank, c->device, nbuf, 0, n_slow, c->n_mid};
  std::memcpy(blob, &h, sizeof(h));
  BlobEntry* e = reinterpret_cast<BlobEntry*>(blob + sizeof(h));
  ST_TRY(ipc_entry(c->flags, &e[0]));
  for (int i = 0; i < nbuf; ++i) ST_TRY(ipc_entry(buffers[i], &e[i + 1]));
  return ST_OK;
}

st_status st_comm_import(st_comm* c, int32_t peer, const uint8_t* blob, int64_t bytes) {
  clear_error();
  ST_RETURN_IF(!c || c->kind != st_comm::IPC || !blob, ST_EINVAL, "st_comm_import: needs an IPC comm and a blob");
  bool neighbour = peer == c->rank - 1 || peer == c->rank + 1;
  if (c->grid_py > 0) {  // pencils: y neighbours in the same grid row, z neighbours +-py
    const int32_t py = c->grid_py;
    neighbour = (peer / py == c->rank / py && (peer == c->rank - 1 || peer == c->rank + 1)) ||
                peer == c->rank - py || peer == c->rank + py;
  }
  if (!neighbour) return ST_OK;  // only neighbours are mapped
  ST_RETURN_IF(bytes < (int64_t)sizeof(BlobHeader), ST_EINVAL, "st_comm_import: short blob");
  BlobHeader h;
  std::memcpy(&h, blob, sizeof(h));
  ST_RETURN_IF(h.magic != kBlobMagic || h.rank != peer || h.nbuf < 0 ||
                   bytes < (int64_t)sizeof(h) + (int64_t)(h.nbuf + 1) * (int64_t)sizeof(BlobEntry),
               ST_EINVAL, "st_comm_import: malformed blob for rank %d", peer);
  st_peer* pp = nullptr;
  for (auto& kv : c->ipc_peers)
    if (kv.first == peer) pp = &kv.second;
  if (!pp) {
    c->ipc_peers.emplace_back(peer, st_peer());
    pp = &c->ipc_peers.back().second;
  }
  st_peer& p = *pp;
  if (!p.opened.empty()) {
    // kernels (fused stores) or copies queued earlier may still write through the old
    // mappings: drain the device before unmapping them
    ST_CHECK_CUDA(cudaSetDevice(c->device));
    ST_CHECK_CUDA(cudaDeviceSynchronize());
  }
  for (void* q : p.opened) cudaIpcCloseMemHandle(q);
  p = st_peer();
  const BlobEntry* e = reinterpret_cast<const BlobEntry*>(blob + sizeof(h));
  std::vector<cudaIpcMemHandle_t> seen;
  std::vector<char*> bases;
  auto map = [&](const BlobEntry& en, void** outp) -> st_status {
    for (size_t i = 0; i < seen.size(); ++i)  // one mapping per allocation
      if (std::memcmp(&seen[i], &en.handle, sizeof(cudaIpcMemHandle_t)) == 0) {
        *outp = bases[i] + en.offset;
        return ST_OK;
      }
    void* base = nullptr;
    ST_CHECK_CUDA(cudaIpcOpenMemHandle(&base, en.handle, cudaIpcMemLazyEnablePeerAccess));
    seen.push_back(en.handle);
    bases.push_back(static_cast<char*>(base));
    p.opened.push_back(base);
    *outp = static_cast<char*>(base) + en.offset;
    return ST_OK;
  };
  void* fp = nullptr;
  ST_TRY(map(e[0], &fp));
  p.flags = static_cast<uint32_t*>(fp);
  for (int i = 0; i < h.nbuf; ++i) {
    void* bp = nullptr;
    ST_TRY(map(e[i + 1], &bp));
    p.bound.push_back(static_cast<double*>(bp));
  }
  p.n_slow = h.n_slow;
  p.n_mid = h.n_mid;
  p.device = h.device;
  p.valid = true;
  return ST_OK;
}

st_status st_comm_set_grid(st_comm* comm, int32_t py, int64_t ny_local) {
  clear_error();
  ST_RETURN_IF(!comm || py < 1 || comm->nranks % py != 0 || ny_local < 1, ST_EINVAL,
               "st_comm_set_grid: py must divide nranks, ny_local >= 1");
  comm->grid_py = py;
  comm->n_mid = ny_local;
  return ST_OK;
}

st_status st_pencil_split(int64_t ny, int64_t nz, int32_t py, int32_t pz, int32_t rank, int64_t* y0, int64_t* nyl,
                          int64_t* z0, int64_t* nzl) {
  clear_error();
  ST_RETURN_IF(py < 1 || pz < 1 || rank < 0 || rank >= py * pz || !y0 || !nyl || !z0 || !nzl, ST_EINVAL,
               "st_pencil_split: bad arguments");
  ST_TRY(st_block_split(ny, py, rank % py, y0, nyl));
  return st_block_split(nz, pz, rank / py, z0, nzl);
}

st_status st_comm_bind(st_comm* comm, double* const* buffers, int32_t nbuffers, int64_t n_slow_local) {
  clear_error();
  ST_RETURN_IF(!comm || nbuffers < 0 || (nbuffers > 0 && !buffers) || n_slow_local < 1, ST_EINVAL,
               "st_comm_bind: bad arguments");
  if (comm->kind == st_comm::NCCL) return ST_OK;
  comm->bound.assign(buffers, buffers + nbuffers);
  comm->bound_n_slow = n_slow_local;
  return ST_OK;
}

st_status st_comm_destroy(st_comm* c) {
  clear_error();
  if (!c) return ST_OK;
  cudaSetDevice(c->device);
  // the caller's streams may still run fused stores through IPC mappings or copies into peers
  if (!c->ipc_peers.empty()) cudaDeviceSynchronize();
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  st_status s = ST_OK;
  if (c->nccl && !c->borrowed && ncclCommDestroy(c->nccl) != ncclSuccess) s = ST_ENCCL;
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  std::set<cudaEvent_t> evs(c->prof_pool.begin(), c->prof_pool.end());
  for (int p = 0; p < ST_PHASES; ++p)
    for (auto& ab : c->prof_ev[p]) evs.insert(ab.first), evs.insert(ab.second);
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  for (auto& kv : c->ipc_peers)
    for (void* p : kv.second.opened) cudaIpcCloseMemHandle(p);
  if (c->flags) cudaFree(c->flags);
  if (c->group) {
    st_local_group* g = c->group;
    g->ranks[(size_t)c->rank] = nullptr;
    if (--g->alive == 0) delete g;
  }
  delete c;
  return s;
}

st_status st_comm_profile(st_comm* c, int32_t enable) {
  clear_error();
  ST_RETURN_IF(!c, ST_EINVAL, "st_comm_profile: null comm");
  c->prof = enable != 0;
  return ST_OK;
}

st_status st_comm_profile_read(st_comm* c, double ms[ST_PHASES], int64_t counts[ST_PHASES]) {
  clear_error();
  ST_RETURN_IF(!c || !ms || !counts, ST_EINVAL, "st_comm_profile_read: null argument");
  ST_CHECK_CUDA(cudaSetDevice(c->device));
  st_status st = ST_OK;
  std::set<cudaEvent_t> used;  // an event may close one interval and open the next
  for (int p = 0; p < ST_PHASES; ++p) {
    double tot = 0.0;
    for (auto& ab : c->prof_ev[p]) {
      float t = 0.f;
      if (cudaEventSynchronize(ab.second) == cudaSuccess && cudaEventElapsedTime(&t, ab.first, ab.second) == cudaSuccess)
        tot += t;
      else
        st = ST_ECUDA;
      used.insert(ab.first);
      used.insert(ab.second);
    }
    ms[p] = tot;
    counts[p] = (int64_t)c->prof_ev[p].size();
    c->prof_ev[p].clear();
  }
  c->prof_pool.insert(c->prof_pool.end(), used.begin(), used.end());
  if (st != ST_OK) {
    cudaGetLastError();
    set_error("st_comm_profile_read: an event could not be timed");
  }
  return st;
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

"""paper_2310_01882_b200 — B200-native stencil hot path (arXiv 2310.01882).

Thin Python binding over the C ABI of ``libstencil.so`` (include/libstencil.h).
It only marshals arguments: every step of the hot path runs in the library's
sm_100a kernels. PyTorch supplies device memory, streams and process groups.

The binding has no fallback: if ``libstencil.so`` is missing or fails to load,
every entry point raises. It never imports the CPU oracle.

Entry points (same names as the C ABI, tensors instead of raw pointers):
    st_jacobi2d_run(a, b, iters, tblock=0, halo=1, comm=None, nx=None) -> result tensor
    st_jacobi3d_run(a, b, iters, tblock=0, halo=1, comm=None, nx=None) -> result tensor
    st_pw_advect3d(u, v, w, su, sv, sw, tcx, tcy, tzc1, tzc2, tzd1, tzd2, comm=None, nx=None)
    st_halo_exchange(comm, fields, n_slow_local, slab_pitch, width)
    st_halo_plan(rank, nranks, n_slow_local, slab_pitch, width) -> (sends, recvs)   [host only]
    st_jacobi2d_schedule(rank, nranks, nx, ny_local, halo, iters, tblock) -> [ops]   [host only]
    st_jacobi3d_schedule(rank, nranks, nx, nz_local, halo, iters, tblock) -> [ops]   [host only]
    st_block_split(n, nranks, rank) -> (start, count)                                [host only]
    Comm.create(rank, nranks, unique_id, device) / Comm.from_process_group(pg, device)
    Comm.local_group(nranks, devices) -> [Comm]; comm.bind(buffers, n_slow_local)
    Comm.create_ipc(rank, nranks, device); comm.bind_ipc(buffers, n_slow_local)      [multi-process]
"""
from __future__ import annotations

import ctypes
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "libstencil.so"
UNIQUE_ID_BYTES = 128

ST_OK, ST_EINVAL, ST_ECUDA, ST_ENCCL, ST_ENOTSUP, ST_EINTERNAL, ST_ETIMEDOUT = range(7)
_STATUS = {1: "EINVAL", 2: "ECUDA", 3: "ENCCL", 4: "ENOTSUP", 5: "EINTERNAL", 6: "ETIMEDOUT"}

_lib = None


class StencilError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn}: ST_{_STATUS.get(code, code)}: {msg}")
        self.code = code


class Xfer(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("offset", ctypes.c_int64), ("count", ctypes.c_int64)]


class Op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("buf", ctypes.c_int32), ("sweeps", ctypes.c_int32),
                ("flag", ctypes.c_int32), ("y_lo", ctypes.c_int64), ("y_hi", ctypes.c_int64),
                ("ring_lo", ctypes.c_int64), ("ring_hi", ctypes.c_int64)]


OP_SWEEP, OP_EXCHANGE, OP_JOIN, OP_SWAP = 1, 2, 3, 4
PHASES = ("boundary", "interior", "join_wait", "swap", "ready_wait")  # ST_PHASE_* order

_vp, _i64, _i32, _dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double

_SIGS = {
    "st_abi_version": (ctypes.c_int32, []),
    "st_last_error": (ctypes.c_char_p, []),
    "st_launch_count": (ctypes.c_uint64, []),
    "st_comm_unique_id": (ctypes.c_int, [_vp]),
    "st_comm_init": (ctypes.c_int, [ctypes.POINTER(_vp), _i32, _i32, _vp, _i32]),
    "st_comm_destroy": (ctypes.c_int, [_vp]),
    "st_comm_from_nccl": (ctypes.c_int, [ctypes.POINTER(_vp), _vp, _i32]),
    "st_comm_wait": (ctypes.c_int, [_vp, _vp, _i32]),
    "st_comm_profile": (ctypes.c_int, [_vp, _i32]),
    "st_comm_profile_read": (ctypes.c_int, [_vp, ctypes.POINTER(_dbl), ctypes.POINTER(_i64)]),
    "st_stencil2d_run": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _i32, _i64, _vp,
                                        ctypes.POINTER(_i32)]),
    "st_stencil2d_expr_halo": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_i32)]),
    "st_pw_fused_expression": (ctypes.c_int, [_dbl, _dbl, _i32, ctypes.c_char_p, _i64, ctypes.POINTER(_i64)]),
    "st_stencil_expr_info": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "st_stencil3d_fused_run": (ctypes.c_int, [ctypes.POINTER(_vp), _i32, ctypes.POINTER(_vp), _i32,
                                              ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(_vp), _i32, _i64, _i64,
                                              _i64, _i64, _vp]),
    "st_stencil3d_expr_run": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_char_p, _i64, _vp,
                                             ctypes.POINTER(_i32)]),
    "st_stencil2d_expr_run": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, ctypes.c_char_p, _i64, _vp,
                                             ctypes.POINTER(_i32)]),
    "st_comm_init_local": (ctypes.c_int, [ctypes.POINTER(_vp), _i32, ctypes.POINTER(_i32)]),
    "st_comm_bind": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), _i32, _i64]),
    "st_comm_init_ipc": (ctypes.c_int, [ctypes.POINTER(_vp), _i32, _i32, _i32]),
    "st_comm_export": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), _i32, _i64, _vp, _i64, ctypes.POINTER(_i64)]),
    "st_comm_import": (ctypes.c_int, [_vp, _i32, _vp, _i64]),
    "st_comm_query": (ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "st_block_split": (ctypes.c_int, [_i64, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "st_halo_plan": (ctypes.c_int, [_i32, _i32, _i64, _i64, _i32, ctypes.POINTER(Xfer),
                                    ctypes.POINTER(_i32), ctypes.POINTER(Xfer), ctypes.POINTER(_i32)]),
    "st_halo_exchange": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), _i32, _i64, _i64, _i32, _vp]),
    "st_jacobi2d_schedule": (ctypes.c_int, [_i32, _i32, _i64, _i64, _i32, _i64, _i32, ctypes.POINTER(Op), _i64,
                                            ctypes.POINTER(_i64)]),
    "st_jacobi3d_schedule": (ctypes.c_int, [_i32, _i32, _i64, _i64, _i32, _i64, _i32, ctypes.POINTER(Op), _i64,
                                            ctypes.POINTER(_i64)]),
    "st_jacobi2d_run": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _i32, _i64, _i32, _vp, _vp,
                                       ctypes.POINTER(_i32)]),
    "st_jacobi3d_run": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i32, _i64, _i32, _vp, _vp,
                                       ctypes.POINTER(_i32)]),
    "st_selftest_div6": (ctypes.c_int, [_vp, _i64, _vp, _vp]),
    "st_gauss_seidel2d_workspace_bytes": (ctypes.c_int64, [_i64, _i64]),
    "st_gauss_seidel2d_run": (ctypes.c_int, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp]),
    "st_comm_set_grid": (ctypes.c_int, [_vp, _i32, _i64]),
    "st_pencil_split": (ctypes.c_int, [_i64, _i64, _i32, _i32, _i32] + [ctypes.POINTER(_i64)] * 4),
    "st_jacobi3d_run_pencils": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i32, _i64, _i32, _vp, _vp,
                                               ctypes.POINTER(_i32)]),
    "st_pw_advect3d_pencils": (ctypes.c_int, [_vp] * 6 + [_i64] * 4 + [_dbl, _dbl] + [_vp] * 4 + [_vp, _vp]),
    "st_pw_advect3d": (ctypes.c_int, [_vp] * 6 + [_i64] * 4 + [_dbl, _dbl] + [_vp] * 4 + [_vp, _vp]),
}
EXPORTS = tuple(_SIGS)


def lib() -> ctypes.CDLL:
    """Load libstencil.so (raises if it is not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is not built: run `make` (or __graft_entry__.build())")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.st_abi_version() != 1:
            raise RuntimeError("libstencil ABI version mismatch")
        _lib = handle
    return _lib


def _check(code: int, fn: str) -> None:
    if code != ST_OK:
        raise StencilError(code, fn, (lib().st_last_error() or b"").decode())


def last_error() -> str:
    return (lib().st_last_error() or b"").decode()


def launch_count() -> int:
    return int(lib().st_launch_count())


def _stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def _f64_cuda(t, name: str):
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    if t.dtype != torch.float64 or not t.is_cuda:
        raise TypeError(f"{name}: expected a float64 CUDA tensor, got {t.dtype} on {t.device}")


# ----------------------------------------------------------------- comm ---
class Comm:
    """Owns an ``st_comm`` (NCCL communicator + comm stream) for one rank."""

    def __init__(self, handle: int, rank: int, nranks: int, device: int):
        self.handle = ctypes.c_void_p(handle)
        self.rank, self.nranks, self.device = rank, nranks, device

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * UNIQUE_ID_BYTES)()
        _check(lib().st_comm_unique_id(ctypes.cast(buf, _vp)), "st_comm_unique_id")
        return bytes(buf)

    @classmethod
    def create(cls, rank: int, nranks: int, uid: bytes, device: int) -> "Comm":
        assert len(uid) == UNIQUE_ID_BYTES
        h = _vp()
        buf = (ctypes.c_uint8 * UNIQUE_ID_BYTES).from_buffer_copy(uid)
        _check(lib().st_comm_init(ctypes.byref(h), nranks, rank, ctypes.cast(buf, _vp), device), "st_comm_init")
        return cls(h.value, rank, nranks, device)

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "Comm":
        """Collective: rank 0 creates the NCCL id and broadcasts it over torch.distributed."""
        import torch.distributed as dist
        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.create(rank, nranks, obj[0], device)

    @classmethod
    def from_nccl(cls, nccl_comm_ptr: int, device: int) -> "Comm":
        """Borrow an existing ncclComm_t (not destroyed by close(); its owner must outlive this Comm)."""
        h = _vp()
        _check(lib().st_comm_from_nccl(ctypes.byref(h), _vp(nccl_comm_ptr), device), "st_comm_from_nccl")
        r, n, d = _i32(), _i32(), _i32()
        _check(lib().st_comm_query(h, ctypes.byref(r), ctypes.byref(n), ctypes.byref(d)), "st_comm_query")
        return cls(h.value, r.value, n.value, d.value)

    @classmethod
    def from_torch_nccl(cls, device: int, group=None) -> "Comm":
        """Borrow torch's own NCCL communicator of `group` (ProcessGroupNCCL._comm_ptr(); the
        group must have run a collective on `device` so that the communicator exists)."""
        import torch
        import torch.distributed as dist
        pg = group if group is not None else dist.group.WORLD
        backend = pg._get_backend(torch.device("cuda", device))
        return cls.from_nccl(int(backend._comm_ptr()), device)

    def wait(self, stream=None, timeout_ms: int = 0) -> None:
        """Failure detection: wait for the queued work (raises StencilError with code
        ST_ETIMEDOUT if it is still pending after timeout_ms, ST_ENCCL on an async NCCL error)."""
        _check(lib().st_comm_wait(self.handle, _stream_ptr(stream), int(timeout_ms)), "st_comm_wait")

    def profile(self, enable: bool = True) -> None:
        """Phase profiler on/off (include/libstencil.h st_comm_profile)."""
        _check(lib().st_comm_profile(self.handle, int(bool(enable))), "st_comm_profile")

    def profile_read(self) -> dict:
        """{phase: (milliseconds, intervals)} since the last read (waits for the events)."""
        ms, cnt = (_dbl * len(PHASES))(), (_i64 * len(PHASES))()
        _check(lib().st_comm_profile_read(self.handle, ms, cnt), "st_comm_profile_read")
        return {p: (ms[i], cnt[i]) for i, p in enumerate(PHASES)}

    @classmethod
    def local_group(cls, nranks: int, devices=None) -> list["Comm"]:
        """A single-process group of ranks (LOCAL transport: copy-engine swaps ordered by
        device-side flags). devices[r] is rank r's CUDA device (default: all on device 0)."""
        devices = [0] * nranks if devices is None else list(devices)
        hs = (_vp * nranks)()
        devs = (_i32 * nranks)(*devices)
        _check(lib().st_comm_init_local(hs, nranks, devs), "st_comm_init_local")
        return [cls(hs[r], r, nranks, devices[r]) for r in range(nranks)]

    @classmethod
    def create_ipc(cls, rank: int, nranks: int, device: int) -> "Comm":
        """One rank of a multi-process IPC group (copy-engine / fused swaps on CUDA-IPC mappings)."""
        h = _vp()
        _check(lib().st_comm_init_ipc(ctypes.byref(h), nranks, rank, device), "st_comm_init_ipc")
        c = cls(h.value, rank, nranks, device)
        c.kind = "ipc"
        return c

    @classmethod
    def ipc_from_process_group(cls, device: int, group=None) -> "Comm":
        import torch.distributed as dist
        return cls.create_ipc(dist.get_rank(group), dist.get_world_size(group), device)

    def bind_ipc(self, buffers, n_slow_local: int, group=None) -> None:
        """Collective (IPC comms): export this rank's buffers, all-gather the blobs over
        torch.distributed, map the neighbours' buffers and flags."""
        import torch.distributed as dist
        for i, t in enumerate(buffers):
            _f64_cuda(t, f"buffers[{i}]")
        arr = (_vp * len(buffers))(*[t.data_ptr() for t in buffers])
        need = _i64()
        _check(lib().st_comm_export(self.handle, arr, len(buffers), n_slow_local, None, 0, ctypes.byref(need)),
               "st_comm_export")
        blob = (ctypes.c_uint8 * need.value)()
        _check(lib().st_comm_export(self.handle, arr, len(buffers), n_slow_local, ctypes.cast(blob, _vp),
                                    need.value, ctypes.byref(need)), "st_comm_export")
        blobs = [None] * self.nranks
        dist.all_gather_object(blobs, bytes(blob), group=group)
        for peer, b in enumerate(blobs):
            buf = (ctypes.c_uint8 * len(b)).from_buffer_copy(b)
            _check(lib().st_comm_import(self.handle, peer, ctypes.cast(buf, _vp), len(b)), "st_comm_import")

    def bind(self, buffers, n_slow_local: int) -> None:
        """Registers the buffers this rank swaps (LOCAL transport; no-op for NCCL)."""
        for i, t in enumerate(buffers):
            _f64_cuda(t, f"buffers[{i}]")
        arr = (_vp * len(buffers))(*[t.data_ptr() for t in buffers])
        _check(lib().st_comm_bind(self.handle, arr, len(buffers), n_slow_local), "st_comm_bind")

    def set_grid(self, py: int, ny_local: int) -> None:
        """Pencil decomposition: py ranks along y (rank = iz*py + iy); this rank owns ny_local rows."""
        _check(lib().st_comm_set_grid(self.handle, py, ny_local), "st_comm_set_grid")

    def close(self) -> None:
        if self.handle:
            _check(lib().st_comm_destroy(self.handle), "st_comm_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _comm_ptr(comm) -> _vp:
    return None if comm is None else comm.handle


# ------------------------------------------------------------- host-only ---
def st_block_split(n: int, nranks: int, rank: int) -> tuple[int, int]:
    s, c = _i64(), _i64()
    _check(lib().st_block_split(n, nranks, rank, ctypes.byref(s), ctypes.byref(c)), "st_block_split")
    return s.value, c.value


def st_pencil_split(ny: int, nz: int, py: int, pz: int, rank: int) -> tuple[int, int, int, int]:
    """(y0, ny_local, z0, nz_local) of `rank` in a py x pz grid (host only)."""
    o = [_i64() for _ in range(4)]
    _check(lib().st_pencil_split(ny, nz, py, pz, rank, *[ctypes.byref(v) for v in o]), "st_pencil_split")
    return tuple(v.value for v in o)


def st_halo_plan(rank: int, nranks: int, n_slow_local: int, slab_pitch: int, width: int):
    sends, recvs = (Xfer * 2)(), (Xfer * 2)()
    ns, nr = _i32(), _i32()
    _check(lib().st_halo_plan(rank, nranks, n_slow_local, slab_pitch, width, sends, ctypes.byref(ns),
                              recvs, ctypes.byref(nr)), "st_halo_plan")
    conv = lambda x: (x.peer, x.offset, x.count)
    return [conv(sends[i]) for i in range(ns.value)], [conv(recvs[i]) for i in range(nr.value)]


def _schedule(name, rank, nranks, nx, n_local, halo, iters, tblock):
    fn = getattr(lib(), name)
    n = _i64()
    _check(fn(rank, nranks, nx, n_local, halo, iters, tblock, None, 0, ctypes.byref(n)), name)
    arr = (Op * max(1, n.value))()
    _check(fn(rank, nranks, nx, n_local, halo, iters, tblock, arr, n.value, ctypes.byref(n)), name)
    return [{f: getattr(arr[i], f) for f, _ in Op._fields_} for i in range(n.value)]


def st_jacobi2d_schedule(rank: int, nranks: int, nx: int, ny_local: int, halo: int, iters: int,
                         tblock: int = 0) -> list[dict]:
    """The step schedule st_jacobi2d_run executes for one rank (host only)."""
    return _schedule("st_jacobi2d_schedule", rank, nranks, nx, ny_local, halo, iters, tblock)


def st_jacobi3d_schedule(rank: int, nranks: int, nx: int, nz_local: int, halo: int, iters: int,
                         tblock: int = 0) -> list[dict]:
    """The step schedule st_jacobi3d_run executes for one rank (host only; rows = planes)."""
    return _schedule("st_jacobi3d_schedule", rank, nranks, nx, nz_local, halo, iters, tblock)


# ------------------------------------------------------------- compute ---
def st_jacobi2d_run(a, b, iters: int, tblock: int = 0, halo: int = 1, comm: Comm | None = None,
                    nx: int | None = None, stream=None):
    """`iters` Jacobi sweeps on (rows, ld) float64 CUDA tensors a, b.

    a, b: (ny_local + 2*halo, ld) row-major; nx defaults to ld - 2. Returns the
    tensor holding the result (b iff iters is odd)."""
    _f64_cuda(a, "a")
    _f64_cuda(b, "b")
    if a.dim() != 2 or a.shape != b.shape or a.stride(1) != 1 or b.stride(1) != 1 or a.stride(0) != b.stride(0):
        raise ValueError("a, b: 2-D row-major tensors of equal shape and row pitch")
    ld = a.stride(0)
    nx = a.shape[1] - 2 if nx is None else nx
    ny = a.shape[0] - 2 * halo
    rib = _i32()
    _check(lib().st_jacobi2d_run(a.data_ptr(), b.data_ptr(), nx, ny, ld, halo, iters, tblock,
                                 _comm_ptr(comm), _stream_ptr(stream), ctypes.byref(rib)), "st_jacobi2d_run")
    return b if rib.value else a


def st_jacobi3d_run(a, b, iters: int, tblock: int = 0, halo: int = 1, comm: Comm | None = None,
                    nx: int | None = None, stream=None):
    """`iters` 7-point Jacobi sweeps on (planes, ny+2, ldx) float64 CUDA tensors.

    a, b: (nz_local + 2*halo, ny+2, ldx), contiguous; nx defaults to ldx - 2.
    Returns the tensor holding the result (b iff iters is odd)."""
    _f64_cuda(a, "a")
    _f64_cuda(b, "b")
    if a.dim() != 3 or a.shape != b.shape or not a.is_contiguous() or not b.is_contiguous():
        raise ValueError("a, b: contiguous 3-D tensors of equal shape")
    ldx = a.shape[2]
    nx = ldx - 2 if nx is None else nx
    ny = a.shape[1] - 2
    nz = a.shape[0] - 2 * halo
    rib = _i32()
    _check(lib().st_jacobi3d_run(a.data_ptr(), b.data_ptr(), nx, ny, nz, ldx, halo, iters, tblock,
                                 _comm_ptr(comm), _stream_ptr(stream), ctypes.byref(rib)), "st_jacobi3d_run")
    return b if rib.value else a


def st_jacobi3d_run_pencils(a, b, iters: int, comm: Comm | None = None, nx: int | None = None, halo: int = 1,
                            tblock: int = 0, stream=None):
    """3-D Jacobi on a pencil block (nz_local+2*halo, ny_local+2*halo, ldx); see include/libstencil.h."""
    _f64_cuda(a, "a")
    _f64_cuda(b, "b")
    if a.dim() != 3 or a.shape != b.shape or not a.is_contiguous() or not b.is_contiguous():
        raise ValueError("a, b: contiguous 3-D tensors of equal shape")
    nzl, nyl, ldx = a.shape[0] - 2 * halo, a.shape[1] - 2 * halo, a.shape[2]
    nx = ldx - 2 if nx is None else nx
    rib = _i32()
    _check(lib().st_jacobi3d_run_pencils(a.data_ptr(), b.data_ptr(), nx, nyl, nzl, ldx, halo, iters, tblock,
                                         _comm_ptr(comm), _stream_ptr(stream), ctypes.byref(rib)),
           "st_jacobi3d_run_pencils")
    return b if rib.value else a


def st_pw_advect3d_pencils(u, v, w, su, sv, sw, tcx: float, tcy: float, tzc1, tzc2, tzd1, tzd2,
                           comm: Comm | None = None, nx: int | None = None, stream=None) -> None:
    """PW advection on a pencil block; u, v, w ghosts (incl. corners) are swapped first."""
    fields = (u, v, w, su, sv, sw)
    for t, name in zip(fields, ("u", "v", "w", "su", "sv", "sw")):
        _f64_cuda(t, name)
        if t.dim() != 3 or t.shape != u.shape or not t.is_contiguous():
            raise ValueError(f"{name}: contiguous 3-D tensor like u")
    coefs = (tzc1, tzc2, tzd1, tzd2)
    for t, name in zip(coefs, ("tzc1", "tzc2", "tzd1", "tzd2")):
        _f64_cuda(t, name)
    nzl, nyl, ldx = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    nx = ldx - 2 if nx is None else nx
    _check(lib().st_pw_advect3d_pencils(*[t.data_ptr() for t in fields], nx, nyl, nzl, ldx, float(tcx), float(tcy),
                                        *[t.data_ptr() for t in coefs], _comm_ptr(comm), _stream_ptr(stream)),
           "st_pw_advect3d_pencils")


def st_pw_advect3d(u, v, w, su, sv, sw, tcx: float, tcy: float, tzc1, tzc2, tzd1, tzd2,
                   comm: Comm | None = None, nx: int | None = None, stream=None) -> None:
    """Fused PW advection on (nz+2, ny+2, ldx) float64 CUDA tensors."""
    fields = (u, v, w, su, sv, sw)
    for t, name in zip(fields, ("u", "v", "w", "su", "sv", "sw")):
        _f64_cuda(t, name)
        if t.dim() != 3 or t.shape != u.shape or t.stride() != u.stride() or t.stride(2) != 1:
            raise ValueError(f"{name}: 3-D (planes, rows, ldx) tensor like u")
        if t.stride(1) != t.shape[2] or t.stride(0) != t.shape[1] * t.shape[2]:
            raise ValueError(f"{name}: must be contiguous (pitch = shape[2])")
    coefs = (tzc1, tzc2, tzd1, tzd2)
    for t, name in zip(coefs, ("tzc1", "tzc2", "tzd1", "tzd2")):
        _f64_cuda(t, name)
        if t.dim() != 1 or t.shape[0] != u.shape[0] or not t.is_contiguous():
            raise ValueError(f"{name}: contiguous vector of nz+2 doubles")
    nz, ny, ldx = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    nx = ldx - 2 if nx is None else nx
    _check(lib().st_pw_advect3d(*[t.data_ptr() for t in fields], nx, ny, nz, ldx, float(tcx), float(tcy),
                                *[t.data_ptr() for t in coefs], _comm_ptr(comm), _stream_ptr(stream)),
           "st_pw_advect3d")


def st_halo_exchange(comm: Comm, fields, n_slow_local: int, slab_pitch: int, width: int, stream=None) -> None:
    for i, t in enumerate(fields):
        _f64_cuda(t, f"fields[{i}]")
    arr = (_vp * len(fields))(*[t.data_ptr() for t in fields])
    _check(lib().st_halo_exchange(comm.handle, arr, len(fields), n_slow_local, slab_pitch, width,
                                  _stream_ptr(stream)), "st_halo_exchange")


def st_gauss_seidel2d_run(a, iters: int, nx: int | None = None, workspace=None, stream=None):
    """`iters` in-place lexicographic Gauss-Seidel sweeps of a (ny+2, ld) float64 CUDA tensor
    (Listing 1 literally). Returns a."""
    import torch
    _f64_cuda(a, "a")
    if a.dim() != 2 or a.stride(1) != 1:
        raise ValueError("a: 2-D row-major tensor")
    ny, ld = a.shape[0] - 2, a.stride(0)
    nx = a.shape[1] - 2 if nx is None else nx
    need = int(lib().st_gauss_seidel2d_workspace_bytes(nx, ny))
    if workspace is None:
        workspace = torch.empty(max(1, need // 8), dtype=torch.int64, device=a.device)
    _check(lib().st_gauss_seidel2d_run(a.data_ptr(), nx, ny, ld, iters, workspace.data_ptr(),
                                       workspace.numel() * workspace.element_size(), _stream_ptr(stream)),
           "st_gauss_seidel2d_run")
    return a


def st_stencil2d_run(a, b, offsets, coeffs, iters: int, nx: int | None = None, stream=None):
    """Generic linear stencil.apply (reading R23): `iters` sweeps of
    sum_i coeffs[i] * a(y + dy_i, x + dx_i), left to right, on (ny + 2R, ld) float64 CUDA
    tensors (R = max |offset|). Returns whichever of a, b holds the result."""
    _f64_cuda(a, "a")
    _f64_cuda(b, "b")
    if a.dim() != 2 or a.shape != b.shape or a.stride() != b.stride() or a.stride(1) != 1:
        raise ValueError("a, b: same-shape 2-D row-major tensors")
    offs = [int(v) for dy_dx in offsets for v in dy_dx]
    n = len(offs) // 2
    if n < 1 or len(coeffs) != n:
        raise ValueError("one coefficient per (dy, dx) offset")
    R = max(abs(v) for v in offs)
    ld = a.stride(0)
    ny = a.shape[0] - 2 * R
    nx = a.shape[1] - 2 * R if nx is None else nx
    o = (_i32 * (2 * n))(*offs)
    c = (_dbl * n)(*[float(v) for v in coeffs])
    in_b = _i32(0)
    _check(lib().st_stencil2d_run(a.data_ptr(), b.data_ptr(), nx, ny, ld, ctypes.cast(o, _vp), ctypes.cast(c, _vp),
                                  n, iters, _stream_ptr(stream), ctypes.byref(in_b)), "st_stencil2d_run")
    return b if in_b.value else a


def st_stencil2d_expr_halo(expr: str) -> int:
    """Validates an expression stencil on the host and returns its halo R = max |offset|."""
    r = _i32(0)
    _check(lib().st_stencil2d_expr_halo(expr.encode(), ctypes.byref(r)), "st_stencil2d_expr_halo")
    return r.value


def st_stencil2d_expr_run(a, b, expr: str, iters: int, nx: int | None = None, stream=None):
    """`iters` sweeps of the expression stencil (reading R24; NVRTC-compiled, cached) on
    (ny + 2R, ld) float64 CUDA tensors. Returns whichever of a, b holds the result."""
    _f64_cuda(a, "a")
    _f64_cuda(b, "b")
    if a.dim() != 2 or a.shape != b.shape or a.stride() != b.stride() or a.stride(1) != 1:
        raise ValueError("a, b: same-shape 2-D row-major tensors")
    R = st_stencil2d_expr_halo(expr)
    ld = a.stride(0)
    ny = a.shape[0] - 2 * R
    nx = a.shape[1] - 2 * R if nx is None else nx
    in_b = _i32(0)
    _check(lib().st_stencil2d_expr_run(a.data_ptr(), b.data_ptr(), nx, ny, ld, expr.encode(), iters,
                                       _stream_ptr(stream), ctypes.byref(in_b)), "st_stencil2d_expr_run")
    return b if in_b.value else a


def st_stencil_expr_info(expr: str) -> tuple[int, int]:
    """(halo R, access arity 2 or 3) of a validated expression stencil."""
    r, d = _i32(0), _i32(0)
    _check(lib().st_stencil_expr_info(expr.encode(), ctypes.byref(r), ctypes.byref(d)), "st_stencil_expr_info")
    return r.value, d.value


def st_stencil3d_expr_run(a, b, expr: str, iters: int, nx: int | None = None, stream=None):
    """3-D expression stencil over a(dz, dy, dx) on (nz + 2R, ny + 2R, ldx) float64 CUDA tensors
    (x fastest). Returns whichever of a, b holds the result."""
    _f64_cuda(a, "a")
    _f64_cuda(b, "b")
    if a.dim() != 3 or a.shape != b.shape or a.stride() != b.stride() or a.stride(2) != 1:
        raise ValueError("a, b: same-shape 3-D tensors, x contiguous")
    R, dims = st_stencil_expr_info(expr)
    if dims != 3:
        raise ValueError("3-D accesses a(dz, dy, dx) expected")
    ldx = a.stride(1)
    if a.stride(0) != (a.shape[1]) * ldx:
        raise ValueError("planes must be contiguous (stride(0) == rows * ldx)")
    nz, ny = a.shape[0] - 2 * R, a.shape[1] - 2 * R
    nx = a.shape[2] - 2 * R if nx is None else nx
    in_b = _i32(0)
    _check(lib().st_stencil3d_expr_run(a.data_ptr(), b.data_ptr(), nx, ny, nz, ldx, expr.encode(), iters,
                                       _stream_ptr(stream), ctypes.byref(in_b)), "st_stencil3d_expr_run")
    return b if in_b.value else a


def st_stencil3d_fused_run(inputs, outputs, exprs, plane_coefs=(), nx: int | None = None, stream=None) -> None:
    """One application of a fused region: outputs[j] = exprs[j] over f<i> = inputs[i] and
    k<c> = plane_coefs[c][z]. Fields: (nz + 2R, ny + 2R, ldx) float64 CUDA tensors."""
    import re
    for i, t in enumerate(list(inputs) + list(outputs) + list(plane_coefs)):
        _f64_cuda(t, f"tensor {i}")
    a0 = inputs[0]
    offs = [int(v) for e in exprs for m in re.findall(r"f[0-7]\(\s*(-?\d+)\s*,\s*(-?\d+)\s*,\s*(-?\d+)\s*\)", e)
            for v in m]
    R = max(abs(v) for v in offs) if offs else 0
    ldx = a0.stride(1)
    nz, ny = a0.shape[0] - 2 * R, a0.shape[1] - 2 * R
    nx = a0.shape[2] - 2 * R if nx is None else nx
    ins = (_vp * len(inputs))(*[t.data_ptr() for t in inputs])
    outs = (_vp * len(outputs))(*[t.data_ptr() for t in outputs])
    ex = (ctypes.c_char_p * len(exprs))(*[e.encode() for e in exprs])
    ks = (_vp * max(1, len(plane_coefs)))(*[t.data_ptr() for t in plane_coefs])
    _check(lib().st_stencil3d_fused_run(ins, len(inputs), outs, len(outputs), ex, ks, len(plane_coefs), nx, ny, nz,
                                        ldx, _stream_ptr(stream)), "st_stencil3d_fused_run")


def st_pw_fused_expression(tcx: float, tcy: float, which: int) -> str:
    """The PW advection's su/sv/sw (which = 0/1/2) as a fused-region expression (C library text)."""
    n = _i64()
    _check(lib().st_pw_fused_expression(float(tcx), float(tcy), which, None, 0, ctypes.byref(n)),
           "st_pw_fused_expression")
    buf = ctypes.create_string_buffer(n.value)
    _check(lib().st_pw_fused_expression(float(tcx), float(tcy), which, buf, n.value, ctypes.byref(n)),
           "st_pw_fused_expression")
    return buf.value.decode()


def pw_fused_expressions(tcx: float, tcy: float) -> list[str]:
    """[su, sv, sw] expressions of the PW fused region (st_pw_fused_expression)."""
    return [st_pw_fused_expression(tcx, tcy, w) for w in range(3)]


def st_selftest_div6(x) -> int:
    """Number of x (float64 CUDA tensor) where the kernels' fast x/6 differs from IEEE division."""
    import torch
    _f64_cuda(x, "x")
    cnt = torch.zeros(1, dtype=torch.int64, device=x.device)
    _check(lib().st_selftest_div6(x.data_ptr(), x.numel(), cnt.data_ptr(), _stream_ptr()), "st_selftest_div6")
    return int(cnt.item())


# Friendlier aliases
jacobi2d = st_jacobi2d_run
jacobi3d = st_jacobi3d_run
gauss_seidel2d = st_gauss_seidel2d_run
stencil2d = st_stencil2d_run
stencil2d_expr = st_stencil2d_expr_run
pw_advect3d = st_pw_advect3d


def halo_exchange(comm: Comm, tensors, width: int = 1, stream=None) -> None:
    """SURVEY.md §8(b) convention: swap the `width` first/last owned slabs of every tensor
    (slabs = the slowest axis: rows of a 2-D field, planes of a 3-D one) with the neighbour
    ranks; each tensor holds n_slow_local + 2*width slabs."""
    t0 = tensors[0]
    if any(t.shape != t0.shape or t.stride() != t0.stride() for t in tensors):
        raise ValueError("all tensors must have the same shape and strides")
    st_halo_exchange(comm, list(tensors), t0.shape[0] - 2 * width, t0.stride(0), width, stream=stream)

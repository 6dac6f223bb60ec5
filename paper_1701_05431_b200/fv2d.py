"""Thin ctypes binding of libfv2d.so (include/fv2d.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; there is no
Python or CPU fallback -- if the library cannot be built/loaded, import of the
binding raises.  Names follow the C ABI (fv2d_create -> Solver(...),
fv2d_step -> Solver.step, ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

OK, E_ARG, E_CFL, E_NONFINITE, E_RECON, E_CUDA, E_NCCL, E_STATE = range(8)
ADVECTION, EULER, SPRAY = 0, 1, 2
BC_PERIODIC, BC_DIRICHLET, BC_WALL = 0, 1, 2
AOS, SOA = 0, 1
FLAG_NAIVE, FLAG_SPLIT_SOURCE, FLAG_ONE_CELL, FLAG_NCCL_LOOPBACK, FLAG_FUSE_SOURCE, FLAG_GRAPH, FLAG_PEER_HALO = (
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40)
FLAG_GHOST_COLUMNS = 0x80
FLAG_PEER_SPLIT = 0x100
PEER_HANDLE_BYTES = 192
NVAR = {ADVECTION: 1, EULER: 4, SPRAY: 6}
_NAMES = {OK: "OK", E_ARG: "E_ARG", E_CFL: "E_CFL", E_NONFINITE: "E_NONFINITE", E_RECON: "E_RECON",
          E_CUDA: "E_CUDA", E_NCCL: "E_NCCL", E_STATE: "E_STATE"}


class Config(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nvar", C.c_int32), ("system", C.c_int32),
                ("bc_x", C.c_int32), ("bc_y", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("param", C.c_double * 8), ("dirichlet", C.c_double * 6),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("nslabs", C.c_int32), ("device", C.c_int32),
                ("flags", C.c_uint32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("nranks_x", C.c_int32), ("reserved", C.c_int32 * 4)]


class Stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("kernel_launches", C.c_int64), ("newton_iters", C.c_int64),
                ("dt", C.c_double), ("step_kernel_ms", C.c_double), ("step_kernels_timed", C.c_int64),
                ("source_kernel_ms", C.c_double), ("source_kernels_timed", C.c_int64),
                ("sms", C.c_int32), ("resident_ctas", C.c_int32), ("strip_rows", C.c_int32),
                ("reserved0", C.c_int32)]


_LIB = None


def lib():
    """Load libfv2d.so (building it in-tree first if missing or stale)."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("FV2D_LIB") or _build.build()  # FV2D_LIB: an alternative build (tuning)
        L = C.CDLL(path)
        P = C.POINTER
        vp = C.c_void_p
        d = P(C.c_double)
        L.fv2d_version.argtypes = [P(C.c_int32), P(C.c_int32)]
        L.fv2d_config_default.argtypes = [P(Config), C.c_int32, C.c_int32, C.c_int32]
        L.fv2d_nccl_unique_id.argtypes = [C.c_char_p]
        L.fv2d_create.argtypes = [P(Config), C.c_char_p, vp, P(vp)]
        L.fv2d_destroy.argtypes = [vp]
        L.fv2d_set_state.argtypes = [vp, vp, C.c_int]
        L.fv2d_set_state_device.argtypes = [vp, vp, C.c_int]
        L.fv2d_get_state.argtypes = [vp, vp, C.c_int]
        L.fv2d_compute_dt.argtypes = [vp, C.c_double, d, d]
        L.fv2d_check_dt.argtypes = [vp, C.c_double, d]
        L.fv2d_step.argtypes = [vp, C.c_double, C.c_int32]
        L.fv2d_step_adaptive.argtypes = [vp, C.c_double, C.c_int32, d]
        L.fv2d_apply_source.argtypes = [vp, C.c_double]
        L.fv2d_synchronize.argtypes = [vp]
        L.fv2d_device_state.argtypes = [vp, C.c_int32, P(vp), P(C.c_int64), P(C.c_int64), P(C.c_int32)]
        L.fv2d_last_error.argtypes = [vp, C.c_char_p, C.c_size_t, P(C.c_int64), P(C.c_int64), d]
        L.fv2d_get_stats.argtypes = [vp, P(Stats)]
        L.fv2d_set_profiling.argtypes = [vp, C.c_int32]
        L.fv2d_snapshot.argtypes = [vp, vp, C.c_int]
        L.fv2d_snapshot_wait.argtypes = [vp]
        L.fv2d_host_alloc.argtypes = [C.c_size_t, P(vp)]
        L.fv2d_host_free.argtypes = [vp]
        L.fv2d_peer_export.argtypes = [vp, C.c_char_p]
        L.fv2d_peer_connect.argtypes = [vp, C.c_char_p]
        L.fv2d_peer_connect_local.argtypes = [vp, P(vp)]
        L.fv2d_step_host.argtypes = [vp, vp, vp, C.c_int, C.c_double, C.c_int32]
        for name in ("fv2d_version", "fv2d_config_default", "fv2d_nccl_unique_id", "fv2d_create", "fv2d_destroy",
                     "fv2d_set_state", "fv2d_set_state_device", "fv2d_get_state", "fv2d_compute_dt",
                     "fv2d_check_dt", "fv2d_step", "fv2d_step_adaptive", "fv2d_apply_source",
                     "fv2d_synchronize", "fv2d_device_state", "fv2d_last_error", "fv2d_get_stats",
                     "fv2d_set_profiling", "fv2d_snapshot", "fv2d_snapshot_wait", "fv2d_host_alloc",
                     "fv2d_host_free", "fv2d_peer_export", "fv2d_peer_connect", "fv2d_peer_connect_local",
                     "fv2d_step_host"):
            getattr(L, name).restype = C.c_int
        _LIB = L
    return _LIB


def lib_path() -> str:
    return _build.LIB


class FV2DError(RuntimeError):
    def __init__(self, code, message="", step=-1, cell=-1, value=float("nan")):
        super().__init__(f"fv2d {_NAMES.get(code, code)}: {message} (step {step}, cell {cell})")
        self.code, self.message, self.step, self.cell, self.value = code, message, step, cell, value


def _preload_nccl():
    """Load torch's NCCL (the nvidia-nccl wheel) globally first, so the library's
    dlopen("libnccl.so.2") resolves to the same single copy torch uses."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        path = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(path):
            C.CDLL(path, mode=C.RTLD_GLOBAL)
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    _preload_nccl()
    buf = C.create_string_buffer(128)
    rc = lib().fv2d_nccl_unique_id(buf)
    if rc != OK:
        raise FV2DError(rc, "ncclGetUniqueId")
    return buf.raw


class PinnedArray:
    """A float64 numpy array in page-locked host memory (fv2d_host_alloc)."""

    def __init__(self, shape):
        n = int(np.prod(shape))
        p = C.c_void_p()
        rc = lib().fv2d_host_alloc(max(8, n * 8), C.byref(p))
        if rc != OK:
            raise FV2DError(rc, "fv2d_host_alloc")
        self._p = p
        self.array = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(n,)).reshape(shape)

    def free(self):
        if getattr(self, "_p", None):
            self.array = None
            lib().fv2d_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Solver:
    """One context of libfv2d (fv2d_create ... fv2d_destroy)."""

    def __init__(self, nx, ny, system=EULER, *, x0=0.0, x1=1.0, y0=0.0, y1=1.0, param=None,
                 bc_x=BC_PERIODIC, bc_y=BC_PERIODIC, dirichlet=(), rank=0, nranks=1, nslabs=1, device=0,
                 flags=0, tiles=(1, 1), nranks_x=1, nccl_id: bytes | None = None, stream: int | None = None):
        L = lib()
        cfg = Config()
        rc = L.fv2d_config_default(C.byref(cfg), nx, ny, system)
        if rc != OK:
            raise FV2DError(rc, "config_default")
        cfg.x0, cfg.x1, cfg.y0, cfg.y1 = x0, x1, y0, y1
        if param is not None:
            for k in range(8):
                cfg.param[k] = 0.0
            for k, v in enumerate(param):
                cfg.param[k] = v
        for k, v in enumerate(dirichlet):
            cfg.dirichlet[k] = v
        cfg.bc_x, cfg.bc_y = bc_x, bc_y
        cfg.rank, cfg.nranks, cfg.nslabs, cfg.device, cfg.flags = rank, nranks, nslabs, device, flags
        cfg.tiles_x, cfg.tiles_y = tiles
        cfg.nranks_x = nranks_x
        self.cfg = cfg
        self.nx, self.ny, self.nv, self.system = nx, ny, NVAR[system], system
        px = max(1, nranks_x)
        self.ny_local = ny // (nranks // px)  # this rank's block (fv2d.h: Layouts)
        self.nx_local = nx // px
        if nranks > 1 or (flags & FLAG_NCCL_LOOPBACK):
            _preload_nccl()
        h = C.c_void_p()
        rc = L.fv2d_create(C.byref(cfg), nccl_id, C.c_void_p(stream or 0), C.byref(h))
        if rc != OK:
            raise FV2DError(rc, "fv2d_create")
        self._h = h

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib().fv2d_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- errors
    def last_error(self):
        buf = C.create_string_buffer(512)
        st, cell = C.c_int64(-1), C.c_int64(-1)
        val = C.c_double(float("nan"))
        lib().fv2d_last_error(self._h, buf, 512, C.byref(st), C.byref(cell), C.byref(val))
        return {"message": buf.value.decode(), "step": st.value, "cell": cell.value, "value": val.value}

    def _check(self, rc, what=""):
        if rc != OK:
            e = self.last_error() if self._h else {"message": what, "step": -1, "cell": -1, "value": float("nan")}
            raise FV2DError(rc, e["message"] or what, e["step"], e["cell"], e["value"])

    # -- state
    def _shape(self, layout):
        return (self.ny_local, self.nx_local, self.nv) if layout == AOS else (self.nv, self.ny_local, self.nx_local)

    def set_state(self, W: np.ndarray, layout: int = AOS):
        W = np.ascontiguousarray(W, dtype=np.float64)
        if W.shape != self._shape(layout):
            raise ValueError(f"state shape {W.shape} != {self._shape(layout)}")
        self._check(lib().fv2d_set_state(self._h, W.ctypes.data, layout), "set_state")

    def set_state_ptr(self, ptr: int, layout: int = AOS, device: bool = False):
        fn = lib().fv2d_set_state_device if device else lib().fv2d_set_state
        self._check(fn(self._h, C.c_void_p(ptr), layout), "set_state")

    def get_state(self, layout: int = AOS, out: np.ndarray | None = None, raise_on_error: bool = True):
        if out is None:
            out = np.empty(self._shape(layout))
        elif out.shape != self._shape(layout) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError(f"get_state buffer must be float64 C-contiguous {self._shape(layout)}")
        rc = lib().fv2d_get_state(self._h, out.ctypes.data, layout)
        if raise_on_error:
            self._check(rc, "get_state")
        return out

    def get_state_ptr(self, ptr: int, layout: int = AOS):
        self._check(lib().fv2d_get_state(self._h, C.c_void_p(ptr), layout), "get_state")

    def device_state(self, slab: int = 0):
        p, pitch, plane, ny = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int32()
        self._check(lib().fv2d_device_state(self._h, slab, C.byref(p), C.byref(pitch), C.byref(plane),
                                            C.byref(ny)))
        return p.value, pitch.value, plane.value, ny.value

    # -- the hot path
    def compute_dt(self, cfl: float):
        dt, s = C.c_double(), C.c_double()
        self._check(lib().fv2d_compute_dt(self._h, cfl, C.byref(dt), C.byref(s)), "compute_dt")
        return dt.value, s.value

    def check_dt(self, dt: float) -> float:
        s = C.c_double()
        self._check(lib().fv2d_check_dt(self._h, dt, C.byref(s)), "check_dt")
        return s.value

    def step(self, dt: float, nsteps: int = 1):
        self._check(lib().fv2d_step(self._h, dt, nsteps), "step")

    def step_adaptive(self, cfl: float, nsteps: int = 1, log: bool = True):
        if log:
            buf = np.zeros(max(1, nsteps))
            self._check(lib().fv2d_step_adaptive(self._h, cfl, nsteps, _dp(buf)), "step_adaptive")
            return buf[:nsteps]
        self._check(lib().fv2d_step_adaptive(self._h, cfl, nsteps, None), "step_adaptive")
        return None

    def step_host(self, W_in, W_out, dt: float, nsteps: int = 1, layout: int = AOS):
        """fv2d_step_host: W^0 from host W_in, nsteps fixed-dt steps, result into host
        W_out (may be W_in); numpy arrays, PinnedArray or raw pointers (ints)."""
        def ptr(x):
            if isinstance(x, int):
                return x
            arr = x.array if isinstance(x, PinnedArray) else x
            if arr.shape != self._shape(layout) or arr.dtype != np.float64 or not arr.flags.c_contiguous:
                raise ValueError(f"host state must be float64 C-contiguous {self._shape(layout)}")
            return arr.ctypes.data
        self._check(lib().fv2d_step_host(self._h, C.c_void_p(ptr(W_in)), C.c_void_p(ptr(W_out)), layout, dt, nsteps),
                    "step_host")

    def apply_source(self, dt: float):
        self._check(lib().fv2d_apply_source(self._h, dt), "apply_source")

    def synchronize(self):
        self._check(lib().fv2d_synchronize(self._h), "synchronize")

    def status(self) -> int:
        return lib().fv2d_synchronize(self._h)

    def snapshot(self, out: "PinnedArray | np.ndarray", layout: int = AOS):
        """Asynchronous copy of the current state into `out`; valid after
        snapshot_wait().  Pass a PinnedArray for a copy that overlaps stepping."""
        arr = out.array if isinstance(out, PinnedArray) else out
        if arr.shape != self._shape(layout) or arr.dtype != np.float64 or not arr.flags.c_contiguous:
            raise ValueError(f"snapshot buffer must be float64 C-contiguous {self._shape(layout)}")
        self._check(lib().fv2d_snapshot(self._h, arr.ctypes.data, layout), "snapshot")

    def snapshot_wait(self):
        self._check(lib().fv2d_snapshot_wait(self._h), "snapshot_wait")

    # -- peer-memory multi-GPU path (FLAG_PEER_HALO)
    def peer_export(self) -> bytes:
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        self._check(lib().fv2d_peer_export(self._h, buf), "peer_export")
        return buf.raw

    def peer_connect(self, all_handles: bytes):
        """all_handles: every rank's peer_export() bytes, concatenated in rank order."""
        self._check(lib().fv2d_peer_connect(self._h, all_handles), "peer_connect")

    def peer_connect_local(self, group):
        """group[r]: the Solver of rank r, all in this process (drive them from separate threads)."""
        arr = (C.c_void_p * len(group))(*[g._h.value for g in group])
        self._check(lib().fv2d_peer_connect_local(self._h, arr), "peer_connect_local")

    def set_profiling(self, enable: bool = True):
        self._check(lib().fv2d_set_profiling(self._h, 1 if enable else 0), "set_profiling")

    def stats(self) -> dict:
        s = Stats()
        self._check(lib().fv2d_get_stats(self._h, C.byref(s)), "get_stats")
        return {"steps": s.steps, "kernel_launches": s.kernel_launches, "newton_iters": s.newton_iters,
                "dt": s.dt, "step_kernel_ms": s.step_kernel_ms, "step_kernels_timed": s.step_kernels_timed,
                "source_kernel_ms": s.source_kernel_ms, "source_kernels_timed": s.source_kernels_timed,
                "sms": s.sms, "resident_ctas": s.resident_ctas, "strip_rows": s.strip_rows}

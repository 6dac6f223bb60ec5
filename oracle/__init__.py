"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle (see fv2d_oracle.c header).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1701_05431_b200``) never imports it.

This module is argument marshalling around ``liboracle.so`` (plain C, fp64,
``-O2 -ffp-contract=off``): numpy arrays in the paper's Cell (AoS) layout
``W[j, i, v]``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fv2d_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, E_ARG, E_CFL, E_NONFINITE, E_RECON = 0, 1, 2, 3, 4
ADVECTION, EULER, SPRAY = 0, 1, 2
BC_PERIODIC, BC_DIRICHLET, BC_WALL = 0, 1, 2
NVAR = {ADVECTION: 1, EULER: 4, SPRAY: 6}


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, strict IEEE: no FMA contraction, no fast-math).
    ``FV2D_ORACLE_LIB`` names a prebuilt oracle instead (tools/mutate_oracle.py
    points it at deliberately broken builds to show that the pins catch them)."""
    if os.environ.get("FV2D_ORACLE_LIB"):
        return os.environ["FV2D_ORACLE_LIB"]
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-D_DEFAULT_SOURCE", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nvar", C.c_int32), ("system", C.c_int32),
                ("bc_x", C.c_int32), ("bc_y", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("param", C.c_double * 8), ("dirichlet", C.c_double * 6)]


class _Err(C.Structure):
    _fields_ = [("code", C.c_int32), ("cell", C.c_int64), ("value", C.c_double)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        d = P(C.c_double)
        cfg = P(_Cfg)
        err = P(_Err)
        _lib.or_phys_flux.argtypes = [cfg, d, C.c_int, d, d]
        _lib.or_lf_flux.argtypes = [cfg, d, d, C.c_int, d]
        _lib.or_smax.argtypes = [cfg, d, d, P(C.c_int64), err]
        _lib.or_speeds.argtypes = [cfg, d, d, d]
        _lib.or_transport_step.argtypes = [cfg, d, d, C.c_double, err]
        _lib.or_source_step.argtypes = [cfg, d, C.c_double, P(C.c_int64), err]
        _lib.or_reconstruct.argtypes = [d, d, d, d, P(C.c_int32)]
        _lib.or_gl24.argtypes = [d, d]
        _lib.or_gl24.restype = None
        _lib.or_spray_guard.argtypes = [cfg, d, C.c_double, err]
        _lib.or_run.argtypes = [cfg, d, C.c_int32, C.c_int32, C.c_double, d, P(C.c_int32),
                                C.c_int32, d, P(C.c_int32), P(C.c_int64), err]
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class Config:
    """Problem statement: system, mesh Nx x Ny over [x0,x1]x[y0,y1], BCs."""
    nx: int
    ny: int
    system: int = EULER
    x0: float = 0.0
    x1: float = 1.0
    y0: float = 0.0
    y1: float = 1.0
    param: tuple = (1.4,)
    bc_x: int = BC_PERIODIC
    bc_y: int = BC_PERIODIC
    dirichlet: tuple = ()

    @property
    def nvar(self) -> int:
        return NVAR[self.system]

    def _c(self) -> _Cfg:
        c = _Cfg()
        c.nx, c.ny, c.nvar, c.system = self.nx, self.ny, self.nvar, self.system
        c.bc_x, c.bc_y = self.bc_x, self.bc_y
        c.x0, c.x1, c.y0, c.y1 = self.x0, self.x1, self.y0, self.y1
        for k, v in enumerate(self.param):
            c.param[k] = v
        for k, v in enumerate(self.dirichlet):
            c.dirichlet[k] = v
        return c


class OracleError(RuntimeError):
    def __init__(self, code, cell=-1, value=float("nan"), steps_done=None):
        super().__init__(f"oracle status {code} at cell {cell} (value {value}), steps_done={steps_done}")
        self.code, self.cell, self.value, self.steps_done = code, cell, value, steps_done


def _check(rc, err: _Err | None = None, steps_done=None):
    if rc != OK:
        if err is not None:
            raise OracleError(rc, err.cell, err.value, steps_done)
        raise OracleError(rc)


def _aos(cfg: Config, W) -> np.ndarray:
    W = np.ascontiguousarray(W, dtype=np.float64)
    if W.shape != (cfg.ny, cfg.nx, cfg.nvar):
        raise ValueError(f"W shape {W.shape} != {(cfg.ny, cfg.nx, cfg.nvar)}")
    return W


def phys_flux(cfg: Config, W, direction: int):
    """F(W).n for n = e_x (0) / e_y (1) and the directional spectral radius."""
    w = np.ascontiguousarray(W, dtype=np.float64)
    F = np.zeros(6)
    s = np.zeros(1)
    rc = _L().or_phys_flux(C.byref(cfg._c()), _dp(w), direction, _dp(F), _dp(s))
    _check(rc)
    return F[: cfg.nvar].copy(), float(s[0])


def lf_flux(cfg: Config, WL, WR, direction: int) -> np.ndarray:
    """Lax-Friedrichs numerical flux F~(WL, WR, n)."""
    L = np.ascontiguousarray(WL, dtype=np.float64)
    R = np.ascontiguousarray(WR, dtype=np.float64)
    F = np.zeros(6)
    rc = _L().or_lf_flux(C.byref(cfg._c()), _dp(L), _dp(R), direction, _dp(F))
    _check(rc)
    return F[: cfg.nvar].copy()


def smax(cfg: Config, W):
    """CFL reduction (eq:CFL_cond): (smax, argmax j*nx+i)."""
    W = _aos(cfg, W)
    s = np.zeros(1)
    a = C.c_int64(-1)
    e = _Err()
    _check(_L().or_smax(C.byref(cfg._c()), _dp(W), _dp(s), C.byref(a), C.byref(e)), e)
    return float(s[0]), int(a.value)


def speeds(cfg: Config, W):
    W = _aos(cfg, W)
    sx = np.zeros((cfg.ny, cfg.nx))
    sy = np.zeros((cfg.ny, cfg.nx))
    _check(_L().or_speeds(C.byref(cfg._c()), _dp(W), _dp(sx), _dp(sy)))
    return sx, sy


def transport_step(cfg: Config, W, dt: float) -> np.ndarray:
    """W* of eq:VF_scheme (one transport step, no source)."""
    W = _aos(cfg, W)
    out = np.empty_like(W)
    e = _Err()
    _check(_L().or_transport_step(C.byref(cfg._c()), _dp(W), _dp(out), dt, C.byref(e)), e)
    return out


def source_step(cfg: Config, W, dt: float):
    """W^{n+1} = W* + dt S(W*) (eq:SourceTerm); returns (W_new, newton_iterations)."""
    W = _aos(cfg, W).copy()
    it = C.c_int64(0)
    e = _Err()
    _check(_L().or_source_step(C.byref(cfg._c()), _dp(W), dt, C.byref(it), C.byref(e)), e)
    return W, int(it.value)


def reconstruct(m):
    """NDF reconstruction -> (lambda[4], n(0), m_-1/2, iterations)."""
    m = np.ascontiguousarray(m, dtype=np.float64)
    lam = np.zeros(4)
    n0 = np.zeros(1)
    mmh = np.zeros(1)
    it = C.c_int32(0)
    rc = _L().or_reconstruct(_dp(m), _dp(lam), _dp(n0), _dp(mmh), C.byref(it))
    _check(rc)
    return lam, float(n0[0]), float(mmh[0]), int(it.value)


def spray_guard(cfg: Config, W, dt: float):
    """S:440 startup guard: raises OracleError(E_ARG, argmin cell, min m3/m1)
    when dt*K > 0.1*min(m3/m1)."""
    W = _aos(cfg, W)
    e = _Err()
    _check(_L().or_spray_guard(C.byref(cfg._c()), _dp(W), dt, C.byref(e)), e)


def gl24():
    t = np.zeros(24)
    w = np.zeros(24)
    _L().or_gl24(_dp(t), _dp(w))
    return t, w


@dataclass
class RunResult:
    W: np.ndarray
    dt_log: np.ndarray
    dumps: dict = field(default_factory=dict)
    steps_done: int = 0
    newton_iters: int = 0


FIXED, ADAPTIVE = 0, 1


def run(cfg: Config, W0, nsteps: int, mode: int = ADAPTIVE, value: float = 0.45,
        dump_steps=(), raise_on_error: bool = True):
    """Time loop: mode FIXED (value = dt, checked each iteration) or
    ADAPTIVE (value = C, dt_n = C*min(dx,dy)/smax(W^n))."""
    W = _aos(cfg, W0).copy()
    dump_steps = sorted(set(int(s) for s in dump_steps))
    ds = (C.c_int32 * max(1, len(dump_steps)))(*dump_steps)
    dumps = np.zeros((max(1, len(dump_steps)),) + W.shape)
    dt_log = np.full(max(1, nsteps), np.nan)
    done = C.c_int32(0)
    it = C.c_int64(0)
    e = _Err()
    rc = _L().or_run(C.byref(cfg._c()), _dp(W), nsteps, mode, value, _dp(dt_log), ds,
                     len(dump_steps), _dp(dumps), C.byref(done), C.byref(it), C.byref(e))
    if rc != OK and raise_on_error:
        raise OracleError(rc, e.cell, e.value, done.value)
    res = RunResult(W=W, dt_log=dt_log[: done.value].copy(),
                    dumps={s: dumps[k].copy() for k, s in enumerate(dump_steps) if s <= done.value},
                    steps_done=int(done.value), newton_iters=int(it.value))
    res.status = rc
    res.err_cell = int(e.cell) if rc else -1
    return res

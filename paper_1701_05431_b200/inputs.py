"""Seeded synthetic initial conditions (the ONLY module shared by the oracle
tests and the CUDA path -- it holds none of the scheme's arithmetic: no flux,
no update, no CFL reduction, no source term).

Every generator returns the paper's Cell layout: a float64 array
``W[j, i, v]`` of shape (ny, nx, nVar) (x fastest, variable innermost), built
on the host once and fed identically to both sides (R23).  Cell centres are
``x_i = x0 + (i + 0.5) dx`` (R24).  Random draws use numpy's PCG64 via
``np.random.default_rng(seed)``.  ``rows=(j0, j1)`` generates only that band of
rows (used to build large grids slab by slab without holding the full array).

Recipes:
  * advection_dyadic  -- u = k/256, k ~ U{0..255} (exact in fp64; CFL=1 pin)
  * advection_smooth  -- u = sin(2 pi x) sin(2 pi y)
  * euler_lax_liu3    -- 2-D Riemann problem, Lax-Liu configuration 3
  * euler_sod_x       -- Sod shock tube along x
  * euler_random      -- rho, p ~ U[0.5, 2], u, v ~ U[-1, 1] per cell
  * euler_bell        -- localized cosine, bell reading R22 of eq:LocalizedCosine
  * euler_cosine_printed -- eq:LocalizedCosine exactly as printed
  * euler_vortex      -- isentropic vortex eq:RotatingGaussian/eq:SetUp (R21)
  * spray_taylor_green -- R16: lambda_true = (0, 1 + sin sin/2, cos/2, 0), u = u_g
"""
from __future__ import annotations

import numpy as np

GAMMA = 1.4


def _centres(nx, ny, rows, x0=0.0, x1=1.0, y0=0.0, y1=1.0):
    j0, j1 = rows if rows is not None else (0, ny)
    dx = (x1 - x0) / nx
    dy = (y1 - y0) / ny
    x = x0 + (np.arange(nx) + 0.5) * dx
    y = y0 + (np.arange(j0, j1) + 0.5) * dy
    return np.meshgrid(x, y, indexing="xy")  # (rows, nx)


def primitive_to_conserved(rho, u, v, p, gamma=GAMMA):
    """(rho, u, v, p) -> (rho, rho u, rho v, rho E), rho E = p/(gamma-1) + rho (u^2+v^2)/2
    (perfect gas law of eq:Euler).  IC construction only."""
    W = np.empty(rho.shape + (4,))
    W[..., 0] = rho
    W[..., 1] = rho * u
    W[..., 2] = rho * v
    W[..., 3] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return W


def advection_dyadic(nx, ny, seed=0, rows=None):
    j0, j1 = rows if rows is not None else (0, ny)
    rng = np.random.default_rng(seed)
    k = rng.integers(0, 256, size=(ny, nx))[j0:j1]
    return (k.astype(np.float64) / 256.0)[..., None]


def advection_smooth(nx, ny, rows=None):
    X, Y = _centres(nx, ny, rows)
    return (np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y))[..., None]


def euler_lax_liu3(nx, ny, rows=None, gamma=GAMMA):
    """Lax & Liu (1998) configuration 3 (external to the paper; BASELINE c2):
    quadrants about (0.5, 0.5), (rho, u, v, p):
    NE (1.5, 0, 0, 1.5), NW (0.5323, 1.206, 0, 0.3),
    SW (0.138, 1.206, 1.206, 0.029), SE (0.5323, 0, 1.206, 0.3)."""
    X, Y = _centres(nx, ny, rows)
    east = X >= 0.5
    north = Y >= 0.5
    rho = np.where(north, np.where(east, 1.5, 0.5323), np.where(east, 0.5323, 0.138))
    u = np.where(north, np.where(east, 0.0, 1.206), np.where(east, 0.0, 1.206))
    v = np.where(north, np.where(east, 0.0, 0.0), np.where(east, 1.206, 1.206))
    p = np.where(north, np.where(east, 1.5, 0.3), np.where(east, 0.3, 0.029))
    return primitive_to_conserved(rho, u, v, p, gamma)


def euler_sod_x(nx, ny, rows=None, gamma=GAMMA):
    """Sod shock tube along x: (1, 0, 0, 1) for x < 0.5, (0.125, 0, 0, 0.1) otherwise."""
    X, _ = _centres(nx, ny, rows)
    left = X < 0.5
    rho = np.where(left, 1.0, 0.125)
    p = np.where(left, 1.0, 0.1)
    z = np.zeros_like(rho)
    return primitive_to_conserved(rho, z, z, p, gamma)


def euler_random(nx, ny, seed=1, rows=None, gamma=GAMMA):
    """Per cell rho, p ~ U[0.5, 2], u, v ~ U[-1, 1] (PCG64, seed)."""
    j0, j1 = rows if rows is not None else (0, ny)
    rng = np.random.default_rng(seed)
    # draw the full field row-block by row-block so that a band equals the
    # corresponding rows of the full draw
    out = np.empty((j1 - j0, nx, 4))
    for j in range(0, ny, 256):
        jb = min(ny, j + 256)
        blk = rng.random(size=(jb - j, nx, 4))
        lo, hi = max(j, j0), min(jb, j1)
        if lo < hi:
            b = blk[lo - j: hi - j]
            rho = 0.5 + 1.5 * b[..., 0]
            p = 0.5 + 1.5 * b[..., 1]
            u = -1.0 + 2.0 * b[..., 2]
            v = -1.0 + 2.0 * b[..., 3]
            out[lo - j0: hi - j0] = primitive_to_conserved(rho, u, v, p, gamma)
        if jb >= j1:
            break
    return out


def euler_bell(nx, ny, rows=None, gamma=GAMMA):
    """Localized cosine, reading R22: rho = 1 + (r<0.25) (1 + cos 4 pi r)/2, u=v=1, p=1/gamma."""
    X, Y = _centres(nx, ny, rows)
    r = np.sqrt((X - 0.5) ** 2 + (Y - 0.5) ** 2)
    rho = 1.0 + np.where(r < 0.25, 0.5 * (1.0 + np.cos(4 * np.pi * r)), 0.0)
    one = np.ones_like(rho)
    return primitive_to_conserved(rho, one, one, one / gamma, gamma)


def euler_bell_exact(nx, ny, t, gamma=GAMMA):
    """eq:LCAnalytic for the bell reading: floor-wrapped advection by (1,1)."""
    X, Y = _centres(nx, ny, None)
    xs = X - t - np.floor(X - t)
    ys = Y - t - np.floor(Y - t)
    r = np.sqrt((xs - 0.5) ** 2 + (ys - 0.5) ** 2)
    rho = 1.0 + np.where(r < 0.25, 0.5 * (1.0 + np.cos(4 * np.pi * r)), 0.0)
    one = np.ones_like(rho)
    return primitive_to_conserved(rho, one, one, one / gamma, gamma)


def euler_cosine_printed(nx, ny, rows=None, gamma=GAMMA):
    """eq:LocalizedCosine as printed: rho = 1 + (r<0.25) cos(4 pi r)."""
    X, Y = _centres(nx, ny, rows)
    r = np.sqrt((X - 0.5) ** 2 + (Y - 0.5) ** 2)
    rho = 1.0 + np.where(r < 0.25, np.cos(4 * np.pi * r), 0.0)
    one = np.ones_like(rho)
    return primitive_to_conserved(rho, one, one, one / gamma, gamma)


def euler_vortex(nx, ny, rows=None, gamma=GAMMA, omega=1.0, R=0.1, ubar=1.0, vbar=1.0, t=0.0):
    """Isentropic vortex (eq:RotatingGaussian, eq:SetUp), coordinates relative to
    the (advected, floor-wrapped) centre (R21); p = rho^gamma / gamma (eq:isentropy)."""
    X, Y = _centres(nx, ny, rows)
    xs = X - ubar * t - np.floor(X - ubar * t) - 0.5
    ys = Y - vbar * t - np.floor(Y - vbar * t) - 0.5
    r2 = xs * xs + ys * ys
    w = omega * np.exp(-r2 / (2 * R * R))
    u = ubar - ys / R * w
    v = vbar + xs / R * w
    rho = (1.0 - (gamma - 1.0) / 2.0 * w * w) ** (1.0 / (gamma - 1.0))
    p = rho ** gamma / gamma
    return primitive_to_conserved(rho, u, v, p, gamma)


def taylor_green(x, y):
    """Gas velocity u_g = (sin 2pi x cos 2pi y, -cos 2pi x sin 2pi y) (R20)."""
    return np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y), -np.cos(2 * np.pi * x) * np.sin(2 * np.pi * y)


def spray_taylor_green(nx, ny, rows=None):
    """R16: lambda_true(x,y) = (0, 1 + sin(2pi x) sin(2pi y)/2, cos(2pi x)/2, 0);
    moments m_k = 2 int_0^1 t^{k+1} exp(-P(t)) dt by 24-node Gauss-Legendre
    (numpy leggauss, independent of both the oracle's and the library's tables);
    velocity u(0) = u_g.  Realizable by construction."""
    X, Y = _centres(nx, ny, rows)
    l1 = 1.0 + 0.5 * np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y)
    l2 = 0.5 * np.cos(2 * np.pi * X)
    xg, wg = np.polynomial.legendre.leggauss(24)
    t = (xg + 1.0) / 2.0
    w = wg / 2.0
    W = np.empty(X.shape + (6,))
    e = np.exp(-(l1[..., None] * t + l2[..., None] * t * t))  # lambda0 = lambda3 = 0
    for k in range(4):
        W[..., k] = 2.0 * np.sum(w * t ** (k + 1) * e, axis=-1)
    ugx, ugy = taylor_green(X, Y)
    W[..., 4] = W[..., 2] * ugx
    W[..., 5] = W[..., 2] * ugy
    return W


def uniform(nx, ny, state):
    state = np.asarray(state, dtype=np.float64)
    return np.broadcast_to(state, (ny, nx, state.size)).copy()

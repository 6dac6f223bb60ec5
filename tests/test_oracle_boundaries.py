"""Pins of the oracle's spray transport flux and of its boundary ghosts
(Dirichlet, wall) against what the paper and mathematics fix -- textbook
upwind, exact rational arithmetic, 50-digit evaluations written in the paper's
primitive notation, and closed forms derived by hand from reading R13.

P:L = PAPER.md line, S:L = SPEC.md line, R<n> = DESIGN.md §3 reading.
"""
import math
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from paper_1701_05431_b200 import inputs

G = 1.4


def _spray_cfg(nx, ny=None, **kw):
    return O.Config(nx=nx, ny=ny or nx, system=O.SPRAY, param=(1.0, 1.0), **kw)


def _fsum_vars(W):
    return np.array([math.fsum(W[..., k].ravel()) for k in range(W.shape[-1])])


# ------------------------------------------------- spray transport = upwind
def _dyadic_spray_uniform_velocity(n, a, seed):
    """Moments k/256 (k = 1..255), m2 a power of two per cell so that
    u = m2u * (1/m2) is exactly a: then every product of the scheme is exact."""
    rng = np.random.default_rng(seed)
    W = np.empty((n, n, 6))
    W[..., 0] = rng.integers(1, 256, size=(n, n)) / 256.0
    W[..., 1] = rng.integers(1, 256, size=(n, n)) / 256.0
    W[..., 2] = 2.0 ** rng.integers(-2, 2, size=(n, n))
    W[..., 3] = rng.integers(1, 256, size=(n, n)) / 256.0
    W[..., 4] = a[0] * W[..., 2]
    W[..., 5] = a[1] * W[..., 2]
    return W


def _upwind_component(u, a, lx, ly):
    """First-order upwind for q_t + a.grad q = 0 (textbook, LeVeque; the scheme
    family P:126 cites), periodic."""
    ax, ay = a
    dxu = u - np.roll(u, 1, axis=1) if ax > 0 else np.roll(u, -1, axis=1) - u
    dyu = u - np.roll(u, 1, axis=0) if ay > 0 else np.roll(u, -1, axis=0) - u
    return u - lx * ax * dxu - ly * ay * dyu


@pytest.mark.parametrize("a", [(0.5, -0.25), (-0.25, 0.5), (1.0, 0.5), (-0.5, -1.0)])
def test_spray_uniform_velocity_is_per_moment_upwind_bitwise(a):
    """eq:Essadki's left-hand side is pure transport at velocity u:
    every one of the six conserved quantities (m0, m1, m2, m3, m2 u, m2 v) obeys
    q_t + div(q u) = 0.  With a uniform velocity field u = a the system is six
    decoupled linear advections, and the LF flux with the directional spectral
    radius |u.n| (R2) is exactly first-order upwind for each of them --
    so one step must equal textbook upwind per moment, bitwise on dyadic data.
    Pins every flux component and the speed sigma = |u.n|."""
    n = 32
    cfg = _spray_cfg(n)
    W = _dyadic_spray_uniform_velocity(n, a, seed=17)
    dt = 0.5 / n                       # lx = ly = 1/2, |a| <= 1: stable, exact
    out = O.transport_step(cfg, W, dt)
    for k in range(6):
        ref = _upwind_component(W[..., k], a, 0.5, 0.5)
        assert np.array_equal(out[..., k], ref), f"moment {k}"
    # and the CFL speed is max(|a_x|, |a_y|) exactly
    s, _ = O.smax(cfg, W)
    assert s == max(abs(a[0]), abs(a[1]))


def test_spray_directional_speed_values():
    """spectral radius with u = (1, 2), n = (0, 1) -> 2; n = (1, 0) -> 1."""
    cfg = _spray_cfg(1)
    m2 = 0.5
    W = np.array([0.9, 0.7, m2, 0.4, 1.0 * m2, 2.0 * m2])
    F, s = O.phys_flux(cfg, W, 1)
    assert s == 2.0
    assert np.array_equal(F, 2.0 * W)       # flux = M * (u.n) component-wise
    F, s = O.phys_flux(cfg, W, 0)
    assert s == 1.0
    assert np.array_equal(F, 1.0 * W)


def _decimal_spray_step(W, dt, ghost):
    """eq:Essadki transport written in the paper's primitive notation in 50-digit
    decimal: velocity u = (m2 u)/m2, flux of m_k is m_k (u.n), flux of the
    momentum m2 u is m2 u (u.n), sigma = |u.n|, LF,
    eq:VF_scheme with dx = dy = 1.  ghost(i, j) gives out-of-range states."""
    getcontext().prec = 50
    D = Decimal
    ny, nx, _ = W.shape

    def cell(i, j):
        if 0 <= i < nx and 0 <= j < ny:
            return [D(float(x)) for x in W[j, i]]
        return [D(float(x)) for x in ghost(i, j)]

    def fn(w, nxn, nyn):
        m2 = w[2]
        ux, uy = w[4] / m2, w[5] / m2
        un = ux * nxn + uy * nyn
        return [w[0] * un, w[1] * un, m2 * un, w[3] * un, m2 * ux * un, m2 * uy * un], abs(un)

    def lf(L, R, nxn, nyn):
        FL, sL = fn(L, nxn, nyn)
        FR, sR = fn(R, nxn, nyn)
        sig = max(sL, sR)
        return [(FL[k] + FR[k]) / 2 - sig / 2 * (R[k] - L[k]) for k in range(6)]

    dtd = D(dt)
    out = np.zeros(W.shape)
    for j in range(ny):
        for i in range(nx):
            C = cell(i, j)
            Fe, Fw = lf(C, cell(i + 1, j), 1, 0), lf(cell(i - 1, j), C, 1, 0)
            Fn, Fs = lf(C, cell(i, j + 1), 0, 1), lf(cell(i, j - 1), C, 0, 1)
            for k in range(6):
                out[j, i, k] = float(C[k] - dtd * (Fe[k] - Fw[k]) - dtd * (Fn[k] - Fs[k]))
    return out


def _wrap(W):
    ny, nx, _ = W.shape
    return lambda i, j: W[j % ny, i % nx]


def test_spray_random_4x5_50_digit():
    """Non-uniform velocity: the oracle's spray step agrees with the 50-digit
    primitive-notation evaluation to rounding (periodic 4x5, dx = dy = 1)."""
    W = inputs.spray_taylor_green(4, 5)
    rng = np.random.default_rng(3)
    W[..., 4] = W[..., 2] * rng.uniform(-1, 1, size=(5, 4))
    W[..., 5] = W[..., 2] * rng.uniform(-1, 1, size=(5, 4))
    cfg = O.Config(nx=4, ny=5, system=O.SPRAY, param=(1.0, 1.0), x1=4.0, y1=5.0)
    out = O.transport_step(cfg, W, 0.125)
    ref = _decimal_spray_step(W, 0.125, _wrap(W))
    scale = np.abs(ref).max(axis=(0, 1))
    assert np.all(np.abs(out - ref) <= 4e-15 * scale)


# --------------------------------------------------------------- spray wall
def _spray_uniform_moving(nx, ny, a, axis):
    m = [0.75, 0.5, 0.375, 0.25]
    st = m + ([a * m[2], 0.0] if axis == 0 else [0.0, a * m[2]])
    return inputs.uniform(nx, ny, st)


@pytest.mark.parametrize("axis", [0, 1])
def test_spray_wall_closed_form(axis):
    """R13 (wall = mirror ghost with the normal momentum negated; spray: m2u at
    an x-wall, m2v at a y-wall).  Uniform moments moving at u.n = a > 0 toward
    the far wall, dyadic data, lambda = 1/2.  By hand from the ghost:
      * near wall (flow leaves it): every component of the wall flux is 0, the
        inner face carries a*W, so W_new = W - lambda a W;
      * far wall (flow enters it): the mass-type fluxes (m0..m3, tangential
        momentum) are 0 and the normal-momentum flux is 2 a^2 m2, the inner face
        carries a*W, so W_new = W + lambda a W except the normal momentum,
        m2 a - lambda a^2 m2;
      * every other cell is unchanged.  Exact in binary64."""
    n = 8
    a = 0.5
    lam = 0.5
    kw = {"bc_x": O.BC_WALL} if axis == 0 else {"bc_y": O.BC_WALL}
    cfg = _spray_cfg(n, **kw)
    W = _spray_uniform_moving(n, n, a, axis)
    out = O.transport_step(cfg, W, lam / n)
    st = W[0, 0]
    near = st - lam * a * st
    far = st + lam * a * st
    nm = 4 + axis
    far[nm] = a * st[2] - lam * a * a * st[2]
    exp = W.copy()
    if axis == 0:
        exp[:, 0] = near
        exp[:, n - 1] = far
    else:
        exp[0, :] = near
        exp[n - 1, :] = far
    assert np.array_equal(out, exp)


def test_spray_wall_zero_mass_flux_and_conservation():
    """R13: with the mirror ghost the LF wall flux of m0..m3 and of the
    tangential momentum is exactly 0 for any state, so with walls on both axes
    sum m_k |K| (k = 0..3) is conserved by transport (S:284 with closed
    boundaries)."""
    n = 32
    cfg = _spray_cfg(n, bc_x=O.BC_WALL, bc_y=O.BC_WALL)
    W = inputs.spray_taylor_green(n, n)
    W[..., 4] += 0.3 * W[..., 2]         # net drift in x and y: the walls must push back
    W[..., 5] -= 0.2 * W[..., 2]
    s0 = _fsum_vars(W)
    scale = np.array([math.fsum(np.abs(W[..., k]).ravel()) for k in range(6)])
    dt = 0.5 / n / O.smax(cfg, W)[0]
    for _ in range(5):
        W = O.transport_step(cfg, W, dt)
    s1 = _fsum_vars(W)
    assert np.all(np.abs(s1[:4] - s0[:4]) <= 1e-12 * scale[:4])
    # the wall pushes on the normal momenta: those sums move
    assert np.all(np.abs(s1[4:] - s0[4:]) > 1e-9 * scale[4:])


# --------------------------------------------------------------- Dirichlet
@pytest.mark.parametrize("a", [(1.0, 0.5), (-1.0, -0.5), (0.5, -1.0)])
def test_dirichlet_3x3_advection_exact_rationals(a):
    """P:397-398 ("the boundary state is prescribed"; R13: constant ghost).  A
    3x3 advection step with the Dirichlet value g = 5/4 on every side, brute
    force in exact rationals with the textbook upwind formula: the inflow
    sides read g, the outflow sides never read the ghost."""
    g = Fraction(5, 4)
    cfg = O.Config(nx=3, ny=3, system=O.ADVECTION, param=a, x1=3.0, y1=3.0,
                   bc_x=O.BC_DIRICHLET, bc_y=O.BC_DIRICHLET, dirichlet=(1.25,))
    u0 = np.array([[3 * j + i + 1 for i in range(3)] for j in range(3)], dtype=float)
    out = O.transport_step(cfg, u0[..., None], 0.5)[..., 0]
    F = Fraction
    u = [[F(3 * j + i + 1) for i in range(3)] for j in range(3)]

    def at(i, j):
        return u[j][i] if 0 <= i < 3 and 0 <= j < 3 else g

    ax, ay, lam = F(a[0]), F(a[1]), F(1, 2)
    exact = []
    for j in range(3):
        row = []
        for i in range(3):
            dxu = at(i, j) - at(i - 1, j) if ax > 0 else at(i + 1, j) - at(i, j)
            dyu = at(i, j) - at(i, j - 1) if ay > 0 else at(i, j + 1) - at(i, j)
            row.append(u[j][i] - lam * ax * dxu - lam * ay * dyu)
        exact.append(row)
    assert [[F(x) for x in r] for r in out.tolist()] == exact


@pytest.mark.parametrize("system", [O.EULER, O.SPRAY])
def test_dirichlet_state_equal_to_interior_is_preserved(system):
    """Constant-state preservation with a Dirichlet frame carrying the
    same state on every side: the boundary faces see (W, W), so every face flux
    equals F(W) and the step leaves W unchanged bitwise.  Any other ghost
    (e.g. one component substituted for another) breaks it."""
    n = 8
    if system == O.EULER:
        st = inputs.primitive_to_conserved(np.array(1.3), np.array(0.4), np.array(-0.2), np.array(0.9))
        cfg = O.Config(nx=n, ny=n, system=O.EULER, param=(G,), bc_x=O.BC_DIRICHLET,
                       bc_y=O.BC_DIRICHLET, dirichlet=tuple(st))
    else:
        st = inputs.spray_taylor_green(7, 5)[2, 3]
        cfg = O.Config(nx=n, ny=n, system=O.SPRAY, param=(1.0, 1.0), bc_x=O.BC_DIRICHLET,
                       bc_y=O.BC_DIRICHLET, dirichlet=tuple(st))
    W = inputs.uniform(n, n, st)
    out = O.transport_step(cfg, W, 1e-3)
    assert np.array_equal(out, W)


def _decimal_euler_step(W, dt, gamma, ghost):
    """eq:VF_scheme + LF in 50-digit decimal in the paper's primitive notation
    (eq:Euler: rho u.n, rho u u.n + p n, rho u.n H; H = E + p/rho,
    E specific; sigma = |u.n| + c), dx = dy = 1; ghost(i, j) for outside cells."""
    getcontext().prec = 50
    D = Decimal
    g = D(gamma)
    ny, nx, _ = W.shape

    def cell(i, j):
        src = W[j, i] if 0 <= i < nx and 0 <= j < ny else ghost(i, j)
        return [D(float(x)) for x in src]

    def fn(w, nxn, nyn):
        rho = w[0]
        u, v, Es = w[1] / rho, w[2] / rho, w[3] / rho
        p = (g - 1) * rho * (Es - (u * u + v * v) / 2)
        c = (g * p / rho).sqrt()
        un = u * nxn + v * nyn
        H = Es + p / rho
        return [rho * un, rho * u * un + p * nxn, rho * v * un + p * nyn, rho * un * H], abs(un) + c

    def lf(L, R, nxn, nyn):
        FL, sL = fn(L, nxn, nyn)
        FR, sR = fn(R, nxn, nyn)
        sig = max(sL, sR)
        return [(FL[k] + FR[k]) / 2 - sig / 2 * (R[k] - L[k]) for k in range(4)]

    dtd = D(dt)
    out = np.zeros(W.shape)
    for j in range(ny):
        for i in range(nx):
            C = cell(i, j)
            Fe, Fw = lf(C, cell(i + 1, j), 1, 0), lf(cell(i - 1, j), C, 1, 0)
            Fn, Fs = lf(C, cell(i, j + 1), 0, 1), lf(cell(i, j - 1), C, 0, 1)
            for k in range(4):
                out[j, i, k] = float(C[k] - dtd * (Fe[k] - Fw[k]) - dtd * (Fn[k] - Fs[k]))
    return out


def test_dirichlet_euler_4x5_50_digit():
    """A random 4x5 Euler grid inside a Dirichlet frame (constant
    ghost state g): the oracle agrees with the 50-digit evaluation whose ghost
    is g on every side (hand-written boundary faces)."""
    W = inputs.euler_random(4, 5, seed=21)
    g = inputs.primitive_to_conserved(np.array(0.8), np.array(0.3), np.array(-0.6), np.array(1.1))
    cfg = O.Config(nx=4, ny=5, system=O.EULER, param=(G,), x1=4.0, y1=5.0,
                   bc_x=O.BC_DIRICHLET, bc_y=O.BC_DIRICHLET, dirichlet=tuple(g))
    out = O.transport_step(cfg, W, 0.05)
    ref = _decimal_euler_step(W, 0.05, G, lambda i, j: g)
    scale = np.abs(ref).max(axis=(0, 1))
    assert np.all(np.abs(out - ref) <= 2e-15 * scale)


def test_wall_euler_4x5_50_digit():
    """R13 Euler wall on both axes: ghost = mirror of the adjacent cell with
    the normal momentum negated, in the 50-digit evaluation."""
    W = inputs.euler_random(4, 5, seed=22)

    def ghost(i, j):
        if i < 0 or i >= 4:
            s = W[j, 0 if i < 0 else 3].copy()
            s[1] = -s[1]
        else:
            s = W[0 if j < 0 else 4, i].copy()
            s[2] = -s[2]
        return s

    cfg = O.Config(nx=4, ny=5, system=O.EULER, param=(G,), x1=4.0, y1=5.0,
                   bc_x=O.BC_WALL, bc_y=O.BC_WALL)
    out = O.transport_step(cfg, W, 0.05)
    ref = _decimal_euler_step(W, 0.05, G, ghost)
    scale = np.abs(ref).max(axis=(0, 1))
    assert np.all(np.abs(out - ref) <= 2e-15 * scale)


def test_spray_dirichlet_and_wall_4x5_50_digit():
    """Spray ghosts in the 50-digit evaluation: Dirichlet in x (constant state
    g), wall in y (mirror, m2v negated; R13)."""
    W = inputs.spray_taylor_green(4, 5)
    rng = np.random.default_rng(4)
    W[..., 4] = W[..., 2] * rng.uniform(-1, 1, size=(5, 4))
    W[..., 5] = W[..., 2] * rng.uniform(-1, 1, size=(5, 4))
    g = inputs.spray_taylor_green(9, 7)[3, 5].copy()
    g[4], g[5] = 0.25 * g[2], -0.5 * g[2]

    def ghost(i, j):
        if i < 0 or i >= 4:
            return g
        s = W[0 if j < 0 else 4, i].copy()
        s[5] = -s[5]
        return s

    cfg = O.Config(nx=4, ny=5, system=O.SPRAY, param=(1.0, 1.0), x1=4.0, y1=5.0,
                   bc_x=O.BC_DIRICHLET, bc_y=O.BC_WALL, dirichlet=tuple(g))
    out = O.transport_step(cfg, W, 0.125)
    ref = _decimal_spray_step(W, 0.125, ghost)
    scale = np.abs(ref).max(axis=(0, 1))
    assert np.all(np.abs(out - ref) <= 4e-15 * scale)

"""Pins of the oracle's transport path (flux, update, CFL reduction) against
what the paper and mathematics fix -- never against the oracle itself.

Each test names the passage it follows (P:L = PAPER.md line, S:L = SPEC.md line,
R<n> = DESIGN.md §3 reading).
"""
import math
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from paper_1701_05431_b200 import inputs

G = 1.4


def euler_cfg(n, **kw):
    return O.Config(nx=n, ny=kw.pop("ny", n), system=O.EULER, param=(G,), **kw)


def adv_cfg(n, a, **kw):
    return O.Config(nx=n, ny=kw.pop("ny", n), system=O.ADVECTION, param=tuple(a), **kw)


# --------------------------------------------------------------------- flux
def test_euler_flux_worked_examples():
    """S:262 / S:366-368: rest state -> (0, 1/gamma, 0, 0), s = c = 1;
    (rho,u,v,p) = (1,1,0,1/gamma) -> (1, 1+1/gamma, 0, H = 3), s = u + c = 2."""
    cfg = euler_cfg(1)
    rest = inputs.primitive_to_conserved(np.array(1.0), np.array(0.0), np.array(0.0), np.array(1 / G))
    F, s = O.phys_flux(cfg, rest, 0)
    assert F[0] == 0.0 and F[2] == 0.0 and F[3] == 0.0
    assert F[1] == pytest.approx(1 / G, rel=4e-16)
    assert s == pytest.approx(1.0, rel=4e-16)
    mov = inputs.primitive_to_conserved(np.array(1.0), np.array(1.0), np.array(0.0), np.array(1 / G))
    F, s = O.phys_flux(cfg, mov, 0)
    assert F[0] == 1.0 and F[2] == 0.0
    assert F[1] == pytest.approx(1 + 1 / G, rel=4e-16)
    assert F[3] == pytest.approx(3.0, rel=1e-15)   # H = E + p/rho = 1/(0.4*1.4) + 0.5 + 1/1.4 = 3
    assert s == pytest.approx(2.0, rel=4e-16)
    # y direction of the same state: u.n = 0 -> (0, 0, p, 0), s = c = 1
    F, s = O.phys_flux(cfg, mov, 1)
    assert F[0] == 0.0 and F[1] == 0.0 and F[3] == 0.0
    assert F[2] == pytest.approx(1 / G, rel=4e-16)
    assert s == pytest.approx(1.0, rel=4e-16)


@pytest.mark.parametrize("system", [O.ADVECTION, O.EULER, O.SPRAY])
def test_lf_consistency_bitwise(system):
    """F~(W, W, n) = F(W).n exactly (the dissipation vanishes)."""
    rng = np.random.default_rng(5)
    if system == O.ADVECTION:
        cfg = adv_cfg(1, (0.7, -1.3))
        states = rng.normal(size=(50, 1))
    elif system == O.EULER:
        cfg = euler_cfg(1)
        states = inputs.euler_random(50, 1, seed=3)[0]
    else:
        cfg = O.Config(nx=1, ny=1, system=O.SPRAY, param=(1.0, 1.0))
        states = inputs.spray_taylor_green(50, 1)[0]
    for W in states:
        for d in (0, 1):
            F, _ = O.phys_flux(cfg, W, d)
            assert np.array_equal(O.lf_flux(cfg, W, W, d), F)


def test_lf_is_upwind_for_advection():
    """Textbook special case (LeVeque, cited P:126): for linear advection the LF
    flux with sigma = |a| IS the upwind flux a*u_upwind."""
    for a in (1.0, -0.5, 2.0, -3.0):
        cfg = adv_cfg(1, (a, a))
        for uL, uR in ((0.25, 0.75), (3.0, -1.0), (1.5, 1.5)):
            up = a * (uL if a > 0 else uR)
            assert O.lf_flux(cfg, [uL], [uR], 0)[0] == up


# ------------------------------------------------------------------- update
def _upwind_step(u, a, lx, ly):
    """First-order upwind scheme (textbook) for u_t + a.grad u = 0, periodic."""
    ax, ay = a
    if ax > 0:
        dxu = u - np.roll(u, 1, axis=1)
    else:
        dxu = np.roll(u, -1, axis=1) - u
    if ay > 0:
        dyu = u - np.roll(u, 1, axis=0)
    else:
        dyu = np.roll(u, -1, axis=0) - u
    return u - lx * ax * dxu - ly * ay * dyu


def test_3x3_advection_exact_rationals():
    """Brute force in exact rational arithmetic on a 3x3 periodic grid
    (SURVEY Appendix A2 setup): a=(1,1/2), dx=dy=1, dt=1/2, u0[j][i] = 3j+i+1.
    All values are dyadic, so the fp64 oracle must reproduce them bitwise."""
    cfg = adv_cfg(3, (1.0, 0.5), x1=3.0, y1=3.0)
    u0 = np.array([[3 * j + i + 1 for i in range(3)] for j in range(3)], dtype=float)
    out = O.transport_step(cfg, u0[..., None], 0.5)[..., 0]
    F = Fraction
    u = [[F(3 * j + i + 1) for i in range(3)] for j in range(3)]
    ax, ay, lam = F(1), F(1, 2), F(1, 2)
    exact = [[u[j][i] - lam * ax * (u[j][i] - u[j][i - 1]) - lam * ay * (u[j][i] - u[j - 1][i])
              for i in range(3)] for j in range(3)]
    assert [[F(x) for x in row] for row in out.tolist()] == exact
    assert out[0].tolist() == [3.5, 3.0, 4.0]
    assert sum(map(sum, exact)) == 45


@pytest.mark.parametrize("a", [(1.0, 0.5), (-1.0, -0.5), (0.5, -1.0), (-0.25, 1.0)])
def test_advection_equals_upwind_bitwise(a):
    """Dyadic data and dyadic lambda: LF == upwind with every op exact (64^2)."""
    n = 64
    cfg = adv_cfg(n, a)
    u0 = inputs.advection_dyadic(n, n, seed=0)
    dt = 0.5 / n
    out = O.transport_step(cfg, u0, dt)[..., 0]
    ref = _upwind_step(u0[..., 0], a, dt * n, dt * n)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("a,shift", [((1.0, 0.0), (0, 1)), ((-1.0, 0.0), (0, -1)),
                                     ((0.0, 1.0), (1, 0)), ((0.0, -1.0), (-1, 0))])
def test_cfl1_exact_translation(a, shift):
    """BASELINE north_star pin: linear advection at CFL=1 (dt = dx) translates
    the data exactly: after 100 steps W = roll(W0, 100).  Needs the directional
    sigma (R2); adaptive mode with C=1 must produce dt = dx exactly."""
    n = 64
    cfg = adv_cfg(n, a)
    u0 = inputs.advection_dyadic(n, n, seed=0)
    res = O.run(cfg, u0, 100, O.ADAPTIVE, 1.0)
    assert np.all(res.dt_log == 1.0 / n)
    expect = np.roll(u0, (100 * shift[0], 100 * shift[1]), axis=(0, 1))
    assert np.array_equal(res.W, expect)
    res2 = O.run(cfg, u0, 100, O.FIXED, 1.0 / n)
    assert np.array_equal(res2.W, expect)


def test_cfl1_diagonal_is_unstable():
    """R4: with a=(1,1) the paper's eq:CFL_cond admits dt = dx, but the unsplit
    2-D scheme is then not positive: the max norm grows (S:319 monotonicity fails)."""
    n = 64
    cfg = adv_cfg(n, (1.0, 1.0))
    u0 = inputs.advection_dyadic(n, n, seed=0)
    res = O.run(cfg, u0, 3, O.ADAPTIVE, 1.0)
    assert np.abs(res.W).max() > 2 * np.abs(u0).max()
    res = O.run(cfg, u0, 50, O.ADAPTIVE, 0.5)      # C = 0.5: monotone
    assert res.W.max() <= u0.max() and res.W.min() >= u0.min()


@pytest.mark.parametrize("system", [O.ADVECTION, O.EULER, O.SPRAY])
def test_constant_state_preserved_bitwise(system):
    """one full step on constant data preserves it exactly (consistency)."""
    n = 16
    if system == O.ADVECTION:
        cfg, st = adv_cfg(n, (0.3, -0.7)), [0.8125]
    elif system == O.EULER:
        cfg = euler_cfg(n)
        st = inputs.primitive_to_conserved(np.array(1.3), np.array(0.4), np.array(-0.2), np.array(0.9))
    else:
        cfg = O.Config(nx=n, ny=n, system=O.SPRAY, param=(1.0, 1.0))
        st = inputs.spray_taylor_green(7, 5)[2, 3]
    W0 = inputs.uniform(n, n, st)
    out = O.transport_step(cfg, W0, 1e-3)
    assert np.array_equal(out, W0)


def _fsum_vars(W):
    return np.array([math.fsum(W[..., k].ravel()) for k in range(W.shape[-1])])


def test_conservation_periodic_euler():
    """periodic, S=0: sum W |K| is invariant to round-off
    (1e-12 relative per step), exact sums via math.fsum."""
    n = 64
    cfg = euler_cfg(n)
    W = inputs.euler_random(n, n, seed=1)
    scale = np.array([math.fsum(np.abs(W[..., k]).ravel()) for k in range(4)])
    for step in range(20):
        s, _ = O.smax(cfg, W)
        dt = 0.45 * (1.0 / n) / s
        W1 = O.transport_step(cfg, W, dt)
        assert np.all(np.abs(_fsum_vars(W1) - _fsum_vars(W)) <= 1e-12 * scale)
        W = W1


def test_conservation_spray_transport():
    n = 32
    cfg = O.Config(nx=n, ny=n, system=O.SPRAY, param=(1.0, 1.0))
    W = inputs.spray_taylor_green(n, n)
    scale = np.array([math.fsum(np.abs(W[..., k]).ravel()) for k in range(6)])
    W1 = O.transport_step(cfg, W, 0.5 / n)
    assert np.all(np.abs(_fsum_vars(W1) - _fsum_vars(W)) <= 1e-12 * scale)


def test_wall_conservation_and_zero_face_flux():
    """R13: wall = mirror ghost with the normal momentum negated.  The LF wall
    flux of mass, tangential momentum and energy is then exactly 0, so with walls
    in x and periodic y, sum(rho) and sum(rho E) are conserved, sum(rho u) is not
    (wall pressure)."""
    cfg = euler_cfg(1)
    rng = np.random.default_rng(9)
    for W in inputs.euler_random(200, 1, seed=4)[0]:
        ghost = W.copy()
        ghost[1] = -ghost[1]
        F = O.lf_flux(cfg, W, ghost, 0)
        assert F[0] == 0.0 and F[2] == 0.0 and F[3] == 0.0
        ghost = W.copy()
        ghost[2] = -ghost[2]
        F = O.lf_flux(cfg, ghost, W, 1)
        assert F[0] == 0.0 and F[1] == 0.0 and F[3] == 0.0
    n = 64
    cfg = euler_cfg(n, bc_x=O.BC_WALL)
    W = inputs.euler_sod_x(n, n)
    res = O.run(cfg, W, 30, O.ADAPTIVE, 0.45)
    s0, s1 = _fsum_vars(W), _fsum_vars(res.W)
    assert abs(s1[0] - s0[0]) <= 1e-12 * abs(s0[0])
    assert abs(s1[3] - s0[3]) <= 1e-12 * abs(s0[3])
    assert abs(s1[1] - s0[1]) > 1e-6            # wall pressure acts on x-momentum
    assert np.all(res.W[..., 2] == 0.0)          # 1-D problem stays 1-D


def test_mirror_and_transpose_symmetry_bitwise():
    """The scheme commutes with the symmetries of the Cartesian mesh: reflection
    i -> nx-1-i with u -> -u, and the transpose x <-> y with (u,v) -> (v,u).
    IEEE negation and commutativity are exact, so this holds bitwise and pins
    direction/index/sign bookkeeping in eq:VF_scheme."""
    n = 24
    cfg = euler_cfg(n)
    W = inputs.euler_random(n, n, seed=7)
    dt = 2e-3
    out = O.transport_step(cfg, W, dt)
    Wm = W[:, ::-1].copy()
    Wm[..., 1] = -Wm[..., 1]
    om = O.transport_step(cfg, Wm, dt)
    exp = out[:, ::-1].copy()
    exp[..., 1] = -exp[..., 1]
    assert np.array_equal(om, exp)
    Wt = W.transpose(1, 0, 2)[..., [0, 2, 1, 3]].copy()
    ot = O.transport_step(cfg, Wt, dt)
    assert np.array_equal(ot, out.transpose(1, 0, 2)[..., [0, 2, 1, 3]])
    # anisotropic mesh: transpose must also swap dx and dy
    cfg2 = O.Config(nx=n, ny=12, system=O.EULER, param=(G,), x1=1.0, y1=0.75)
    W2 = inputs.euler_random(n, 12, seed=8)
    o2 = O.transport_step(cfg2, W2, dt)
    cfg2t = O.Config(nx=12, ny=n, system=O.EULER, param=(G,), x1=0.75, y1=1.0)
    o2t = O.transport_step(cfg2t, W2.transpose(1, 0, 2)[..., [0, 2, 1, 3]].copy(), dt)
    assert np.array_equal(o2t, o2.transpose(1, 0, 2)[..., [0, 2, 1, 3]])


def _decimal_euler_step(W, dt, gamma):
    """eq:VF_scheme + LF flux in 50-digit decimal arithmetic, written in the
    paper's primitive notation (eq:Euler: rho u.n, rho u u.n + p n_x, ...,
    rho u.n H with H = E + p/rho, E specific; lambda = u.n -+ c, c^2 = gamma p/rho)."""
    getcontext().prec = 50
    D = Decimal
    g = D(gamma)
    ny, nx, _ = W.shape
    Wd = [[[D(float(x)) for x in W[j, i]] for i in range(nx)] for j in range(ny)]

    def prim(w):
        rho = w[0]
        u = w[1] / rho
        v = w[2] / rho
        Espec = w[3] / rho
        p = (g - 1) * rho * (Espec - (u * u + v * v) / 2)
        c = (g * p / rho).sqrt()
        return rho, u, v, Espec, p, c

    def fn(w, nxn, nyn):
        rho, u, v, Es, p, c = prim(w)
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
            C = Wd[j][i]
            Fe = lf(C, Wd[j][(i + 1) % nx], 1, 0)
            Fw = lf(Wd[j][i - 1], C, 1, 0)
            Fn = lf(C, Wd[(j + 1) % ny][i], 0, 1)
            Fs = lf(Wd[j - 1][i], C, 0, 1)
            for k in range(4):
                out[j, i, k] = float(C[k] - dtd * (Fe[k] - Fw[k]) - dtd * (Fn[k] - Fs[k]))
    return out


def test_3x3_euler_50_digit():
    """SURVEY Appendix A3 setup: dx=dy=1, dt=1/8, gamma=1.4, periodic 3x3,
    W[j][i] = (1+(3j+i)/8, (i-1)/4, (j-1)/8, 2+(i+2j)/16).  The fp64 oracle must
    agree with a 50-digit evaluation to within rounding (1e-15 relative)."""
    W = np.array([[[1 + (3 * j + i) / 8, (i - 1) / 4, (j - 1) / 8, 2 + (i + 2 * j) / 16]
                   for i in range(3)] for j in range(3)])
    cfg = O.Config(nx=3, ny=3, system=O.EULER, param=(G,), x1=3.0, y1=3.0)
    out = O.transport_step(cfg, W, 0.125)
    ref = _decimal_euler_step(W, 0.125, G)
    scale = np.abs(ref).max(axis=(0, 1))
    assert np.all(np.abs(out - ref) <= 1e-15 * scale)
    # and conservation is exact up to rounding
    assert abs(math.fsum(out[..., 0].ravel()) - 13.5) < 1e-14


def test_random_euler_50_digit_4x5():
    """Same 50-digit brute force on a random, anisotropic 4x5 grid (dx != dy)."""
    W = inputs.euler_random(4, 5, seed=11)
    cfg = O.Config(nx=4, ny=5, system=O.EULER, param=(G,), x1=4.0, y1=5.0)
    dt = 0.05
    out = O.transport_step(cfg, W, dt)
    ref = _decimal_euler_step(W, dt, G)
    scale = np.abs(ref).max(axis=(0, 1))
    assert np.all(np.abs(out - ref) <= 2e-15 * scale)


# ----------------------------------------------------------------- CFL / dt
def test_smax_bell_and_advection():
    """S:272 (bell reading R22): s_max = |u| + c = 1 + 1 = 2 where rho = 1; the
    fp64 value is 2 up to a few ulps.  Advection: smax = max(|ax|,|ay|) exactly."""
    n = 128
    s, arg = O.smax(euler_cfg(n), inputs.euler_bell(n, n))
    assert s == pytest.approx(2.0, abs=1e-14)
    s, _ = O.smax(adv_cfg(8, (0.25, -0.75)), inputs.advection_dyadic(8, 8))
    assert s == 0.75


def test_smax_argmax_lowest_index_and_fixed_dt_check():
    """eq:CFL_cond: max over cells; fixed dt is checked at the
    beginning of each iteration and a violation leaves W^k unchanged (R14);
    argmax = lowest j*nx+i among ties (DESIGN §3.1 step 1)."""
    n = 8
    cfg = euler_cfg(n)
    base = inputs.primitive_to_conserved(np.array(1.0), np.array(0.0), np.array(0.0), np.array(1 / G))
    W = inputs.uniform(n, n, base)
    fast = inputs.primitive_to_conserved(np.array(1.0), np.array(3.0), np.array(0.0), np.array(1 / G))
    W[5, 2] = fast
    W[6, 1] = fast
    s, arg = O.smax(cfg, W)
    assert arg == 5 * n + 2
    assert s == pytest.approx(4.0, rel=1e-15)
    dt_ok = (1.0 / n) / 4.0 * 0.999
    O.run(cfg, W, 1, O.FIXED, dt_ok)
    res = O.run(cfg, W, 3, O.FIXED, (1.0 / n) / 4.0 * 1.01, raise_on_error=False)
    assert res.status == O.E_CFL and res.steps_done == 0 and res.err_cell == 5 * n + 2
    assert np.array_equal(res.W, W)


def test_cfl_c1_euler_blows_up_c045_stable():
    """R4: Euler bell at 128^2 with dt = 1.0*h/smax loses positivity within ~20
    steps, with C = 0.45 it runs 100 steps with rho, p > 0."""
    n = 128
    cfg = euler_cfg(n)
    W0 = inputs.euler_bell(n, n)
    res = O.run(cfg, W0, 40, O.ADAPTIVE, 1.0, raise_on_error=False)
    assert res.status == O.E_NONFINITE and res.steps_done < 40
    res = O.run(cfg, W0, 100, O.ADAPTIVE, 0.45)
    assert res.W[..., 0].min() > 0.99 and res.W[..., 0].max() < 2.0 + 1e-12


def test_first_order_convergence_bell():
    """fig:Convergence: the scheme is first order, L1 slopes ~0.95.
    Bell reading (R22), T = 0.1, fixed dt = 0.45 h/2 adjusted to hit T exactly,
    compared with eq:LCAnalytic; slopes over 64 -> 128 -> 256 in [0.85, 1.05]."""
    errs = []
    T = 0.1
    for n in (64, 128, 256):
        cfg = euler_cfg(n)
        nsteps = int(math.ceil(T / (0.45 / n / 2.0)))
        dt = T / nsteps
        res = O.run(cfg, inputs.euler_bell(n, n), nsteps, O.FIXED, dt)
        ex = inputs.euler_bell_exact(n, n, T)
        errs.append(np.abs(res.W[..., 0] - ex[..., 0]).sum() / n / n)
    slopes = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert all(0.85 <= s <= 1.05 for s in slopes), slopes

"""Pins of the oracle's spray source path (NDF reconstruction + eq:SourceTerm)
against closed forms and independent quadrature."""
import math

import numpy as np
import pytest
from scipy import integrate

import oracle as O
from paper_1701_05431_b200 import inputs


def test_gl24_exactness():
    """24-node Gauss-Legendre integrates t^k exactly on [0,1] for k <= 47."""
    t, w = O.gl24()
    assert np.all(np.diff(t) > 0) and t[0] > 0 and t[-1] < 1
    for k in range(48):
        assert math.fsum(w * t ** k) == pytest.approx(1.0 / (k + 1), rel=5e-15, abs=0)
    xg, wg = np.polynomial.legendre.leggauss(24)
    assert np.allclose(t, (xg + 1) / 2, rtol=0, atol=2e-16)
    assert np.allclose(w, wg / 2, rtol=2e-13, atol=0)  # numpy weights carry ~1e-13 error


def test_uniform_ndf_reconstruction():
    """uniform NDF n = 1 on [0,1]: m_k/2 = 2/(k+2) = (1, 2/3, 1/2, 2/5)
    -> lambda = 0, n(0) = 1, m_-1/2 = int S^-1/2 dS = 2."""
    lam, n0, mmh, it = O.reconstruct([1.0, 2 / 3, 0.5, 0.4])
    assert np.all(np.abs(lam) < 1e-12)
    assert n0 == pytest.approx(1.0, abs=1e-12)
    assert mmh == pytest.approx(2.0, abs=1e-12)
    assert it == 0  # lambda0 = -ln(1) = 0 already solves the system


def _closed_form_moments_exp_sqrt():
    """n(S) = exp(-sqrt S) (lambda = (0,1,0,0)): m_k/2 = 2 int_0^1 t^{k+1} e^{-t} dt
    = 2 (k+1)! (1 - e^{-1} sum_{i<=k+1} 1/i!)  (lower incomplete gamma)."""
    m = []
    for k in range(4):
        s = sum(1.0 / math.factorial(i) for i in range(k + 2))
        m.append(2.0 * math.factorial(k + 1) * (1.0 - math.exp(-1.0) * s))
    return np.array(m)


def test_exp_sqrt_ndf_recovered():
    """moments of n = exp(-S^1/2) -> lambda recovered to 1e-8;
    closed-form check of the printed values (0.52848224, 0.32120559, 0.22785788, 0.17567265)."""
    m = _closed_form_moments_exp_sqrt()
    assert np.allclose(m, [0.52848224, 0.32120559, 0.22785788, 0.17567265], atol=5e-9)
    lam, n0, mmh, it = O.reconstruct(m)
    assert np.allclose(lam, [0.0, 1.0, 0.0, 0.0], atol=1e-8)
    assert n0 == pytest.approx(1.0, abs=1e-8)
    assert mmh == pytest.approx(2.0 * (1.0 - math.exp(-1.0)), rel=1e-10)
    assert 1 <= it <= 50


def _quad_moments(lam, ks=range(-1, 4)):
    """Independent adaptive quadrature (scipy.integrate.quad) of
    m_k/2 = int_0^1 S^{k/2} exp(-(l0 + l1 S^1/2 + l2 S + l3 S^3/2)) dS, via S = t^2."""
    out = []
    for k in ks:
        f = lambda t, k=k: 2.0 * t ** (k + 1) * math.exp(-(lam[0] + lam[1] * t + lam[2] * t * t + lam[3] * t ** 3))
        out.append(integrate.quad(f, 0.0, 1.0, epsabs=0, epsrel=2e-14, limit=200)[0])
    return np.array(out)


def test_round_trip_random_realizable():
    """forward/inverse round trip on 50 realizable moment sets
    (generated from random lambda by independent quadrature) holds to 1e-8."""
    rng = np.random.default_rng(2024)
    worst = 0.0
    for _ in range(50):
        lam_true = np.array([rng.uniform(-1, 1), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-1, 1)])
        mm = _quad_moments(lam_true)
        lam, n0, mmh, it = O.reconstruct(mm[1:])
        assert n0 == pytest.approx(math.exp(-lam_true[0]), rel=1e-8)
        assert mmh == pytest.approx(mm[0], rel=1e-8)
        back = _quad_moments(lam)
        worst = max(worst, np.max(np.abs(back - mm) / mm))
    assert worst <= 1e-8


def test_non_realizable_rejected():
    with pytest.raises(O.OracleError) as e:
        O.reconstruct([1.0, 2.0, 0.5, 0.4])   # m1^2 > m0 m2: no positive measure on [0,1]
    assert e.value.code == O.E_RECON
    with pytest.raises(O.OracleError):
        O.reconstruct([1.0, -0.5, 0.5, 0.4])


def _spray_cfg(n, K=1.0, theta=1.0):
    return O.Config(nx=n, ny=n, system=O.SPRAY, param=(K, theta))


def test_source_uniform_ndf_closed_form():
    """uniform NDF, K=1, theta -> infinity: S = (-1, -1, -1, -1, -u, -v)
    (n(0)=1, m_-1/2=2, m0=1, m1=2/3)."""
    n = 4
    cfg = _spray_cfg(n, K=1.0, theta=1e300)
    u, v = 0.3, -0.6
    st = [1.0, 2 / 3, 0.5, 0.4, 0.5 * u, 0.5 * v]
    W = inputs.uniform(n, n, st)
    dt = 1e-3
    out, it = O.source_step(cfg, W, dt)
    S = np.array([-1.0, -1.0, -1.0, -1.0, -u, -v])
    assert np.allclose(out, np.array(st) + dt * S, rtol=0, atol=1e-14)


def test_source_drag_only_closed_form():
    """K = 0 leaves only drag, d(m2 u)/dt = m0 (u_g - u)/theta, whose exact
    solution is u(t) = u_g + (u0 - u_g) exp(-m0 t/(m2 theta)).  One forward-Euler
    step (eq:SourceTerm) has local error O(dt^2): halving dt quarters it."""
    n = 4
    theta = 0.7
    cfg = _spray_cfg(n, K=0.0, theta=theta)
    m = [0.9, 0.55, 0.4, 0.3]
    u0, v0 = 0.25, -0.4
    W = inputs.uniform(n, n, m + [m[2] * u0, m[2] * v0])
    x = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(x, x, indexing="xy")
    ugx, ugy = inputs.taylor_green(X, Y)
    errs = []
    for dt in (1e-2, 5e-3, 2.5e-3):
        out, _ = O.source_step(cfg, W, dt)
        assert np.array_equal(out[..., :4], W[..., :4])            # K=0: moments frozen
        ex_u = ugx + (u0 - ugx) * np.exp(-m[0] * dt / (m[2] * theta))
        ex_v = ugy + (v0 - ugy) * np.exp(-m[0] * dt / (m[2] * theta))
        errs.append(max(np.abs(out[..., 4] / m[2] - ex_u).max(), np.abs(out[..., 5] / m[2] - ex_v).max()))
    assert errs[0] / errs[1] == pytest.approx(4.0, rel=0.02)
    assert errs[1] / errs[2] == pytest.approx(4.0, rel=0.02)


def test_evaporation_of_moments_matches_reconstruction_values():
    """Source moment rows of eq:Essadki with drag off: the (n(0), m_-1/2) used by
    the step equal the reconstruction of the cell's moments."""
    cfg = _spray_cfg(2, K=0.8, theta=1e300)
    W = inputs.spray_taylor_green(2, 2)
    dt = 1e-3
    out, _ = O.source_step(cfg, W, dt)
    for j in range(2):
        for i in range(2):
            m = W[j, i, :4]
            lam, n0, mmh, _ = O.reconstruct(m)
            expect = m + dt * np.array([-0.8 * n0, -0.4 * mmh, -0.8 * m[0], -1.2 * m[1]])
            assert np.allclose(out[j, i, :4], expect, rtol=1e-15, atol=0)


def _realizable(W):
    m0, m1, m2, m3 = (W[..., k] for k in range(4))
    return bool(np.all(m0 > 0) and np.all(m1 > 0) and np.all(m2 > 0) and np.all(m3 > 0)
                and np.all(m3 <= m2) and np.all(m2 <= m1) and np.all(m1 <= m0)
                and np.all(m1 * m1 <= m0 * m2) and np.all(m2 * m2 <= m1 * m3))


def test_spray_run_stays_realizable():
    """S:353-356, S:433, P:1007-1008 ("the set of moments is everywhere realizable"):
    Taylor-Green spray IC (R16), fixed dt = 0.5 h/smax(W0) (R17), 20 steps."""
    n = 32
    cfg = _spray_cfg(n)
    W0 = inputs.spray_taylor_green(n, n)
    assert _realizable(W0)
    s0, _ = O.smax(cfg, W0)
    dt = 0.5 * (1.0 / n) / s0
    t_sum = 0
    W = W0
    for _ in range(20):
        W = O.run(cfg, W, 1, O.FIXED, dt).W
        assert _realizable(W)
    assert W[..., 0].sum() < W0[..., 0].sum()   # evaporation removes droplets


def test_spray_guard_closed_form_boundary():
    """S:440 (SPEC "Design decisions"): reject a run whose dt has
    dt*K > 0.1*min over cells of m3/m1, erroring at startup with the state
    untouched.  Uniform moments with m3/m1 = 1/2 and K = 1 put the boundary at
    dt = 0.1*0.5 = 0.05 (0.1*0.5 is fl(0.1)/2 = fl(0.05): halving is exact):
    dt = 0.05 runs, the next double above is rejected; the argmin cell is the
    lowest-index cell with the smallest ratio."""
    n = 4
    cfg = _spray_cfg(n)
    st = [0.75, 0.5, 0.375, 0.25, 0.0, 0.0]
    W = inputs.uniform(n, n, st)
    O.spray_guard(cfg, W, 0.05)
    with pytest.raises(O.OracleError) as e:
        O.spray_guard(cfg, W, np.nextafter(0.05, 1.0))
    assert e.value.code == O.E_ARG and e.value.value == 0.5 and e.value.cell == 0
    W2 = W.copy()
    W2[2, 1, 3] = 0.125          # m3/m1 = 1/4 at cell (i=1, j=2): boundary dt = 0.025
    W2[3, 2, 3] = 0.125
    with pytest.raises(O.OracleError) as e:
        O.spray_guard(cfg, W2, 0.03)
    assert e.value.cell == 2 * n + 1 and e.value.value == 0.25
    # through the time loop: E_ARG at startup, W^0 returned, no step taken
    res = O.run(cfg, W2, 3, O.FIXED, 0.03, raise_on_error=False)
    assert res.status == O.E_ARG and res.steps_done == 0 and np.array_equal(res.W, W2)
    # K scales the boundary: K = 2 halves it
    cfg2 = _spray_cfg(n, K=2.0)
    O.spray_guard(cfg2, W, 0.025)
    with pytest.raises(O.OracleError):
        O.spray_guard(cfg2, W, 0.026)


def test_spray_guard_adaptive_first_dt_and_r16_ic():
    """The guard applies to the first dt of an adaptive run too; the R16 IC at
    64^2 with the paper's fixed dt passes it (7.8e-3 <= 5.0e-2)."""
    n = 64
    W0 = inputs.spray_taylor_green(n, n)
    cfg = _spray_cfg(n)
    s0, _ = O.smax(cfg, W0)
    dt = 0.5 * (1.0 / n) / s0
    rmin = float(np.min(W0[..., 3] / W0[..., 1]))
    assert dt * 1.0 <= 0.1 * rmin
    O.run(cfg, W0, 1, O.FIXED, dt)
    big_k = _spray_cfg(n, K=0.2 * rmin / dt)      # dt*K = 2 * 0.1 rmin
    res = O.run(big_k, W0, 2, O.ADAPTIVE, 0.5, raise_on_error=False)
    assert res.status == O.E_ARG and res.steps_done == 0


def _decimal_newton_iterations(m):
    """S:401-409 + R19 in 40-digit decimal, step by step: lambda = (-ln m0, 0, 0, 0);
    mu_j = 2 sum_q w_q t_q^j exp(-P(t_q)) on GL-24 mapped to [0,1] (numpy
    leggauss nodes); while max_k |mu_{k+1} - m_k|/m_k > 1e-10: solve
    H d = mu_{1..4} - m (H_kl = mu_{k+l+1}, Gaussian elimination), backtrack
    alpha = 1, 1/2, ... until the residual decreases.  Returns the count."""
    from decimal import Decimal as D, getcontext
    getcontext().prec = 40
    xg, wg = np.polynomial.legendre.leggauss(24)
    t = [(D(float(x)) + 1) / 2 for x in xg]
    w = [D(float(x)) / 2 for x in wg]
    md = [D(float(x)) for x in m]

    def mom(lam):
        mu = [D(0)] * 8
        for q in range(24):
            e = (-(lam[0] + t[q] * (lam[1] + t[q] * (lam[2] + t[q] * lam[3])))).exp()
            for j in range(8):
                mu[j] += 2 * w[q] * t[q] ** j * e
        return mu

    def res(mu):
        return max(abs(mu[k + 1] - md[k]) / md[k] for k in range(4))

    lam = [-md[0].ln(), D(0), D(0), D(0)]
    mu = mom(lam)
    r0 = res(mu)
    it = 0
    while r0 > D("1e-10"):
        A = [[mu[k + l + 1] for l in range(4)] + [mu[k + 1] - md[k]] for k in range(4)]
        for c in range(4):
            for r in range(c + 1, 4):
                f = A[r][c] / A[c][c]
                A[r] = [A[r][k] - f * A[c][k] for k in range(5)]
        d = [D(0)] * 4
        for c in range(3, -1, -1):
            d[c] = (A[c][4] - sum(A[c][k] * d[k] for k in range(c + 1, 4))) / A[c][c]
        a = D(1)
        for _ in range(31):
            lt = [lam[k] + a * d[k] for k in range(4)]
            mt = mom(lt)
            rt = res(mt)
            if rt < r0:
                lam, mu, r0 = lt, mt, rt
                break
            a /= 2
        it += 1
        assert it <= 50
    return it


def test_newton_iteration_counts_match_decimal_algorithm():
    """S:405's stopping rule (max relative moment residual <= 1e-10, residual of
    moment k relative to m_k) and the backtracking of R19: on 50 random
    realizable sets (SURVEY A6 distribution) the oracle takes exactly as many
    Newton iterations as the same algorithm run in 40-digit decimal."""
    rng = np.random.default_rng(2024)
    for _ in range(50):
        lam_true = np.array([rng.uniform(-1, 1), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-1, 1)])
        mm = _quad_moments(lam_true)
        assert O.reconstruct(mm[1:])[3] == _decimal_newton_iterations(mm[1:])


def test_polished_reconstruction_reaches_the_root():
    """R19: after convergence one undamped Newton step polishes lambda, so
    (n(0), m_-1/2) reach the GL-24 root to conditioning x rounding -- within
    1e-11 (n0) and 1e-12 (m_-1/2) of the true values exp(-lambda0_true) and the
    adaptive-quadrature m_-1/2 (stopping at 1e-10 alone leaves up to ~5e-9)."""
    rng = np.random.default_rng(2024)
    for _ in range(50):
        lam_true = np.array([rng.uniform(-1, 1), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-1, 1)])
        mm = _quad_moments(lam_true)
        lam, n0, mmh, _ = O.reconstruct(mm[1:])
        assert n0 == pytest.approx(math.exp(-lam_true[0]), rel=1e-11, abs=0)
        assert mmh == pytest.approx(mm[0], rel=1e-12, abs=0)

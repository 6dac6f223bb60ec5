"""Checks of the seeded input generators (shared by oracle tests and the GPU path)."""
import numpy as np
import pytest

from paper_1701_05431_b200 import inputs

G = 1.4


def _prim(W):
    rho = W[..., 0]
    u = W[..., 1] / rho
    v = W[..., 2] / rho
    p = (G - 1) * (W[..., 3] - 0.5 * rho * (u * u + v * v))
    return rho, u, v, p


def test_vortex_isentropic_and_centre():
    """eq:isentropy: p/rho^gamma = 1/gamma everywhere (1e-12);
    S:386-388: centre rho = 0.8^2.5, far corner ~ (1, 1, 1, 1/gamma)."""
    n = 64
    W = inputs.euler_vortex(n + 1, n + 1)   # odd size: a cell centre sits at (0.5, 0.5)
    rho, u, v, p = _prim(W)
    assert np.allclose(p / rho ** G, 1 / G, rtol=1e-12, atol=0)
    c = n // 2
    assert rho[c, c] == pytest.approx(0.8 ** 2.5, rel=1e-12)
    assert rho[0, 0] == pytest.approx(1.0, abs=1e-9) and u[0, 0] == pytest.approx(1.0, abs=1e-9)


def test_bell_range_and_printed_cosine_degeneracy():
    """R22: the bell reading stays in [1, 2] (c <= 1); the printed formula reaches rho ~ 0."""
    n = 1024
    W = inputs.euler_bell(n, n, rows=(400, 624))
    assert W[..., 0].min() >= 1.0 and W[..., 0].max() <= 2.0
    Wp = inputs.euler_cosine_printed(n, n, rows=(400, 624))
    assert Wp[..., 0].min() < 1e-3


def test_rows_band_matches_full_grid():
    full = inputs.euler_random(40, 600, seed=1)
    band = inputs.euler_random(40, 600, seed=1, rows=(250, 530))
    assert np.array_equal(full[250:530], band)
    assert np.array_equal(inputs.euler_lax_liu3(32, 32)[5:9], inputs.euler_lax_liu3(32, 32, rows=(5, 9)))
    assert np.array_equal(inputs.advection_dyadic(16, 16, seed=0)[3:7], inputs.advection_dyadic(16, 16, seed=0, rows=(3, 7)))


def test_spray_ic_realizable():
    W = inputs.spray_taylor_green(48, 48)
    m0, m1, m2, m3 = (W[..., k] for k in range(4))
    assert np.all(m3 < m2) and np.all(m2 < m1) and np.all(m1 < m0)
    assert np.all(m1 * m1 < m0 * m2) and np.all(m2 * m2 < m1 * m3)


def test_tfv1_roundtrip(tmp_path):
    """SPEC's solution file: magic, LE int64 Nx Ny nVar, f64 t, data."""
    from paper_1701_05431_b200 import output
    W = inputs.euler_random(7, 5, seed=2)
    p = tmp_path / "s.tfv1"
    output.write_tfv1(str(p), W, 0.125)
    raw = p.read_bytes()
    assert raw[:4] == b"TFV1" and len(raw) == 4 + 32 + W.size * 8
    W2, t = output.read_tfv1(str(p))
    assert t == 0.125 and np.array_equal(W2, W)

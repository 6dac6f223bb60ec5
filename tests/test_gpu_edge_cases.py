"""GPU parity on the method's edge cases, through the C ABI, against the oracle:
the S:440 startup guard, a non-realizable cell (E_RECON), cold-start Newton on
random realizable moment sets (backtracking, several iterations), mixed
fixed/adaptive time stepping, full-size c3 on random data with every strip
seam sampled, and the launch geometry the library derives from the device."""
import numpy as np
import pytest

import oracle as O
from paper_1701_05431_b200 import fv2d, inputs

pytestmark = pytest.mark.gpu
G = 1.4


def relerr(a, b):
    e = 0.0
    for v in range(b.shape[-1]):
        nb = np.abs(b[..., v]).max()
        d = np.abs(a[..., v] - b[..., v]).max()
        if nb == 0:
            assert d == 0
        else:
            e = max(e, d / nb)
    return e


def solver_for(cfg: O.Config, **kw):
    return fv2d.Solver(cfg.nx, cfg.ny, cfg.system, x0=cfg.x0, x1=cfg.x1, y0=cfg.y0, y1=cfg.y1,
                       param=cfg.param, bc_x=cfg.bc_x, bc_y=cfg.bc_y, dirichlet=cfg.dirichlet, **kw)


def spray_case(n, K=1.0):
    cfg = O.Config(nx=n, ny=n, system=O.SPRAY, param=(K, 1.0))
    W0 = inputs.spray_taylor_green(n, n)
    s0, _ = O.smax(cfg, W0)
    return cfg, W0, 0.5 * (1.0 / n) / s0


# ------------------------------------------------------------ S:440 guard
@pytest.mark.parametrize("flags", [0, fv2d.FLAG_NAIVE])
def test_spray_guard_fixed_dt(flags):
    """dt*K > 0.1*min(m3/m1) is rejected at startup with E_ARG, the
    argmin cell and value of the oracle, W^0 untouched and no step taken; a
    K at the boundary runs and matches the oracle."""
    cfg, W0, dt = spray_case(48)
    rmin = float(np.min(W0[..., 3] / W0[..., 1]))
    K_bad = 0.2 * rmin / dt                     # dt*K = 2 x 0.1*rmin
    bad = O.Config(nx=48, ny=48, system=O.SPRAY, param=(K_bad, 1.0))
    ref = O.run(bad, W0, 3, O.FIXED, dt, raise_on_error=False)
    assert ref.status == O.E_ARG and ref.steps_done == 0
    with solver_for(bad, flags=flags) as s:
        s.set_state(W0)
        with pytest.raises(fv2d.FV2DError) as e:
            s.step(dt, 3)
        assert e.value.code == fv2d.E_ARG and e.value.cell == ref.err_cell
        assert W0.reshape(-1, 6)[ref.err_cell, 3] / W0.reshape(-1, 6)[ref.err_cell, 1] == rmin
        assert e.value.value == rmin
        assert np.array_equal(s.get_state(), W0)
        assert s.stats()["steps"] == 0
    # the boundary itself: dt*K == 0.1*rmin exactly is accepted by both sides
    K_edge = (0.1 * rmin) / dt
    while dt * K_edge > 0.1 * rmin:
        K_edge = np.nextafter(K_edge, 0.0)
    edge = O.Config(nx=48, ny=48, system=O.SPRAY, param=(K_edge, 1.0))
    ref = O.run(edge, W0, 2, O.FIXED, dt)
    with solver_for(edge, flags=flags) as s:
        s.set_state(W0)
        s.step(dt, 2)
        W = s.get_state()
    assert relerr(W, ref.W) <= 1e-12


def test_spray_guard_adaptive_and_step_host():
    """The guard checks the first adaptive dt too, and fv2d_step_host (which
    starts every call from a host W^0) returns E_ARG with W^0 in the output."""
    cfg, W0, dt = spray_case(40)
    s0, _ = O.smax(cfg, W0)
    dt0 = (0.5 * (1.0 / 40)) / s0
    rmin = float(np.min(W0[..., 3] / W0[..., 1]))
    bad = O.Config(nx=40, ny=40, system=O.SPRAY, param=(0.3 * rmin / dt0, 1.0))
    ref = O.run(bad, W0, 2, O.ADAPTIVE, 0.5, raise_on_error=False)
    assert ref.status == O.E_ARG
    with solver_for(bad) as s:
        s.set_state(W0)
        with pytest.raises(fv2d.FV2DError) as e:
            s.step_adaptive(0.5, 2)
        assert e.value.code == fv2d.E_ARG and e.value.cell == ref.err_cell
        out = np.full_like(W0, np.nan)
        with pytest.raises(fv2d.FV2DError) as e:
            s.step_host(W0, out, dt0, 2)
        assert e.value.code == fv2d.E_ARG
        assert np.array_equal(out, W0)


def test_spray_guard_after_cfl_precedence():
    """Oracle order (or_run): a fixed-dt CFL violation is reported
    before the guard, at step 0, with W^0 readable."""
    cfg, W0, dt = spray_case(32)
    big = 6.0 * dt                              # dt*smax = 3 hmin
    rmin = float(np.min(W0[..., 3] / W0[..., 1]))
    both = O.Config(nx=32, ny=32, system=O.SPRAY, param=(rmin / big, 1.0))
    ref = O.run(both, W0, 1, O.FIXED, big, raise_on_error=False)
    assert ref.status == O.E_CFL
    with solver_for(both) as s:
        s.set_state(W0)
        s.step(big, 1)
        with pytest.raises(fv2d.FV2DError) as e:
            s.synchronize()
        assert e.value.code == fv2d.E_CFL and e.value.step == 0
        assert np.array_equal(s.get_state(raise_on_error=False), W0)


# ------------------------------------------------------------ E_RECON
@pytest.mark.parametrize("flags", [0, fv2d.FLAG_NAIVE])
def test_nonrealizable_cell_latches_recon(flags):
    """A cell whose moments violate m1^2 <= m0 m2 (no positive measure, S:402
    precondition): the source step's reconstruction fails there; both sides
    report E_RECON at step 0 with the same (lowest) cell, and W^0 stays
    readable (ping-pong, R14)."""
    cfg, W0, dt = spray_case(64)
    W0 = W0.copy()
    for (j, i) in ((41, 9), (12, 50)):
        W0[j, i, 1] = 1.5 * np.sqrt(W0[j, i, 0] * W0[j, i, 2])
    ref = O.run(cfg, W0, 3, O.FIXED, dt, raise_on_error=False)
    assert ref.status == O.E_RECON and ref.steps_done == 0
    with solver_for(cfg, flags=flags) as s:
        s.set_state(W0)
        s.step(dt, 3)
        with pytest.raises(fv2d.FV2DError) as e:
            s.synchronize()
        assert e.value.code == fv2d.E_RECON and e.value.step == 0
        assert e.value.cell == ref.err_cell
        assert np.array_equal(s.get_state(raise_on_error=False), W0)


# ------------------------------------------- Newton on random moment sets
def _moments_from_lambda(lam):
    """m_k = 2 int_0^1 t^{k+1} exp(-P(t)) dt, k = 0..3, by GL-24 (numpy
    leggauss): the R16 recipe with a general lambda (input generation only)."""
    xg, wg = np.polynomial.legendre.leggauss(24)
    t = (xg + 1.0) / 2.0
    w = wg / 2.0
    P = lam[..., 0:1] + t * (lam[..., 1:2] + t * (lam[..., 2:3] + t * lam[..., 3:4]))
    e = np.exp(-P)
    return np.stack([2.0 * np.sum(w * t ** (k + 1) * e, axis=-1) for k in range(4)], axis=-1)


def test_apply_source_on_random_realizable_sets():
    """50 random realizable moment sets (lambda uniform in
    [-1,1]x[-2,2]^2x[-1,1], 4-8 cold-start Newton iterations, backtracking)
    through fv2d_apply_source (cold start after set_state) against the oracle's
    source step at <= 1e-12 -- exercises the full moment evaluation, the
    incremental trial points and their fallback, and the polishing step."""
    rng = np.random.default_rng(77)
    nx, ny = 10, 5
    lam = np.stack([rng.uniform(-1, 1, (ny, nx)), rng.uniform(-2, 2, (ny, nx)),
                    rng.uniform(-2, 2, (ny, nx)), rng.uniform(-1, 1, (ny, nx))], axis=-1)
    W0 = np.empty((ny, nx, 6))
    W0[..., :4] = _moments_from_lambda(lam)
    W0[..., 4] = W0[..., 2] * rng.uniform(-1, 1, (ny, nx))
    W0[..., 5] = W0[..., 2] * rng.uniform(-1, 1, (ny, nx))
    cfg = O.Config(nx=nx, ny=ny, system=O.SPRAY, param=(1.0, 1.0), x1=2.0)
    for dt in (1e-3, 3e-2):
        ref, iters = O.source_step(cfg, W0, dt)
        assert iters >= 4 * nx * ny
        with solver_for(cfg) as s:
            s.set_state(W0)
            s.apply_source(dt)
            W = s.get_state()
        assert relerr(W, ref) <= 1e-12
        # per cell, the reconstruction's outputs: the source rows relative to dt*S
        dS = np.abs((W - W0)[..., :4] - (ref - W0)[..., :4]) / np.abs((ref - W0)[..., :4])
        assert dS.max() <= 1e-10


# ------------------------------------------------ mixed fixed / adaptive dt
def test_mixed_fixed_and_adaptive_dt_log():
    """adaptive(C1) -> fixed(dt) -> adaptive(C2): every adaptive step uses
    dt_n = (C*hmin)/smax(W^n) of its own C and of the current state (the
    fixed steps must not leave a stale dt behind); dt logs ==, state bitwise."""
    n = 96
    cfg = O.Config(nx=n, ny=n, system=O.EULER, param=(G,))
    W0 = inputs.euler_lax_liu3(n, n)
    r1 = O.run(cfg, W0, 3, O.ADAPTIVE, 0.45)
    fixed = 0.3 * (1.0 / n) / 2.6
    r2 = O.run(cfg, r1.W, 2, O.FIXED, fixed)
    r3 = O.run(cfg, r2.W, 3, O.ADAPTIVE, 0.3)
    r4 = O.run(cfg, r3.W, 2, O.ADAPTIVE, 0.45)
    with solver_for(cfg) as s:
        s.set_state(W0)
        l1 = s.step_adaptive(0.45, 3)
        s.step(fixed, 2)
        l3 = s.step_adaptive(0.3, 3)
        l4 = s.step_adaptive(0.45, 2)
        W = s.get_state()
    assert np.array_equal(l1, r1.dt_log)
    assert np.array_equal(l3, r3.dt_log)
    assert np.array_equal(l4, r4.dt_log)
    assert np.array_equal(W, r4.W)


# ------------------------------------------------------------ ABI hygiene
def test_get_state_rejects_a_wrong_buffer():
    cfg = O.Config(nx=16, ny=8, system=O.EULER, param=(G,))
    with solver_for(cfg) as s:
        s.set_state(inputs.euler_random(16, 8, seed=3))
        for bad in (np.empty((8, 16, 3)), np.empty((8, 16, 4), dtype=np.float32),
                    np.empty((16, 8, 4)).transpose(1, 0, 2)):
            with pytest.raises(ValueError):
                s.get_state(out=bad)


def test_launch_geometry_from_the_device():
    """The strip-height cost model uses the device's SM count and the step
    kernel's occupancy (not constants): 148 SMs on a B200, and the wave size is
    SMs x resident CTAs per SM of the launched kernel."""
    import torch
    props = torch.cuda.get_device_properties(0)
    for system, param in ((O.EULER, (G,)), (O.SPRAY, (1.0, 1.0)), (O.ADVECTION, (1.0, 0.5))):
        cfg = O.Config(nx=2048, ny=2048, system=system, param=param)
        with solver_for(cfg) as s:
            st = s.stats()
        assert st["sms"] == props.multi_processor_count
        assert st["resident_ctas"] % st["sms"] == 0 and st["resident_ctas"] >= st["sms"]
        assert 4 <= st["strip_rows"] <= 128
    if props.multi_processor_count == 148:
        cfg = O.Config(nx=16384, ny=16384, system=O.EULER, param=(G,))
        with solver_for(cfg) as s:
            st = s.stats()
        assert st["resident_ctas"] == 148 * 3      # the pair kernel: 3 CTAs of 4 warps per SM


# ------------------------------------------ full-size c3, random data
def test_full_size_random_euler_every_seam():
    """BASELINE configs[2] at 16384^2 on euler_random (every cell different, so
    a wrong-neighbour read shows anywhere, unlike piecewise-constant Lax-Liu):
    one fixed-dt step in the bench's launch configuration, then 10 row bands
    recomputed by the oracle -- the first and last rows, bands straddling the
    first, a middle and the last strip seam of the launch, and random bands."""
    n = 16384
    cfg = O.Config(nx=n, ny=n, system=O.EULER, param=(G,))
    W0 = inputs.euler_random(n, n, seed=1)
    dt = 0.45 * (1.0 / n) / 3.5
    with solver_for(cfg) as s:
        s.set_state(W0)
        s.step(dt, 1)
        W1 = s.get_state()
        rps = s.stats()["strip_rows"]
    rng = np.random.default_rng(5)
    starts = [0, rps - 4, (n // rps // 2) * rps - 4, n - rps - 4, n - 8]
    starts += [int(x) for x in rng.integers(8, n - 16, size=5)]
    for j0 in starts:
        lo, hi = j0 - 1, j0 + 9
        rows = [r % n for r in range(lo, hi)]
        bcfg = O.Config(nx=n, ny=len(rows), system=O.EULER, param=(G,), y1=len(rows) / n)
        out = O.transport_step(bcfg, W0[rows], dt)
        assert np.array_equal(W1[[r % n for r in range(j0, j0 + 8)]], out[1:-1]), j0
    del W0, W1


# ------------------------------------------------- FAST kernel range fallback
@pytest.mark.parametrize("mode", [O.FIXED, O.ADAPTIVE])
@pytest.mark.parametrize("flags", [0, fv2d.FLAG_GRAPH])
def test_fast_division_out_of_range_cells_rerun_exactly(mode, flags, capfd, monkeypatch):
    """The adaptive-dt Euler pair kernel divides and takes square roots
    branch-free (the compiler's fast paths, same bits inside their range).  Admissible cells
    whose operands fall outside that range -- a subnormal density (1/rho still
    finite) and a subnormal gamma*p/rho -- make the step re-run with the exact
    kernel: state and dt log stay bitwise the oracle's, and the library reports
    the re-run (FV2D_DEBUG_FAST)."""
    monkeypatch.setenv("FV2D_DEBUG_FAST", "1")
    nx, ny = 70, 44
    cfg = O.Config(nx=nx, ny=ny, system=O.EULER, param=(G,))
    W0 = inputs.euler_random(nx, ny, seed=11).copy()
    W0[5, 7] = (1e-308, 0.0, 0.0, 1e-308)      # rho subnormal: 1/rho = 1e308, c = sqrt(0.56)
    W0[30, 40] = (1.0, 0.0, 0.0, 1e-310)       # gamma*p/rho subnormal
    value = 0.45 if mode == O.ADAPTIVE else 0.5 * 0.45 * (1.0 / nx) / O.smax(cfg, W0)[0]
    ref = O.run(cfg, W0, 6, mode, value)
    assert ref.status == 0
    with solver_for(cfg, flags=flags) as s:
        s.set_state(W0)
        log = s.step_adaptive(value, 6) if mode == O.ADAPTIVE else s.step(value, 6)
        W = s.get_state()
    assert np.array_equal(W, ref.W)
    if mode == O.ADAPTIVE:  # (fixed dt runs the exact kernel: nothing to re-run)
        assert np.array_equal(log, ref.dt_log)
        assert "fast-path recovery" in capfd.readouterr().err


def test_fast_division_genuine_error_still_reported():
    """A non-admissible cell (p < 0) in a FAST step is re-run exactly and then
    reported as the oracle reports it: E_NONFINITE at the same step, W^k kept."""
    nx, ny = 64, 40
    cfg = O.Config(nx=nx, ny=ny, system=O.EULER, param=(G,))
    W0 = inputs.euler_random(nx, ny, seed=12).copy()
    W0[10, 20, 3] = 0.0                          # E = 0 -> p < 0
    dt = 1e-4
    ref = O.run(cfg, W0, 3, O.FIXED, dt, raise_on_error=False)
    assert ref.status == O.E_NONFINITE
    with solver_for(cfg) as s:
        s.set_state(W0)
        s.step(dt, 3)
        with pytest.raises(fv2d.FV2DError) as e:
            s.synchronize()
        assert e.value.code == fv2d.E_NONFINITE and e.value.step == ref.steps_done
        assert e.value.cell == ref.err_cell
        assert np.array_equal(s.get_state(raise_on_error=False), ref.W)


@pytest.mark.parametrize("seed", range(12))
def test_fast_division_recovery_randomized(seed):
    """Random Euler meshes, boundary conditions, slab counts, tiles and graph
    mode with 1-3 admissible cells whose operands leave the branch-free range
    (subnormal rho or subnormal gamma*p/rho), adaptive dt mixed with fixed-dt
    runs: state and dt logs bitwise the oracle's."""
    rng = np.random.default_rng(500 + seed)
    nslabs = int(rng.choice([1, 1, 2]))
    ny = int(rng.integers(4, 40)) * nslabs
    nx = int(rng.integers(5, 200))
    bcs = [O.BC_PERIODIC, O.BC_WALL, O.BC_DIRICHLET]
    cfg = O.Config(nx=nx, ny=ny, system=O.EULER, param=(G,), bc_x=int(rng.choice(bcs)), bc_y=int(rng.choice(bcs)),
                   dirichlet=(1.0, 0.1, -0.2, 2.6))
    W0 = inputs.euler_random(nx, ny, seed=seed + 40).copy()
    for _ in range(int(rng.integers(1, 4))):
        j, i = int(rng.integers(0, ny)), int(rng.integers(0, nx))
        W0[j, i] = (1e-308, 0.0, 0.0, 1e-308) if rng.random() < 0.5 else (1.0, 0.0, 0.0, 1e-310)
    flags = int(rng.choice([0, fv2d.FLAG_GRAPH]))
    tiles = (1, 1) if rng.random() < 0.6 or nx < 8 else (2, 2)
    n1, n2 = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    C = 0.4
    ref1 = O.run(cfg, W0, n1, O.ADAPTIVE, C, raise_on_error=False)
    if ref1.status != O.OK:
        pytest.skip(f"oracle status {ref1.status}")
    dt = 0.5 * C * min(cfg.x1 - cfg.x0, cfg.y1 - cfg.y0) / max(nx, ny) / O.smax(cfg, ref1.W)[0]
    ref2 = O.run(cfg, ref1.W, n2, O.FIXED, dt, raise_on_error=False)
    ref3 = O.run(cfg, ref2.W, n1, O.ADAPTIVE, C, raise_on_error=False)
    if ref2.status != O.OK or ref3.status != O.OK:
        pytest.skip("oracle status")
    with solver_for(cfg, nslabs=nslabs, flags=flags, tiles=tiles) as s:
        s.set_state(W0)
        l1 = s.step_adaptive(C, n1)
        s.step(dt, n2)
        l3 = s.step_adaptive(C, n1)
        W = s.get_state()
    assert np.array_equal(l1, ref1.dt_log) and np.array_equal(l3, ref3.dt_log)
    assert np.array_equal(W, ref3.W)

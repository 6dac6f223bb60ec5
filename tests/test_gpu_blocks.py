"""2-D rank blocks (nranks_x > 1) -- the paper's NPartX x NPartY decomposition
with its four overlaps -- and the
ghost-column machinery they use (FV2D_FLAG_GHOST_COLUMNS), through the C ABI,
against the oracle on the same seeded inputs.  The scheme is a per-cell closed
form (R25), so any decomposition must give the oracle's bits and dt sequence.

Ranks run as contexts of this process on the pool's single GPU, each driven by
its own host thread and stream (the peer-memory path: step kernels store their
boundary rows AND columns into the neighbours' ghost rows/columns); the NCCL
column exchange (pack, send/recv, unpack) runs as a 1-rank self exchange."""
import threading

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


def solver_for(cfg, **kw):
    return fv2d.Solver(cfg.nx, cfg.ny, cfg.system, x0=cfg.x0, x1=cfg.x1, y0=cfg.y0, y1=cfg.y1,
                       param=cfg.param, bc_x=cfg.bc_x, bc_y=cfg.bc_y, dirichlet=cfg.dirichlet, **kw)


def run_single(cfg, W0, nsteps, mode, value, **kw):
    with solver_for(cfg, **kw) as s:
        s.set_state(W0)
        log = s.step_adaptive(value, nsteps) if mode == O.ADAPTIVE else s.step(value, nsteps)
        return s.get_state(), log


def run_blocks(cfg, W0, px, py, nsteps, mode, value, flags=0, tiles=(1, 1)):
    """px x py ranks (rank = ry*px + rx) of the peer-memory path on one GPU."""
    import torch
    P = px * py
    H, Wd = cfg.ny // py, cfg.nx // px
    streams = [torch.cuda.Stream() for _ in range(P)]
    solvers = [solver_for(cfg, rank=r, nranks=P, nranks_x=px, flags=fv2d.FLAG_PEER_HALO | flags, tiles=tiles,
                          stream=streams[r].cuda_stream) for r in range(P)]
    for s in solvers:
        s.peer_connect_local(solvers)
    out, logs, errs = [None] * P, [None] * P, []

    def work(r):
        try:
            rx, ry = r % px, r // px
            s = solvers[r]
            s.set_state(W0[ry * H:(ry + 1) * H, rx * Wd:(rx + 1) * Wd])
            if mode == O.ADAPTIVE:
                logs[r] = s.step_adaptive(value, nsteps)
            else:
                s.step(value, nsteps)
            out[r] = s.get_state()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for s in solvers:
        s.close()
    assert not errs, errs
    W = np.concatenate([np.concatenate(out[ry * px:(ry + 1) * px], axis=1) for ry in range(py)], axis=0)
    return W, logs


def euler(nx, ny, bc_x=O.BC_PERIODIC, bc_y=O.BC_PERIODIC, seed=3):
    cfg = O.Config(nx=nx, ny=ny, system=O.EULER, param=(G,), bc_x=bc_x, bc_y=bc_y, x1=nx / ny,
                   dirichlet=(1.0, 0.1, -0.2, 2.6) if O.BC_DIRICHLET in (bc_x, bc_y) else ())
    return cfg, inputs.euler_random(nx, ny, seed=seed)


BLOCK_CASES = [
    # (px, py, bc_x, bc_y, nx, ny)
    (2, 1, O.BC_PERIODIC, O.BC_PERIODIC, 150, 64),    # odd local width (75)
    (2, 2, O.BC_PERIODIC, O.BC_PERIODIC, 160, 96),
    (2, 2, O.BC_WALL, O.BC_PERIODIC, 132, 80),
    (2, 2, O.BC_WALL, O.BC_WALL, 140, 64),
    (4, 2, O.BC_PERIODIC, O.BC_WALL, 256, 64),
    (3, 2, O.BC_DIRICHLET, O.BC_DIRICHLET, 138, 70),
    (8, 1, O.BC_PERIODIC, O.BC_PERIODIC, 136, 40),   # 17-column blocks: every warp straddles a block edge
    (1, 4, O.BC_WALL, O.BC_PERIODIC, 96, 96),        # y-slabs through the same code (px = 1)
]


@pytest.mark.parametrize("px,py,bc_x,bc_y,nx,ny", BLOCK_CASES)
def test_block_decomposition_bitwise(px, py, bc_x, bc_y, nx, ny):
    """2-D blocks over peer memory: same bits and dt sequence as the oracle."""
    cfg, W0 = euler(nx, ny, bc_x, bc_y, seed=px * 10 + py)
    ref = O.run(cfg, W0, 20, O.ADAPTIVE, 0.45)
    W, logs = run_blocks(cfg, W0, px, py, 20, O.ADAPTIVE, 0.45)
    for lg in logs:
        assert np.array_equal(lg, ref.dt_log)
    assert np.array_equal(W, ref.W)


@pytest.mark.parametrize("flags", [fv2d.FLAG_ONE_CELL, fv2d.FLAG_NAIVE])
def test_block_decomposition_other_kernels(flags):
    cfg, W0 = euler(120, 64, O.BC_WALL, O.BC_PERIODIC, seed=9)
    ref = O.run(cfg, W0, 12, O.ADAPTIVE, 0.45)
    W, logs = run_blocks(cfg, W0, 2, 2, 12, O.ADAPTIVE, 0.45, flags=flags)
    assert np.array_equal(logs[0], ref.dt_log)
    assert np.array_equal(W, ref.W)


def test_block_decomposition_tiled_sub_launches():
    cfg, W0 = euler(200, 96, O.BC_PERIODIC, O.BC_PERIODIC, seed=12)
    ref = O.run(cfg, W0, 10, O.ADAPTIVE, 0.45)
    W, _ = run_blocks(cfg, W0, 2, 2, 10, O.ADAPTIVE, 0.45, tiles=(2, 3))
    assert np.array_equal(W, ref.W)


def test_block_decomposition_advection_fixed_dt():
    cfg = O.Config(nx=128, ny=64, system=O.ADVECTION, param=(1.0, 0.5), x1=2.0)
    W0 = inputs.advection_dyadic(128, 64, seed=0)
    dt = 0.5 / 64
    ref = O.run(cfg, W0, 30, O.FIXED, dt)
    W, _ = run_blocks(cfg, W0, 4, 2, 30, O.FIXED, dt)
    assert np.array_equal(W, ref.W)


@pytest.mark.parametrize("flags", [0, fv2d.FLAG_NAIVE])
def test_block_decomposition_spray(flags):
    """Spray: tolerance parity (device exp/sincospi vs glibc); the source's
    Taylor-Green drag uses the block's global cell centres."""
    n = 48
    cfg = O.Config(nx=n, ny=n, system=O.SPRAY, param=(1.0, 1.0))
    W0 = inputs.spray_taylor_green(n, n)
    s0, _ = O.smax(cfg, W0)
    dt = 0.5 * (1.0 / n) / s0
    ref = O.run(cfg, W0, 5, O.FIXED, dt)
    W, _ = run_blocks(cfg, W0, 2, 2, 5, O.FIXED, dt, flags=flags)
    assert relerr(W, ref.W) <= 1e-10


def test_block_cfl_error_latched_on_every_rank():
    """A fixed dt violating eq:CFL_cond is detected through the peer max-all-reduce
    on every block; the readable state stays W^0."""
    cfg, W0 = euler(64, 64, seed=4)
    s0, _ = O.smax(cfg, W0)
    dt = 1.5 * (1.0 / 64) / s0
    with pytest.raises(AssertionError) as ei:
        run_blocks(cfg, W0, 2, 2, 3, O.FIXED, dt)
    assert "E_CFL" in str(ei.value)


# ---------------------------------------------------------------- one context, ghost columns

@pytest.mark.parametrize("bc_x", [O.BC_PERIODIC, O.BC_WALL, O.BC_DIRICHLET])
@pytest.mark.parametrize("nslabs", [1, 3])
def test_ghost_columns_single_context(bc_x, nslabs):
    """FV2D_FLAG_GHOST_COLUMNS on one context: x-neighbours through the stored
    ghost columns (own columns for periodic x) -- same bits as the oracle."""
    cfg, W0 = euler(126, 60, bc_x, O.BC_PERIODIC, seed=17)
    ref = O.run(cfg, W0, 15, O.ADAPTIVE, 0.45)
    W, log = run_single(cfg, W0, 15, O.ADAPTIVE, 0.45, flags=fv2d.FLAG_GHOST_COLUMNS, nslabs=nslabs)
    assert np.array_equal(log, ref.dt_log)
    assert np.array_equal(W, ref.W)


@pytest.mark.parametrize("bc_x,nx,ny", [(O.BC_PERIODIC, 100, 48), (O.BC_WALL, 100, 48), (O.BC_PERIODIC, 300, 80),
                                        (O.BC_WALL, 258, 72)])
def test_ghost_columns_nccl_loopback(bc_x, nx, ny):
    """The NCCL column exchange (packed send columns, grouped send/recv, unpack
    into the ghost columns) as a 1-rank self exchange; from nx >= 256 the
    boundary rows and column strips run first and the exchange overlaps the
    interior launch on the comm stream."""
    cfg, W0 = euler(nx, ny, bc_x, O.BC_PERIODIC, seed=23)
    ref = O.run(cfg, W0, 12, O.ADAPTIVE, 0.45)
    W, log = run_single(cfg, W0, 12, O.ADAPTIVE, 0.45, nccl_id=fv2d.nccl_unique_id(),
                        flags=fv2d.FLAG_GHOST_COLUMNS | fv2d.FLAG_NCCL_LOOPBACK)
    assert np.array_equal(log, ref.dt_log)
    assert np.array_equal(W, ref.W)


def test_ghost_columns_graph_and_spray():
    cfg, W0 = euler(90, 50, O.BC_PERIODIC, O.BC_WALL, seed=29)
    ref = O.run(cfg, W0, 10, O.ADAPTIVE, 0.45)
    W, _ = run_single(cfg, W0, 10, O.ADAPTIVE, 0.45, flags=fv2d.FLAG_GHOST_COLUMNS | fv2d.FLAG_GRAPH)
    assert np.array_equal(W, ref.W)
    n = 40
    scfg = O.Config(nx=n, ny=n, system=O.SPRAY, param=(1.0, 1.0))
    S0 = inputs.spray_taylor_green(n, n)
    s0, _ = O.smax(scfg, S0)
    dt = 0.5 * (1.0 / n) / s0
    sref = O.run(scfg, S0, 4, O.FIXED, dt)
    SW, _ = run_single(scfg, S0, 4, O.FIXED, dt, flags=fv2d.FLAG_GHOST_COLUMNS)
    assert relerr(SW, sref.W) <= 1e-10


def _random_block_case(seed):
    rng = np.random.default_rng(1000 + seed)
    while True:
        px, py = int(rng.integers(1, 5)), int(rng.integers(1, 3))
        if 2 <= px * py <= 8:
            break
    wl, hl = int(rng.integers(2, 70)), int(rng.integers(3, 40))
    nx, ny = px * wl, py * hl
    system = O.EULER if rng.random() < 0.7 else O.ADVECTION
    bcs = [O.BC_PERIODIC, O.BC_DIRICHLET] + ([O.BC_WALL] if system == O.EULER else [])
    bc_x, bc_y = int(rng.choice(bcs)), int(rng.choice(bcs))
    flags = int(rng.choice([0, 0, fv2d.FLAG_ONE_CELL, fv2d.FLAG_NAIVE, fv2d.FLAG_PEER_SPLIT]))
    if system == O.EULER:
        cfg = O.Config(nx=nx, ny=ny, system=O.EULER, param=(G,), bc_x=bc_x, bc_y=bc_y, x1=nx / ny,
                       dirichlet=(1.1, 0.2, -0.1, 2.4))
        W0 = inputs.euler_random(nx, ny, seed=seed)
    else:
        a = (float(rng.choice([-1.0, 0.5, 1.0])), float(rng.choice([-0.75, 0.25, 1.0])))
        cfg = O.Config(nx=nx, ny=ny, system=O.ADVECTION, param=a, bc_x=bc_x, bc_y=bc_y, x1=nx / ny,
                       dirichlet=(0.375,))
        W0 = inputs.advection_dyadic(nx, ny, seed=seed)
    return cfg, W0, px, py, flags


@pytest.mark.parametrize("seed", range(24))
def test_randomized_block_grids_bitwise(seed):
    """Random block grids (1..4 x 1..2 ranks), block sizes (2..69 x 3..39 cells,
    odd and even), systems, boundary conditions, kernels and the fused/split
    peer all-reduce: bitwise the oracle, identical dt logs."""
    cfg, W0, px, py, flags = _random_block_case(seed)
    ref = O.run(cfg, W0, 12, O.ADAPTIVE, 0.4, raise_on_error=False)
    if ref.status != O.OK:
        pytest.skip(f"oracle status {ref.status} for this random state")
    W, logs = run_blocks(cfg, W0, px, py, 12, O.ADAPTIVE, 0.4, flags=flags)
    for lg in logs:
        assert np.array_equal(lg, ref.dt_log), (px, py, cfg.nx, cfg.ny, flags)
    assert np.array_equal(W, ref.W), (px, py, cfg.nx, cfg.ny, flags)

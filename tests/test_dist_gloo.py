"""The N>1 host path on CPU with the gloo backend (world size 2 and 4): the
y-slab partition, the halo-row protocol the library posts to NCCL, the
max-all-reduce of the CFL speed, the id broadcast.  Each rank advances its slab
with the oracle on [ghost_s; slab; ghost_n]; the gathered result must equal the
single-domain oracle bitwise, with an identical dt sequence."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_1701_05431_b200 import dist as D
from paper_1701_05431_b200 import inputs


def test_slab_rows_and_neighbours():
    assert D.slab_rows(0, 4, 16) == (0, 4) and D.slab_rows(3, 4, 16) == (12, 16)
    with pytest.raises(ValueError):
        D.slab_rows(0, 3, 16)
    assert D.neighbours(0, 4, True) == (3, 1)
    assert D.neighbours(3, 4, True) == (2, 0)
    assert D.neighbours(0, 4, False) == (None, 1)
    assert D.neighbours(3, 4, False) == (2, None)
    assert D.neighbours(0, 2, True) == (1, 1)
    assert D.neighbours(0, 1, True) == (0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mirror(row, var):
    r = row.copy()
    r[..., var] = -r[..., var]
    return r


def _worker(rank, world, port, bc_y, nsteps, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny = 40, 32
        periodic = bc_y == O.BC_PERIODIC
        W = inputs.euler_random(nx, ny, seed=21)
        j0, j1 = D.slab_rows(rank, world, ny)
        loc = W[j0:j1].copy()
        cfg_loc = O.Config(nx=nx, ny=j1 - j0, system=O.EULER, param=(1.4,))
        hmin = min(1.0 / nx, 1.0 / ny)
        band_cfg = O.Config(nx=nx, ny=j1 - j0 + 2, system=O.EULER, param=(1.4,),
                            y1=(j1 - j0 + 2) / ny)
        ident = D.broadcast_bytes(b"nccl-id-from-rank-0" if rank == 0 else None)
        assert ident == b"nccl-id-from-rank-0"
        dts = []
        for _ in range(nsteps):
            s_loc, _ = O.smax(cfg_loc, loc)
            (smax,) = D.max_over_ranks([s_loc])
            dt = (0.45 * hmin) / smax
            dts.append(dt)
            gs, gn = D.exchange_halo_rows(loc[0], loc[-1], rank, world, periodic)
            if gs is None:
                gs = _mirror(loc[0], 2)          # wall: mirror, normal momentum negated (R13)
            if gn is None:
                gn = _mirror(loc[-1], 2)
            band = np.concatenate([gs[None], loc, gn[None]], axis=0)
            loc = O.transport_step(band_cfg, band, dt)[1:-1]
        out = [None] * world
        dist.all_gather_object(out, loc)
        if rank == 0:
            q.put((np.concatenate(out, axis=0), dts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,bc_y", [(2, O.BC_PERIODIC), (2, O.BC_WALL), (4, O.BC_PERIODIC)])
def test_gloo_slab_exchange_matches_single_domain(world, bc_y):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    nsteps = 12
    procs = [ctx.Process(target=_worker, args=(r, world, port, bc_y, nsteps, q)) for r in range(world)]
    for p in procs:
        p.start()
    W, dts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = O.Config(nx=40, ny=32, system=O.EULER, param=(1.4,), bc_y=bc_y)
    ref = O.run(cfg, inputs.euler_random(40, 32, seed=21), nsteps, O.ADAPTIVE, 0.45)
    assert np.array_equal(np.array(dts), ref.dt_log)
    assert np.array_equal(W, ref.W)


def test_block_of_and_block_neighbours():
    assert D.block_of(0, 2, 2, 40, 32) == (0, 16, 0, 20)
    assert D.block_of(3, 2, 2, 40, 32) == (16, 32, 20, 40)
    assert D.block_of(5, 4, 2, 40, 32) == (16, 32, 10, 20)
    with pytest.raises(ValueError):
        D.block_of(0, 3, 1, 40, 32)
    with pytest.raises(ValueError):
        D.block_of(4, 2, 2, 40, 32)
    # 2x2 periodic: (south, north, west, east)
    assert D.block_neighbours(0, 2, 2) == (2, 2, 1, 1)
    assert D.block_neighbours(3, 2, 2) == (1, 1, 2, 2)
    # 4x2, walls in x, periodic y
    assert D.block_neighbours(4, 4, 2, periodic_x=False) == (0, 0, None, 5)
    assert D.block_neighbours(7, 4, 2, periodic_x=False) == (3, 3, 6, None)
    assert D.block_neighbours(1, 4, 2, periodic_y=False) == (None, 5, 0, 2)


def _worker_2d(rank, px, py, port, bc_x, bc_y, nsteps, q):
    """One 2-D block per rank: the oracle advances [ghost frame; block] each step
    with ghosts from exchange_halo_2d (the library's NCCL group pattern)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    world = px * py
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny = 40, 32
        W = inputs.euler_random(nx, ny, seed=31)
        j0, j1, i0, i1 = D.block_of(rank, px, py, nx, ny)
        loc = W[j0:j1, i0:i1].copy()
        h, w = loc.shape[:2]
        # dx = dy = 1/32 (dyadic), so every sub-domain has bitwise the global mesh size
        cfg_loc = O.Config(nx=w, ny=h, system=O.EULER, param=(1.4,), x1=w / 32, y1=h / 32)
        pad_cfg = O.Config(nx=w + 2, ny=h + 2, system=O.EULER, param=(1.4,), x1=(w + 2) / 32, y1=(h + 2) / 32)
        hmin = 1.0 / 32
        dts = []
        for _ in range(nsteps):
            s_loc, _ = O.smax(cfg_loc, loc)
            (smax,) = D.max_over_ranks([s_loc])
            dt = (0.45 * hmin) / smax
            dts.append(dt)
            gs, gn, gw, ge = D.exchange_halo_2d(loc, rank, px, py, bc_x == O.BC_PERIODIC, bc_y == O.BC_PERIODIC)
            gs = _mirror(loc[0], 2) if gs is None else gs        # walls (R13)
            gn = _mirror(loc[-1], 2) if gn is None else gn
            gw = _mirror(loc[:, 0], 1) if gw is None else gw
            ge = _mirror(loc[:, -1], 1) if ge is None else ge
            pad = np.empty((h + 2, w + 2, 4))
            pad[1:-1, 1:-1] = loc
            pad[0, 1:-1], pad[-1, 1:-1], pad[1:-1, 0], pad[1:-1, -1] = gs, gn, gw, ge
            # corners are never read by the 5-point stencil; any admissible state
            pad[0, 0], pad[0, -1], pad[-1, 0], pad[-1, -1] = loc[0, 0], loc[0, -1], loc[-1, 0], loc[-1, -1]
            loc = O.transport_step(pad_cfg, pad, dt)[1:-1, 1:-1]
        out = [None] * world
        dist.all_gather_object(out, loc)
        if rank == 0:
            rows = [np.concatenate(out[ry * px:(ry + 1) * px], axis=1) for ry in range(py)]
            q.put((np.concatenate(rows, axis=0), dts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("px,py,bc_x,bc_y", [(2, 2, O.BC_PERIODIC, O.BC_PERIODIC), (2, 2, O.BC_WALL, O.BC_PERIODIC),
                                             (2, 1, O.BC_WALL, O.BC_PERIODIC), (4, 1, O.BC_PERIODIC, O.BC_WALL)])
def test_gloo_2d_block_exchange_matches_single_domain(px, py, bc_x, bc_y):
    """2-D blocks with the four overlaps: bitwise the single-domain
    oracle with an identical dt sequence."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    nsteps = 8
    procs = [ctx.Process(target=_worker_2d, args=(r, px, py, port, bc_x, bc_y, nsteps, q)) for r in range(px * py)]
    for p in procs:
        p.start()
    W, dts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = O.Config(nx=40, ny=32, system=O.EULER, param=(1.4,), bc_x=bc_x, bc_y=bc_y, x1=40 / 32)
    ref = O.run(cfg, inputs.euler_random(40, 32, seed=31), nsteps, O.ADAPTIVE, 0.45)
    assert np.array_equal(np.array(dts), ref.dt_log)
    assert np.array_equal(W, ref.W)

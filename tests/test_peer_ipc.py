"""The peer-memory multi-GPU path across PROCESSES (CUDA IPC), as two ranks
sharing this box's single GPU: handles exchanged with torch.distributed (gloo),
fv2d_peer_export / fv2d_peer_connect, then stepping -- the same code path one
process per GPU takes on an 8-GPU node.  Results must be bitwise the oracle's."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_1701_05431_b200 import inputs

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, bc_y, nsteps, q, px=1):
    import torch
    import torch.distributed as dist

    from paper_1701_05431_b200 import fv2d
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny = 140, 64
        W0 = inputs.euler_random(nx, ny, seed=77)
        H, Wd = ny // (world // px), nx // px
        rx, ry = rank % px, rank // px
        st = torch.cuda.Stream()
        s = fv2d.Solver(nx, ny, fv2d.EULER, param=(1.4,), bc_y=bc_y, rank=rank, nranks=world, nranks_x=px,
                        flags=fv2d.FLAG_PEER_HALO, stream=st.cuda_stream)
        handles = [None] * world
        dist.all_gather_object(handles, s.peer_export())
        s.peer_connect(b"".join(handles))
        dist.barrier()
        s.set_state(W0[ry * H:(ry + 1) * H, rx * Wd:(rx + 1) * Wd])
        log = s.step_adaptive(0.45, nsteps)
        W = s.get_state()
        out = [None] * world
        dist.all_gather_object(out, (W, log))
        dist.barrier()
        s.close()
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bc_y,px", [(O.BC_PERIODIC, 1), (O.BC_WALL, 1), (O.BC_WALL, 2)])
def test_peer_ipc_two_processes_bitwise(bc_y, px):
    """px = 1: two y-slabs; px = 2: two x-blocks (east/west ghost columns over IPC)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    nsteps = 15
    ps = [ctx.Process(target=_rank, args=(r, 2, port, bc_y, nsteps, q, px)) for r in range(2)]
    for p in ps:
        p.start()
    out = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = O.Config(nx=140, ny=64, system=O.EULER, param=(1.4,), bc_y=bc_y)
    ref = O.run(cfg, inputs.euler_random(140, 64, seed=77), nsteps, O.ADAPTIVE, 0.45)
    W = np.concatenate([o[0] for o in out], axis=1 if px == 2 else 0)
    for o in out:
        assert np.array_equal(o[1], ref.dt_log)
    assert np.array_equal(W, ref.W)

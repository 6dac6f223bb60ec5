"""Small runs for compute-sanitizer (memcheck / racecheck / initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1701_05431_b200 import fv2d, inputs

cases = [
    dict(nx=130, ny=70, system=fv2d.EULER, param=(1.4,), bc_x=fv2d.BC_DIRICHLET, bc_y=fv2d.BC_DIRICHLET,
         dirichlet=(1.0, 0.1, -0.2, 2.6), W=inputs.euler_random(130, 70, seed=5)),
    dict(nx=125, ny=64, system=fv2d.EULER, param=(1.4,), bc_x=fv2d.BC_WALL, bc_y=fv2d.BC_WALL,
         W=inputs.euler_random(125, 64, seed=6)),
    dict(nx=125, ny=64, system=fv2d.EULER, param=(1.4,), nslabs=4, W=inputs.euler_random(125, 64, seed=7)),
    dict(nx=64, ny=64, system=fv2d.ADVECTION, param=(1.0, 0.5), W=inputs.advection_dyadic(64, 64)),
    dict(nx=33, ny=32, system=fv2d.SPRAY, param=(1.0, 1.0), W=inputs.spray_taylor_green(33, 32)),
    dict(nx=33, ny=32, system=fv2d.SPRAY, param=(1.0, 1.0), flags=fv2d.FLAG_NAIVE,
         W=inputs.spray_taylor_green(33, 32)),
    # spray with two slabs and with CUDA-graph replay (the three multiplier levels
    # rotate with the device step counter)
    dict(nx=40, ny=32, system=fv2d.SPRAY, param=(1.0, 1.0), nslabs=2, W=inputs.spray_taylor_green(40, 32)),
    dict(nx=40, ny=32, system=fv2d.SPRAY, param=(1.0, 1.0), flags=fv2d.FLAG_GRAPH,
         W=inputs.spray_taylor_green(40, 32)),
    dict(nx=100, ny=40, system=fv2d.EULER, param=(1.4,), flags=fv2d.FLAG_NAIVE, W=inputs.euler_random(100, 40)),
    dict(nx=100, ny=40, system=fv2d.EULER, param=(1.4,), flags=fv2d.FLAG_ONE_CELL, W=inputs.euler_random(100, 40)),
    dict(nx=130, ny=60, system=fv2d.EULER, param=(1.4,), tiles=(3, 4), W=inputs.euler_random(130, 60)),
    dict(nx=130, ny=60, system=fv2d.EULER, param=(1.4,), flags=fv2d.FLAG_GRAPH, tiles=(2, 2),
         W=inputs.euler_random(130, 60)),
    dict(nx=130, ny=64, system=fv2d.EULER, param=(1.4,), flags=fv2d.FLAG_NCCL_LOOPBACK, W=inputs.euler_random(130, 64)),
    # stored ghost columns (the 2-D rank blocks' layout and kernels' xghost mode)
    dict(nx=126, ny=60, system=fv2d.EULER, param=(1.4,), flags=fv2d.FLAG_GHOST_COLUMNS, nslabs=2,
         W=inputs.euler_random(126, 60, seed=8)),
    dict(nx=125, ny=64, system=fv2d.EULER, param=(1.4,), bc_x=fv2d.BC_WALL, flags=fv2d.FLAG_GHOST_COLUMNS,
         W=inputs.euler_random(125, 64, seed=9)),
    dict(nx=130, ny=70, system=fv2d.EULER, param=(1.4,), bc_x=fv2d.BC_DIRICHLET, dirichlet=(1.0, 0.1, -0.2, 2.6),
         flags=fv2d.FLAG_GHOST_COLUMNS | fv2d.FLAG_ONE_CELL, W=inputs.euler_random(130, 70, seed=10)),
    dict(nx=33, ny=32, system=fv2d.SPRAY, param=(1.0, 1.0), flags=fv2d.FLAG_GHOST_COLUMNS,
         W=inputs.spray_taylor_green(33, 32)),
    dict(nx=300, ny=80, system=fv2d.EULER, param=(1.4,), flags=fv2d.FLAG_GHOST_COLUMNS | fv2d.FLAG_NCCL_LOOPBACK,
         W=inputs.euler_random(300, 80, seed=11)),
]
for c in cases:
    W = c.pop("W")
    if c.get("flags", 0) & fv2d.FLAG_NCCL_LOOPBACK:
        c["nccl_id"] = fv2d.nccl_unique_id()
    with fv2d.Solver(**c) as s:
        s.set_state(W)
        snap = fv2d.PinnedArray(W.shape)
        s.snapshot(snap)
        s.step_adaptive(0.4, 3)
        dt, _ = s.compute_dt(0.4)
        s.step(dt * 0.9, 2)
        if c["system"] == fv2d.SPRAY:
            s.apply_source(1e-4)
        out = s.get_state()
        s.snapshot_wait()
        assert np.array_equal(snap.array, W)
        snap.free()
        assert np.all(np.isfinite(out))
# the pipelined host -> host step (banded H2D / step / D2H on three streams)
W = inputs.euler_random(256, 160, seed=12)
with fv2d.Solver(256, 160, fv2d.EULER, param=(1.4,)) as s:
    s.set_state(W)
    dt, _ = s.compute_dt(0.4)
    pin = fv2d.PinnedArray(W.shape)
    pin.array[:] = W
    s.step_host(pin, pin, dt, 1)
    s.step_host(pin, pin, dt, 2)
    assert np.all(np.isfinite(pin.array))
    pin.free()
# FAST pair kernel: a subnormal density makes the library re-run the steps with
# the exact kernel (recover_fast)
W = inputs.euler_random(96, 64, seed=13).copy()
W[5, 7] = (1e-308, 0.0, 0.0, 1e-308)
with fv2d.Solver(96, 64, fv2d.EULER, param=(1.4,)) as s:
    s.set_state(W)
    s.step_adaptive(0.45, 3)
    dt, _ = s.compute_dt(0.4)
    s.step(dt, 2)
    assert np.all(np.isfinite(s.get_state()))
print("sanitize cases ok")

"""Per-GPU share of the c3 strong-scaling run measured on one GPU: the
16384 x (16384/P) slab a rank owns at P = 1, 2, 4, 8 (y-slabs) and the 2-D
blocks of a 4x2 grid, stepped alone (fixed dt, the bench's kernel).  Gives the
compute-only strong-scaling efficiency T1 / (P * T_P) -- the ceiling the
multi-GPU run can reach before communication (the fused peer-memory path adds
one in-kernel all-reduce and in-kernel halo stores per step).  JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1701_05431_b200 import fv2d, inputs

N = 16384


def step_ms(nx, ny, steps=50):
    W0 = np.empty((ny, nx, 4))
    for j in range(0, ny, 1024):
        W0[j:j + 1024] = inputs.euler_lax_liu3(nx, ny, rows=(j, min(ny, j + 1024)))
    st = torch.cuda.current_stream()
    with fv2d.Solver(nx, ny, fv2d.EULER, param=(1.4,), stream=st.cuda_stream) as s:
        s.set_state(W0)
        dt, _ = s.compute_dt(0.45)
        s.step(dt, 5)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        s.step(dt, steps)
        e1.record(st)
        torch.cuda.synchronize()
        s.synchronize()
    return e0.elapsed_time(e1) / steps


t1 = None
for P, (nx, ny) in [(1, (N, N)), (2, (N, N // 2)), (4, (N, N // 4)), (8, (N, N // 8)), (8, (N // 4, N // 2))]:
    ms = step_ms(nx, ny)
    if t1 is None:
        t1 = ms
    print(json.dumps({"P": P, "block": f"{nx}x{ny}", "ms_per_step": ms, "cell_updates_per_s_per_gpu": nx * ny / (ms * 1e-3),
                      "compute_only_strong_efficiency": t1 / (P * ms)}), flush=True)

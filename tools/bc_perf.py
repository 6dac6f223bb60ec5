"""c3-size step time per boundary-condition mode of the pair kernel (periodic
x: wrap loads; wall / Dirichlet x: ghosts built in registers; stored ghost
columns of 2-D blocks), Lax-Liu 3, fixed dt.  JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1701_05431_b200 import fv2d, inputs

n = 16384
W0 = np.empty((n, n, 4))
for j in range(0, n, 1024):
    W0[j:j + 1024] = inputs.euler_lax_liu3(n, n, rows=(j, j + 1024))
for name, kw in [("periodic", {}), ("wall_x", {"bc_x": fv2d.BC_WALL}), ("wall_xy", {"bc_x": fv2d.BC_WALL, "bc_y": fv2d.BC_WALL}),
                 ("dirichlet_x", {"bc_x": fv2d.BC_DIRICHLET, "dirichlet": (1.0, 0.0, 0.0, 2.5)}),
                 ("ghost_columns", {"flags": fv2d.FLAG_GHOST_COLUMNS})]:
    st = torch.cuda.current_stream()
    with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,), stream=st.cuda_stream, **kw) as s:
        s.set_state(W0)
        dt, _ = s.compute_dt(0.45)
        s.step(dt, 3)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.step(dt, 30)
        e1.record(st)
        torch.cuda.synchronize()
        s.synchronize()
        ms = e0.elapsed_time(e1) / 30
    print(json.dumps({"bc": name, "ms_per_step": ms, "cell_updates_per_s": n * n / (ms * 1e-3)}), flush=True)

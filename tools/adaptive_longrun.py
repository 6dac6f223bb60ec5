"""c3 (16384^2 Lax-Liu 3) for 1000 adaptive steps with the branch-free adaptive
kernel: wall-clock throughput, exact conservation of the sums, the dt range, and
whether any step needed the exact re-run (run with FV2D_DEBUG_FAST=1: the
library reports every re-run on stderr)."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1701_05431_b200 import fv2d, inputs

n, steps = 16384, 1000
W0 = np.empty((n, n, 4))
for j in range(0, n, 1024):
    W0[j:j + 1024] = inputs.euler_lax_liu3(n, n, rows=(j, min(n, j + 1024)))
s0 = [math.fsum(W0[..., v].ravel()) for v in range(4)]
with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,)) as s:
    s.set_state(W0)
    s.step_adaptive(0.45, 5, log=False)
    s.synchronize()
    t = time.perf_counter()
    log = s.step_adaptive(0.45, steps)
    el = time.perf_counter() - t
    W = s.get_state()
s1 = [math.fsum(W[..., v].ravel()) for v in range(4)]
print(json.dumps({"case": "c3_lax_liu3_adaptive", "steps": steps, "wall_s": el, "cell_updates_per_s": n * n * steps / el,
                  "dt_min": float(log.min()), "dt_max": float(log.max()),
                  "rel_change_sum": [abs(b - a) / abs(a) for a, b in zip(s0, s1)],
                  "rho_min": float(W[..., 0].min()), "finite": bool(np.isfinite(W).all())}))

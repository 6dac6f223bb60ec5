"""Profiling driver: set up an Euler (or spray) state and run a few steps (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1701_05431_b200 import fv2d, inputs

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--system", default="euler")
ap.add_argument("--naive", action="store_true")
ap.add_argument("--adaptive", action="store_true")
ap.add_argument("--one-cell", action="store_true")
a = ap.parse_args()
n = a.n
flags = (fv2d.FLAG_NAIVE if a.naive else 0) | (fv2d.FLAG_ONE_CELL if a.one_cell else 0)
if a.system == "euler":
    W0 = np.empty((n, n, 4))
    for j in range(0, n, 1024):
        W0[j:j + 1024] = inputs.euler_lax_liu3(n, n, rows=(j, min(n, j + 1024)))
    s = fv2d.Solver(n, n, fv2d.EULER, param=(1.4,), flags=flags)
else:
    W0 = inputs.spray_taylor_green(n, n)
    s = fv2d.Solver(n, n, fv2d.SPRAY, param=(1.0, 1.0), flags=flags)
s.set_state(W0)
dt, smax = s.compute_dt(0.45)
if a.system == "spray":
    dt = 0.5 * (1.0 / n) / smax
for _ in range(a.steps):
    if a.adaptive:
        s.step_adaptive(0.45, 1, log=False)
    else:
        s.step(dt, 1)
s.synchronize()
print("ok", s.stats())

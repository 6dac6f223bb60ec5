"""Adaptive-dt step time on several initial conditions (tuning A/B of the
adaptive pair kernel): Lax-Liu 3 (piecewise constant: most cells unchanged per
step), the isentropic vortex and random Euler data (every cell changes).

  python tools/adapt_ic_bench.py [--n 8192] [--steps 50] [--lib PATH]
Prints one JSON line per IC: event-timed step-kernel ms (mean), fixed vs adaptive.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1701_05431_b200 import fv2d, inputs

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
n = a.n


def ic(name):
    W = np.empty((n, n, 4))
    f = {"lax_liu3": inputs.euler_lax_liu3, "vortex": inputs.euler_vortex, "random": inputs.euler_random}[name]
    for j in range(0, n, 1024):
        W[j:j + 1024] = f(n, n, rows=(j, min(n, j + 1024)))
    return W


for name in ("lax_liu3", "vortex", "random"):
    W0 = ic(name)
    out = {"ic": name, "n": n, "lib": os.environ.get("FV2D_LIB", "default")}
    with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,)) as s:
        for mode in ("fixed", "adaptive"):
            s.set_state(W0)
            dt, _ = s.compute_dt(0.45)
            run = (lambda k: s.step(0.5 * dt, k)) if mode == "fixed" else (lambda k: s.step_adaptive(0.45, k, log=False))
            run(5)
            s.synchronize()
            s.set_profiling(True)
            run(a.steps)
            s.synchronize()
            st = s.stats()
            s.set_profiling(False)
            out[mode + "_ms"] = round(st["step_kernel_ms"] / max(1, st["step_kernels_timed"]), 4)
    print(json.dumps(out), flush=True)

"""fig:Convergence on the GPU: L1/L2 errors of rho
against the analytic solutions at T, for the localized cosine (bell reading R22,
eq:LCAnalytic) and the isentropic vortex (eq:RotatingGaussian, advected by (1,1)),
fixed dt = T/ceil(T/(C h/2)) hitting T exactly, C = 0.45.  Prints JSON lines."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1701_05431_b200 import fv2d, inputs


def errors(case, n, T, C=0.45, smax=2.0):
    W0 = inputs.euler_bell(n, n) if case == "bell" else inputs.euler_vortex(n, n)
    ex = inputs.euler_bell_exact(n, n, T) if case == "bell" else inputs.euler_vortex(n, n, t=T)
    with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,)) as s:
        s.set_state(W0)
        _, s0 = s.compute_dt(C)
        nsteps = int(math.ceil(T / (C * (1.0 / n) / s0)))
        s.step(T / nsteps, nsteps)
        W = s.get_state()
    d = W[..., 0] - ex[..., 0]
    h2 = 1.0 / (n * n)
    return {"case": case, "n": n, "T": T, "steps": nsteps, "L1": float(np.abs(d).sum() * h2),
            "L2": float(math.sqrt((d * d).sum() * h2)), "Linf": float(np.abs(d).max())}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=float, default=0.1)
    ap.add_argument("--sizes", default="128,256,512,1024,2048")
    a = ap.parse_args()
    for case in ("bell", "vortex"):
        prev = None
        for n in [int(x) for x in a.sizes.split(",")]:
            r = errors(case, n, a.T)
            if prev:
                r["slope_L1"] = math.log2(prev["L1"] / r["L1"])
                r["slope_L2"] = math.log2(prev["L2"] / r["L2"])
            prev = r
            print(json.dumps(r), flush=True)

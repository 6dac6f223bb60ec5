"""Long runs at full size (evidence beyond the parity tests):
c3 16384^2 Euler Lax-Liu 3, 1000 fixed-dt steps: no CFL/admissibility error,
sum(W) conserved (exact sums with math.fsum per row, periodic, S = 0);
c4 4096^2 spray, 1000 fixed-dt steps: realizable moments everywhere
(positivity, monotonicity, Hankel), total m0 decays (evaporation).
JSON lines."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1701_05431_b200 import fv2d, inputs


def fsum_vars(W):
    return [math.fsum(math.fsum(r) for r in W[..., k]) for k in range(W.shape[-1])]


def euler(n=16384, steps=1000):
    W0 = np.empty((n, n, 4))
    for j in range(0, n, 1024):
        W0[j:j + 1024] = inputs.euler_lax_liu3(n, n, rows=(j, j + 1024))
    s0 = fsum_vars(W0)
    a0 = [math.fsum(np.abs(W0[..., k]).ravel()) for k in range(4)]
    with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,)) as s:
        s.set_state(W0)
        dt, smax = s.compute_dt(0.45)
        t0 = time.perf_counter()
        s.step(dt, steps)
        s.synchronize()
        el = time.perf_counter() - t0
        W = s.get_state(out=W0)
    s1 = fsum_vars(W)
    rho = W[..., 0]
    return {"case": "c3_euler_16384_lax_liu3", "steps": steps, "dt": dt, "wall_s": el,
            "cell_updates_per_s": n * n * steps / el,
            "rel_change_sum": [abs(b - a) / c for a, b, c in zip(s0, s1, a0)],
            "rho_min": float(rho.min()), "rho_max": float(rho.max()), "finite": bool(np.isfinite(W).all())}


def spray(n=4096, steps=1000):
    W0 = inputs.spray_taylor_green(n, n)
    with fv2d.Solver(n, n, fv2d.SPRAY, param=(1.0, 1.0)) as s:
        s.set_state(W0)
        _, smax = s.compute_dt(0.5)
        dt = 0.5 * (1.0 / n) / smax
        t0 = time.perf_counter()
        s.step(dt, steps)
        s.synchronize()
        el = time.perf_counter() - t0
        it = s.stats()["newton_iters"]
        W = s.get_state()
    m0, m1, m2, m3 = (W[..., k] for k in range(4))
    real = bool(np.all(m0 > 0) & np.all(m1 > 0) & np.all(m2 > 0) & np.all(m3 > 0) & np.all(m3 <= m2) &
                np.all(m2 <= m1) & np.all(m1 <= m0) & np.all(m1 * m1 <= m0 * m2) & np.all(m2 * m2 <= m1 * m3))
    return {"case": "c4_spray_4096_taylor_green", "steps": steps, "dt": dt, "wall_s": el,
            "cell_updates_per_s": n * n * steps / el, "realizable": real,
            "m0_total_ratio": float(W[..., 0].sum() / W0[..., 0].sum()),
            "newton_iters_per_cell_step": it / (n * n * steps), "finite": bool(np.isfinite(W).all())}


if __name__ == "__main__":
    print(json.dumps(euler()), flush=True)
    print(json.dumps(spray()), flush=True)

"""Cost of the asynchronous output pipeline (fig:GanttWithOutput) on
an 8192^2 Euler run: wall time per step with no output, with a snapshot every
`every` steps taken but not written (device conversion + PCIe D2H overlapped
with stepping), and with the TFV1 files written by the background thread."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1701_05431_b200 import fv2d, inputs, output

n, steps, every, nbuf = 8192, 400, 100, 4
W0 = np.empty((n, n, 4))
for j in range(0, n, 1024):
    W0[j:j + 1024] = inputs.euler_lax_liu3(n, n, rows=(j, j + 1024))
res = {}
for mode in ("none", "snapshot_only", "snapshot_and_disk"):
    with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,)) as s:
        s.set_state(W0)
        dt, _ = s.compute_dt(0.45)
        s.step(dt, 3)
        s.synchronize()
        d = tempfile.mkdtemp()
        w = None
        if mode != "none":
            w = output.AsyncWriter(s, os.path.join(d, "s_{step:05d}.tfv1") if mode == "snapshot_and_disk" else None,
                                   nbuf=nbuf)
        t0 = time.perf_counter()
        for k in range(steps):
            s.step(dt, 1)
            if w and (k + 1) % every == 0:
                w.submit(k + 1, (k + 1) * dt)
        s.synchronize()
        t_steps = time.perf_counter() - t0
        files = w.close() if w else []
        t_all = time.perf_counter() - t0
        for f in files:
            if f:
                os.remove(f)
        res[mode] = {"wall_ms_per_step_while_stepping": t_steps / steps * 1e3, "wall_s_until_all_written": t_all,
                     "snapshots": len(files)}
print(json.dumps({"n": n, "steps": steps, "every": every, "snapshot_gb": n * n * 32 / 1e9, **res,
                  "stepping_overhead_snapshot_only": res["snapshot_only"]["wall_ms_per_step_while_stepping"] /
                  res["none"]["wall_ms_per_step_while_stepping"] - 1}))

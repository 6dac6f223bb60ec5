"""c4 (4096^2 spray) over a long run: source-pass time and Newton iterations
per cell-step in blocks of steps (does the per-step cost drift as the spray
evaporates?).  JSON lines: block index, steps so far, source / transport
kernel ms (library events), Newton iterations per cell-step in the block."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_05431_b200 import fv2d, inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 12
per = int(sys.argv[3]) if len(sys.argv) > 3 else 200
W0 = inputs.spray_taylor_green(n, n)
with fv2d.Solver(n, n, fv2d.SPRAY, param=(1.0, 1.0)) as s:
    s.set_state(W0)
    _, smax = s.compute_dt(0.5)
    dt = 0.5 * (1.0 / n) / smax
    done = 0
    for b in range(blocks):
        st0 = s.stats()
        s.set_profiling(True)
        s.step(dt, per)
        s.synchronize()
        st1 = s.stats()
        s.set_profiling(False)
        done += per
        src = (st1["source_kernel_ms"] - st0["source_kernel_ms"]) / max(1, st1["source_kernels_timed"] - st0["source_kernels_timed"])
        tr = (st1["step_kernel_ms"] - st0["step_kernel_ms"]) / max(1, st1["step_kernels_timed"] - st0["step_kernels_timed"])
        print(json.dumps({"block": b, "steps_done": done, "t": done * dt, "source_ms": src, "transport_ms": tr,
                          "newton_per_cell_step": (st1["newton_iters"] - st0["newton_iters"]) / (n * n * per)}),
              flush=True)

"""Strip-height sweep of the pair kernel (FV2D_RPS) over domain shapes,
Lax-Liu 3, fixed dt, device time per step.  Usage: rps_sweep.py nx ny [rps...]
(rps 0 = the built-in choice).  JSON lines."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    from paper_1701_05431_b200 import fv2d, inputs
    nx, ny = int(sys.argv[2]), int(sys.argv[3])
    W0 = np.empty((ny, nx, 4))
    for j in range(0, ny, 1024):
        W0[j:j + 1024] = inputs.euler_lax_liu3(nx, ny, rows=(j, min(ny, j + 1024)))
    st = torch.cuda.current_stream()
    with fv2d.Solver(nx, ny, fv2d.EULER, param=(1.4,), stream=st.cuda_stream) as s:
        s.set_state(W0)
        dt, _ = s.compute_dt(0.45)
        s.step(dt, 3)
        s.synchronize()
        steps = max(20, int(2e9 / (nx * ny)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.step(dt, steps)
        e1.record(st)
        torch.cuda.synchronize()
        s.synchronize()
        ms = e0.elapsed_time(e1) / steps
    print(json.dumps({"nx": nx, "ny": ny, "rps": os.environ.get("FV2D_RPS", "0"), "ms": ms,
                      "G": nx * ny / ms / 1e6}), flush=True)
else:
    nx, ny = sys.argv[1], sys.argv[2]
    for r in sys.argv[3:]:
        env = dict(os.environ, FV2D_RPS=r)
        subprocess.run([sys.executable, __file__, "--one", nx, ny], env=env)

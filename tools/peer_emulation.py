"""The fused peer-memory multi-GPU path with P ranks as contexts of ONE process
on one GPU (each rank its own host thread and stream; kernels of different
ranks run concurrently, as they would on P GPUs, but share one GPU's SMs and
HBM).  c3 (16384^2 Euler, Lax-Liu 3, fixed dt) split into P y-slabs (or
PX x PY blocks): total cell-updates/s vs P = 1 measures what the decomposition
itself costs -- halo rows/columns stored into the neighbours' ghost cells and
the max-all-reduce in each step kernel's last CTA (spinning while the other
ranks finish) -- with the GPU's bandwidth held fixed.  JSON lines."""
import json
import os
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1701_05431_b200 import fv2d, inputs

N = int(os.environ.get("EMU_N", "16384"))
STEPS = int(os.environ.get("EMU_STEPS", "50"))


def ic():
    W = np.empty((N, N, 4))
    for j in range(0, N, 1024):
        W[j:j + 1024] = inputs.euler_lax_liu3(N, N, rows=(j, min(N, j + 1024)))
    return W


def run(W0, px, py, flags=0):
    P = px * py
    H, Wd = N // py, N // px
    streams = [torch.cuda.Stream() for _ in range(P)]
    peer = fv2d.FLAG_PEER_HALO if P > 1 else 0
    solvers = [fv2d.Solver(N, N, fv2d.EULER, param=(1.4,), rank=r, nranks=P, nranks_x=px, flags=peer | flags,
                           stream=streams[r].cuda_stream) for r in range(P)]
    if P > 1:
        for s in solvers:
            s.peer_connect_local(solvers)
    dts = [None] * P
    bar = threading.Barrier(P)
    errs = []

    def setup(r):
        try:
            rx, ry = r % px, r // px
            s = solvers[r]
            s.set_state(np.ascontiguousarray(W0[ry * H:(ry + 1) * H, rx * Wd:(rx + 1) * Wd]))
            dts[r], _ = s.compute_dt(0.45)
            s.step(dts[r], 3)
            s.synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    def work(r):
        try:
            bar.wait()
            solvers[r].step(dts[r], STEPS)
            solvers[r].synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    for fn in (setup, work):
        th = [threading.Thread(target=fn, args=(r,)) for r in range(P)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        el = time.perf_counter() - t0
    for s in solvers:
        s.close()
    assert not errs, errs
    return el


if __name__ == "__main__":
    W0 = ic()
    base = None
    for px, py, flags in [(1, 1, 0), (1, 2, 0), (1, 4, 0), (1, 8, 0), (2, 4, 0), (1, 8, fv2d.FLAG_PEER_SPLIT)]:
        el = run(W0, px, py, flags)
        v = N * N * STEPS / el
        base = base or v
        print(json.dumps({"ranks": f"{px}x{py}", "split_allreduce": bool(flags), "steps": STEPS, "wall_s": el,
                          "cell_updates_per_s": v, "relative_to_1_rank": v / base}), flush=True)

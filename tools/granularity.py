"""GPU analog of the paper's task-granularity study (
SURVEY §8d c5): (a) throughput vs per-GPU domain size 256^2 .. 16384^2; (b) one
8192^2 Euler domain launched as k x k sub-launches ("tasks", like NPart = k^2),
with plain stream launches and with a CUDA graph.  Device time per step by CUDA
events on the stream.  JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1701_05431_b200 import fv2d, inputs


def ic(n):
    W = np.empty((n, n, 4))
    for j in range(0, n, 1024):
        W[j:j + 1024] = inputs.euler_lax_liu3(n, n, rows=(j, min(n, j + 1024)))
    return W


def measure(n, W0, steps, tiles=(1, 1), flags=0):
    st = torch.cuda.current_stream()
    with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,), tiles=tiles, flags=flags, stream=st.cuda_stream) as s:
        s.set_state(W0)
        dt, _ = s.compute_dt(0.45)
        s.step(dt, 3)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        s.step(dt, steps)
        e1.record(st)
        torch.cuda.synchronize()
        s.synchronize()
        ms = e0.elapsed_time(e1) / steps
    return ms


if __name__ == "__main__":
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    for n in (() if only == "tiles" else (256, 512, 1024, 2048, 4096, 8192, 16384)):
        W0 = ic(n)
        steps = max(20, min(2000, int(4e9 / (n * n))))
        for graph in (False, True):
            ms = measure(n, W0, steps, flags=fv2d.FLAG_GRAPH if graph else 0)
            print(json.dumps({"study": "size", "n": n, "graph": graph, "ms_per_step": ms,
                              "cell_updates_per_s": n * n / (ms * 1e-3)}), flush=True)
    n = 8192
    W0 = ic(n)
    for k in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        for graph in (False, True):
            steps = 20 if k <= 64 else 5
            ms = measure(n, W0, steps, tiles=(k, k), flags=fv2d.FLAG_GRAPH if graph else 0)
            tile = n // k
            print(json.dumps({"study": "tiles", "n": n, "k": k, "tasks": k * k, "tile": tile, "graph": graph,
                              "ms_per_step": ms, "us_per_task": ms * 1e3 / (k * k),
                              "cell_updates_per_s": n * n / (ms * 1e-3)}), flush=True)

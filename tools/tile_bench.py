"""Small-domain step time, tile kernel vs marching pair kernel (FV2D_TILE_MAX_CELLS
decides; this script runs one mode per process):
  FV2D_TILE_MAX_CELLS=0 python tools/tile_bench.py      # pair kernel
  FV2D_TILE_MAX_CELLS=1e12 python tools/tile_bench.py   # tile kernel wherever eligible
One JSON line per (size, mode): ms per step from CUDA events around K steps
(stream launches, then CUDA-graph replay), Lax-Liu 3, fixed and adaptive dt."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1701_05431_b200 import fv2d, inputs

tile = os.environ.get("FV2D_TILE_MAX_CELLS", "default")
for n in (64, 256, 512, 1024, 2048, 4096):
    W0 = inputs.euler_lax_liu3(n, n)
    for graph in (False, True):
        with fv2d.Solver(n, n, fv2d.EULER, param=(1.4,), flags=fv2d.FLAG_GRAPH if graph else 0) as s:
            s.set_state(W0)
            dt, _ = s.compute_dt(0.45)
            out = {"n": n, "tile_max_cells": tile, "graph": graph}
            for mode in ("fixed", "adaptive"):
                run = (lambda k: s.step(0.5 * dt, k)) if mode == "fixed" else (lambda k: s.step_adaptive(0.45, k, log=False))
                K = 2000 if n <= 1024 else 200
                run(20)
                s.synchronize()
                st = torch.cuda.current_stream()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                run(K)
                e1.record(st)
                s.synchronize()
                torch.cuda.synchronize()
                out[mode + "_us"] = round(e0.elapsed_time(e1) / K * 1000, 3)
            print(json.dumps(out), flush=True)

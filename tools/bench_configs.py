"""Device-time throughput of every BASELINE config on one GPU (JSONL to stdout).

c1 advection 64^2, c2 Euler 1024^2 (Lax-Liu 3), c3 Euler 16384^2 (also in bench.py),
c4 spray 4096^2 (Taylor-Green), c5 Euler 8192^2 per GPU, plus
the fused kernel variants (pair / one-cell / paper-style naive) and adaptive dt.
Timing: CUDA events on the library stream around K steps after W warm-up steps.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1701_05431_b200 import fv2d, inputs


def timed(s, stepfn, K, W):
    stepfn(W)
    s.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.set_profiling(True)
    torch.cuda.synchronize()
    e0.record(st)
    stepfn(K)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    stats = s.stats()
    s.set_profiling(False)
    s.synchronize()
    return ms / K, stats["step_kernel_ms"] / max(1, stats["step_kernels_timed"])


def euler_ic(n):
    W = np.empty((n, n, 4))
    for j in range(0, n, 1024):
        W[j:j + 1024] = inputs.euler_lax_liu3(n, n, rows=(j, min(n, j + 1024)))
    return W


def run(name, system, n, W0, K, Wu, flags=0, adaptive=False, cfl=0.45, param=None, fixed_dt=None):
    stream = torch.cuda.current_stream().cuda_stream
    with fv2d.Solver(n, n, system, param=param, flags=flags, stream=stream) as s:
        s.set_state(W0)
        dt, smax = s.compute_dt(cfl)
        if fixed_dt is not None:
            dt = fixed_dt(smax)
        fn = (lambda k: s.step_adaptive(cfl, k, log=False)) if adaptive else (lambda k: s.step(dt, k))
        ms, kms = timed(s, fn, K, Wu)
        st = s.stats()
    nv = fv2d.NVAR[system]
    cells = n * n
    rec = {"config": name, "n": n, "nvar": nv, "flags": flags, "adaptive": adaptive, "ms_per_step": ms,
           "kernel_ms": kms, "cell_updates_per_s": cells / (ms * 1e-3),
           "hbm_gbs_alg": 16 * nv * cells / (kms * 1e-3) / 1e9, "newton_iters": st["newton_iters"]}
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    want = lambda k: not a.only or k in a.only.split(",")
    torch.cuda.init()
    if want("c1"):
        run("c1_advection_64", fv2d.ADVECTION, 64, inputs.advection_dyadic(64, 64), 100, 5, cfl=0.5, param=(1.0, 0.5))
    if want("c2"):
        W = euler_ic(1024)
        run("c2_euler_1024", fv2d.EULER, 1024, W, 100, 5)
        run("c2_euler_1024_adaptive", fv2d.EULER, 1024, W, 100, 5, adaptive=True)
        run("c2_euler_1024_naive", fv2d.EULER, 1024, W, 100, 5, flags=fv2d.FLAG_NAIVE)
        run("c2_euler_1024_onecell", fv2d.EULER, 1024, W, 100, 5, flags=fv2d.FLAG_ONE_CELL)
        run("c2_euler_1024_graph", fv2d.EULER, 1024, W, 100, 5, flags=fv2d.FLAG_GRAPH)
    if want("c3"):
        W = euler_ic(16384)
        run("c3_euler_16384_pair", fv2d.EULER, 16384, W, 50, 3)
        run("c3_euler_16384_pair_adaptive", fv2d.EULER, 16384, W, 50, 3, adaptive=True)
        run("c3_euler_16384_onecell", fv2d.EULER, 16384, W, 50, 3, flags=fv2d.FLAG_ONE_CELL)
        run("c3_euler_16384_naive", fv2d.EULER, 16384, W, 20, 3, flags=fv2d.FLAG_NAIVE)
        del W
    if want("c4"):
        n = 4096
        W = inputs.spray_taylor_green(n, n)
        fd = lambda smax: 0.5 * (1.0 / n) / smax
        run("c4_spray_4096", fv2d.SPRAY, n, W, 10, 3, param=(1.0, 1.0), fixed_dt=fd)
    if want("paper"):
        # the paper's own workloads (context: PAPER.md 889-900 Euler 16384^2 x 50 iterations in
        # 61 s on 4 CPU workers + 4 GPUs; 1063-1071 spray 200^2 x 100 iterations in 5.81 s)
        n = 200
        W = inputs.spray_taylor_green(n, n)
        fd = lambda smax: 0.5 * (1.0 / n) / smax
        run("paper_spray_200_100it", fv2d.SPRAY, n, W, 100, 3, param=(1.0, 1.0), fixed_dt=fd)
        run("paper_euler_16384_50it", fv2d.EULER, 16384, euler_ic(16384), 50, 3)
    if want("c5"):
        run("c5_euler_8192", fv2d.EULER, 8192, euler_ic(8192), 100, 5)

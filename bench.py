#!/usr/bin/env python
"""Benchmark of the FV hot path (BASELINE.json metric: fp64 cell-updates/s and
% of HBM roofline at 1/2/4/8 B200).

Workload (config.workload): BASELINE configs[2] -- 2-D Euler, 16384 x 16384
cells, Lax-Liu configuration 3 (synthetic, seeded/analytic), periodic, the
paper's constant dt checked every step, y-slabs over N GPUs
(strong scaling).  A "step" is one pass of the whole hot path: CFL reduction
(fused check), x/y Lax-Friedrichs fluxes, conservative update (+ halo exchange
and max-all-reduce for N > 1: by default fused into the step kernel over peer
memory, --nccl for the NCCL baseline).  The state (2 x 8.6 GB) is far larger
than L2, so no flush is needed between steps.  --workload c4_spray_4096 times
the spray (BASELINE configs[3]) with the source pass's FP64 roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload ...] [--nranks-x PX] [--nccl]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 cell-updates/sec and % of HBM roofline at 1/2/4/8 B200"
UNIT = "cell-updates/s"
GAMMA = 1.4
CFL = 0.45
BYTES_PER_CELL = {"euler": 64, "advection": 16, "spray": 96}   # algorithmic: read W^n + write W^{n+1}

WORKLOADS = {
    # name: (system, nx, ny, description)
    "c3_euler_16384": ("euler", 16384, 16384, "BASELINE configs[2]: 2D Euler nVar=4, 16384x16384, Lax-Liu 3, "
                                              "periodic, fixed dt checked each step, y-slabs (strong scaling)"),
    "c2_euler_1024": ("euler", 1024, 1024, "BASELINE configs[1]: 2D Euler nVar=4, 1024x1024, Lax-Liu 3"),
    "c5_euler_8192_per_gpu": ("euler", 8192, 8192, "BASELINE configs[4]: 8192^2 cells per GPU (weak scaling)"),
    "c4_spray_4096": ("spray", 4096, 4096, "BASELINE configs[3]: evaporating spray nVar=6 (eq:Essadki), 4096x4096, "
                                           "Taylor-Green IC (R16), K=theta=1, the paper's fixed dt (R17), split "
                                           "source with the NDF reconstruction (S:401-419)"),
}
# FP64 peak of the spray source kernel's roofline (bound "alu"): 148 SMs x 64
# FP64 lanes (measured 64 DFMA/DADD/DMUL per SM per clock, tools/microbench.cu)
# x 2 flop per DFMA x 1.965 GHz max SM clock (B200_PROFILING.md unit counts)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel_key):
    """dram bytes per launch of the step kernel from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel_key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def gen_ic(system, nx, ny, rows):
    """Lax-Liu 3 (Euler) or the R16 Taylor-Green spray state, in row chunks
    (bounded temporaries) into one AoS array."""
    from paper_1701_05431_b200 import inputs
    j0, j1 = rows
    nv = 6 if system == "spray" else 4
    out = np.empty((j1 - j0, nx, nv))
    for a in range(j0, j1, 1024):
        b = min(j1, a + 1024)
        out[a - j0:b - j0] = (inputs.spray_taylor_green(nx, ny, rows=(a, b)) if system == "spray" else
                              inputs.euler_lax_liu3(nx, ny, rows=(a, b), gamma=GAMMA))
    return out


def spray_band_oracle(nx, ny, rows, budget_s, steps=None):
    """The oracle's spray step (transport + source, cold-start Newton as R19) on a
    full-width row band of the c4 workload: (cell-updates/s, steps, seconds)."""
    import oracle as O
    from paper_1701_05431_b200 import inputs
    j0 = ny // 2 - rows // 2
    band = inputs.spray_taylor_green(nx, ny, rows=(j0, j0 + rows))
    cfg = O.Config(nx=nx, ny=rows, system=O.SPRAY, param=(1.0, 1.0), y0=j0 / ny, y1=(j0 + rows) / ny)
    s0, _ = O.smax(cfg, band)
    dt = 0.5 * (1.0 / nx) / s0
    W = band
    t0 = time.perf_counter()
    n = 0
    while True:
        W = O.transport_step(cfg, W, dt)
        W, _ = O.source_step(cfg, W, dt)
        n += 1
        el = time.perf_counter() - t0
        if (steps is not None and n >= steps) or (steps is None and el > budget_s):
            break
    return nx * rows * n / el, n, el


def cpu_baseline(nx, ny, budget_s=12.0, system="euler"):
    """The oracle as it stands (single-threaded C, -O2 -ffp-contract=off) on a
    bounded sample: full-width row bands of the same workload, periodic."""
    import oracle as O
    from paper_1701_05431_b200 import inputs
    if system == "spray":
        v, n, el = spray_band_oracle(nx, ny, 8, budget_s)
        return {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"{n} spray steps (transport + source, cold-start Newton) on a {nx}x8 full-width row "
                          f"band of the workload, {el:.1f} s, 1 thread"}
    rows = min(ny, 256)
    band = inputs.euler_lax_liu3(nx, ny, rows=(ny // 2 - rows // 2, ny // 2 + rows // 2), gamma=GAMMA)
    cfg = O.Config(nx=nx, ny=rows, system=O.EULER, param=(GAMMA,), y1=rows / ny)
    dt = CFL * (1.0 / nx) / 2.5
    t0 = time.perf_counter()
    steps = 0
    W = band
    while True:
        W = O.transport_step(cfg, W, dt)
        steps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return {"value": nx * rows * steps / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{steps} transport steps on a {nx}x{rows} full-width row band of the workload "
                      f"(periodic band), {el:.1f} s, 1 thread"}


def run_reference(args, rank, world):
    """--impl reference: the oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return
    system, nx, ny, desc = WORKLOADS[args.workload]
    import oracle as O
    from paper_1701_05431_b200 import inputs
    if system == "spray":
        # ~1 M cell-updates/s: a 2-row band keeps the whole run within minutes
        spray_band_oracle(nx, ny, 2, 0.0, steps=args.warmup)
        val, n, el = spray_band_oracle(nx, ny, 2, 0.0, steps=args.steps)
        sample = f"each step = one oracle spray step (transport + source) on a {nx}x2 full-width row band"
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.workload, "description": desc, "nx": nx, "ny": ny,
                                            "sample_rows": 2},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    # size the band so that warmup + steps take ~60 s of CPU at ~10 M cell-updates/s
    total = max(1, args.steps + args.warmup)
    rows = int(max(2, min(ny, 60e6 / total / nx)))
    band = inputs.euler_lax_liu3(nx, ny, rows=(ny // 2 - rows // 2, ny // 2 - rows // 2 + rows), gamma=GAMMA)
    cfg = O.Config(nx=nx, ny=rows, system=O.EULER, param=(GAMMA,), y1=rows / ny)
    dt = CFL * (1.0 / nx) / 2.5
    W = band
    for _ in range(args.warmup):
        W = O.transport_step(cfg, W, dt)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        W = O.transport_step(cfg, W, dt)
    el = time.perf_counter() - t0
    val = nx * rows * args.steps / el
    sample = f"each step = one oracle transport step on a {nx}x{rows} full-width row band of the workload"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.workload, "description": desc, "nx": nx, "ny": ny,
                                        "sample_rows": rows},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3_euler_16384", choices=sorted(WORKLOADS))
    ap.add_argument("--naive", action="store_true", help="paper's one-thread-per-cell kernel (baseline)")
    ap.add_argument("--one-cell", action="store_true", help="one-cell-per-lane fused kernel (default: two)")
    ap.add_argument("--peer-halo", action="store_true",
                    help="N>1: peer-memory path (the default for N>1; kept for compatibility)")
    ap.add_argument("--nccl", action="store_true",
                    help="N>1: the NCCL baseline (halo send/recv overlapped with the interior, ncclAllReduce) "
                         "instead of the fused peer-memory path")
    ap.add_argument("--adaptive", action="store_true", help="adaptive dt (smax reduced in the epilogue)")
    ap.add_argument("--nranks-x", type=int, default=1,
                    help="N>1: the ranks as a PX x (N/PX) grid of 2-D blocks (E/W ghost columns) instead of y-slabs")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--shared-gpu", action="store_true",
                    help="test mode: every rank on cuda:0 with gloo for the host-side collectives "
                         "(peer-memory path only: NCCL refuses two ranks on one GPU); not a scaling measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1701_05431_b200 import dist as D
    from paper_1701_05431_b200 import fv2d

    if args.shared_gpu:
        if world > 1 and args.nccl:
            raise SystemExit("--shared-gpu needs the peer-memory path (NCCL refuses two ranks on one GPU)")
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if args.shared_gpu else "cuda"  # device of the max-over-ranks reductions
    system, nx, ny_global, desc = WORKLOADS[args.workload]
    weak = args.workload.startswith("c5")
    ny = ny_global * world if weak else ny_global
    px = max(1, args.nranks_x)
    if world % px or ny % (world // px) or nx % px:
        raise SystemExit(f"{nx}x{ny} cells do not split into {px}x{world // px} blocks")
    j0, j1, i0, i1 = D.block_of(rank, px, world // px, nx, ny)
    H = j1 - j0
    # N > 1: the fused peer-memory path by default (each step ONE kernel: flux,
    # update, halo rows/columns stored into the neighbours' ghost cells over
    # NVLink, CFL max-all-reduce by system-scope atomics in its last CTA); the
    # NCCL path is the baseline (--nccl) and the fallback if CUDA IPC between
    # the ranks fails (decided collectively, so every rank takes the same path)
    peer = world > 1 and not args.nccl
    stream = torch.cuda.current_stream()
    spray = system == "spray"
    base_flags = (fv2d.FLAG_NAIVE if args.naive else 0) | (fv2d.FLAG_ONE_CELL if args.one_cell else 0)

    def make_solver(use_peer):
        nid = None
        if world > 1 and not use_peer:
            nid = D.broadcast_bytes(fv2d.nccl_unique_id() if rank == 0 else None)
        return fv2d.Solver(nx, ny, fv2d.SPRAY if spray else fv2d.EULER, param=(1.0, 1.0) if spray else (GAMMA,),
                           rank=rank, nranks=world, device=local,
                           flags=base_flags | (fv2d.FLAG_PEER_HALO if use_peer else 0), nranks_x=px,
                           nccl_id=nid, stream=stream.cuda_stream)

    s = None
    if peer:
        # every rank reaches every collective below whatever fails where
        h = None
        try:
            s = make_solver(True)
            h = s.peer_export()
        except fv2d.FV2DError as e:
            print(f"rank {rank}: peer-memory path unavailable ({e})", file=sys.stderr, flush=True)
        handles = [None] * world
        dist.all_gather_object(handles, h)
        ok = 1.0 if all(x is not None for x in handles) else 0.0
        if ok:
            try:
                s.peer_connect(b"".join(handles))
            except fv2d.FV2DError as e:
                print(f"rank {rank}: peer_connect failed ({e})", file=sys.stderr, flush=True)
                ok = 0.0
        (neg_ok,) = D.max_over_ranks([-ok], device="cpu" if args.shared_gpu else "cuda")
        if -neg_ok < 1.0:  # some rank failed: all take the NCCL path
            if rank == 0:
                print("peer-memory path unavailable on some rank: using NCCL", file=sys.stderr, flush=True)
            if s is not None:
                s.close()
            s, peer = None, False
    if s is None:
        s = make_solver(False)
    W0 = gen_ic(system, nx, ny, (j0, j1))
    if px > 1:
        W0 = np.ascontiguousarray(W0[:, i0:i1])
    s.set_state(W0)
    dt, smax0 = s.compute_dt(CFL)    # the paper's constant dt, set at start
    if spray:
        dt = 0.5 * min(1.0 / nx, 1.0 / ny) / smax0   # R17

    def steps(k):
        if args.adaptive:
            s.step_adaptive(CFL, k, log=False)
        else:
            s.step(dt, k)

    steps(args.warmup)
    s.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed
    st0 = s.stats()
    s.set_profiling(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        steps(args.steps)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    st1 = s.stats()
    s.set_profiling(False)
    s.synchronize()                      # no latched CFL/non-finite error in the timed steps
    kern_ms = st1["step_kernel_ms"] / max(1, st1["step_kernels_timed"])
    src_ms = st1["source_kernel_ms"] / max(1, st1["source_kernels_timed"])
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    ms_max, kern_max, src_max = D.max_over_ranks([ms, kern_ms, src_ms], device=red_dev)
    cells_total = nx * ny
    value = cells_total * args.steps / (ms_max * 1e-3)

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        hostbuf = torch.empty(W0.size, dtype=torch.float64, pin_memory=True)
        hostbuf.numpy()[:] = W0.ravel()
        ptr = hostbuf.data_ptr()
        s.set_state_ptr(ptr)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            # one step host -> host: H2D of W^n (pinned AoS), step, D2H of W^{n+1},
            # in place; row bands pipelined so both copy directions and the kernels overlap
            s.step_host(ptr, ptr, dt, 1)
        e1.record(stream)
        barrier()
        (et,) = D.max_over_ranks([e0.elapsed_time(e1)], device=red_dev)
        nbytes = W0.size * 8
        e2e = {"value": cells_total * args.e2e_steps / (et * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "api": "fv2d_step_host(host AoS in -> host AoS out, pinned, in place; banded copy/compute overlap" +
                      ("; a new W^0 each step, so the source's Newton starts cold)" if spray else ")")}
        del hostbuf

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(nx, ny, system=system)

    if rank == 0:
        peak, peak_src = measured_peaks()
        bpc = BYTES_PER_CELL[system]
        cells_per_launch = (i1 - i0) * H
        achieved = bpc * cells_per_launch / (kern_max * 1e-3) / 1e9
        kernel = ("fv_step_naive_kernel<Euler>" if args.naive else
                  "fv_step_kernel<Euler> (one cell/lane)" if args.one_cell else "fv_step_pair_kernel<Euler>")
        traffic = ncu_traffic(kernel)
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                    "bytes_per_cell": bpc, "kernel_ms": kern_max, "cells_per_launch": cells_per_launch}
        if spray:
            # the dominant kernel is the source pass: FP64-bound (arithmetic intensity
            # ~14 flop/B, far above the FP64 ridge of ~5.7 flop/B)
            kernel = "spray_source_step_kernel (+ fv_step_kernel<Spray> transport)"
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))["spray_source_step_kernel"]
            fpc = prof["fp64_flops_per_cell"]
            ach = fpc * cells_per_launch / (src_max * 1e-3) / 1e12
            roofline = {"bound": "alu", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": ach / FP64_PEAK_TFLOPS, "traffic": prof["dram_bytes_per_launch"],
                        "peak_source": "derived: 148 SMs x 64 FP64 lanes x 2 flop (DFMA) x 1.965 GHz",
                        "flops_per_cell": fpc, "flops_per_cell_source": "ncu DFMA/DADD/DMUL counts "
                        "(profiles/ncu_summary.json), steady state", "kernel_ms": src_max,
                        "cells_per_launch": cells_per_launch,
                        "arithmetic_intensity_flop_per_byte": prof["arithmetic_intensity_flop_per_byte"],
                        "transport_kernel": {"bound": "hbm", "achieved_gbs": achieved, "peak_gbs": peak,
                                             "frac": achieved / peak, "bytes_per_cell": bpc,
                                             "kernel_ms": kern_max}}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "description": desc, "nx": nx, "ny": ny,
                       "rows_per_gpu": H, "cols_per_gpu": i1 - i0,
                       "mode": "adaptive dt" if args.adaptive else "fixed dt (checked)",
                       "dt": dt, "kernel": kernel,
                       **({"newton_iters_per_cell_step": (st1["newton_iters"] - st0["newton_iters"]) /
                           (cells_per_launch * args.steps)} if spray else {}),
                       "parallelism": (f"y-slabs x{world}" if px == 1 else f"2-D blocks {px}x{world // px}") + (
                           (" (peer memory: halo stores + all-reduce fused in the step kernel)" if peer else
                            " (NCCL halo overlapped + all-reduce)")
                           if world > 1 else ""),
                       "l2": "state 2 x %.1f GB >> 126 MB L2, no flush needed" % ((i1 - i0) * H * bpc / 2 / 1e9),
                       **({"test_mode": "all ranks share cuda:0 (--shared-gpu): not a scaling measurement"}
                          if args.shared_gpu else {})},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

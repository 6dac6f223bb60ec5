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
    """GPU clocks, power and clock-event (throttle) reasons, sampled in-process
    through NVML every 10 ms from before the warm-up to the end of the run.
    Each sample carries the phase label current when it was taken, so the
    summary covers exactly the timed repetitions (or the sustained run)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device):
        self.device = device
        self.phase = "setup"
        self.samples = []            # (phase, sm_mhz, reasons bitmask, power_w)
        self.sm_max = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            # CUDA device index -> NVML index (NVML ignores CUDA_VISIBLE_DEVICES)
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
            if vis and vis[0].strip() and self.device < len(vis) and vis[self.device].strip().isdigit():
                idx = int(vis[self.device])
            h = N.nvmlDeviceGetHandleByIndex(idx)
            self._nvml, self._h = N, h
            self.sm_max = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # no NVML: clocks stay unmeasured (reported as such)
            self._err = repr(e)
        return self

    def sample_now(self):
        """One sample from the calling thread (the timed loop calls this right
        after issuing a repetition's steps, while the GPU runs them, so even a
        repetition shorter than the 10 ms period has a sample)."""
        if self._nvml is None:
            return
        N, h = self._nvml, self._h
        try:
            sm = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
            rs = int(N.nvmlDeviceGetCurrentClocksEventReasons(h))
            pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
            self.samples.append((self.phase, sm, rs, pw))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample_now()
            self._stop.wait(0.01)

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)
            try:
                self._nvml.nvmlShutdown()
            except Exception:
                pass

    def summary(self, phase="timed"):
        rows = [x for x in self.samples if x[0] == phase]
        reasons = sorted(n for n, bit in self.REASONS.items() if any(r & bit for _, _, r, _ in rows))
        sm = [x[1] for x in rows]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.sm_max,
                "sm_mhz_min": min(sm) if sm else None, "reasons": reasons, "samples": len(rows),
                "power_w_median": float(np.median([x[3] for x in rows])) if rows else None,
                "source": "NVML in-process, 10 ms" if self._nvml is not None else
                          f"unavailable ({getattr(self, '_err', '?')})"}


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cores": os.cpu_count(), "cpu_model": model}


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
        return {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", **host_info(),
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
    return {"value": nx * rows * steps / el, "unit": UNIT, "cores": 1, "kind": "oracle", **host_info(),
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
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             **host_info()},
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
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             **host_info()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def sha_state(W):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(W).tobytes()).hexdigest()


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
    ap.add_argument("--reps", type=int, default=5, help="timed repetitions of --steps steps (median reported)")
    ap.add_argument("--sustained-s", type=float, default=1.5,
                    help="length of the extra sustained run (power-cap steady state), 0 to skip")
    ap.add_argument("--check-steps", type=int, default=3,
                    help="N>1: steps of the peer-path self-check against a reference path before timing")
    ap.add_argument("--inject-peer-fault", action="store_true",
                    help="test: rank 1 reports a self-check mismatch (exercises the fallback decision)")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="test mode: every rank on cuda:0 with gloo for the host-side collectives "
                         "(peer-memory path only: NCCL refuses two ranks on one GPU); not a scaling measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.reps = max(1, args.reps)

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
    # NCCL path is the measured baseline (nccl_baseline in the line; --nccl to
    # time it alone) and the fallback if CUDA IPC between the ranks fails or
    # the peer path's self-check disagrees (decided collectively, so every rank
    # takes the same path)
    peer = world > 1 and not args.nccl
    have_nccl = world > 1 and not args.shared_gpu
    stream = torch.cuda.current_stream()
    spray = system == "spray"
    base_flags = (fv2d.FLAG_NAIVE if args.naive else 0) | (fv2d.FLAG_ONE_CELL if args.one_cell else 0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def make_solver(use_peer):
        nid = None
        if world > 1 and not use_peer:
            nid = D.broadcast_bytes(fv2d.nccl_unique_id() if rank == 0 else None)
        return fv2d.Solver(nx, ny, fv2d.SPRAY if spray else fv2d.EULER, param=(1.0, 1.0) if spray else (GAMMA,),
                           rank=rank, nranks=world, device=local,
                           flags=base_flags | (fv2d.FLAG_PEER_HALO if use_peer else 0), nranks_x=px,
                           nccl_id=nid, stream=stream.cuda_stream)

    clk = ClockSampler(local).__enter__()     # sampling from before the warm-up
    s = None
    s_nccl = None
    peer_check = None
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
        (neg_ok,) = D.max_over_ranks([-ok], device=red_dev)
        if -neg_ok < 1.0:  # some rank failed: all take the NCCL path
            if rank == 0:
                print("peer-memory path unavailable on some rank: using NCCL", file=sys.stderr, flush=True)
            if s is not None:
                s.close()
            s, peer = None, False
            peer_check = {"ok": False, "reason": "CUDA IPC setup failed on some rank", "fallback": "nccl"}
    if s is None:
        if args.shared_gpu and world > 1:
            raise SystemExit("--shared-gpu: the peer-memory path is unavailable and NCCL cannot share one GPU")
        s = make_solver(False)
    elif have_nccl:
        s_nccl = make_solver(False)   # the baseline, the self-check reference and the fallback
    W0 = gen_ic(system, nx, ny, (j0, j1))
    if px > 1:
        W0 = np.ascontiguousarray(W0[:, i0:i1])
    s.set_state(W0)
    dt, smax0 = s.compute_dt(CFL)    # the paper's constant dt, set at start
    if spray:
        dt = 0.5 * min(1.0 / nx, 1.0 / ny) / smax0   # R17

    def run_steps(sol, k):
        if args.adaptive:
            sol.step_adaptive(CFL, k, log=False)
        else:
            sol.step(dt, k)

    # ------------------------------------------- N > 1: peer-path self-check
    if peer:
        k = max(1, args.check_steps)
        err = None
        hp = ""
        try:
            s.set_state(W0)
            run_steps(s, k)
            hp = sha_state(s.get_state())
        except fv2d.FV2DError as e:
            err = str(e)
        if s_nccl is not None:
            ref_kind = "the NCCL path on the same ranks"
            s_nccl.set_state(W0)
            run_steps(s_nccl, k)
            hr = sha_state(s_nccl.get_state())
        else:
            # --shared-gpu (no NCCL): rank 0 steps the whole domain as one rank
            ref_kind = "one rank over the whole domain (rank 0)"
            blocks = None
            if rank == 0:
                Wf = gen_ic(system, nx, ny, (0, ny))
                with fv2d.Solver(nx, ny, fv2d.SPRAY if spray else fv2d.EULER,
                                 param=(1.0, 1.0) if spray else (GAMMA,), device=local, flags=base_flags) as r1:
                    r1.set_state(Wf)
                    run_steps(r1, k)
                    Wr = r1.get_state()
                blocks = []
                for r in range(world):
                    b0, b1, c0, c1 = D.block_of(r, px, world // px, nx, ny)
                    blocks.append(sha_state(Wr[b0:b1, c0:c1]))
                del Wf, Wr
            obj = [blocks]
            dist.broadcast_object_list(obj, src=0)
            hr = obj[0][rank]
        bad = err is not None or hp != hr or (args.inject_peer_fault and rank == 1)
        flags_bad = [0.0] * world
        flags_bad[rank] = 1.0 if bad else 0.0
        bad_ranks = [r for r, v in enumerate(D.max_over_ranks(flags_bad, device=red_dev)) if v > 0]
        peer_check = {"ok": not bad_ranks, "steps": k, "reference": ref_kind, "compared": "sha256 of each rank's "
                      "state after the steps", "mismatch_ranks": bad_ranks,
                      **({"injected_fault": True} if args.inject_peer_fault else {})}
        if bad_ranks:
            if rank == 0:
                print(f"peer-memory path self-check failed on ranks {bad_ranks}" +
                      (" (injected)" if args.inject_peer_fault else "") + ": falling back to NCCL" +
                      ("" if s_nccl is not None else " -- unavailable (--shared-gpu)"), file=sys.stderr, flush=True)
            if s_nccl is None:
                peer_check["fallback"] = "none available (--shared-gpu: no NCCL on one GPU)"
                if rank == 0:
                    print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                                      "error": "peer-memory self-check failed", "peer_check": peer_check}),
                          flush=True)
                clk.__exit__()
                s.close()
                dist.destroy_process_group()
                return
            peer_check["fallback"] = "nccl"
            s.close()
            s, s_nccl, peer = s_nccl, None, False

    # ---------------------------------------------------------------- timed
    def timed(sol, phase, k, reps):
        """reps repetitions of exactly k steps, each bracketed by a barrier and a
        device synchronize; CUDA events on the library's stream; per repetition
        the max over ranks.  Returns (per-rep ms list, kernel ms, source ms, launches)."""
        st0 = sol.stats()
        sol.set_profiling(True)
        per_rep = []
        for _ in range(reps):
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            barrier()
            clk.phase = phase
            ev0.record(stream)
            run_steps(sol, k)
            clk.sample_now()
            ev1.record(stream)
            barrier()
            clk.phase = "between"
            per_rep.append(ev0.elapsed_time(ev1))
        st1 = sol.stats()
        sol.set_profiling(False)
        sol.synchronize()                      # no latched CFL/non-finite error in the timed steps
        kern = st1["step_kernel_ms"] / max(1, st1["step_kernels_timed"])
        src = st1["source_kernel_ms"] / max(1, st1["source_kernels_timed"])
        red = D.max_over_ranks(per_rep + [kern, src], device=red_dev)
        return red[:reps], red[reps], red[reps + 1], (st1["kernel_launches"] - st0["kernel_launches"]) / reps, st0, st1

    s.set_state(W0)
    run_steps(s, args.warmup)
    s.synchronize()
    reps_ms, kern_max, src_max, launches, st0, st1 = timed(s, "timed", args.steps, args.reps)
    ms_max = float(np.median(reps_ms))
    cells_total = nx * ny
    value = cells_total * args.steps / (ms_max * 1e-3)
    newton = (st1["newton_iters"] - st0["newton_iters"]) / ((i1 - i0) * H * args.steps * args.reps)

    sustained = None
    if args.sustained_s > 0:
        nsus = max(args.steps, int(np.ceil(args.sustained_s * 1e3 / (ms_max / args.steps))))
        sus_ms, sus_kern, sus_src, _, _, _ = timed(s, "sustained", nsus, 1)
        sustained = {"steps": nsus, "seconds": sus_ms[0] / 1e3, "ms_per_step": sus_ms[0] / nsus,
                     "value": cells_total * nsus / (sus_ms[0] * 1e-3), "kernel_ms": sus_kern,
                     "source_kernel_ms": sus_src if spray else None, "clocks": clk.summary("sustained")}

    nccl_baseline = None
    if s_nccl is not None:
        # the north_star's mechanism, timed on the same ranks and workload
        s_nccl.set_state(W0)
        run_steps(s_nccl, args.warmup)
        s_nccl.synchronize()
        n_ms, n_kern, _, n_launch, _, _ = timed(s_nccl, "nccl", args.steps, args.reps)
        nm = float(np.median(n_ms))
        nccl_baseline = {"ms_per_step": nm / args.steps, "value": cells_total * args.steps / (nm * 1e-3),
                         "ms_per_step_min": min(n_ms) / args.steps, "ms_per_step_max": max(n_ms) / args.steps,
                         "interior_kernel_ms": n_kern, "gpu_launches": n_launch,
                         "path": "boundary rows + NCCL send/recv on a comm stream overlapped with the interior "
                                 "launch, ncclAllReduce(max) of [smax, status], finalize kernel"}
        s_nccl.close()
        s_nccl = None

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        hostbuf = torch.empty(W0.size, dtype=torch.float64, pin_memory=True)
        hostbuf.numpy()[:] = W0.ravel()
        ptr = hostbuf.data_ptr()
        s.set_state_ptr(ptr)
        barrier()
        clk.phase = "e2e"
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            # one step host -> host: H2D of W^n (pinned AoS), step, D2H of W^{n+1},
            # in place; row bands pipelined so both copy directions and the kernels overlap
            s.step_host(ptr, ptr, dt, 1)
        e1.record(stream)
        barrier()
        clk.phase = "between"
        (et,) = D.max_over_ranks([e0.elapsed_time(e1)], device=red_dev)
        nbytes = W0.size * 8
        e2e = {"value": cells_total * args.e2e_steps / (et * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "api": "fv2d_step_host(host AoS in -> host AoS out, pinned, in place" +
                      ("; the spray's first step needs all of W^0 on the device for the S:440 guard, so its "
                       "copies are not overlapped; a new W^0 each step, so the source's Newton starts cold)"
                       if spray else "; banded copy/compute overlap)")}
        del hostbuf
    clk.__exit__()

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
                    "bytes_per_cell": bpc, "kernel_ms": kern_max, "cells_per_launch": cells_per_launch,
                    **({"sustained_frac": bpc * cells_per_launch / (sustained["kernel_ms"] * 1e-3) / 1e9 / peak}
                       if sustained else {})}
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
                        # the same kernel against the FP64 pipe's INSTRUCTION rate (a DADD or DMUL
                        # occupies the pipe like a DFMA but counts 1 flop, so a mixed kernel cannot
                        # reach the DFMA flop peak): 148 SMs x 64 lanes x 1.965 GHz
                        "fp64_instr_per_cell": prof["fp64_instr_per_cell"],
                        "fp64_instr_frac": prof["fp64_instr_per_cell"] * cells_per_launch / (src_max * 1e-3)
                        / (FP64_PEAK_TFLOPS * 1e12 / 2),
                        **({"sustained_frac": fpc * cells_per_launch / (sustained["source_kernel_ms"] * 1e-3)
                            / 1e12 / FP64_PEAK_TFLOPS} if sustained else {}),
                        "transport_kernel": {"bound": "hbm", "achieved_gbs": achieved, "peak_gbs": peak,
                                             "frac": achieved / peak, "bytes_per_cell": bpc,
                                             "kernel_ms": kern_max}}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "repetitions": args.reps, "ms_per_step_min": min(reps_ms) / args.steps,
            "ms_per_step_max": max(reps_ms) / args.steps,
            "timing": f"median of {args.reps} repetitions of exactly {args.steps} steps, each bracketed by a "
                      "barrier + cudaDeviceSynchronize, CUDA events on the library's stream, max over ranks",
            "config": {"workload": args.workload, "description": desc, "nx": nx, "ny": ny,
                       "rows_per_gpu": H, "cols_per_gpu": i1 - i0,
                       "mode": "adaptive dt" if args.adaptive else "fixed dt (checked)",
                       "dt": dt, "kernel": kernel,
                       **({"newton_iters_per_cell_step": newton} if spray else {}),
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
            "clocks": clk.summary("timed"),
            "sustained": sustained,
            **({"peer_check": peer_check, "nccl_baseline": nccl_baseline} if world > 1 else {}),
        }
        print(json.dumps(out), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

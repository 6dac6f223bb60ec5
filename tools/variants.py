"""Build / time compile-time variants of libfv2d.so (tuning A/B).

  python tools/variants.py build NAME=DEF[,DEF...] ...      # here (nvcc cross-compiles)
  python tools/variants.py run --workload W [--steps K] NAME ...   # on the GPU box

Variants live in paper_1701_05431_b200/lib/variants/lib<NAME>.so (git-ignored,
shipped by gpurun).  `run` times each with bench.py (FV2D_LIB=...) and prints
one JSON line per variant with the median ms/step, the dominant kernel's time
and roofline fraction; `base` means the default build.
"""
from __future__ import annotations

import concurrent.futures as cf
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_1701_05431_b200", "lib", "variants")


def build(specs):
    from paper_1701_05431_b200 import build as b
    os.makedirs(VDIR, exist_ok=True)

    def one(spec):
        name, _, defs = spec.partition("=")
        out = os.path.join(VDIR, f"lib{name}.so")
        b.build(out=out, defines=[d for d in defs.split(",") if d])
        return name

    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        for name in ex.map(one, specs):
            print("built", name, flush=True)


def run(names, workload, steps, extra):
    for name in names:
        env = dict(os.environ)
        if name != "base":
            env["FV2D_LIB"] = os.path.join(VDIR, f"lib{name}.so")
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", workload, "--steps", str(steps),
               "--warmup", "5", "--no-cpu-baseline", "--no-e2e", *extra]
        r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        if r.returncode or not line:
            print(json.dumps({"variant": name, "error": r.stderr[-800:]}), flush=True)
            continue
        d = json.loads(line[0])
        rf = d["roofline"]
        out = {"variant": name, "ms_per_step": d["ms_per_step"], "min": d["ms_per_step_min"],
               "max": d["ms_per_step_max"], "kernel_ms": rf["kernel_ms"], "frac": rf["frac"],
               "sm_mhz": d["clocks"]["sm_mhz"], "reasons": d["clocks"]["reasons"]}
        if d.get("sustained"):
            out["sustained_ms_per_step"] = d["sustained"]["ms_per_step"]
            out["sustained_frac"] = rf.get("sustained_frac")
        if "newton_iters_per_cell_step" in d["config"]:
            out["newton"] = d["config"]["newton_iters_per_cell_step"]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("names", nargs="+")
        ap.add_argument("--workload", default="c4_spray_4096")
        ap.add_argument("--steps", type=int, default=50)
        ap.add_argument("--sustained-s", default="0")
        ap.add_argument("--adaptive", action="store_true")
        a = ap.parse_args()
        run(a.names, a.workload, a.steps, ["--sustained-s", a.sustained_s] + (["--adaptive"] if a.adaptive else []))

"""bench.py's reference arm runs on CPU (the oracle, bounded sample) and prints
the contract's JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "cell-updates/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "c3_euler_16384"


import pytest


@pytest.mark.gpu
def test_bench_json_contract_on_gpu():
    """bench.py (our arm) prints one JSON line with the driver contract's keys,
    the roofline and cpu_baseline objects, e2e through host buffers, clocks."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c2_euler_1024", "--steps", "20",
                        "--warmup", "3", "--e2e-steps", "2"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 1e9 and d["n_gpus"] == 1 and d["dtype"] == "f64" and d["gpu_launches"] == 20
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and 0 < rf["frac"] < 1.5 and rf["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 1024 * 1024 * 32 and d["e2e"]["value"] > 0
    assert d["config"]["workload"] == "c2_euler_1024"

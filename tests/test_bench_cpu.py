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
    assert d["cpu_baseline"]["host_cores"] >= 1 and "cpu_model" in d["cpu_baseline"]
    assert d["e2e"]["h2d_bytes_per_step"] == 1024 * 1024 * 32 and d["e2e"]["value"] > 0
    assert d["config"]["workload"] == "c2_euler_1024"
    # protocol: median of repetitions, in-process clock samples inside the timed region, sustained run
    assert d["repetitions"] == 5 and d["ms_per_step_min"] <= d["ms_per_step"] <= d["ms_per_step_max"]
    assert d["clocks"]["samples"] > 0 and d["clocks"]["sm_mhz"] > 0
    assert d["sustained"]["seconds"] >= 1.0 and d["sustained"]["clocks"]["samples"] > 50
    assert 0 < d["roofline"]["sustained_frac"] < 1.5


@pytest.mark.gpu
@pytest.mark.parametrize("px", [1, 2])
def test_bench_multi_rank_launch_on_one_gpu(px):
    """The N>1 bench flow under torch.distributed.run (2 ranks), as far as one
    GPU allows: --shared-gpu puts both ranks on cuda:0 with the peer-memory path
    (CUDA IPC) and gloo for the host collectives.  One JSON line from rank 0,
    n_gpus = 2, max-over-ranks timing; y-slabs (px = 1) or 2-D blocks (px = 2)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--shared-gpu", "--nranks-x", str(px), "--workload", "c2_euler_1024", "--steps", "10", "--warmup", "3",
           "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["test_mode"].startswith("all ranks share cuda:0")
    assert ("2-D blocks 2x1" if px == 2 else "y-slabs x2") in d["config"]["parallelism"]
    assert d["cpu_baseline"] is None and d["e2e"]["value"] > 0
    pc = d["peer_check"]
    assert pc["ok"] is True and pc["steps"] == 3 and pc["reference"].startswith("one rank over the whole domain")
    assert d["nccl_baseline"] is None        # NCCL cannot put two ranks on one GPU


@pytest.mark.gpu
def test_bench_peer_self_check_forced_failure():
    """--inject-peer-fault: rank 1 reports a self-check mismatch; every rank
    takes the same decision (fall back to NCCL -- which --shared-gpu cannot
    provide, so the line reports the failed check instead of a number) and the
    run exits cleanly instead of timing a path it cannot trust."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--shared-gpu", "--workload", "c2_euler_1024", "--steps", "5", "--warmup", "3", "--inject-peer-fault"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["value"] is None and d["peer_check"]["ok"] is False and d["peer_check"]["mismatch_ranks"] == [1]
    assert d["peer_check"]["fallback"].startswith("none available")
    assert "falling back to NCCL" in r.stderr


def test_reference_arm_spray_workload():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                        "c4_spray_4096", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == "c4_spray_4096"


@pytest.mark.gpu
def test_bench_spray_workload_fp64_roofline():
    """bench.py --workload c4_spray_4096: the source pass is the dominant kernel;
    its roofline is FP64 ("alu", TFLOP/s) with the measured arithmetic intensity."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c4_spray_4096", "--steps", "10",
                        "--warmup", "3", "--e2e-steps", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    rf = d["roofline"]
    assert rf["bound"] == "alu" and rf["unit"] == "TFLOP/s" and 0 < rf["frac"] < 1
    assert rf["arithmetic_intensity_flop_per_byte"] > 5.7        # above the FP64 ridge
    assert 0 < rf["fp64_instr_frac"] < 1 and rf["fp64_instr_per_cell"] > 0   # the pipe's instruction rate
    assert rf["transport_kernel"]["bound"] == "hbm"
    assert d["value"] > 1e9 and d["e2e"]["value"] > 0 and d["cpu_baseline"]["value"] > 0
    assert 0.5 < d["config"]["newton_iters_per_cell_step"] < 3

"""Build libfv2d.so in-tree for sm_100a (nvcc; cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "lib", "libfv2d.so")
SOURCES = [os.path.join(HERE, "csrc", "fv2d_api.cu")]
DEPS = SOURCES + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "fv2d.h")]


def nccl_include() -> str:
    import nvidia.nccl  # torch's NCCL wheel (headers + libnccl.so.2)
    base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include")


def nvcc_cmd(out: str, verbose_ptxas: bool = False, defines=()) -> list[str]:
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", *[f"-D{d}" for d in defines],
           "--fmad=false",                 # exact build: no FMA contraction
           "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", nccl_include(),
           *SOURCES, "-o", out, "-ldl"]
    if verbose_ptxas:
        cmd += ["-Xptxas", "-v"]
    return cmd


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libfv2d.so (or, with `out`, a tuning variant with extra -D defines)."""
    target = out or LIB
    if out is None and not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    tmp = target + f".tmp{os.getpid()}"
    cmd = nvcc_cmd(tmp, verbose, defines)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libfv2d.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

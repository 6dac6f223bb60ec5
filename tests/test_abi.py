"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads, and
exports every symbol include/fv2d.h declares; host-side argument validation.
(No compute calls: there is no GPU here.)"""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1701_05431_b200 import fv2d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fv2d.h")).read()
    return sorted(set(re.findall(r"^fv2d_status\s+(fv2d_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = fv2d.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", fv2d.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fv2d_\w+)", out))
    for s in syms:
        assert s in exported, s
        assert getattr(L, s) is not None


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", fv2d.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_struct_matches_header():
    # 6 int32 + 4 doubles + 8 + 6 doubles + 4 int32 + uint32 + 7 int32 (with padding)
    assert C.sizeof(fv2d.Config) == 24 + 32 + 64 + 48 + 16 + 4 + 28
    cfg = fv2d.Config()
    assert fv2d.lib().fv2d_config_default(C.byref(cfg), 64, 32, fv2d.EULER) == fv2d.OK
    assert (cfg.nx, cfg.ny, cfg.nvar, cfg.param[0], cfg.nranks, cfg.nslabs) == (64, 32, 4, 1.4, 1, 1)
    assert fv2d.lib().fv2d_config_default(C.byref(cfg), 64, 32, 7) == fv2d.E_ARG


def test_create_validates_before_touching_the_device():
    L = fv2d.lib()
    h = C.c_void_p()
    cfg = fv2d.Config()
    L.fv2d_config_default(C.byref(cfg), 64, 30, fv2d.EULER)
    cfg.nslabs = 4                      # 30 % 4 != 0
    assert L.fv2d_create(C.byref(cfg), None, None, C.byref(h)) == fv2d.E_ARG
    cfg.nslabs = 1
    cfg.nvar = 3                        # nvar mismatch
    assert L.fv2d_create(C.byref(cfg), None, None, C.byref(h)) == fv2d.E_ARG
    cfg.nvar = 4
    cfg.param[0] = 1.0                  # gamma <= 1
    assert L.fv2d_create(C.byref(cfg), None, None, C.byref(h)) == fv2d.E_ARG
    L.fv2d_config_default(C.byref(cfg), 8, 8, fv2d.ADVECTION)
    cfg.bc_x = fv2d.BC_WALL             # wall undefined for advection
    assert L.fv2d_create(C.byref(cfg), None, None, C.byref(h)) == fv2d.E_ARG
    L.fv2d_config_default(C.byref(cfg), 8, 8, fv2d.SPRAY)
    cfg.flags = fv2d.FLAG_FUSE_SOURCE       # removed one-pass spray step (reserved bit)
    assert L.fv2d_create(C.byref(cfg), None, None, C.byref(h)) == fv2d.E_ARG
    assert L.fv2d_step(None, 1e-3, 1) == fv2d.E_ARG
    assert L.fv2d_destroy(None) == fv2d.OK


def test_create_validates_2d_rank_blocks():
    """nranks_x (2-D blocks): nranks % nranks_x == 0, nx % nranks_x == 0, blocks
    at least 2 columns wide, ny divisible by the block rows, one slab per rank."""
    L = fv2d.lib()
    h = C.c_void_p()
    cfg = fv2d.Config()
    for (nx, ny, nranks, px, nslabs) in [(64, 32, 4, 3, 1),   # 4 % 3
                                         (66, 32, 4, 4, 1),   # 66 % 4
                                         (6, 32, 4, 4, 1),    # 6 % 4 (and < 2 columns)
                                         (4, 32, 4, 4, 1),    # 1-column blocks
                                         (64, 30, 8, 2, 1),   # 30 % (8/2)
                                         (64, 32, 4, 2, 2),   # slabs with blocks
                                         (64, 32, 4, -1, 1),
                                         (64, 32, 2, 4, 1),   # nranks_x > nranks (was a SIGFPE)
                                         (64, 32, 1, 2, 1)]:  # nranks_x > nranks = 1
        L.fv2d_config_default(C.byref(cfg), nx, ny, fv2d.EULER)
        cfg.nranks, cfg.nranks_x, cfg.nslabs = nranks, px, nslabs
        cfg.flags = fv2d.FLAG_PEER_HALO
        assert L.fv2d_create(C.byref(cfg), None, None, C.byref(h)) == fv2d.E_ARG, (nx, ny, nranks, px, nslabs)
    L.fv2d_config_default(C.byref(cfg), 64, 32, fv2d.EULER)
    cfg.reserved[0] = 1                 # reserved words must be 0
    assert L.fv2d_create(C.byref(cfg), None, None, C.byref(h)) == fv2d.E_ARG


def test_c_client_compiles_against_the_header():
    """The ABI is usable from plain C (examples/c_client.c): header + .so only."""
    exe = os.path.join(ROOT, "examples", "c_client")
    r = subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "c_client.c"), "-L", os.path.dirname(fv2d.lib_path()),
                        "-lfv2d", f"-Wl,-rpath,{os.path.dirname(fv2d.lib_path())}", "-lm", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_c_client_runs():
    exe = os.path.join(ROOT, "examples", "c_client")
    test_c_client_compiles_against_the_header()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_client ok" in r.stdout


def test_struct_layouts_match_the_c_header(tmp_path):
    """The ctypes mirrors of fv2d_config / fv2d_stats have the C header's size
    and field offsets (compiled and measured with gcc)."""
    src = tmp_path / "layout.c"
    cfg_fields = [f for f, _ in fv2d.Config._fields_]
    st_fields = [f for f, _ in fv2d.Stats._fields_]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "fv2d.h"', "int main(void) {",
             'printf("%zu %zu\\n", sizeof(fv2d_config), sizeof(fv2d_stats));']
    lines += [f'printf("%zu\\n", offsetof(fv2d_config, {f}));' for f in cfg_fields]
    lines += [f'printf("%zu\\n", offsetof(fv2d_stats, {f}));' for f in st_fields]
    lines += ["return 0; }"]
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    r = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()
    sizes, offs = out[:2], [int(x) for x in out[2:]]
    assert int(sizes[0]) == C.sizeof(fv2d.Config) and int(sizes[1]) == C.sizeof(fv2d.Stats)
    got = [getattr(fv2d.Config, f).offset for f in cfg_fields] + [getattr(fv2d.Stats, f).offset for f in st_fields]
    assert offs == got

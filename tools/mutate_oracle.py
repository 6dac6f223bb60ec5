"""Mutation check of the oracle's pins (test infrastructure).

Each mutation is one plausible slip in oracle/fv2d_oracle.c (a dropped term, a
wrong sign, index or operand).  For each, a mutated copy is compiled to a
scratch .so, and the CPU pins (tests/test_oracle_*.py, tests/test_inputs.py)
are run against it through FV2D_ORACLE_LIB.  A mutation must make at least one
pin fail ("caught"); the run fails if any survives.

    python tools/mutate_oracle.py [--out profiles/r2_oracle_mutations.txt]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "fv2d_oracle.c")

# (id, what, old, new): `old` must occur exactly once in the oracle source.
MUTATIONS = [
    ("M1", "Euler x-momentum flux drops the pressure",
     "F[1] = (mx * u) + p;", "F[1] = (mx * u);"),
    ("M2", "spray x-speed |u| -> |u| + |v|/4",
     "F[4] = m2u * u; F[5] = m2v * u;\n      *s = fabs(u);",
     "F[4] = m2u * u; F[5] = m2v * u;\n      *s = fabs(u) + 0.25 * fabs(v);"),
    ("M3", "Dirichlet ghost uses component 0 for every variable",
     "else if (c->bc_x == OR_BC_DIRICHLET) { for (int k = 0; k < nv; ++k) out[k] = c->dirichlet[k]; return; }",
     "else if (c->bc_x == OR_BC_DIRICHLET) { for (int k = 0; k < nv; ++k) out[k] = c->dirichlet[0]; return; }"),
    ("M3b", "Dirichlet y ghost uses component 0 for every variable",
     "else if (c->bc_y == OR_BC_DIRICHLET) { for (int k = 0; k < nv; ++k) out[k] = c->dirichlet[k]; return; }",
     "else if (c->bc_y == OR_BC_DIRICHLET) { for (int k = 0; k < nv; ++k) out[k] = c->dirichlet[0]; return; }"),
    ("M4", "spray wall mirrors index 4 on both axes",
     "else if (c->system == OR_SPRAY) out[4 + mirror_dir] = -out[4 + mirror_dir];",
     "else if (c->system == OR_SPRAY) out[4] = -out[4];"),
    ("M5", "spray y-flux of m2u uses u instead of v",
     "F[4] = m2u * v; F[5] = m2v * v;", "F[4] = m2u * u; F[5] = m2v * v;"),
    ("M6", "Euler wall mirrors index 1 on both axes",
     "if (c->system == OR_EULER) out[1 + mirror_dir] = -out[1 + mirror_dir];",
     "if (c->system == OR_EULER) out[1] = -out[1];"),
    ("M7", "LF uses min instead of max of the speeds",
     "const double hs = 0.5 * dmax(sL, sR);", "const double hs = 0.5 * fmin(sL, sR);"),
    ("M8", "update uses dt/dx in y", "const double ly = dt / dy;", "const double ly = dt / dx;"),
    ("M9", "update sign (+ residual, eq:RHSFilling as printed)",
     "out[k] = C[k] + (-((lx * (Fe[k] - Fw[k])) + (ly * (Fn[k] - Fs[k]))));",
     "out[k] = C[k] + ((lx * (Fe[k] - Fw[k])) + (ly * (Fn[k] - Fs[k])));"),
    ("M10", "sound speed without gamma", "const double cs = sqrt((gamma * p) * inv);",
     "const double cs = sqrt(p * inv);"),
    ("M11", "CFL argmax takes the last tie", "if (s > best) { best = s;", "if (s >= best) { best = s;"),
    ("M12", "fixed-dt check against 2*hmin", "if (dt * smax > hmin) {", "if (dt * smax > 2.0 * hmin) {"),
    ("M13", "Newton Jacobian index mu[k+l]", "A[k][l] = mu[k + l + 1];", "A[k][l] = mu[k + l];"),
    ("M14", "n(0) = exp(+lambda0)", "*n0 = exp(-lam[0]);", "*n0 = exp(lam[0]);"),
    ("M15", "drag sign reversed (x)", "S[4] = (-((K * m0) * u)) + ((m0 * (ugx - u)) / theta);",
     "S[4] = (-((K * m0) * u)) + ((m0 * (u - ugx)) / theta);"),
    ("M16", "m_-1/2 evaporation factor K instead of K/2", "S[1] = -((0.5 * K) * mmh);", "S[1] = -(K * mmh);"),
    ("M17", "m1 evaporation factor K instead of 3K/2", "S[3] = -((1.5 * K) * m1);", "S[3] = -(K * m1);"),
    ("M18", "GL weights not halved", "gl_w[n - 1 - k] = w / 2.0;", "gl_w[n - 1 - k] = w;"),
    ("M19", "Taylor-Green v sign", "*ugy = -(cos(tp * x) * sin(tp * y));", "*ugy = (cos(tp * x) * sin(tp * y));"),
    ("M20", "no polishing Newton step",
     "for (int k = 0; k < 4; ++k) lam[k] = lam[k] + d[k];\n  moments8(lam, mu);",
     "moments8(lam, mu);"),
    ("M21", "S:440 guard factor 1.0 instead of 0.1", "if ((dt * K) > (0.1 * rmin)) {", "if ((dt * K) > (1.0 * rmin)) {"),
    ("M22", "spray mass flux m0*u -> m1*u", "F[0] = m0 * u; F[1] = m1 * u;", "F[0] = m1 * u; F[1] = m1 * u;"),
    ("M23", "Euler energy flux E*u (drops p)", "F[3] = (E + p) * u;", "F[3] = E * u;"),
    ("M24", "kinetic energy without the 1/2", "const double ke = 0.5 * ((mx * u) + (my * v));",
     "const double ke = ((mx * u) + (my * v));"),
    ("M25", "relative residual divided by m[0]", "const double rk = fabs(mu[k + 1] - m[k]) / m[k];",
     "const double rk = fabs(mu[k + 1] - m[k]) / m[0];"),
    ("M26", "y ghost periodic wrap shifted by one", "if (c->bc_y == OR_BC_PERIODIC) jj = ((j % ny) + ny) % ny;",
     "if (c->bc_y == OR_BC_PERIODIC) jj = ((j % ny) + ny + 1) % ny;"),
]

PINS = ["tests/test_oracle_transport.py", "tests/test_oracle_source.py", "tests/test_oracle_boundaries.py",
        "tests/test_inputs.py"]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="comma-separated mutation ids")
    args = ap.parse_args()
    src = open(SRC).read()
    only = set(args.only.split(",")) if args.only else None
    lines, survived = [], []
    with tempfile.TemporaryDirectory() as tmp:
        for mid, what, old, new in MUTATIONS:
            if only and mid not in only:
                continue
            n = src.count(old)
            if n != 1:
                raise SystemExit(f"{mid}: pattern occurs {n} times in the oracle")
            c = os.path.join(tmp, f"{mid}.c")
            so = os.path.join(tmp, f"lib{mid}.so")
            open(c, "w").write(src.replace(old, new))
            subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                                   "-D_DEFAULT_SOURCE", "-shared", "-fPIC", "-o", so, c, "-lm"])
            env = dict(os.environ, FV2D_ORACLE_LIB=so)
            t0 = time.time()
            r = subprocess.run([sys.executable, "-m", "pytest", *PINS, "-x", "-q", "-m", "not gpu",
                                "-p", "no:randomly"], cwd=ROOT, env=env, capture_output=True, text=True,
                               timeout=1800)
            failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            caught = r.returncode != 0
            if not caught:
                survived.append(mid)
            line = (f"{mid:4s} {'caught  ' if caught else 'SURVIVED'} {time.time() - t0:5.1f}s  {what}"
                    + (f"\n       first failing pin: {failed[0]}" if failed else ""))
            print(line, flush=True)
            lines.append(line)
    summary = f"{len(lines) - len(survived)}/{len(lines)} mutations caught" + (
        f"; SURVIVED: {', '.join(survived)}" if survived else "")
    print(summary)
    if args.out:
        with open(args.out, "w") as f:
            f.write("# tools/mutate_oracle.py: each mutation of oracle/fv2d_oracle.c vs the CPU pins\n")
            f.write("\n".join(lines) + "\n" + summary + "\n")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())

"""The pins catch the oracle slips the round-1 review found unpinned (M2 spray
speed, M3 Dirichlet component, M4 spray wall index) and the reconstruction
details of R19 (M20 polishing step, M25 residual normalisation): each mutated
oracle build must fail at least one CPU pin.  The full list (27 mutations) is
`python tools/mutate_oracle.py`, output in profiles/r2_oracle_mutations.txt."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_named_mutations_are_caught():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "mutate_oracle.py"),
                        "--only", "M2,M3,M3b,M4,M20,M25"], cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "6/6 mutations caught" in r.stdout

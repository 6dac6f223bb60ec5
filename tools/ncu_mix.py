"""Per-cell SASS instruction mix of a kernel from an ncu report's source page
(thread instructions executed / cells), e.g. DFMA/DADD/DMUL counts for §8(d)."""
import collections
import csv
import io
import json
import re
import subprocess
import sys

rep, cells = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
isrc, iex = hdr.index("Source"), hdr.index("Thread Instructions Executed")
mix = collections.Counter()
for r in rows[2:]:
    if len(r) > iex and r[iex].isdigit():
        op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split()[0] if r[isrc].strip() else "?"
        mix[op.split(".")[0]] += int(r[iex])
per = {k: round(v / cells, 2) for k, v in mix.most_common()}
fp64 = sum(v for k, v in per.items() if k in ("DADD", "DMUL", "DFMA"))
print(json.dumps({"report": rep, "cells": cells, "thread_instr_per_cell": round(sum(mix.values()) / cells, 1),
                  "fp64_per_cell": round(fp64, 1), "mix_per_cell": per}, indent=1))

"""Summarise the SASS source page of an ncu report: warp-stall samples and
executed instructions aggregated by opcode, the top instructions, and (with
cuda,sass correlation) the top CUDA source lines.  Run where ncu is available.
Usage: ncu_source_top.py REP [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40


def page(view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


rows = page("sass")
hdr = next((r for r in rows if "Address" in r and "Source" in r), None)
if hdr is None:
    print("\n".join(",".join(r) for r in rows[:10]))
    sys.exit(0)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
kst = next((k for k in hdr if k.startswith("Warp Stall Sampling (All")), None)
kex = next((k for k in hdr if k.startswith("Instructions Executed")), None)
print("columns:", hdr)
tot_s = sum(num(d[kst]) for d in data) or 1.0
tot_e = sum(num(d[kex]) for d in data) or 1.0
agg = collections.defaultdict(lambda: [0.0, 0.0])
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1] if len(d["Source"].split()) > 1 else op
    op = op.split(".")[0]
    agg[op][0] += num(d[kst])
    agg[op][1] += num(d[kex])
print(f"\nby opcode (stall samples %, executed %), total executed {tot_e:.4g}")
for op, (st, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{op:12s} {100 * st / tot_s:6.2f}% {100 * ex / tot_e:6.2f}%")
print("\ntop instructions by stall samples")
for d in sorted(data, key=lambda d: -num(d[kst]))[:n]:
    print(f"{100 * num(d[kst]) / tot_s:6.2f}% {d['Address']:>8s} {d['Source'][:90]}")
rows = page("cuda,sass")
hdr2 = next((r for r in rows if "Source" in r and len(r) > 3), None)
if hdr2:
    k2 = next((k for k in hdr2 if k.startswith("Warp Stall Sampling (All")), None)
    lines = [dict(zip(hdr2, r)) for r in rows[rows.index(hdr2) + 1:] if len(r) == len(hdr2)]
    if k2:
        tot = sum(num(d[k2]) for d in lines) or 1.0
        print("\ntop CUDA lines (cuda,sass view)")
        for d in sorted(lines, key=lambda d: -num(d[k2]))[:n]:
            print(f"{100 * num(d[k2]) / tot:6.2f}% {d.get('#', d.get('Line No', ''))} {d['Source'][:100]}")

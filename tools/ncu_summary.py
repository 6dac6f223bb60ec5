"""Summarise an ncu report: key throughput / stall metrics per kernel (reads here, no GPU)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__occupancy_limit_registers",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__cycles_active.avg"]
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "not_selected", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "barrier", "branch_resolving", "dispatch_stall", "no_instruction", "selected", "membar"]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in d:
                e[k] = d[k] + " " + units[hdr.index(k)]
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d:
                e["stall_" + s] = d[k]
        res.append(e)
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        for e in summarise(rep):
            print(json.dumps(e, indent=1))

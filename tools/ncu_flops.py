"""Fold an ncu FP64-count capture of the spray source pass into
profiles/ncu_summary.json (read by bench.py for the c4 roofline).

  python tools/ncu_flops.py profiles/r2_ncu_spray_flops_c4.csv 4096

The CSV comes from tools/r2_variants_run.sh (ncu --metrics
smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum, DRAM bytes,
duration, FP64 pipe; one steady-state launch at c4).  flops = 2 DFMA + DADD + DMUL.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, n):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr, body = rows[0], rows[1:]
    mi, vi = hdr.index("Metric Name"), hdr.index("Metric Value")
    m = {r[mi]: float(r[vi].replace(",", "")) for r in body}
    cells = n * n
    dfma = m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
    dadd = m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
    dmul = m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    flops = 2 * dfma + dadd + dmul
    ent = {
        "fp64_flops_per_launch": flops, "cells_per_launch": cells, "fp64_flops_per_cell": flops / cells,
        "fp64_instr_per_cell": (dfma + dadd + dmul) / cells,
        "dfma_dadd_dmul_per_cell": [dfma / cells, dadd / cells, dmul / cells],
        "warp_instr_per_cell": m["smsp__inst_executed.sum"] / cells,
        "dram_bytes_per_launch": dram, "dram_bytes_per_cell": dram / cells,
        "arithmetic_intensity_flop_per_byte": flops / dram,
        "fp64_pipe_pct_active": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
        "duration_ns_ncu_cold_serialised": m["gpu__time_duration.sum"],
        "source": f"{os.path.relpath(path, ROOT)} (ncu --metrics smsp__sass_thread_inst_executed_op_"
                  "{dfma,dadd,dmul}_pred_on.sum, dram bytes; c4 4096^2, 6th source launch: steady state of "
                  "the extrapolated warm start); flops = 2 DFMA + DADD + DMUL",
    }
    sp = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(sp))
    summ["spray_source_step_kernel"] = ent
    json.dump(summ, open(sp, "w"), indent=1)
    print(json.dumps(ent, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))

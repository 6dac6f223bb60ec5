#!/bin/bash
# Round evidence on one B200 (run through gpurun from the repo root):
#   default bench line, all-config table, ncu launch list of the bench,
#   ncu --set full summaries of the c3 step kernel and the spray source kernel.
# Outputs under gpurun_out/ (copy what is judged into profiles/).
set -u
mkdir -p gpurun_out /tmp/nc
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/ev_smi.txt 2>&1
nproc > gpurun_out/ev_host.txt; lscpu | grep "Model name" >> gpurun_out/ev_host.txt
timeout 400 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 900 python tools/bench_configs.py > gpurun_out/ev_configs.jsonl 2> gpurun_out/ev_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ev_launches_bench.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ev_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fv_step_pair -s 3 -c 1 \
  -o /tmp/nc/c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu_c3.log 2>&1
python tools/ncu_summary.py /tmp/nc/c3.ncu-rep > gpurun_out/ev_ncu_c3.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spray_source_step -s 3 -c 1 \
  -o /tmp/nc/spray python tools/prof_step.py --system spray --n 2048 --steps 5 > gpurun_out/ev_ncu_spray.log 2>&1
python tools/ncu_summary.py /tmp/nc/spray.ncu-rep > gpurun_out/ev_ncu_spray.json 2>&1
python tools/ncu_source_top.py /tmp/nc/spray.ncu-rep 30 > gpurun_out/ev_ncu_spray_source.txt 2>&1
echo done

# Session-3 evidence on one B200 (gpurun from the repo root); outputs in gpurun_out/
set -u
mkdir -p gpurun_out /tmp/nc
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/f_smi.txt 2>&1
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/f_pytest_gpu.txt)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench_c3_20.json 2> gpurun_out/f_bench_c3_20.err
timeout 400 python bench.py > gpurun_out/f_bench_c3.json 2> gpurun_out/f_bench_c3.err
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:spray_source_step -s 5 -c 1 --csv --log-file gpurun_out/f_ncu_spray_flops_c4.csv python bench.py --workload c4_spray_4096 --steps 2 --warmup 5 --reps 1 --sustained-s 0 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_flops.log 2>&1
python tools/ncu_flops.py gpurun_out/f_ncu_spray_flops_c4.csv 4096 > gpurun_out/f_ncu_flops_fold.txt 2>&1
timeout 400 python bench.py --workload c4_spray_4096 > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/f_launches_bench.csv python bench.py --steps 10 --warmup 3 --reps 1 --sustained-s 0 \
  --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spray_source_step -s 5 -c 1 \
  -o /tmp/nc/spray python bench.py --workload c4_spray_4096 --steps 2 --warmup 5 --reps 1 --sustained-s 0 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_spray.log 2>&1
python tools/ncu_summary.py /tmp/nc/spray.ncu-rep > gpurun_out/f_ncu_spray.json 2>&1
python tools/ncu_source_top.py /tmp/nc/spray.ncu-rep 40 > gpurun_out/f_ncu_spray_source.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fv_step_pair -s 3 -c 1 \
  -o /tmp/nc/c3 python bench.py --steps 2 --warmup 3 --reps 1 --sustained-s 0 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_c3.log 2>&1
python tools/ncu_summary.py /tmp/nc/c3.ncu-rep > gpurun_out/f_ncu_c3.json 2>&1
cp /tmp/nc/spray.ncu-rep /tmp/nc/c3.ncu-rep gpurun_out/ 2>/dev/null
echo done

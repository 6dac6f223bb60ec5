# Evidence for the current build (gpurun from the repo root); outputs in gpurun_out/
set -u
mkdir -p gpurun_out /tmp/nc
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/g_pytest_gpu.txt)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.txt 2>&1
timeout 400 python bench.py --workload c4_spray_4096 > gpurun_out/g_bench_c4.json 2> gpurun_out/g_bench_c4.err
timeout 400 python bench.py > gpurun_out/g_bench_c3.json 2> gpurun_out/g_bench_c3.err
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:spray_source_step -s 5 -c 1 --csv --log-file gpurun_out/g_ncu_spray_flops_c4.csv python bench.py --workload c4_spray_4096 --steps 2 --warmup 5 --reps 1 --sustained-s 0 --no-cpu-baseline --no-e2e > gpurun_out/g_ncu_flops.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spray_source_step -s 5 -c 1 \
  -o /tmp/nc/src python tools/prof_step.py --system spray --n 4096 --steps 8 > gpurun_out/g_ncu_src.log 2>&1
python tools/ncu_summary.py /tmp/nc/src.ncu-rep > gpurun_out/g_ncu_src_c4.json 2>&1
python tools/ncu_source_top.py /tmp/nc/src.ncu-rep 40 > gpurun_out/g_ncu_src_c4_sass.txt 2>&1
timeout 600 python tools/c4_drift.py 4096 12 200 > gpurun_out/g_c4_drift.jsonl 2>&1
echo done

# Session-3 final evidence on one B200 (gpurun from the repo root); outputs in gpurun_out/
set -u
mkdir -p gpurun_out /tmp/nc
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/g_smi.txt 2>&1
(timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/g_pytest_gpu.txt)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench_c3_20.json 2> gpurun_out/g_bench_c3_20.err
timeout 400 python bench.py > gpurun_out/g_bench_c3.json 2> gpurun_out/g_bench_c3.err
timeout 400 python bench.py --adaptive --no-cpu-baseline --no-e2e > gpurun_out/g_bench_c3_adaptive.json 2> gpurun_out/g_bench_c3_adaptive.err
FV2D_EXACT_DIV=1 timeout 400 python bench.py --adaptive --no-cpu-baseline --no-e2e > gpurun_out/g_bench_c3_adaptive_exact.json 2> gpurun_out/g_bench_c3_adaptive_exact.err
timeout 400 python bench.py --workload c4_spray_4096 > gpurun_out/g_bench_c4.json 2> gpurun_out/g_bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/g_launches_bench.csv python bench.py --steps 10 --warmup 3 --reps 1 --sustained-s 0 \
  --no-cpu-baseline --no-e2e > gpurun_out/g_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fv_step_pair -s 3 -c 1 \
  -o /tmp/nc/adapt python tools/prof_step.py --n 16384 --steps 5 --adaptive > gpurun_out/g_ncu_adapt.log 2>&1
python tools/ncu_summary.py /tmp/nc/adapt.ncu-rep > gpurun_out/g_ncu_adapt.json 2>&1
FV2D_EXACT_DIV=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:fv_step_pair -s 3 -c 1 \
  -o /tmp/nc/adapt_exact python tools/prof_step.py --n 16384 --steps 5 --adaptive > gpurun_out/g_ncu_adapt_exact.log 2>&1
python tools/ncu_summary.py /tmp/nc/adapt_exact.ncu-rep > gpurun_out/g_ncu_adapt_exact.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fv_step_pair -s 3 -c 1 \
  -o /tmp/nc/c3 python bench.py --steps 2 --warmup 3 --reps 1 --sustained-s 0 --no-cpu-baseline --no-e2e > gpurun_out/g_ncu_c3.log 2>&1
python tools/ncu_summary.py /tmp/nc/c3.ncu-rep > gpurun_out/g_ncu_c3.json 2>&1
cp /tmp/nc/adapt.ncu-rep /tmp/nc/adapt_exact.ncu-rep gpurun_out/ 2>/dev/null
echo done

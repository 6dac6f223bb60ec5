# Round-2 evidence on one B200 (gpurun from the repo root); outputs in gpurun_out/
set -u
mkdir -p gpurun_out /tmp/nc
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/e_pytest_gpu.txt)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.txt 2>&1
timeout 400 python bench.py > gpurun_out/e_bench_c3.json 2> gpurun_out/e_bench_c3.err
timeout 400 python bench.py --workload c4_spray_4096 > gpurun_out/e_bench_c4.json 2> gpurun_out/e_bench_c4.err
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/e_bench_c3_20.json 2> gpurun_out/e_bench_c3_20.err
timeout 600 python tools/c4_drift.py 4096 12 200 > gpurun_out/e_c4_drift.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/e_launches_bench.csv python bench.py --steps 10 --warmup 3 --reps 1 --sustained-s 0 \
  --no-cpu-baseline --no-e2e > gpurun_out/e_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fv_step_pair -s 3 -c 1 \
  -o /tmp/nc/adapt python tools/prof_step.py --n 16384 --steps 5 --adaptive > gpurun_out/e_ncu_adapt.log 2>&1
python tools/ncu_summary.py /tmp/nc/adapt.ncu-rep > gpurun_out/e_ncu_adapt.json 2>&1
python tools/ncu_source_top.py /tmp/nc/adapt.ncu-rep 40 > gpurun_out/e_ncu_adapt_source.txt 2>&1
cp /tmp/nc/adapt.ncu-rep gpurun_out/ 2>/dev/null
echo done

set -u
mkdir -p gpurun_out
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/s3_pytest_gpu.txt)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/s3_bench_c3_20.json 2> gpurun_out/s3_bench_c3_20.err
timeout 400 python bench.py --workload c4_spray_4096 > gpurun_out/s3_bench_c4.json 2> gpurun_out/s3_bench_c4.err
echo done

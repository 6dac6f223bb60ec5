set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/fdcheck tools/fastdiv_check.cu && timeout 120 /tmp/fdcheck > gpurun_out/s3f_fdcheck.txt 2>&1; echo "exit $?" >> gpurun_out/s3f_fdcheck.txt
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3f_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/s3f_pytest.txt)
python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3f_ic_fast.jsonl 2>&1
FV2D_EXACT_DIV=1 python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3f_ic_exact.jsonl 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s3f_c3_fast.json 2>&1
FV2D_EXACT_DIV=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s3f_c3_exact.json 2>&1
python bench.py --steps 100 --warmup 5 --adaptive --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/s3f_c3ad_fast.json 2>&1
FV2D_EXACT_DIV=1 python bench.py --steps 100 --warmup 5 --adaptive --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/s3f_c3ad_exact.json 2>&1
echo done

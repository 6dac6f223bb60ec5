set -u
mkdir -p gpurun_out
(FV2D_SPRAY_OVERLAP=1 timeout 900 python -m pytest tests -m gpu -x -q -k "spray or source or recon" > gpurun_out/s3y_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/s3y_pytest.txt)
for r in 1 2; do
FV2D_SPRAY_OVERLAP=0 python bench.py --workload c4_spray_4096 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/s3y_off_$r.json 2>&1
FV2D_SPRAY_OVERLAP=1 python bench.py --workload c4_spray_4096 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --sustained-s 0 > gpurun_out/s3y_on_$r.json 2>&1
done
echo done

set -u
mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q -k "spray or source or recon or edge or smoke" > gpurun_out/s3s_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/s3s_pytest.txt)
python tools/variants.py run r2orig hslow hfast r2orig hslow hfast --workload c4_spray_4096 --steps 200 > gpurun_out/s3s_c4.jsonl 2>&1
for k in "" "--naive" "--one-cell"; do
python bench.py --workload c2_euler_1024 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --sustained-s 0 $k > gpurun_out/s3s_c2$k.json 2>&1
done
echo done

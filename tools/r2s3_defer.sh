set -u
mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q -k "adapt or trajectory or near_ties or full_size or mixed or blocks or random or c2" > gpurun_out/s3d_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/s3d_pytest.txt)
for v in defer nodefer; do
FV2D_LIB=paper_1701_05431_b200/lib/variants/lib$v.so python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3d_ic_$v.jsonl 2>&1
done
python tools/variants.py run base nodefer --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/s3d_ad.jsonl 2>&1
echo done

set -u
mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q -k "adapt or trajectory or near_ties or full_size or mixed or blocks or random" > gpurun_out/s3r_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/s3r_pytest.txt)
python tools/variants.py run base noreuse --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/s3r_ad.jsonl 2>&1
python tools/variants.py run base noreuse --workload c5_euler_8192_per_gpu --steps 100 --adaptive > gpurun_out/s3r_ad_c5.jsonl 2>&1
echo done
python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3r_ic_base.jsonl 2>&1
FV2D_LIB=paper_1701_05431_b200/lib/variants/libnoreuse.so python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3r_ic_noreuse.jsonl 2>&1

mkdir -p gpurun_out
python tools/variants.py run base --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/fd2_ad.jsonl 2>&1
FV2D_EXACT_DIV=1 python tools/variants.py run base --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/fd2_ad_exact.jsonl 2>&1
python tools/variants.py run base --workload c3_euler_16384 --steps 100 > gpurun_out/fd2_fix.jsonl 2>&1
FV2D_EXACT_DIV=1 python tools/variants.py run base --workload c3_euler_16384 --steps 100 > gpurun_out/fd2_fix_exact.jsonl 2>&1
python tools/variants.py run base --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/fd2_ad2.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fd2_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/fd2_pytest.txt

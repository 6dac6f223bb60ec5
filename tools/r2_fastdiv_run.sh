mkdir -p gpurun_out
python tools/variants.py run nofast base nofb --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/fd_ad.jsonl 2>&1
python tools/variants.py run nofast base nofb --workload c3_euler_16384 --steps 100 > gpurun_out/fd_fix.jsonl 2>&1
python tools/variants.py run nofast base nofb --workload c4_spray_4096 --steps 100 > gpurun_out/fd_c4.jsonl 2>&1
python -c "from paper_1701_05431_b200 import fv2d; print(fv2d.selftest_divsqrt(1<<26, 12345))" > gpurun_out/fd_selftest.txt 2>&1

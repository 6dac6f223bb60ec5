set -u
mkdir -p gpurun_out
python tools/variants.py run base ad1 ad2 ff1 ff2 ff3 base ff1 --workload c3_euler_16384 --steps 20 --sustained-s 0 > gpurun_out/s3q_fixed.jsonl 2>&1
python tools/variants.py run base ad1 ad2 ff1 base --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/s3q_adapt.jsonl 2>&1
for v in ad1 ff1; do
FV2D_LIB=paper_1701_05431_b200/lib/variants/lib$v.so python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3q_ic_$v.jsonl 2>&1
done
python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3q_ic_base.jsonl 2>&1
echo done

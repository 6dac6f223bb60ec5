set -u
mkdir -p gpurun_out
for v in noreuse floor screen; do
FV2D_LIB=paper_1701_05431_b200/lib/variants/lib$v.so python tools/adapt_ic_bench.py --n 8192 --steps 50 > gpurun_out/s3e_ic_$v.jsonl 2>&1
done
echo done

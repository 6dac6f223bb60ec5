set -u
mkdir -p gpurun_out
python tools/variants.py run base ng4 ng8 ng12 base --workload c4_spray_4096 --steps 200 > gpurun_out/s3w_c4.jsonl 2>&1
echo done

set -u
mkdir -p gpurun_out
python tools/variants.py run base c6 base c6 --workload c4_spray_4096 --steps 200 > gpurun_out/s3z_c4.jsonl 2>&1
echo done

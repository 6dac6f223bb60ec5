# compute-sanitizer over tools/sanitize.py, a 2-process spray bench on one GPU, long runs
mkdir -p gpurun_out
( for t in memcheck racecheck initcheck; do echo "$t:"; timeout 900 compute-sanitizer --tool $t python tools/sanitize.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|sanitize cases|Error|error" | head -20; done ) > gpurun_out/s3r_sanitizers.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --shared-gpu --workload c4_spray_4096 --steps 20 --warmup 3 --reps 2 --sustained-s 0 --no-cpu-baseline --no-e2e > gpurun_out/s3r_bench_c4_2rank.json 2> gpurun_out/s3r_bench_c4_2rank.err
timeout 900 python tools/longrun.py > gpurun_out/s3r_longrun.jsonl 2>&1
echo done

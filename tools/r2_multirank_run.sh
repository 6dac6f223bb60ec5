# N > 1 bench flow with 4 and 8 processes sharing one GPU (functional check of the
# peer path + self-check at the ranks the driver's scaling run uses), and the new tests
mkdir -p gpurun_out
for n in 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) \
    bench.py --gpus $n --shared-gpu --workload c2_euler_1024 --steps 10 --warmup 3 --reps 2 --sustained-s 0 --no-cpu-baseline --no-e2e \
    > gpurun_out/m_bench_${n}rank.json 2> gpurun_out/m_bench_${n}rank.err
  echo "n=$n exit $?" >> gpurun_out/m_status.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 \
  bench.py --gpus 4 --shared-gpu --nranks-x 2 --workload c2_euler_1024 --steps 10 --warmup 3 --reps 2 --sustained-s 0 --no-cpu-baseline --no-e2e \
  > gpurun_out/m_bench_4rank_blocks.json 2> gpurun_out/m_bench_4rank_blocks.err
echo "blocks exit $?" >> gpurun_out/m_status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "randomized_spray" > gpurun_out/m_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/m_pytest.txt

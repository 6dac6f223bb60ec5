set -u
mkdir -p gpurun_out
(timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/m_pytest_gpu.txt 2>&1; echo "exit $?" >> gpurun_out/m_pytest_gpu.txt)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/m_bench_c3_20.json 2> gpurun_out/m_bench_c3_20.err
echo done

set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/fdcheck tools/fastdiv_check.cu && timeout 120 /tmp/fdcheck > gpurun_out/s3u_fdcheck.txt 2>&1; echo "exit $?" >> gpurun_out/s3u_fdcheck.txt
(timeout 900 python -m pytest tests -m gpu -x -q -k "spray or source or recon or edge or smoke" > gpurun_out/s3u_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/s3u_pytest.txt)
python tools/variants.py run nosrcrcp srcrcp bothrcp nosrcrcp srcrcp bothrcp --workload c4_spray_4096 --steps 200 > gpurun_out/s3u_c4.jsonl 2>&1
echo done

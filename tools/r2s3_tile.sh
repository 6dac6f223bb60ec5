set -u
mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q -k "spray or source or recon or edge or smoke" > gpurun_out/s3t_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/s3t_pytest.txt)
python tools/variants.py run hfastc base hfastc base --workload c4_spray_4096 --steps 200 > gpurun_out/s3t_c4.jsonl 2>&1
echo done

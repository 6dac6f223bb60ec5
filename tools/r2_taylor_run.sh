mkdir -p gpurun_out
python tools/variants.py run base ex1 t2 t2b --workload c4_spray_4096 --steps 200 > gpurun_out/t_c4.jsonl 2>&1
FV2D_LIB=paper_1701_05431_b200/lib/variants/libt2.so timeout 600 python tools/c4_drift.py 4096 12 200 > gpurun_out/t_drift_t2.jsonl 2>&1
FV2D_LIB=paper_1701_05431_b200/lib/variants/libt2.so timeout 900 python -m pytest tests -m gpu -q -x -k "spray or source or recon or guard or Spray" > gpurun_out/t_pytest_t2.txt 2>&1; echo "exit $?" >> gpurun_out/t_pytest_t2.txt

mkdir -p gpurun_out
python tools/variants.py run base ex1 --workload c4_spray_4096 --steps 200 > gpurun_out/q_c4.jsonl 2>&1
python tools/variants.py run q9 q8 q7 q6 q5 q4 --workload c4_spray_4096 --steps 50 > gpurun_out/q_bhist.jsonl 2>&1
timeout 600 python tools/c4_drift.py 4096 12 200 > gpurun_out/q_drift_quad.jsonl 2>&1
FV2D_LIB=paper_1701_05431_b200/lib/variants/libex1.so timeout 600 python tools/c4_drift.py 4096 12 200 > gpurun_out/q_drift_lin.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "spray or source or recon or guard or Spray" > gpurun_out/q_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/q_pytest.txt

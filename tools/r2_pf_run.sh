mkdir -p gpurun_out
python tools/variants.py run base pf base pf --workload c4_spray_4096 --steps 200 > gpurun_out/pf_c4.jsonl 2>&1
python tools/variants.py run base unc base unc --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/unc_ad.jsonl 2>&1
FV2D_LIB=paper_1701_05431_b200/lib/variants/libpf.so timeout 900 python -m pytest tests -m gpu -q -x -k "spray or source or recon or guard or Spray" > gpurun_out/pf_pytest.txt 2>&1; echo "exit $?" >> gpurun_out/pf_pytest.txt

mkdir -p gpurun_out
python tools/variants.py run base sm5 sm6 ng6 ng12 --workload c4_spray_4096 --steps 200 > gpurun_out/v_c4.jsonl 2>&1
python tools/variants.py run base ad2 ad4 --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/v_ad.jsonl 2>&1
FV2D_RING_DEPTH=6 python tools/variants.py run base ad2 --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/v_ad6.jsonl 2>&1
FV2D_RING_DEPTH=8 python tools/variants.py run base ad2 --workload c3_euler_16384 --steps 100 --adaptive > gpurun_out/v_ad8.jsonl 2>&1
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:spray_source_step -s 5 -c 1 --csv --log-file gpurun_out/r2_ncu_spray_flops_c4.csv python bench.py --workload c4_spray_4096 --steps 2 --warmup 5 --reps 1 --sustained-s 0 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_flops.log 2>&1
echo done

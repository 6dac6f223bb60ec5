# ncu --set full of the fused spray step and of the split source pass at c4 (4096^2, steady state)
set -u
mkdir -p gpurun_out /tmp/nc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spray_fused_step -s 4 -c 1 \
  -o /tmp/nc/fused python tools/prof_step.py --system spray --n 4096 --steps 6 --fuse > gpurun_out/ncu_fused.log 2>&1
python tools/ncu_summary.py /tmp/nc/fused.ncu-rep > gpurun_out/ncu_fused.json 2>&1
python tools/ncu_source_top.py /tmp/nc/fused.ncu-rep 40 > gpurun_out/ncu_fused_source.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spray_source_step -s 4 -c 1 \
  -o /tmp/nc/src python tools/prof_step.py --system spray --n 4096 --steps 6 > gpurun_out/ncu_src.log 2>&1
python tools/ncu_summary.py /tmp/nc/src.ncu-rep > gpurun_out/ncu_src4096.json 2>&1
python tools/ncu_source_top.py /tmp/nc/src.ncu-rep 40 > gpurun_out/ncu_src4096_source.txt 2>&1
cp /tmp/nc/fused.ncu-rep /tmp/nc/src.ncu-rep gpurun_out/ 2>/dev/null
echo done

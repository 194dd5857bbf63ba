# Final-code ncu evidence for the chunk-flag reduction path (virtual bf16
# reduce-scatter): the live line, the launch list and one full capture.
for dt in bfloat16 float32; do
  python tools/virtual_rs_roofline.py --mib 64 --dtype $dt 2>&1 | tail -1 > gpurun_out/r02_rs_${dt}_line.json
  cat gpurun_out/r02_rs_${dt}_line.json
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_rs_launches.csv python tools/virtual_rs_roofline.py --mib 64 --iters 3 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fc_forest_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/r02_rs_bf16_virtual8 -f python tools/virtual_rs_roofline.py --mib 64 --iters 2 --warmup 3 > gpurun_out/ncu_rs.log 2>&1
tail -1 gpurun_out/ncu_rs.log

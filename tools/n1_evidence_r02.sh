# N=1 evidence (round 2): bench line, ncu launch list, one --set full capture
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.log 2>&1
grep "^{" gpurun_out/r02_bench_n1.log > gpurun_out/r02_bench_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_n1_launches.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_n1_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fc_forest_kernel --launch-skip 10 --launch-count 1 \
    -o gpurun_out/r02_n1_virtual8_allgather -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_n1_full.log 2>&1
tail -2 gpurun_out/ncu_n1_full.log

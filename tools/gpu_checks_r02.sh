set -x
timeout 900 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_production.py tests/test_gpu_api.py -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -4
python tools/virtual_rs_roofline.py --mib 64 2>&1 | tail -2
python tools/virtual_rs_roofline.py --mib 64 --dtype float32 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | grep "^{" > gpurun_out/bench_n1.json; python -c "
import json; d=json.load(open('gpurun_out/bench_n1.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['configs0_8x1MiB'], d['local_copy_sanity'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_rs_launches.csv python tools/virtual_rs_roofline.py --mib 64 --iters 3 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fc_forest_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/r02_rs_bf16_virtual8 -f python tools/virtual_rs_roofline.py --mib 64 --iters 2 --warmup 3 > gpurun_out/ncu_rs.log 2>&1
tail -3 gpurun_out/ncu_rs.log
ls -la gpurun_out/

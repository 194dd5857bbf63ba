# Round-2 multi-GPU evidence run: parity/NVLS/DDP/FSDP/soak tests, the bench
# line (sweep, NVLS points, sparse stress) and the full message-size sweep.
N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -p no:cacheprovider -rfE 2>&1 | tail -4 > gpurun_out/r02_multiproc_n$N.txt
cat gpurun_out/r02_multiproc_n$N.txt
timeout 900 $R --master-port 29611 bench.py --gpus $N 2>&1 | grep "^{" | tail -1 > gpurun_out/r02_bench_n$N.json
timeout 1800 $R --master-port 29613 tools/sweep.py --out gpurun_out/r02_sweep_n$N.jsonl > gpurun_out/r02_sweep_n$N.log 2>&1
tail -2 gpurun_out/r02_sweep_n$N.log; wc -l gpurun_out/r02_sweep_n$N.jsonl

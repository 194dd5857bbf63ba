N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1"
PTS=""
for c in 96 128 148; do for w in 4 8; do
  PTS="$PTS ag:1024:f32:0:ctas_per_rank=$c:worker_warps=$w rs:1024:bf16:0:ctas_per_rank=$c:worker_warps=$w"
done; PTS="$PTS ag:256:f32:1:ctas_per_rank=$c ar:25:bf16:1:ctas_per_rank=$c"; done
$R --master-port 29601 tools/ab_time.py $PTS 2>&1 | grep "GB/s\|rror"

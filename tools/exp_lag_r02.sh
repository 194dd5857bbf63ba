N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1"
PTS=""
for sz in ag:32:f32 ag:64:f32 ag:256:f32 ar:25:bf16 rs:64:bf16 ar:4:bf16; do
  for lag in 1 2 4 8 16 64; do PTS="$PTS $sz:-1:lag=$lag"; done
done
$R --master-port 29571 tools/ab_time.py $PTS 2>&1 | grep "GB/s"

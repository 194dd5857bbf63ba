N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1"
PTS=""
for sz in ar:4:bf16 ar:8:bf16 ar:16:bf16 ar:25:bf16 rs:4:bf16 rs:8:bf16 rs:16:bf16; do
  PTS="$PTS $sz:-1:twohop_max=67108864 $sz:-1:twohop_max=0"
done
$R --master-port 29581 tools/ab_time.py $PTS 2>&1 | grep "GB/s\|rror"

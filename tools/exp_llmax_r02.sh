# LL128 vs chunk flags around the ll_max threshold (512 MiB moved per rank)
N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1"
PTS=""
for sz in ag:256:f32 ag:512:f32 ag:768:f32 rs:256:f32 rs:512:f32 rs:768:bf16 ar:128:bf16 ar:256:bf16 ar:512:bf16; do
  PTS="$PTS $sz:1 $sz:0"
done
$R --master-port 29591 tools/ab_time.py $PTS 2>&1 | grep "GB/s\|rror"

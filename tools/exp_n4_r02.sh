R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
PTS=""
for sz in ag:64:f32 ar:25:bf16 rs:64:bf16; do
  for c in 128 148; do for w in 2 4; do for ch in 32768 65536; do
    PTS="$PTS $sz:1:ctas_per_rank=$c:ll_worker_warps=$w:ll_chunk_max=$ch"
  done; done; done
done
PTS="$PTS rs:256:f32:-1 rs:256:f32:0 rs:256:bf16:-1 rs:256:bf16:0 ag:256:f32:-1 ag:256:f32:0 ar:256:bf16:-1 ar:256:bf16:0 ar:1024:bf16:-1 ar:1024:bf16:0 ag:1024:f32:-1"
$R --master-port 29561 tools/ab_time.py $PTS 2>&1 | grep "GB/s"

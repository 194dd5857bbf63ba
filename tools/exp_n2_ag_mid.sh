R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
PTS=""
for m in 16 24 32 48 64 96; do PTS="$PTS ag:$m:f32:-1 ag:$m:f32:-1:oneshot_ag_max=268435456 ag:$m:f32:-1:ce_min=1 ag:$m:f32:-1:oneshot_ag_max=0"; done
$R --master-port 29541 tools/ab_time.py $PTS 2>&1 | grep "GB/s"

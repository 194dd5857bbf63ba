R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
PTS="ag:1024:f32:-1 ag:1024:f32:0 rs:256:f32:0 rs:256:bf16:0 rs:256:f32:-1 ar:1024:bf16:-1 ar:25:bf16:-1 ag:64:f32:-1 ag:16:f32:-1 ag:4:f32:-1"
for i in 1 2; do
echo "--- current"; $R --master-port 2954$i tools/ab_time.py $PTS 2>&1 | grep "GB/s"
echo "--- r01"; (cd _r01 && $R --master-port 2956$i tools/ab_time.py $PTS 2>&1 | grep "GB/s")
done

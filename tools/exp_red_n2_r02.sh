# Reduction A/B at N GPUs: tools/bin/var/old.so (before the bulk_reduce
# changes) vs new.so; chunk-flag (proto 0) and automatic paths.
L=paper_2402_06787_b200/lib/libforestcoll.so
cp $L /tmp/orig.so
N=$(nvidia-smi -L | wc -l)
for rep in 1 2; do
  for V in old new; do
    cp tools/bin/var/$V.so $L
    echo "== $V rep=$rep N=$N"
    torchrun --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/ab_time.py \
      rs:256:f32:0 rs:1024:bf16:0 ar:256:bf16:0 ar:1024:bf16:0 ar:1024:f32:0 ar:25:bf16:-1 ar:64:bf16:-1 2>&1 | grep " us "
  done
done
cp /tmp/orig.so $L

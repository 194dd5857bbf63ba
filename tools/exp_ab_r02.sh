R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
for i in 1 2; do
echo "--- current"; $R --master-port 2954$i tools/host_overhead_probe.py --mib 64,25 2>&1 | grep MiB
echo "--- variant (local dl)"; (cd _var && $R --master-port 2955$i tools/host_overhead_probe.py --mib 64,25 2>&1 | grep MiB)
echo "--- r01"; (cd _r01 && $R --master-port 2956$i tools/trace_multi.py --coll allgather --mib 64 2>&1 | grep "N=2"; $R --master-port 2957$i tools/trace_multi.py --coll allgather --mib 25 2>&1 | grep "N=2")
done

R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
$R --master-port 29531 tools/host_overhead_probe.py 2>&1 | grep MiB
echo "--- r01 tree"
(cd _r01 && $R --master-port 29532 tools/trace_multi.py --coll allgather --mib 64 2>&1 | grep "N=2")
(cd _r01 && $R --master-port 29533 tools/trace_multi.py --coll allreduce --mib 25 2>&1 | grep "N=2")
echo "--- current tree"
$R --master-port 29534 tools/trace_multi.py --coll allgather --mib 64 2>&1 | grep "N=2"
$R --master-port 29535 tools/trace_multi.py --coll allreduce --mib 25 2>&1 | grep "N=2"

# N=2/4 medium-size experiments (round 2): traces and option grids for the
# 25 MiB allreduce (DDP bucket) and 64 MiB allgather.
N=${N:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1"
$R --master-port 29521 tools/trace_multi.py --coll allreduce --mib 25 2>&1 | grep -v "^\*\|OMP\|^W1" | head -40
$R --master-port 29522 tools/trace_multi.py --coll allgather --mib 64 2>&1 | grep -v "^\*\|OMP\|^W1" | head -30
$R --master-port 29523 tools/tune_multi.py --colls allreduce --sizes 25 --ctas 64,128,148 --chunks 16384,32768,65536,131072 --ww 2,4,8 --proto 1 --iters 20 2>&1 | grep "^allreduce"
$R --master-port 29524 tools/tune_multi.py --colls allgather --sizes 64 --ctas 64,128,148 --chunks 16384,65536,131072 --ww 2,4,8 --proto 1 --iters 20 2>&1 | grep "^allgather"

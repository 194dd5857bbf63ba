"""torchrun: trace one collective call on every rank and print the summary
of rank 0 (and the slowest rank).  python -m torch.distributed.run ... tools/trace_multi.py
    --coll allgather --mib 64 --opt ctas_per_rank=32 ..."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import MIB, gbs, timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402
from tools.trace_report import report  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coll", default="allgather")
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--opt", action="append", default=[])
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    for o in args.opt:
        k, v = o.split("=")
        comm.set_option(k, int(v))
    M = args.mib * MIB
    if args.coll == "allgather":
        S = M // n // 4
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S, dtype=torch.float32)
        fn = lambda: comm.all_gather(out, inp)  # noqa: E731
    elif args.coll == "reduce_scatter":
        R = M // n // 4
        inp = torch.randn(R * n, device=dev)
        out = torch.empty(R, device=dev)
        fn = lambda: comm.reduce_scatter(out, inp)  # noqa: E731
    else:
        buf = comm.empty(M // 2, dtype=torch.bfloat16)
        buf.normal_()
        fn = lambda: comm.all_reduce(buf)  # noqa: E731
    ms = timed(fn, 10, 3, dist)
    t = comm.t_star(args.coll, M)
    comm.enable_trace(1 << 20)
    comm.reset_trace()
    dist.barrier()
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    rec = comm.read_trace()
    reps = [None] * n
    dist.all_gather_object(reps, report(rec, comm.plan(args.coll)))
    if rank == 0:
        print(f"{args.coll} {args.mib} MiB N={n}: {ms * 1e3:.1f} us, algbw {gbs(M, ms):.1f} GB/s, "
              f"T* {t * 1e6:.1f} us (frac {t * 1e3 / ms:.3f}) {comm.last_call_info()}")
        for r, txt in enumerate(reps):
            if r in (0, n - 1):
                print(f"--- rank {r}\n{txt}")
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

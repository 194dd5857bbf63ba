"""Single-GPU probe: time the virtual-rank forest kernel and print a trace
summary.   python tools/probe_virtual.py [--coll allgather] [--mib 64] [--opt k=v ...]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import MIB, gbs, timed  # noqa: E402
from paper_2402_06787_b200 import VirtualComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402
from tools.trace_report import report  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coll", default="allgather")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--mib", default="1,64")
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--trace", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    comm = VirtualComm(nvswitch_doc(args.n), device=0)
    for o in args.opt:
        k, v = o.split("=")
        comm.set_option(k, int(v))
    n = args.n
    for mib in [int(x) for x in args.mib.split(",")]:
        S = mib * MIB // 4
        if args.coll == "allgather":
            ins = [torch.randn(S, device=dev) for _ in range(n)]
            outs = [torch.empty(n * S, device=dev) for _ in range(n)]
            fn = lambda: comm.all_gather(outs, ins)  # noqa: E731
            M = n * S * 4
        elif args.coll == "reduce_scatter":
            ins = [torch.randn(n * S, device=dev) for _ in range(n)]
            outs = [torch.empty(S, device=dev) for _ in range(n)]
            fn = lambda: comm.reduce_scatter(outs, ins)  # noqa: E731
            M = n * S * 4
        else:
            bufs = [torch.randn(n * S, device=dev).to(torch.bfloat16) for _ in range(n)]
            fn = lambda: comm.all_reduce(bufs)  # noqa: E731
            M = n * S * 2
        ms = timed(fn, 10, 3)
        info = comm.last_call_info()
        print(f"{args.coll} {mib} MiB/rank-shard: {ms * 1e3:9.1f} us  algbw {gbs(M, ms):8.1f} GB/s  {info}",
              flush=True)
        if args.trace:
            comm.enable_trace(1 << 20)
            comm.reset_trace()
            fn()
            rec = comm.read_trace()
            print(report(rec, comm.plan(args.coll)))
            comm.disable_trace()
    comm.check()


if __name__ == "__main__":
    main()

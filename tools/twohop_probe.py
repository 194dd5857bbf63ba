"""Virtual-rank probe of the two-hop reduction kernel (one GPU; for ncu).
    python tools/twohop_probe.py [--n 4] [--mib 16] [--coll allreduce]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import MIB, gbs, timed  # noqa: E402
from paper_2402_06787_b200 import VirtualComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--mib", type=int, default=16)
    ap.add_argument("--coll", default="allreduce")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    n = args.n
    comm = VirtualComm(nvswitch_doc(n), device=0, options={"twohop_max": 1 << 30})
    cnt = args.mib * MIB // 2
    if args.coll == "allreduce":
        bufs = [torch.randn(cnt, device=dev).to(torch.bfloat16) for _ in range(n)]
        fn = lambda: comm.all_reduce(bufs)  # noqa: E731
    else:
        ins = [torch.randn(cnt, device=dev).to(torch.bfloat16) for _ in range(n)]
        outs = [torch.empty(cnt // n, device=dev, dtype=torch.bfloat16) for _ in range(n)]
        fn = lambda: comm.reduce_scatter(outs, ins)  # noqa: E731
    ms = timed(fn, args.iters, 3)
    print(f"{args.coll} {args.mib} MiB x {n} virtual ranks: {ms * 1e3:.1f} us "
          f"({gbs(args.mib * MIB, ms):.1f} GB/s per rank) {comm.last_call_info()}", flush=True)
    comm.check()
    comm.close()


if __name__ == "__main__":
    main()

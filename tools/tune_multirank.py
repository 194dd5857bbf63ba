"""torchrun (P processes): an N-rank forest with N/P ranks per GPU over real
NVLink (MultiRankComm) -- e.g. the nvswitch(8) forest on 4 GPUs -- timed
across chunk sizes, to see depth-7 pipeline effects before an 8-GPU box.
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/tune_multirank.py --mib 1024 --chunks 131072,262144,524288"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import MIB, gbs, timed  # noqa: E402
from paper_2402_06787_b200 import MultiRankComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--coll", default="allgather")
    ap.add_argument("--mib", default="64,1024")
    ap.add_argument("--chunks", default="131072,262144,524288")
    ap.add_argument("--proto", default="-1")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--tail", default="4")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("gloo")
    p, P = dist.get_rank(), dist.get_world_size()
    N = args.n
    mine = list(range(p * N // P, (p + 1) * N // P))
    comm = MultiRankComm(nvswitch_doc(N), local_ranks=mine, world_size=N, device=local,
                         scratch_bytes=2 << 30)
    for mib in [int(x) for x in args.mib.split(",")]:
        M = mib * MIB
        if args.coll == "allgather":
            S = M // N // 4
            ins = [torch.randn(S, device=dev) for _ in mine]
            outs = [torch.empty(N * S, device=dev) for _ in mine]
            fn = lambda: comm.all_gather(outs, ins)  # noqa: E731
        else:
            R = M // N // 4
            ins = [torch.randn(N * R, device=dev) for _ in mine]
            outs = [torch.empty(R, device=dev) for _ in mine]
            fn = lambda: comm.reduce_scatter(outs, ins)  # noqa: E731
        t = comm.t_star(args.coll, M)
        for proto in [int(x) for x in args.proto.split(",")]:
            for ch, tail in [(int(x), int(y)) for x in args.chunks.split(",") for y in args.tail.split(",")]:
                comm.set_option("chunk_tail", tail)
                comm.set_option("proto", proto)
                comm.set_option("chunk_max", ch)
                comm.set_option("ll_chunk_max", min(ch, 1 << 20))
                ms = timed(fn, args.iters, 2, dist)
                info = comm.last_call_info()
                if p == 0:
                    print(f"{args.coll} N={N} on {P} GPUs {mib} MiB proto={info['proto']} chunk={ch >> 10}K tail={tail} "
                          f"n={info['nchunks']} L={info['launches']}: {ms * 1e3:.1f} us "
                          f"algbw {gbs(M, ms):.1f} GB/s (T* frac {t * 1e3 / ms:.3f})", flush=True)
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

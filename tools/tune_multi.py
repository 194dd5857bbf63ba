"""Option sweep for the multi-GPU path (torchrun, one process per GPU).

    torchrun --nproc-per-node N tools/tune_multi.py [--colls allgather,reduce_scatter]
Prints one line per (collective, size, option set): ms, algbw, frac of T*.
"""
import argparse
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import MIB, gbs, timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--colls", default="allgather")
    ap.add_argument("--sizes", default="64,1024")
    ap.add_argument("--ctas", default="16,32,64,128")
    ap.add_argument("--chunks", default="262144,524288,1048576,2097152")
    ap.add_argument("--ipw", default="4")
    ap.add_argument("--lag", default="2")
    ap.add_argument("--mode", default="1")
    ap.add_argument("--dma", default="0")
    ap.add_argument("--ww", default="4")
    ap.add_argument("--proto", default="-1")
    ap.add_argument("--pdl", default="1")
    ap.add_argument("--chunk-min", default="16384")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--tail", default="4")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    for coll in args.colls.split(","):
        for mib in [int(x) for x in args.sizes.split(",")]:
            M = mib * MIB
            if coll == "allgather":
                S = M // n // 4
                inp = torch.randn(S, device=dev)
                out = comm.empty(n * S, dtype=torch.float32)
                fn = lambda: comm.all_gather(out, inp)  # noqa: E731
            elif coll == "reduce_scatter":
                dt = getattr(torch, args.dtype)
                R = M // n // torch.tensor([], dtype=dt).element_size()
                inp = torch.randn(R * n, device=dev).to(dt)
                out = torch.empty(R, device=dev, dtype=dt)
                fn = lambda: comm.reduce_scatter(out, inp)  # noqa: E731
            else:
                buf = comm.empty(M // 2, dtype=torch.bfloat16)
                buf.normal_()
                fn = lambda: comm.all_reduce(buf)  # noqa: E731
            tstar = comm.t_star(coll, M)
            for ctas, ch, ipw, lag, mode, dma, ww, proto in itertools.product(
                    args.ctas.split(","), args.chunks.split(","), args.ipw.split(","),
                    args.lag.split(","), args.mode.split(","), args.dma.split(","),
                    args.ww.split(","), args.proto.split(",")):
              for pdl, cmin, tail in itertools.product(args.pdl.split(","), args.chunk_min.split(","),
                                                       args.tail.split(",")):
                comm.set_option("chunk_min", int(cmin))
                comm.set_option("chunk_tail", int(tail))
                comm.set_option("pdl", int(pdl))
                comm.set_option("proto", int(proto))
                comm.set_option("worker_warps", int(ww))
                comm.set_option("ll_worker_warps", int(ww))
                comm.set_option("dma_root_copy", int(dma))
                comm.set_option("lag", int(lag))
                comm.set_option("copy_mode", int(mode))
                comm.set_option("ctas_per_rank", int(ctas))
                comm.set_option("chunk_max", int(ch))
                comm.set_option("ll_chunk_max", int(ch))
                comm.set_option("items_per_worker", int(ipw))
                ms = timed(fn, args.iters, 3, dist)
                info = comm.last_call_info()
                if rank == 0:
                    print(f"{coll:15s} {mib:6d}MiB ctas={ctas:>4s} chunk={int(ch)//1024:5d}K ipw={ipw} lag={lag:>3s} ww={ww} p={info["proto"]} pdl={pdl} cmin={int(cmin)//1024}K tail={tail} "
                          f"n={info['nchunks']:5d} L={info['launches']} ms={ms:8.4f} "
                          f"algbw={gbs(M, ms):8.1f} frac_T*={tstar*1e3/ms:6.3f}", flush=True)
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

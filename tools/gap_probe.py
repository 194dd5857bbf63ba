"""torchrun: per-launch timeline of back-to-back small allgathers from the
item trace (globaltimer): item span of each launch and the gap to the next
launch, eager vs CUDA graph.  Rank 0 prints percentiles.
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/gap_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def timeline(rec):
    out = []
    for L in np.unique(rec["launch"]):
        x = rec[rec["launch"] == L]
        out.append((int(x["t_start"].min()), int(x["t_end"].max()), int(L)))
    out.sort()
    spans = np.array([b - a for a, b, _ in out]) / 1e3
    gaps = np.array([out[i + 1][0] - out[i][1] for i in range(len(out) - 1)]) / 1e3
    period = (out[-1][0] - out[0][0]) / 1e3 / max(1, len(out) - 1)
    return spans, gaps, period


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,65536", help="elements per rank (fp32)")
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--reps", type=int, default=300)
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
    for S in [int(x) for x in args.sizes.split(",")]:
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S)
        f = lambda: comm.all_gather(out, inp)  # noqa: E731
        for _ in range(50):
            f()
        torch.cuda.synchronize()
        for mode in ("eager", "graph"):
            comm.enable_trace(1 << 20)
            if mode == "eager":
                dist.barrier()
                torch.cuda.synchronize()
                for _ in range(args.reps):
                    f()
            else:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                g = torch.cuda.CUDAGraph()
                comm.disable_trace()
                comm.enable_trace(1 << 20)
                with torch.cuda.graph(g):
                    for _ in range(100):
                        f()
                comm.reset_trace()
                dist.barrier()
                torch.cuda.synchronize()
                for _ in range(3):
                    g.replay()
            torch.cuda.synchronize()
            rec = comm.read_trace()
            comm.disable_trace()
            spans, gaps, period = timeline(rec[rec["rank"] == rank])
            if rank == 0:
                q = lambda a: " ".join(f"{v:5.1f}" for v in np.percentile(a, [10, 50, 90]))  # noqa: E731
                print(f"AG {S*4*n:8d} B {mode:5s}: period {period:5.2f} us | span p10/50/90 {q(spans)} | "
                      f"gap p10/50/90 {q(gaps)}", flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

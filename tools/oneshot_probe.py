"""torchrun: tree-engine allreduce / reduce-scatter at small sizes with the
one-shot path enabled up to a given size vs disabled (forest kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import gbs, steps_for, timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    for kib in (64, 256, 512, 1024, 2048, 4096):
        M = kib * 1024
        buf = comm.empty(M // 2, dtype=torch.bfloat16)
        buf.normal_()
        inp = torch.randn(M // 2, device=dev).to(torch.bfloat16)
        out = torch.empty(M // 2 // n, device=dev, dtype=torch.bfloat16)
        row = []
        for lim in (0, 16 << 20):
            comm.set_option("oneshot_max", lim)
            a = timed(lambda: comm.all_reduce(buf), steps_for(M, 20), 3, dist)
            pa = comm.last_call_info()["proto"]
            r = timed(lambda: comm.reduce_scatter(out, inp), steps_for(M, 20), 3, dist)
            pr = comm.last_call_info()["proto"]
            row.append(f"AR {pa:7s} {gbs(M, a):6.1f}  RS {pr:7s} {gbs(M, r):6.1f}")
        if rank == 0:
            print(f"{kib:5d} KiB | " + " | ".join(row), flush=True)
        comm.deregister(buf)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

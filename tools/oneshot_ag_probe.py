"""torchrun: tree-engine allgather with the one-hop (one-shot) path on vs off."""
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
    for kib in (64, 1024, 2048, 4096, 8192, 16384, 32768):
        M = kib * 1024
        S = M // n // 4
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S)
        row = []
        for lim in (0, 64 << 20):
            comm.set_option("oneshot_ag_max", lim)
            ms = timed(lambda: comm.all_gather(out, inp), steps_for(M, 20), 3, dist)
            row.append(f"{comm.last_call_info()['proto']:7s} {gbs(M, ms):7.1f}")
        if rank == 0:
            print(f"AG {kib:6d} KiB | " + " | ".join(row), flush=True)
        comm.deregister(out)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

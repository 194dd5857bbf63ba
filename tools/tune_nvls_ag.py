"""torchrun: NVLS-engine LL multicast allgather latency/bandwidth over sizes."""
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
    c = ForestCollComm(nvswitch_doc(n, multicast=True), rank=rank, world_size=n, device=local,
                       scratch_bytes=64 << 20, nvls_bytes=256 << 20)
    for kib in (16, 64, 256, 1024, 2048):
        M = kib * 1024
        S = M // n // 4
        inp = torch.randn(S, device=dev)
        out = torch.empty(n * S, device=dev)
        ms = timed(lambda: c.all_gather(out, inp), steps_for(M, 20), 3, dist)
        if rank == 0:
            print(f"AG {kib:5d} KiB {c.last_call_info()['proto']}: {ms * 1e3:7.2f} us {gbs(M, ms):7.1f} GB/s",
                  flush=True)
    c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

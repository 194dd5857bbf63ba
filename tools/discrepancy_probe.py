"""Why does the bench line's 64 MiB allgather read lower than the sweep's?
(587 vs 702.6 GB/s at N=4.)  torchrun, N ranks.

Times the 64 MiB LL128 allgather (a) on a fresh communicator, (b) after a
1 GiB chunk-flag allgather, (c) after NCCL Ring / NVLS communicators exist
and have run, (d) after an NCCL NVLS all-gather ran right before -- each
with the bench's timing helper.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import MIB, gbs, nccl_group, steps_for, timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(None, rank=rank, world_size=n, device=local)
    M = 64 * MIB
    S = M // n // 4
    inp = torch.randn(S, device=dev)
    out = comm.empty(n * S, dtype=torch.float32)

    def t(tag):
        ms = timed(lambda: comm.all_gather(out, inp), steps_for(M, 20), 3, dist)
        if rank == 0:
            print(f"{tag:50s} {ms * 1e3:7.1f} us {gbs(M, ms):7.1f} GB/s "
                  f"{comm.last_call_info()['proto']} scratch={comm.scratch_bytes >> 20} MiB", flush=True)

    t("fresh communicator")
    t("again")
    big_i = torch.randn((1 << 30) // n // 4, device=dev)
    big_o = comm.empty(n * big_i.numel(), dtype=torch.float32)
    timed(lambda: comm.all_gather(big_o, big_i), 10, 3, dist)
    t("after 1 GiB chunk-flag allgathers")
    o2 = torch.empty_like(out)
    g_ring = nccl_group(dist, "Ring")
    t("after NCCL Ring comm created")
    timed(lambda: dist.all_gather_into_tensor(o2, inp, group=g_ring), 50, 3, dist)
    t("after NCCL Ring all-gathers")
    g_nvls = nccl_group(dist, "NVLS")
    t("after NCCL NVLS comm created")
    timed(lambda: dist.all_gather_into_tensor(o2, inp, group=g_nvls), 50, 3, dist)
    t("after NCCL NVLS all-gathers")
    timed(lambda: dist.all_gather_into_tensor(o2, inp), 50, 3, dist)
    t("after NCCL default all-gathers")
    timed(lambda: comm.all_gather(big_o, big_i), 10, 3, dist, soak_s=1.0)
    t("after a 1 s soak of 1 GiB allgathers")
    from bench import pipelined_e2e

    h_in = torch.empty(big_i.numel(), pin_memory=True)
    h_out = torch.empty(big_o.numel(), pin_memory=True)
    d_sets = [([big_i], [big_o]), ([torch.empty_like(big_i)], [comm.empty(big_o.numel())])]
    pipelined_e2e([h_in], [h_out], d_sets, lambda o, i: comm.all_gather(o[0], i[0]), 5, 1, dist)
    t("after the pipelined e2e phase")
    small_i = torch.randn((1 << 20) // n // 4, device=dev)
    small_o = comm.empty(n * small_i.numel())
    timed(lambda: comm.all_gather(small_o, small_i), 100, 3, dist)
    t("after 1 MiB one-hop allgathers")
    comm.enable_trace(1 << 20)
    comm.all_gather(big_o, big_i)
    comm.disable_trace()
    t("after a traced call")
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""PyTorch DDP integration: a communication hook that all-reduces gradient
buckets over the ForestColl forest (the paper's FSDP /
DDP motivation).

    comm = ForestCollComm()
    model = DDP(model, device_ids=[local_rank])
    model.register_comm_hook(state=comm, hook=forestcoll_allreduce_hook)

Buckets are averaged in place in one kernel (op avg: each tree root scales
its fp32 sum by 1/N before rounding), matching DDP's default hook, which sums
and divides by the world size.  A bucket tensor is registered with the peers on first use —
DDP reuses its bucket buffers, so registration happens once per bucket.
"""

import torch


def forestcoll_allreduce_hook(
    comm, bucket: torch.distributed.GradBucket
) -> torch.futures.Future[torch.Tensor]:
    buf = bucket.buffer()
    comm.all_reduce(buf, op="avg")
    fut = torch.futures.Future()
    fut.set_result(buf)
    return fut

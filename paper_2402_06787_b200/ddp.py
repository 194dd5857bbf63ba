"""PyTorch DDP integration: a communication hook that all-reduces gradient
buckets over the ForestColl forest (the paper's FSDP /
DDP motivation).

    comm = ForestCollComm()
    model = DDP(model, device_ids=[local_rank])
    model.register_comm_hook(state=comm, hook=forestcoll_allreduce_hook)

Buckets are reduced in place (sum, then divided by world size like DDP's
default hook).  A bucket tensor is registered with the peers on first use —
DDP reuses its bucket buffers, so registration happens once per bucket.
"""

import torch


def forestcoll_allreduce_hook(
    comm, bucket: torch.distributed.GradBucket
) -> torch.futures.Future[torch.Tensor]:
    buf = bucket.buffer()
    comm.all_reduce(buf)
    buf.div_(comm.nranks)
    fut = torch.futures.Future()
    fut.set_result(buf)
    return fut

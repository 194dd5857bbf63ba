"""Process-group setup shared by the torchrun workers.

Default: one process per GPU (LOCAL_RANK -> cuda:LOCAL_RANK) over NCCL.
FC_SAMEDEV=1: every rank process on cuda:0 (the driver's 1-GPU box) with a
gloo process group -- NCCL refuses two ranks on one device, while the
ForestColl communicator itself takes its production path there exactly as
on N GPUs (own CUDA context per process, CUDA IPC peer mappings).
"""

import os

import torch
import torch.distributed as dist


def samedev() -> bool:
    return os.environ.get("FC_SAMEDEV") == "1"


def init():
    """Initialise the default process group; returns the local device index.
    FC_RANKS_PER_GPU=k packs k rank processes per GPU (gloo), e.g. the
    8-rank forest on a 4-GPU box."""
    k = int(os.environ.get("FC_RANKS_PER_GPU", "0"))
    if samedev() or k > 1:
        local = 0 if samedev() else int(os.environ["LOCAL_RANK"]) // k
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return local

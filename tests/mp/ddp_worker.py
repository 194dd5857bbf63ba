"""torchrun worker: DDP with the ForestColl all-reduce comm hook gives the
same gradients (within fp32 reassociation tolerance) as DDP's default NCCL
all-reduce."""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from torch.nn.parallel import DistributedDataParallel as DDP  # noqa: E402

from _common import init  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.ddp import forestcoll_allreduce_hook  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def grads(model, comm=None, steps=3):
    torch.manual_seed(0)
    net = model().cuda()
    ddp = DDP(net, device_ids=[torch.cuda.current_device()], bucket_cap_mb=1)
    if comm is not None:
        ddp.register_comm_hook(state=comm, hook=forestcoll_allreduce_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.1)
    g = torch.Generator(device="cuda").manual_seed(1 + dist.get_rank())
    for _ in range(steps):
        x = torch.randn(64, 512, device="cuda", generator=g)
        loss = ddp(x).square().mean()
        opt.zero_grad()
        loss.backward()
        opt.step()
    return [p.detach().clone() for p in net.parameters()]


def main():
    local = init()
    n = dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=dist.get_rank(), world_size=n, device=local)

    def model():
        return torch.nn.Sequential(torch.nn.Linear(512, 1024), torch.nn.GELU(),
                                   torch.nn.Linear(1024, 512))

    ref = grads(model)
    got = grads(model, comm)
    ok = all(torch.allclose(a, b, rtol=1e-4, atol=1e-5) for a, b in zip(ref, got))
    print(f"DDP rank {dist.get_rank()} {'OK' if ok else 'FAIL'}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

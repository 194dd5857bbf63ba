"""torchrun worker: FSDP2 (fully_shard) with the ForestColl all-gather /
reduce-scatter adapters trains to the same parameters (within fp32
reassociation tolerance) as stock FSDP2 over NCCL, in fp32 and in bf16 mixed
precision; the all-gather outputs come from the symmetric pool."""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from torch.distributed.fsdp import FSDPModule, MixedPrecisionPolicy, fully_shard  # noqa: E402

from _common import init  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.fsdp import ForestCollAllGather, ForestCollReduceScatter  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def build(mp):
    torch.manual_seed(0)
    net = torch.nn.Sequential(*[torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.GELU(),
                                                    torch.nn.Linear(512, 256)) for _ in range(4)]).cuda()
    kw = {"mp_policy": MixedPrecisionPolicy(param_dtype=torch.bfloat16, reduce_dtype=torch.bfloat16)} if mp else {}
    for blk in net:
        fully_shard(blk, **kw)
    fully_shard(net, **kw)
    return net


def train(net, steps=4):
    opt = torch.optim.SGD(net.parameters(), lr=0.05)
    g = torch.Generator(device="cuda").manual_seed(10 + dist.get_rank())
    for _ in range(steps):
        x = torch.randn(32, 256, device="cuda", generator=g)
        loss = net(x).float().square().mean()
        opt.zero_grad()
        loss.backward()
        opt.step()
    return [full(p) for p in net.parameters()]


def full(p):
    """The unsharded parameter.  DTensor.full_tensor() on a gloo group with
    CUDA shards (FC_SAMEDEV) crashes inside gloo, so there the dim-0 shards
    travel through host memory instead."""
    from _common import samedev

    if not samedev():
        return p.full_tensor().detach().float().clone()
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, p.to_local().detach().float().cpu())
    return torch.cat(parts, dim=0).cuda()


def main():
    local = init()
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    # a small first segment: the pool must grow (collectively) during training
    ag = ForestCollAllGather(comm, pool_bytes=1 << 20)
    rs = ForestCollReduceScatter(comm)
    fails = []
    for mp, tol in ((False, 1e-5), (True, 2e-2)):
        ref = train(build(mp))
        net = build(mp)
        for m in net.modules():
            if isinstance(m, FSDPModule):
                m.set_custom_all_gather(ag)
                m.set_custom_reduce_scatter(rs)
        got = train(net)
        comm.check()
        if not all(torch.allclose(a, b, rtol=tol, atol=tol) for a, b in zip(ref, got)):
            worst = max(float((a - b).abs().max()) for a, b in zip(ref, got))
            fails.append(f"mp={mp} max|diff|={worst:.3g}")
    if len(ag.pools) < 2:
        fails.append("pool never grew")
    used = sum(p.nbytes - p.free_bytes for p in ag.pools)
    print(f"FSDP rank {rank} {'OK' if not fails else 'FAIL ' + '; '.join(fails)} "
          f"segments={len(ag.pools)} in_use={used}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if not fails else 1)


if __name__ == "__main__":
    main()

"""torchrun worker: forests with more ranks than GPUs over real NVLink —
ranks_per_gpu ranks per process (one cooperative grid), e.g. the 8-GPU
NVSwitch and the sparse 2x4 forests on 4 GPUs.  Bit-exact against the oracle."""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import forest_oracle as fo  # noqa: E402
from paper_2402_06787_b200 import MultiRankComm  # noqa: E402
from paper_2402_06787_b200.topology import groups_switch_doc, nvswitch_doc  # noqa: E402


def host(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("gloo")
    p, P = dist.get_rank(), dist.get_world_size()
    fails = []
    for name, doc in (("nvs8", nvswitch_doc(8)), ("groups300", groups_switch_doc(300)),
                      ("groups100", groups_switch_doc(100))):
        N = 8
        per = N // P
        mine = list(range(p * per, (p + 1) * per))
        comm = MultiRankComm(doc, local_ranks=mine, world_size=N, device=local,
                             options={"timeout_ms": 20000})
        for proto in (-1, 0):
            comm.set_option("proto", proto)
            for S in (1000, 1 << 18, 1 << 20):  # one-hop / one-shot, two-hop, LL128 / flags
                g = torch.Generator().manual_seed(S + proto)
                sends = [torch.randn(S, generator=g) for _ in range(N)]
                outs = [torch.empty(N * S, device=dev) for _ in mine]
                comm.all_gather(outs, [sends[r].to(dev) for r in mine])
                ref = fo.allgather(comm.schedule("allgather"), [x.numpy() for x in sends])
                for i, r in enumerate(mine):
                    if not np.array_equal(host(outs[i]).view(np.uint32), ref[r].view(np.uint32)):
                        fails.append(f"{name} allgather proto={proto} S={S} rank {r}")
                ins = [torch.empty(N * S).uniform_(-1, 1, generator=g).to(torch.bfloat16) for _ in range(N)]
                outs = [torch.empty(S, device=dev, dtype=torch.bfloat16) for _ in mine]
                comm.reduce_scatter(outs, [ins[r].to(dev) for r in mine])
                ref = fo.reduce_scatter(comm.schedule("reduce_scatter"), [host(x) for x in ins], "bfloat16")
                for i, r in enumerate(mine):
                    if not np.array_equal(host(outs[i]), ref[r]):
                        fails.append(f"{name} reduce_scatter proto={proto} S={S} rank {r}")
                ins = [torch.empty(N * S).uniform_(-1, 1, generator=g) for _ in range(N)]
                bufs = [ins[r].to(dev) for r in mine]
                comm.all_reduce(bufs)
                ref = fo.allreduce(comm.schedule("allreduce"), [x.numpy() for x in ins], "float32")
                for i, r in enumerate(mine):
                    if not np.array_equal(host(bufs[i]).view(np.uint32), ref[r].view(np.uint32)):
                        fails.append(f"{name} allreduce proto={proto} S={S} rank {r}")
        comm.check()
        comm.close()
    print(f"MULTIRANK proc {p} {'OK' if not fails else 'FAIL ' + '; '.join(fails[:6])}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

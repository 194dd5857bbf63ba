"""torchrun worker: ranks that pass differently registered output buffers to
one allgather get a loud device error (FC_DEVERR_BUFFER_MISMATCH), not
silently misplaced data.  Only the chunk-flag protocol stores straight into
peers' output buffers (LL128 stores land in the library's staging), so the
check is exercised with that protocol.  Prints `MISMATCH rank r OK|FAIL`."""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.errors import DeviceError  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local,
                          options={"timeout_ms": 3000, "proto": 0})
    S = 4096
    inp = torch.full((S,), float(rank), device=dev)
    a = comm.empty(n * S)
    b = comm.empty(n * S)
    comm.all_gather(a, inp)          # matched call: fine
    comm.check()
    ok = torch.equal(a.view(n, S)[:, 0].cpu(), torch.arange(n, dtype=torch.float32))
    comm.all_gather(a if rank == 0 else b, inp)  # rank 0 disagrees with everyone else
    err = ""
    try:
        comm.check()
    except DeviceError as exc:
        err = str(exc)
    dist.barrier()
    good = ok and ("different output buffer" in err or "timed out" in err)
    print(f"MISMATCH rank {rank} {'OK' if good else 'FAIL'} err={err!r}", flush=True)
    dist.barrier()
    os._exit(0 if good else 1)  # the communicator is poisoned by design


if __name__ == "__main__":
    main()

"""torchrun: eager vs CUDA-graph time per small allgather across launch
options (PDL, CTAs per rank), 2000-call windows.
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/eager_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402
from tools.latency_probe import graph_us  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    for S in (64, 1 << 16):
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S)
        f = lambda: comm.all_gather(out, inp)  # noqa: E731
        side = torch.cuda.Stream()
        for ctas in (128,):
            for pdl in (1, 0):
                comm.set_option("ctas_per_rank", ctas)
                comm.set_option("pdl", pdl)
                e = timed(f, 2000, 50, dist) * 1e3
                with torch.cuda.stream(side):
                    e2 = timed(f, 2000, 50, dist) * 1e3
                g = graph_us(f)
                if rank == 0:
                    print(f"AG {S*4*n:8d} B ctas={ctas:3d} pdl={pdl}: eager(default stream) {e:6.2f} "
                          f"eager(side stream) {e2:6.2f} graph {g:6.2f} us", flush=True)
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

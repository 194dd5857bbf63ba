"""torchrun (N ranks): is a mid-size one-hop allgather's occasional slow
window (N=4, 2 MiB: 10 us usually, 15.7 us in one of three runs) device- or
host-side?  Times several windows of back-to-back eager calls, and of CUDA
graph replays of the same calls, reallocating the output between windows.

    torchrun --nproc-per-node 4 tools/bimodal_probe.py [MiB] [option=value ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def window(fn, k, dist, host=None):
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    fn(k)
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    x = torch.tensor([e0.elapsed_time(e1) / k * 1e3, (t1 - t0) / k * 1e6], device="cuda")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    if host is not None:
        host.append(float(x[1].item()))
    return float(x[0].item())


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    mib = float(sys.argv[1]) if len(sys.argv) > 1 else 2
    for o in sys.argv[2:]:  # name=value executor options
        k, v = o.split("=")
        comm.set_option(k, int(v))
    S = int(mib * (1 << 20)) // n // 4
    inp = torch.randn(S, device=dev)
    eager, graph, host = [], [], []
    for w in range(8):
        out = comm.empty(n * S)

        def run(k):
            for _ in range(k):
                comm.all_gather(out, inp)
        run(5)
        eager.append(window(run, 200, dist, host))
        side = torch.cuda.Stream()
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            run(3)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                run(20)
        torch.cuda.synchronize()
        g.replay()
        graph.append(window(lambda k: [g.replay() for _ in range(k // 20)], 200, dist))
    if rank == 0:
        print(f"N={n} {mib} MiB proto={comm.last_call_info()['proto']}")
        print("eager us/call:", " ".join(f"{x:5.1f}" for x in eager))
        print("graph us/call:", " ".join(f"{x:5.1f}" for x in graph))
        print("host issue us/call (eager, max over ranks):", " ".join(f"{x:5.1f}" for x in host))
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

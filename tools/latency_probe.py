"""torchrun: per-call latency of small collectives -- eager (host + device),
host-side cost per call, and CUDA-graph replay (device only) -- for the
forest kernel and NCCL.
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/latency_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import timed  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def host_us(fn, iters=200):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(iters):
        fn()
    h = (time.perf_counter() - t) / iters * 1e6
    torch.cuda.synchronize()
    return h


def graph_us(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ms = timed(g.replay, 10, 3, dist)
    return ms * 1e3 / reps


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    for k, v in (a.split("=") for a in sys.argv[1:]):
        comm.set_option(k, int(v))
    for S in (16, 1024, 4096, 16384, 65536, 1 << 20):
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S)
        o2 = torch.empty(n * S, device=dev)
        f = lambda: comm.all_gather(out, inp)  # noqa: E731
        g = lambda: dist.all_gather_into_tensor(o2, inp)  # noqa: E731
        e1 = timed(f, 200, 20, dist) * 1e3
        e1b = timed(f, 2000, 20, dist) * 1e3
        h1 = host_us(f)
        try:
            g1 = graph_us(f)
        except Exception as exc:  # noqa: BLE001
            g1 = float("nan")
            if rank == 0:
                print("graph capture failed:", exc, flush=True)
        ref = out.clone()
        e2 = timed(g, 200, 20, dist) * 1e3
        h2 = host_us(g)
        try:
            g2 = graph_us(g)
        except Exception as exc:  # noqa: BLE001
            g2 = float("nan")
            if rank == 0:
                print("nccl graph capture failed:", exc, flush=True)
        ok = torch.equal(out, ref) and torch.equal(o2, ref)
        if rank == 0:
            print(f"AG {S*4*n:9d} B  forest: eager {e1:6.1f} (x2000 {e1b:6.1f}) host {h1:5.1f} graph {g1:6.1f} us"
                  f" | nccl: eager {e2:6.1f} host {h2:5.1f} graph {g2:6.1f} us  ok={ok}", flush=True)
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

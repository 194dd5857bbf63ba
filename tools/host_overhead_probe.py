"""Host issue cost per collective call vs device time (torchrun, N ranks).

    torchrun --nproc-per-node N tools/host_overhead_probe.py [--mib 64,25]

For each size: wall time to ISSUE K calls (no synchronisation inside), device
time per call (CUDA events), and the same through the raw C ABI
(fc_allgather / fc_allreduce via ctypes) -- if host issue time exceeds
device time, back-to-back timing measures the host, not the kernel.
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import MIB, gbs  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.executor import _raw_stream  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def measure(fn, k=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    host = (time.perf_counter() - t0) / k * 1e6
    e1.record(s)
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / k * 1e3
    return host, dev


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", default="64,25,1")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=local)
    lib = comm._lib
    for mib in [int(x) for x in args.mib.split(",")]:
        M = mib * MIB
        S = M // n // 4
        inp = torch.randn(S, device=dev)
        out = comm.empty(n * S, dtype=torch.float32)
        comm.all_gather(out, inp)
        st = _raw_stream(local)
        h1, d1 = measure(lambda: comm.all_gather(out, inp))
        h2, d2 = measure(lambda: lib.fc_allgather(comm._comm, inp.data_ptr(), out.data_ptr(), S, 7, st))
        buf = comm.empty(M // 2, dtype=torch.bfloat16)
        buf.normal_()
        comm.all_reduce(buf)
        h3, d3 = measure(lambda: comm.all_reduce(buf))
        h4, d4 = measure(lambda: lib.fc_allreduce(comm._comm, buf.data_ptr(), buf.data_ptr(),
                                                  M // 2, 9, 0, st))
        if rank == 0:
            print(f"{mib:5d} MiB  allgather python: host {h1:7.1f} us dev {d1:7.1f} us ({gbs(M, d1 / 1e3):7.1f} GB/s)"
                  f" | C ABI: host {h2:7.1f} dev {d2:7.1f} ({gbs(M, d2 / 1e3):7.1f} GB/s) proto {comm.last_call_info()['proto']}",
                  flush=True)
            print(f"{mib:5d} MiB  allreduce python: host {h3:7.1f} us dev {d3:7.1f} us ({gbs(M, d3 / 1e3):7.1f} GB/s)"
                  f" | C ABI: host {h4:7.1f} dev {d4:7.1f} ({gbs(M, d4 / 1e3):7.1f} GB/s)", flush=True)
        comm.deregister(out)
        comm.deregister(buf)
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

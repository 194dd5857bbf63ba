"""Is NCCL under-configured on this box?  (N=2 allgather 4 GiB at
only 475 GB/s busbw.)  torchrun, N ranks: NCCL default vs more channels
(NCCL_MIN_NCHANNELS / NCCL_MAX_NCHANNELS) and protocol / algorithm pins, on
large allgather / reduce-scatter / allreduce."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import MIB, gbs, timed  # noqa: E402

VARIANTS = [
    ("default", {}),
    ("min_ch32", {"NCCL_MIN_NCHANNELS": "32"}),
    ("min_ch64", {"NCCL_MIN_NCHANNELS": "64", "NCCL_MAX_NCHANNELS": "64"}),
    ("ring_simple_ch32", {"NCCL_ALGO": "Ring", "NCCL_PROTO": "Simple", "NCCL_MIN_NCHANNELS": "32"}),
    ("nvls", {"NCCL_ALGO": "NVLS"}),
]


def group_with(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        g = dist.new_group(backend="nccl")
        x = torch.ones(1024, device="cuda")
        dist.all_reduce(x, group=g)
        torch.cuda.synchronize()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return g


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    n = dist.get_world_size()
    groups = []
    for name, env in VARIANTS:
        try:
            groups.append((name, group_with(env)))
        except Exception as exc:  # noqa: BLE001
            if dist.get_rank() == 0:
                print(f"# {name}: {exc}", flush=True)
    for mib in (1024, 4096):
        M = mib * MIB
        S = M // n // 4
        inp = torch.randn(S, device="cuda")
        out = torch.empty(n * S, device="cuda")
        for name, g in groups:
            ms = timed(lambda: dist.all_gather_into_tensor(out, inp, group=g), 10, 3, dist)
            if dist.get_rank() == 0:
                print(f"allgather {mib:5d} MiB {name:18s} {gbs(M, ms):8.1f} GB/s algbw", flush=True)
        del inp, out
    M = 1024 * MIB
    rin = torch.randn(M // 4, device="cuda")
    rout = torch.empty(M // 4 // n, device="cuda")
    buf = torch.randn(M // 2, device="cuda").to(torch.bfloat16)
    for name, g in groups:
        ms = timed(lambda: dist.reduce_scatter_tensor(rout, rin, group=g), 10, 3, dist)
        ms2 = timed(lambda: dist.all_reduce(buf, group=g), 10, 3, dist)
        if dist.get_rank() == 0:
            print(f"reduce_scatter 1024 MiB {name:18s} {gbs(M, ms):8.1f} GB/s | allreduce bf16 1 GiB "
                  f"{gbs(M, ms2):8.1f} GB/s", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

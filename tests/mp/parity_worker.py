"""torchrun worker: multi-GPU parity of ForestCollComm against the oracle.

Every rank regenerates all ranks' seeded inputs on the host, so it can run
the CPU oracle itself and compare its own device output bit-for-bit.
Launched by tests/test_gpu_multiproc.py (one process per GPU).
"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import forest_oracle as fo  # noqa: E402
from _common import init  # noqa: E402
from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def host(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def seeded(n_el, dtype, seed, bits=False):
    g = torch.Generator().manual_seed(seed)
    if dtype == torch.int32:
        return torch.randint(-2**20, 2**20, (n_el,), generator=g, dtype=torch.int32)
    if bits:
        # raw bit patterns (NaN / denormal / inf included) for byte-exact checks
        return torch.randint(0, 2**31 - 1, (n_el,), generator=g, dtype=torch.int32).view(torch.float32)
    return torch.empty(n_el).uniform_(-1, 1, generator=g).to(dtype)


def main():
    local = init()
    dev = torch.device(f"cuda:{local}")
    rank, n = dist.get_rank(), dist.get_world_size()
    topo = nvswitch_doc(n)
    comm = ForestCollComm(topo, rank=rank, world_size=n, device=local,
                          options={"timeout_ms": 20000})
    fails = []
    # auto (one-hop / one-shot, else LL128 where aligned), auto with the
    # one-hop paths off (the forest's LL128 lines), the chunk-flag protocol,
    # and (N=2) every allgather through the copy-engine path (ce_min=1)
    twohop_default = comm.get_option("twohop_max")
    for proto, onehop, ce in ((-1, True, 0), (-1, False, 0), (0, True, 0), (-1, True, 1)):
        comm.set_option("proto", proto)
        comm.set_option("oneshot_ag_max", (16 << 20) if onehop else 0)
        comm.set_option("oneshot_max", (2 << 20) if onehop else 0)
        comm.set_option("twohop_max", twohop_default if onehop else 0)
        comm.set_option("ce_min", ce)
        fails += [f"proto={proto} onehop={onehop} ce={ce}: {f}" for f in run_all(comm, rank, n, dev)]
        if ce and n == 2 and comm.last_call_info()["proto"] not in ("ce", "oneshot", "flags", "ll128"):
            fails.append("unexpected path")
    comm.check()
    print(f"RANK {rank} {'OK' if not fails else 'FAIL ' + '; '.join(fails)}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


def run_all(comm, rank, n, dev):
    fails = []
    # allgather: odd and aligned sizes, bit patterns
    for S in (1, 333, 4096, 1 << 20, (1 << 22) + 5):
        for seed in (10, 11):
            sends = [seeded(S, torch.float32, seed * 100 + r, bits=seed % 2 == 1) for r in range(n)]
            out = comm.empty(n * S, dtype=torch.float32)
            out.fill_(-7.0)
            comm.all_gather(out, sends[rank].to(dev))
            torch.cuda.synchronize()
            got = comm.last_call_info()["proto"]
            enabled = comm.get_option("proto") < 0 and comm.get_option("oneshot_ag_max") > 0
            ce = n == 2 and comm.get_option("ce_min") == 1 and comm.get_option("proto") < 0
            if ce and got != "ce":
                fails.append(f"allgather S={S} took {got}, expected the copy-engine path")
            if enabled and not ce and S == 4096 and got != "oneshot":
                fails.append(f"allgather S={S} took {got}, expected the one-hop path")
            if not enabled and got in ("oneshot", "ce"):
                fails.append(f"allgather S={S} took the one-hop path although it is off")
            ref = fo.allgather(comm.schedule("allgather"), [host(x) for x in sends])[rank]
            if not np.array_equal(host(out).view(np.uint8), ref.view(np.uint8)):
                fails.append(f"allgather S={S} seed={seed}")
    # reduce-scatter
    for dtype, name in ((torch.float32, "float32"), (torch.bfloat16, "bfloat16"), (torch.int32, "int32")):
        for S in (7, 1000, (1 << 20) + 3):
            ins = [seeded(n * S, dtype, 500 + r + 2 * S) for r in range(n)]
            out = torch.zeros(S, dtype=dtype, device=dev)
            comm.reduce_scatter(out, ins[rank].to(dev))
            torch.cuda.synchronize()
            ref = fo.reduce_scatter(comm.schedule("reduce_scatter"), [host(x) for x in ins], name)[rank]
            if not np.array_equal(host(out).view(np.uint8), ref.view(np.uint8)):
                fails.append(f"reduce_scatter {name} S={S}")
    # allreduce (in place)
    for dtype, name in ((torch.bfloat16, "bfloat16"), (torch.float32, "float32"), (torch.int32, "int32")):
        for count in (5, 12345, 1 << 22):
            ins = [seeded(count, dtype, 900 + r + count) for r in range(n)]
            buf = comm.empty(count, dtype=dtype)
            buf.copy_(ins[rank].to(dev))
            comm.all_reduce(buf)
            torch.cuda.synchronize()
            ref = fo.allreduce(comm.schedule("allreduce"), [host(x) for x in ins], name)[rank]
            if not np.array_equal(host(buf).view(np.uint8), ref.view(np.uint8)):
                fails.append(f"allreduce {name} count={count}")
    # one-shot path (small reductions: peer stores of every input + local in-tree
    # evaluation): must be bit-identical to the forest kernel / oracle
    for dtype, name in ((torch.float32, "float32"), (torch.bfloat16, "bfloat16"), (torch.int32, "int32")):
        for count in (8 * n, 4096, 16 * 1024, 150 * 1024 + 8 * n):  # last: LL128-line format
            ins = [seeded(count, dtype, 1700 + r + count) for r in range(n)]
            buf = comm.empty(count, dtype=dtype)
            buf.copy_(ins[rank].to(dev))
            comm.all_reduce(buf)
            want = "oneshot" if comm.get_option("oneshot_max") > 0 else None
            if comm.get_option("proto") < 0 and want and comm.last_call_info()["proto"] != want:
                fails.append(f"allreduce {name} count={count} did not take the one-shot path")
            torch.cuda.synchronize()
            ref = fo.allreduce(comm.schedule("allreduce"), [host(x) for x in ins], name)[rank]
            if not np.array_equal(host(buf).view(np.uint8), ref.view(np.uint8)):
                fails.append(f"one-shot allreduce {name} count={count}")
            S = count // n
            out = torch.zeros(S, dtype=dtype, device=dev)
            comm.reduce_scatter(out, ins[rank].to(dev))
            torch.cuda.synchronize()
            ref = fo.reduce_scatter(comm.schedule("reduce_scatter"), [host(x) for x in ins], name)[rank]
            if not np.array_equal(host(out).view(np.uint8), ref.view(np.uint8)):
                fails.append(f"one-shot reduce_scatter {name} S={S}")
    # two-hop path (mid sizes: shards to their roots, in-tree evaluated at the
    # root, reduced shards to everyone): bit-identical as well
    for dtype, name in ((torch.float32, "float32"), (torch.bfloat16, "bfloat16"), (torch.int32, "int32")):
        es = torch.tensor([], dtype=dtype).element_size()
        count = (3 << 20) // es // (64 * n) * (64 * n)  # 3 MiB, equal 256-byte-aligned shards
        ins = [seeded(count, dtype, 2300 + r) for r in range(n)]
        buf = comm.empty(count, dtype=dtype)
        buf.copy_(ins[rank].to(dev))
        comm.all_reduce(buf)
        torch.cuda.synchronize()
        got = comm.last_call_info()["proto"]
        if comm.get_option("proto") < 0 and comm.get_option("oneshot_max") > 0 and got not in ("twohop", "ce"):
            fails.append(f"allreduce {name} count={count} took {got}, expected the two-hop path")
        ref = fo.allreduce(comm.schedule("allreduce"), [host(x) for x in ins], name)[rank]
        if not np.array_equal(host(buf).view(np.uint8), ref.view(np.uint8)):
            fails.append(f"two-hop allreduce {name} count={count}")
        out = torch.zeros(count // n, dtype=dtype, device=dev)
        comm.reduce_scatter(out, ins[rank].to(dev))
        torch.cuda.synchronize()
        ref = fo.reduce_scatter(comm.schedule("reduce_scatter"), [host(x) for x in ins], name)[rank]
        if not np.array_equal(host(out).view(np.uint8), ref.view(np.uint8)):
            fails.append(f"two-hop reduce_scatter {name} S={count // n}")
    # op avg (fp dtypes): the root scales its fp32 sum by fp32(1/N) once
    for dtype, name in ((torch.bfloat16, "bfloat16"), (torch.float32, "float32")):
        for S in (999, (1 << 19) + 8):
            ins = [seeded(n * S, dtype, 1300 + r + S) for r in range(n)]
            out = torch.zeros(S, dtype=dtype, device=dev)
            comm.reduce_scatter(out, ins[rank].to(dev), op="avg")
            buf = comm.empty(n * S, dtype=dtype)
            buf.copy_(ins[rank].to(dev))
            comm.all_reduce(buf, op=dist.ReduceOp.AVG)
            torch.cuda.synchronize()
            hs = [host(x) for x in ins]
            ref = fo.reduce_scatter(comm.schedule("reduce_scatter"), hs, name, op="avg")[rank]
            if not np.array_equal(host(out).view(np.uint8), ref.view(np.uint8)):
                fails.append(f"reduce_scatter avg {name} S={S}")
            ref = fo.allreduce(comm.schedule("allreduce"), hs, name, op="avg")[rank]
            if not np.array_equal(host(buf).view(np.uint8), ref.view(np.uint8)):
                fails.append(f"allreduce avg {name} count={n * S}")
    # CUDA graph: capture an allgather + allreduce once, replay with new inputs
    S = 5000
    gin = torch.empty(S, device=dev)
    gout = comm.empty(n * S, dtype=torch.float32)
    gbuf = comm.empty(n * S, dtype=torch.float32)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        comm.all_gather(gout, gin)
        comm.all_reduce(gbuf)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        comm.all_gather(gout, gin)
        comm.all_reduce(gbuf)
    for rep in range(3):
        sends = [seeded(S, torch.float32, 8100 + 10 * rep + r) for r in range(n)]
        ins = [seeded(n * S, torch.float32, 8500 + 10 * rep + r) for r in range(n)]
        gin.copy_(sends[rank].to(dev))
        gbuf.copy_(ins[rank].to(dev))
        dist.barrier()
        graph.replay()
        torch.cuda.synchronize()
        ref = fo.allgather(comm.schedule("allgather"), [host(x) for x in sends])[rank]
        if not np.array_equal(host(gout).view(np.uint8), ref.view(np.uint8)):
            fails.append(f"graph replay {rep} allgather")
        ref = fo.allreduce(comm.schedule("allreduce"), [host(x) for x in ins], "float32")[rank]
        if not np.array_equal(host(gbuf).view(np.uint8), ref.view(np.uint8)):
            fails.append(f"graph replay {rep} allreduce")
    # back-to-back calls reusing buffers (entry barrier / epoch reuse)
    S = 1 << 18
    out = comm.empty(n * S, dtype=torch.float32)
    for it in range(20):
        sends = [seeded(S, torch.float32, 7000 + it * 16 + r) for r in range(n)]
        comm.all_gather(out, sends[rank].to(dev))
        got = host(out).copy()
        ref = fo.allgather(comm.schedule("allgather"), [host(x) for x in sends])[rank]
        if not np.array_equal(got.view(np.uint8), ref.view(np.uint8)):
            fails.append(f"allgather repeat {it}")
            break
    return fails


if __name__ == "__main__":
    main()

"""torchrun worker: the NVLS (multicast) engine on a multicast/aggregation
NVSwitch topology — parity and timing against the tree engine.

Parity: allgather bit-exact; int32 reductions exact; fp32/bf16 reductions
within tolerance (the switch's accumulation order is not the tree order).
Prints one `NVLS rank r OK|FAIL|SKIP` line per rank and, on rank 0, timings.
"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import forest_oracle as fo  # noqa: E402

from paper_2402_06787_b200 import ForestCollComm  # noqa: E402
from paper_2402_06787_b200.topology import nvswitch_doc  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    rank, n = dist.get_rank(), dist.get_world_size()
    comm = ForestCollComm(nvswitch_doc(n, multicast=True), rank=rank, world_size=n, device=local,
                          nvls_bytes=3 << 30, options={"timeout_ms": 20000},
                          reduction_order="switch")
    if not comm.nvls_enabled:
        print(f"NVLS rank {rank} SKIP (no multicast)", flush=True)
        return
    fails = []
    g = torch.Generator().manual_seed(100)
    # allgather: bit-exact
    for S in (4, 1000, 1 << 20):
        allin = [torch.randint(0, 2**31 - 1, (S,), generator=g, dtype=torch.int32).view(torch.float32)
                 for _ in range(n)]
        out = comm.nvls_empty(n * S, torch.float32)
        comm.all_gather(out, allin[rank].to(dev))
        torch.cuda.synchronize()
        if comm.last_call_info()["proto"] not in ("nvls", "nvls_ll"):
            fails.append("allgather did not use NVLS")
        if not torch.equal(out.cpu().view(torch.int32), torch.cat(allin).view(torch.int32)):
            fails.append(f"allgather S={S}")
    # small allgathers: LL over multicast into ordinary (non-pool) buffers, queued
    # back to back without a host sync (staging halves alternate by epoch)
    pend = []
    for it in range(12):
        S = [2, 64, 1000, 4096, 65536][it % 5]
        allin = [torch.randint(0, 2**31 - 1, (S,), generator=g, dtype=torch.int32).view(torch.float32)
                 for _ in range(n)]
        out = torch.full((n * S,), -1.0, device=dev)
        comm.all_gather(out, allin[rank].to(dev))
        if comm.last_call_info()["proto"] != "nvls_ll":
            fails.append(f"small allgather S={S} did not use the LL multicast protocol")
        pend.append((S, out, torch.cat(allin)))
    torch.cuda.synchronize()
    for S, out, want in pend:
        if not torch.equal(out.cpu().view(torch.int32), want.view(torch.int32)):
            fails.append(f"LL multicast allgather S={S}")
    # small reductions: LL multicast + local in-tree evaluation, bit-exact with
    # the oracle (the tree engine's arithmetic), ordinary buffers
    def host(t):
        return (t.view(torch.int16).cpu().numpy().view(np.uint16) if t.dtype == torch.bfloat16
                else t.cpu().numpy())

    red_default = comm.get_option("nvls_ll_red_max")
    comm.set_option("nvls_ll_red_max", 8 << 20)  # route every size below through the LL path
    for dtype, name in ((torch.float32, "float32"), (torch.bfloat16, "bfloat16"), (torch.int32, "int32")):
        for S, op in ((16, "sum"), (1000, "sum"), (4096, "avg"), (20000, "sum")):
            if op == "avg" and dtype == torch.int32:
                continue
            allin = [(torch.randint(-1000, 1000, (n * S,), generator=g).to(dtype)
                      if dtype == torch.int32 else torch.empty(n * S).uniform_(-1, 1, generator=g).to(dtype))
                     for _ in range(n)]
            hs = [host(x) for x in allin]
            out = torch.empty(S, dtype=dtype, device=dev)
            comm.reduce_scatter(out, allin[rank].to(dev), op=op)
            if comm.last_call_info()["proto"] != "nvls_ll":
                fails.append(f"small reduce_scatter {name} S={S} did not use LL multicast")
            want = fo.reduce_scatter(comm.schedule("reduce_scatter"), hs, name, op=op)[rank]
            if not np.array_equal(host(out).view(np.uint8), want.view(np.uint8)):
                fails.append(f"LL reduce_scatter {name} S={S} op={op} not bit-exact")
            buf = allin[rank].to(dev)
            comm.all_reduce(buf, op=op)
            if comm.last_call_info()["proto"] != "nvls_ll":
                fails.append(f"small allreduce {name} n={n * S} did not use LL multicast")
            want = fo.allreduce(comm.schedule("allreduce"), hs, name, op=op)[rank]
            if not np.array_equal(host(buf).view(np.uint8), want.view(np.uint8)):
                fails.append(f"LL allreduce {name} count={n * S} op={op} not bit-exact")
    comm.set_option("nvls_ll_red_max", red_default)
    # reduce-scatter / allreduce
    for dtype, tol in ((torch.int32, 0), (torch.float32, 1e-5), (torch.bfloat16, 2e-2)):
        for S in (64, 1 << 18):
            allin = [(torch.randint(-1000, 1000, (n * S,), generator=g).to(dtype)
                      if dtype == torch.int32 else torch.empty(n * S).uniform_(-1, 1, generator=g).to(dtype))
                     for _ in range(n)]
            ref = torch.stack([x.double() for x in allin]).sum(0)
            inp = comm.nvls_empty(n * S, dtype)
            inp.copy_(allin[rank].to(dev))
            out = torch.empty(S, dtype=dtype, device=dev)
            comm.reduce_scatter(out, inp)
            got = out.double().cpu()
            want = ref[rank * S:(rank + 1) * S]
            if not torch.allclose(got, want, rtol=tol, atol=tol * n):
                fails.append(f"reduce_scatter {dtype} S={S}")
            buf = comm.nvls_empty(n * S, dtype)
            buf.copy_(allin[rank].to(dev))
            comm.all_reduce(buf)
            if not torch.allclose(buf.double().cpu(), ref, rtol=tol, atol=tol * n):
                fails.append(f"allreduce {dtype} S={S}")
            if dtype != torch.int32:  # op avg: switch sum scaled by 1/N
                inp.copy_(allin[rank].to(dev))
                comm.reduce_scatter(out, inp, op="avg")
                if not torch.allclose(out.double().cpu(), want / n, rtol=tol, atol=tol):
                    fails.append(f"reduce_scatter avg {dtype} S={S}")
                buf.copy_(allin[rank].to(dev))
                comm.all_reduce(buf, op="avg")
                if not torch.allclose(buf.double().cpu(), ref / n, rtol=tol, atol=tol):
                    fails.append(f"allreduce avg {dtype} S={S}")
    # the same pool tensors with order="tree": the forest's order, bit-exact
    # vs the oracle (the in-switch order is opt-in only)
    for dtype, name in ((torch.bfloat16, "bfloat16"), (torch.float32, "float32")):
        for S in (64, 1 << 18, 1 << 22):
            allin = [torch.empty(n * S).uniform_(-1, 1, generator=g).to(dtype) for _ in range(n)]
            hs = [x.view(torch.int16).numpy().view(np.uint16) if dtype == torch.bfloat16 else x.numpy()
                  for x in allin]
            buf = comm.nvls_empty(n * S, dtype)
            buf.copy_(allin[rank].to(dev))
            comm.all_reduce(buf, order="tree")
            torch.cuda.synchronize()
            if comm.last_call_info()["order"] != "tree":
                fails.append(f"tree-order allreduce {name} S={S} reported {comm.last_call_info()}")
            got = buf.cpu()
            got = got.view(torch.int16).numpy().view(np.uint16) if dtype == torch.bfloat16 else got.numpy()
            want = fo.allreduce(comm.schedule("allreduce"), hs, name)[rank]
            if not np.array_equal(got.view(np.uint8), want.view(np.uint8)):
                fails.append(f"tree-order allreduce {name} S={S} not bit-exact")
            inp = comm.nvls_empty(n * S, dtype)
            inp.copy_(allin[rank].to(dev))
            out = torch.empty(S, dtype=dtype, device=dev)
            comm.reduce_scatter(out, inp, order="tree")
            torch.cuda.synchronize()
            got = out.cpu()
            got = got.view(torch.int16).numpy().view(np.uint16) if dtype == torch.bfloat16 else got.numpy()
            want = fo.reduce_scatter(comm.schedule("reduce_scatter"), hs, name)[rank]
            if not np.array_equal(got.view(np.uint8), want.view(np.uint8)):
                fails.append(f"tree-order reduce_scatter {name} S={S} not bit-exact")
    comm.check()
    print(f"NVLS rank {rank} {'OK' if not fails else 'FAIL ' + '; '.join(fails)}", flush=True)
    # timing: NVLS engine vs tree engine on the same sizes
    if "--time" in sys.argv:
        from bench import MIB, gbs, timed

        res = []
        for coll, mib in (("allgather", 64), ("allgather", 1024), ("reduce_scatter", 256),
                          ("allreduce", 25), ("allreduce", 1024)):
            M = mib * MIB
            if coll == "allgather":
                S = M // n // 4
                inp = torch.randn(S, device=dev)
                o_n = comm.nvls_empty(n * S, torch.float32)
                o_t = comm.empty(n * S, dtype=torch.float32)
                f_n = lambda: comm.all_gather(o_n, inp)  # noqa: E731
                f_t = lambda: comm.all_gather(o_t, inp)  # noqa: E731
            elif coll == "reduce_scatter":
                R = M // n // 4
                i_n = comm.nvls_empty(n * R, torch.float32)
                i_n.normal_()
                i_t = torch.randn(n * R, device=dev)
                out = torch.empty(R, device=dev)
                f_n = lambda: comm.reduce_scatter(out, i_n)  # noqa: E731
                f_t = lambda: comm.reduce_scatter(out, i_t)  # noqa: E731
            else:
                cnt = M // 2
                b_n = comm.nvls_empty(cnt, torch.bfloat16)
                b_n.normal_()
                b_t = comm.empty(cnt, dtype=torch.bfloat16)
                b_t.normal_()
                f_n = lambda: comm.all_reduce(b_n)  # noqa: E731
                f_t = lambda: comm.all_reduce(b_t)  # noqa: E731
            ms_n = 1e9
            for ctas in (32, 64, 128):
                comm.set_option("nvls_ctas", ctas)
                m = timed(f_n, 10, 3, dist)
                if rank == 0:
                    print(f"   {coll} {mib} MiB nvls ctas={ctas}: {m * 1e3:.1f} us", flush=True)
                ms_n = min(ms_n, m)
            ms_t = timed(f_t, 10, 3, dist)
            t = comm.t_star(coll, M)
            res.append((coll, mib, ms_n, gbs(M, ms_n), t * 1e3 / ms_n, ms_t, gbs(M, ms_t)))
        if rank == 0:
            for r in res:
                print(f"{r[0]:15s} {r[1]:5d} MiB  nvls {r[2]*1e3:8.1f} us {r[3]:8.1f} GB/s "
                      f"(T* frac {r[4]:.3f})   tree {r[5]*1e3:8.1f} us {r[6]:8.1f} GB/s", flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""torchrun worker: N rank processes on ONE GPU (cuda:0), real peer mapping.

Every rank is its own process with its own CUDA context, so the
communicator takes the production path exactly as on N GPUs: workspace and
output-buffer CUDA IPC handles exchanged over gloo, cudaIpcOpenMemHandle of
the peers' memory (same device), the entry barrier with the output-buffer
tag check, programmatic dependent launch, and the one-hop / one-shot paths
(which virtual mode reaches only inside one grid).  Contexts of different
processes time-slice the GPU, so every cross-rank wait spans a context
switch: sizes stay small.  Launched by tests/test_gpu_samedev.py.
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


def host(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def seeded(n_el, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    if dtype == torch.int32:
        return torch.randint(-2**20, 2**20, (n_el,), generator=g, dtype=torch.int32)
    return torch.empty(n_el).uniform_(-1, 1, generator=g).to(dtype)


def main():
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    dist.init_process_group("gloo")
    rank, n = dist.get_rank(), dist.get_world_size()
    mode = sys.argv[1] if len(sys.argv) > 1 else "parity"
    comm = ForestCollComm(nvswitch_doc(n), rank=rank, world_size=n, device=0,
                          scratch_bytes=None if mode == "grow" else 64 << 20,
                          max_scratch_bytes=512 << 20, options={"timeout_ms": 60000})
    fails = []
    if mode == "grow":
        fails = grow(comm, rank, n, dev)
    if mode == "parity":
        fails = parity(comm, rank, n, dev)
    elif mode == "fresh_outputs":
        fails = fresh_outputs(comm, rank, n, dev)
    elif mode == "mismatch":
        fails = mismatch(comm, rank, n, dev)
    elif mode == "guards":
        fails = guards(comm, rank, n, dev)
    elif mode == "mismatch_ce":
        fails = mismatch(comm, rank, n, dev, ce=True)
    comm.check() if not mode.startswith("mismatch") else None
    print(f"RANK {rank} {'OK' if not fails else 'FAIL ' + '; '.join(fails)}", flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


def _check(got, ref, what, fails):
    if not np.array_equal(np.ascontiguousarray(got).view(np.uint8),
                          np.ascontiguousarray(ref).view(np.uint8)):
        fails.append(what)


def parity(comm, rank, n, dev):
    fails = []
    s_ag, s_rs, s_ar = (comm.schedule(c) for c in ("allgather", "reduce_scatter", "allreduce"))
    cases = [(-1, 1 << 12, "oneshot"), (-1, (1 << 12) + 1, None), (1, 1 << 14, "ll128"),
             (0, (1 << 14) + 3, "flags")]
    for proto, S, want in cases:
        comm.set_option("proto", proto)
        ins = [seeded(S, torch.float32, 100 + r + S) for r in range(n)]
        out = torch.empty(n * S, device=dev)
        comm.all_gather(out, ins[rank].to(dev))
        torch.cuda.synchronize()
        got = comm.last_call_info()["proto"]
        if want and got != want:
            fails.append(f"allgather S={S}: path {got}, expected {want}")
        _check(out.cpu().numpy(), fo.allgather(s_ag, [x.numpy() for x in ins])[rank],
               f"allgather proto={proto} S={S}", fails)
        for dt, dname in ((torch.bfloat16, "bfloat16"), (torch.int32, "int32")):
            ins = [seeded(n * S, dt, 200 + r + S) for r in range(n)]
            out = torch.empty(S, device=dev, dtype=dt)
            comm.reduce_scatter(out, ins[rank].to(dev))
            torch.cuda.synchronize()
            _check(host(out), fo.reduce_scatter(s_rs, [host(x) for x in ins], dname)[rank],
                   f"reduce_scatter proto={proto} {dname} S={S}", fails)
            buf = seeded(n * S, dt, 300 + rank + S).to(dev)
            hosts = [host(seeded(n * S, dt, 300 + r + S)) for r in range(n)]
            comm.all_reduce(buf)
            torch.cuda.synchronize()
            _check(host(buf), fo.allreduce(s_ar, hosts, dname)[rank],
                   f"allreduce proto={proto} {dname} S={S}", fails)
    comm.set_option("proto", -1)
    return fails


def fresh_outputs(comm, rank, n, dev):
    """The NCCL idiom: a fresh output tensor every call.  Registrations track
    allocator segments, never tensors: their number stays bounded and no
    tensor is kept alive."""
    fails = []
    comm.set_option("proto", 0)  # the chunk-flag protocol writes peers' outputs
    S = 1 << 12
    inp = torch.full((S,), float(rank), device=dev)
    ref = torch.cat([torch.full((S,), float(r)) for r in range(n)])
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(dev)
    for i in range(1000):
        out = torch.empty(n * S + (i % 7), device=dev)[: n * S]
        comm.all_gather(out, inp)
        if i % 97 == 0 and not torch.equal(out.cpu(), ref):
            fails.append(f"call {i}: wrong output")
        del out
    torch.cuda.synchronize()
    grown = torch.cuda.memory_allocated(dev) - base
    if grown > (1 << 20):
        fails.append(f"allocated memory grew by {grown} bytes over 1000 calls")
    nreg = comm.registration_count()
    if nreg > 4:
        fails.append(f"{nreg} registrations after 1000 calls")
    return fails


def grow(comm, rank, n, dev):
    """The workspace starts small and grows collectively when a call's path
    needs more (LL128 staging, reduce-scatter windows), up to the cap;
    results stay bit-exact across re-allocations, and a capture that would
    need growth fails loudly instead of re-allocating inside the graph."""
    fails = []
    s_ag, s_rs = comm.schedule("allgather"), comm.schedule("reduce_scatter")
    start = comm.scratch_bytes
    sizes = []
    for S, dt, dname in ((1 << 12, torch.float32, "float32"), (12 << 20, torch.float32, "float32"),
                         (1 << 12, torch.float32, "float32"), (20 << 20, torch.bfloat16, "bfloat16")):
        ins = [seeded(S, torch.float32, 700 + r + S) for r in range(n)]
        out = torch.empty(n * S, device=dev)
        comm.all_gather(out, ins[rank].to(dev))
        torch.cuda.synchronize()
        _check(out.cpu().numpy(), fo.allgather(s_ag, [x.numpy() for x in ins])[rank],
               f"allgather S={S}", fails)
        rin = [seeded(n * S, dt, 900 + r + S) for r in range(n)]
        rout = torch.empty(S, device=dev, dtype=dt)
        comm.reduce_scatter(rout, rin[rank].to(dev))
        torch.cuda.synchronize()
        _check(host(rout), fo.reduce_scatter(s_rs, [host(x) for x in rin], dname)[rank],
               f"reduce_scatter S={S} {dname}", fails)
        sizes.append(comm.scratch_bytes)
    if not (start == 64 << 20 and sizes[-1] > start and sizes[-1] <= 512 << 20):
        fails.append(f"workspace did not grow as expected: start {start}, then {sizes}")
    # a capture whose size needs a larger workspace raises instead of growing
    S = comm.scratch_bytes // 8  # LL128 staging ~1.07 x the shard in each half: > scratch
    a = torch.empty(S, device=dev)
    b = torch.empty(n * S, device=dev)
    g = torch.cuda.CUDAGraph()
    raised = False
    try:
        with torch.cuda.graph(g):
            comm.set_option("proto", 1)
            comm.all_gather(b, a)
    except Exception as e:  # noqa: BLE001
        raised = "outside CUDA-graph capture" in str(e)
    comm.set_option("proto", -1)
    if not raised:
        fails.append("capture needing a larger workspace did not raise")
    torch.cuda.synchronize()
    return fails


def guards(comm, rank, n, dev):
    """Peer stores land only inside each peer's output: guard words around
    the outputs (same allocation, so inside the registered segment) stay
    untouched on the copy-engine, chunk-flag and LL128 paths, allgather and
    allreduce."""
    fails = []
    G = 8192
    s_ag, s_ar = comm.schedule("allgather"), comm.schedule("allreduce")
    for label, opts in (("ce", {"ce_min": 1, "proto": -1}), ("flags", {"ce_min": 0, "proto": 0}),
                        ("ll128", {"ce_min": 0, "proto": 1})):
        for k, v in opts.items():
            comm.set_option(k, v)
        S = 3 * 65536
        ins = [seeded(S, torch.float32, 4000 + r) for r in range(n)]
        big = torch.full((n * S + 2 * G,), -7.0, device=dev)
        out = big[G:G + n * S]
        comm.all_gather(out, ins[rank].to(dev))
        torch.cuda.synchronize()
        if not (torch.all(big[:G] == -7.0) and torch.all(big[G + n * S:] == -7.0)):
            fails.append(f"{label} allgather wrote outside its output")
        _check(out.cpu().numpy(), fo.allgather(s_ag, [x.numpy() for x in ins])[rank],
               f"{label} allgather", fails)
        if label != "ce":
            cnt = n * S
            ains = [seeded(cnt, torch.float32, 5000 + r) for r in range(n)]
            big = torch.full((cnt + 2 * G,), -7.0, device=dev)
            buf = big[G:G + cnt]
            buf.copy_(ains[rank].to(dev))
            comm.all_reduce(buf)
            torch.cuda.synchronize()
            if not (torch.all(big[:G] == -7.0) and torch.all(big[G + cnt:] == -7.0)):
                fails.append(f"{label} allreduce wrote outside its buffer")
            _check(buf.cpu().numpy(), fo.allreduce(s_ar, [x.numpy() for x in ains], "float32")[rank],
                   f"{label} allreduce", fails)
    comm.set_option("proto", -1)
    return fails


def mismatch(comm, rank, n, dev, ce=False):
    """Rank 0 passes a different (registered) output than its peers: the
    device check fails loudly instead of receiving misplaced stores (chunk
    flags), or right after them (copy engine: the tag check runs beside the
    copy, which stays inside the peer's registered segment)."""
    from paper_2402_06787_b200 import DeviceError

    comm.set_option("proto", -1 if ce else 0)
    comm.set_option("ce_min", 1 if ce else 0)
    comm.set_option("timeout_ms", 4000)
    S = 1 << 12
    a = torch.empty(n * S, device=dev)
    b = torch.empty(n * S, device=dev)
    inp = torch.ones(S, device=dev)
    comm.all_gather(a, inp)  # registers the segment(s)
    comm.all_gather(b, inp)
    torch.cuda.synchronize()
    comm.all_gather(b if rank == 0 else a, inp)
    if ce and comm.last_call_info()["proto"] != "ce":
        return [f"took {comm.last_call_info()['proto']}, not the copy-engine path"]
    try:
        comm.check()
    except DeviceError as e:
        print(f"RANK {rank} detected: {e}", flush=True)
        return []
    return ["mismatch not detected"] if rank == 0 else []


if __name__ == "__main__":
    main()

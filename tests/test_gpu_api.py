"""GPU API behaviour: argument checking, dtype/op support, unaligned views,
empty calls, the Executor surface, tracing, and device-side fault detection."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _vc(name, **kw):
    from paper_2402_06787_b200 import VirtualComm

    s = load_golden(name)
    return VirtualComm(schedules={s.collective: s}, scratch_bytes=256 << 20, **kw)


def test_argument_errors(dev):
    from paper_2402_06787_b200 import InvalidArgument, Unsupported

    comm = _vc("nvs4_reduce_scatter")
    n = comm.nranks
    ins = [torch.zeros(n * 8, device=dev) for _ in range(n)]
    outs = [torch.zeros(8, device=dev) for _ in range(n)]
    with pytest.raises(InvalidArgument):
        comm.reduce_scatter(outs[:-1], ins)
    with pytest.raises(InvalidArgument):
        comm.reduce_scatter([torch.zeros(8, device=dev, dtype=torch.bfloat16)] * n, ins)
    with pytest.raises(Unsupported):
        comm.reduce_scatter(outs, ins, op="max")
    with pytest.raises(Unsupported):
        comm.reduce_scatter([o.double() for o in outs], [i.double() for i in ins])
    with pytest.raises(InvalidArgument):
        comm.reduce_scatter([o.cpu() for o in outs], ins)


def test_empty_and_bytes(dev):
    comm = _vc("nvs4_allgather")
    n = comm.nranks
    comm.all_gather([torch.empty(0, device=dev) for _ in range(n)],
                    [torch.empty(0, device=dev) for _ in range(n)])
    for dt in (torch.uint8, torch.int8, torch.float64, torch.float8_e4m3fn):
        S = 333
        sends = [torch.randint(0, 255, (S,), dtype=torch.uint8).view(torch.uint8).to(dev).view(dt)
                 if dt.itemsize == 1 else torch.randn(S, dtype=torch.float64, device=dev)
                 for _ in range(n)]
        outs = [torch.empty(n * S, dtype=dt, device=dev) for _ in range(n)]
        comm.all_gather(outs, sends)
        cat = torch.cat([s.view(torch.uint8) for s in sends])
        for o in outs:
            assert torch.equal(o.view(torch.uint8), cat)
    comm.check()


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_unaligned_views(dev, offset):
    """Views whose data pointers are not 16-byte aligned take the scalar /
    narrow-vector paths (LL128 needs 8-byte alignment) and stay exact."""
    from oracle import forest_oracle as fo

    comm = _vc("nvs8_reduce_scatter")
    s = comm.schedule("reduce_scatter")
    n, S = comm.nranks, 4099
    base = [torch.randn(n * S + offset, device=dev) for _ in range(n)]
    ins = [b[offset:] for b in base]
    obase = [torch.zeros(S + offset, device=dev) for _ in range(n)]
    outs = [b[offset:] for b in obase]
    comm.reduce_scatter(outs, ins)
    ref = fo.reduce_scatter(s, [x.cpu().numpy() for x in ins], "float32")
    for r in range(n):
        assert np.array_equal(outs[r].cpu().numpy().view(np.uint32), ref[r].view(np.uint32))
    comm.check()


def test_executor_from_json_path(dev):
    import os

    from paper_2402_06787_b200 import Executor

    path = os.path.join(GOLDEN, "schedules", "groups450_allreduce.json")
    ex = Executor(path, virtual=True, validate=False)
    n = ex.comm.nranks
    bufs = [torch.full((1000,), float(r + 1), device=dev) for r in range(n)]
    ex.all_reduce(bufs)
    for b in bufs:
        assert torch.all(b == n * (n + 1) / 2)
    ex.close()


def test_trace_records(dev):
    comm = _vc("nvs8_allgather")
    comm.set_option("oneshot_ag_max", 0)  # the forest kernel traces items; one-hop has none
    n = comm.nranks
    comm.enable_trace(1 << 16)
    sends = [torch.randn(1 << 16, device=dev) for _ in range(n)]
    outs = [torch.empty(n << 16, device=dev) for _ in range(n)]
    comm.all_gather(outs, sends)
    rec = comm.read_trace()
    assert rec.size > 0
    assert set(np.unique(rec["rank"])) == set(range(n))
    assert np.all(rec["t_end"] >= rec["t_start"])
    # peer bytes: every rank receives (N-1) shards; LL128 adds 8 of 128 bytes
    payload = (n - 1) * n * (1 << 16) * 4
    total = int(rec["peer_bytes"].astype(np.int64).sum())
    assert payload <= total <= payload * 1.08, (total, payload)
    comm.disable_trace()


def test_device_timeout_is_reported_not_hung(dev):
    """Fault injection: a forest whose root never sends.  The leaf's wait
    times out on the device, the kernel exits, check() raises DeviceError."""
    import ctypes

    from paper_2402_06787_b200 import DeviceError, _lib
    from paper_2402_06787_b200 import compiler as C

    comm = _vc("nvs2_allgather", options={"timeout_ms": 300, "proto": 0})
    plan = comm.plan("allgather")
    bad = plan.table.copy()
    task0 = C.HEADER_WORDS + plan.nranks * C.RANKDESC_WORDS
    for i in range(sum(map(len, plan.tasks))):
        row = bad[task0 + i * C.TASK_WORDS:task0 + (i + 1) * C.TASK_WORDS]
        if row[C.TW_KIND] == C.K_AG_ROOT and row[C.TW_ROOT] == 0:
            row[C.TW_N_AG_CHILD] = 0  # root 0 "forgets" its child
    _lib.check(comm._lib.fc_plan_load(comm._comm, 0, bad.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                      bad.size), comm._comm)
    sends = [torch.randn(4096, device=dev) for _ in range(2)]
    outs = [torch.empty(8192, device=dev) for _ in range(2)]
    comm.all_gather(outs, sends)
    with pytest.raises(DeviceError):
        comm.check()


@pytest.mark.parametrize("proto", [-1, 0])
def test_cuda_graph_capture_and_replay(dev, proto):
    """The launch epoch lives in device memory, so captured collectives replay
    correctly: every replay with fresh inputs matches the oracle bit-for-bit."""
    from oracle import forest_oracle as fo
    from paper_2402_06787_b200 import VirtualComm
    from paper_2402_06787_b200.topology import nvswitch_doc

    comm = VirtualComm(nvswitch_doc(4), device=0, scratch_bytes=256 << 20,
                       options={"proto": proto, "timeout_ms": 20000})
    n, S = comm.nranks, 3000
    sends = [torch.empty(S, device=dev) for _ in range(n)]
    outs = [torch.empty(n * S, device=dev) for _ in range(n)]
    rs_in = [torch.empty(n * S, device=dev) for _ in range(n)]
    rs_out = [torch.empty(S, device=dev) for _ in range(n)]
    ar = [torch.empty(n * S, device=dev, dtype=torch.bfloat16) for _ in range(n)]
    ar_out = [torch.empty_like(x) for x in ar]

    def calls():
        comm.all_gather(outs, sends)
        comm.reduce_scatter(rs_out, rs_in, op="avg")
        comm.all_reduce(ar, outs=ar_out)

    for t in sends + rs_in + ar:
        t.normal_()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        calls()  # warm-up: plans loaded, buffers registered before capture
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        calls()
    for rep in range(3):
        gen = torch.Generator().manual_seed(50 + rep)
        hs = [torch.randn(S, generator=gen) for _ in range(n)]
        hr = [torch.randn(n * S, generator=gen) for _ in range(n)]
        ha = [torch.randn(n * S, generator=gen).to(torch.bfloat16) for _ in range(n)]
        for d, h in zip(sends + rs_in + ar, hs + hr + ha):
            d.copy_(h)
        g.replay()
        torch.cuda.synchronize()
        comm.check()
        ref = fo.allgather(comm.schedule("allgather"), [h.numpy() for h in hs])
        for r in range(n):
            assert np.array_equal(outs[r].cpu().numpy(), ref[r]), f"replay {rep} AG rank {r}"
        ref = fo.reduce_scatter(comm.schedule("reduce_scatter"), [h.numpy() for h in hr],
                                "float32", op="avg")
        for r in range(n):
            assert np.array_equal(rs_out[r].cpu().numpy(), ref[r]), f"replay {rep} RS rank {r}"
        hb = [h.view(torch.int16).numpy().view(np.uint16) for h in ha]
        ref = fo.allreduce(comm.schedule("allreduce"), hb, "bfloat16")
        for r in range(n):
            got = ar_out[r].view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(got, ref[r]), f"replay {rep} AR rank {r}"
    comm.close()


def test_cli_run_subcommand(dev, tmp_path):
    """`python -m paper_2402_06787_b200 run` times a forest on virtual ranks."""
    import json
    import subprocess
    import sys

    from conftest import REPO
    from paper_2402_06787_b200.topology import nvswitch_doc

    topo = tmp_path / "nvs4.json"
    topo.write_text(json.dumps(nvswitch_doc(4)))
    for coll in ("allgather", "reduce_scatter", "allreduce"):
        r = subprocess.run([sys.executable, "-m", "paper_2402_06787_b200", "run", "-t", str(topo),
                            "--collective", coll, "--mib", "4", "--steps", "3"],
                           cwd=REPO, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        line = json.loads(r.stdout.strip().splitlines()[-1])
        assert line["collective"] == coll and line["ranks"] == 4 and line["ms"] > 0


def test_cli_run_executes_a_schedule_json(dev):
    """`run -s` executes a schedule given in the reference's wire format
    (parse_schedule, schedule.py:439-448), here the sparse groups forest."""
    import json
    import os
    import subprocess
    import sys

    from conftest import GOLDEN, REPO

    for name, coll in (("groups300_allgather", "allgather"), ("nvs4_allreduce", "allreduce")):
        path = os.path.join(GOLDEN, "schedules", name + ".json")
        r = subprocess.run([sys.executable, "-m", "paper_2402_06787_b200", "run", "-s", path,
                            "--collective", coll, "--mib", "8", "--steps", "3"],
                           cwd=REPO, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        line = json.loads(r.stdout.strip().splitlines()[-1])
        assert line["collective"] == coll and line["ms"] > 0

"""GPU parity: the sm_100a forest kernel (virtual ranks, one device) against
the CPU oracle, bit-exact, on reference-generated forests."""

import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

TORCH_DT = {"float32": torch.float32, "bfloat16": torch.bfloat16, "float16": torch.float16,
            "int32": torch.int32}


def _np(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _rand(n, dtype, gen, dev):
    if dtype == "int32":
        return torch.randint(-2**20, 2**20, (n,), generator=gen, dtype=torch.int32).to(dev)
    return torch.empty(n).uniform_(-1, 1, generator=gen).to(TORCH_DT[dtype]).to(dev)


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8)


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _comm(s, proto="auto", **kw):
    from paper_2402_06787_b200 import VirtualComm

    opts = {"timeout_ms": 20000}
    if proto == "flags":
        opts["proto"] = 0
    return VirtualComm(schedules={s.collective: s}, options=opts, **kw)


PROTOS = ["auto", "flags"]  # auto: one-hop / one-shot (single-switch forests), else LL128
# (odd counts end in a partial payload word; allgathers need 4-byte aligned
# slices); the forest LL128 path at production widths is pinned in
# test_gpu_production.py


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", golden_names("allgather"))
@pytest.mark.parametrize("S", [1, 37, 4096, 262144 + 3])
def test_allgather_virtual(dev, name, S, proto):
    from oracle import forest_oracle as fo

    s = load_golden(name)
    comm = _comm(s, proto)
    n = comm.nranks
    gen = torch.Generator().manual_seed(1234)
    sends = [torch.randint(0, 2**31 - 1, (S,), generator=gen, dtype=torch.int32).view(torch.float32).to(dev)
             for _ in range(n)]
    outs = [torch.full((n * S,), float("nan"), device=dev) for _ in range(n)]
    comm.all_gather(outs, sends)
    comm.check()
    ref = fo.allgather(s, [_np(x) for x in sends])
    for r in range(n):
        assert np.array_equal(_bits(_np(outs[r])), _bits(ref[r])), f"rank {r}"


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", golden_names("reduce_scatter"))
@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "int32", "float16"])
@pytest.mark.parametrize("S", [5, 1000, 65536 + 8])
def test_reduce_scatter_virtual(dev, name, dtype, S, proto):
    from oracle import forest_oracle as fo

    s = load_golden(name)
    comm = _comm(s, proto)
    n = comm.nranks
    gen = torch.Generator().manual_seed(99)
    ins = [_rand(n * S, dtype, gen, dev) for _ in range(n)]
    outs = [torch.zeros(S, dtype=TORCH_DT[dtype], device=dev) for _ in range(n)]
    comm.reduce_scatter(outs, ins)
    comm.check()
    ref = fo.reduce_scatter(s, [_np(x) for x in ins], dtype)
    for r in range(n):
        assert np.array_equal(_bits(_np(outs[r])), _bits(ref[r])), f"rank {r}"


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", golden_names("allreduce"))
@pytest.mark.parametrize("dtype", ["bfloat16", "float32", "int32"])
@pytest.mark.parametrize("count", [3, 1001, 1 << 18])
def test_allreduce_virtual(dev, name, dtype, count, proto):
    from oracle import forest_oracle as fo

    s = load_golden(name)
    comm = _comm(s, proto)
    n = comm.nranks
    gen = torch.Generator().manual_seed(7)
    ins = [_rand(count, dtype, gen, dev) for _ in range(n)]
    outs = [torch.zeros(count, dtype=TORCH_DT[dtype], device=dev) for _ in range(n)]
    comm.all_reduce(ins, outs=outs)
    comm.check()
    ref = fo.allreduce(s, [_np(x) for x in ins], dtype)
    for r in range(n):
        assert np.array_equal(_bits(_np(outs[r])), _bits(ref[r])), f"rank {r}"


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", ["nvs4_reduce_scatter", "nvs8_reduce_scatter",
                                  "groups300_reduce_scatter", "groups100_reduce_scatter"])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16"])
@pytest.mark.parametrize("S", [5, 65536 + 8])
def test_reduce_scatter_avg_virtual(dev, name, dtype, S, proto):
    """op avg: the root scales its fp32 sum by fp32(1/N) once (FC_AVG)."""
    from oracle import forest_oracle as fo

    s = load_golden(name)
    comm = _comm(s, proto)
    n = comm.nranks
    gen = torch.Generator().manual_seed(31)
    ins = [_rand(n * S, dtype, gen, dev) for _ in range(n)]
    outs = [torch.zeros(S, dtype=TORCH_DT[dtype], device=dev) for _ in range(n)]
    comm.reduce_scatter(outs, ins, op="avg")
    comm.check()
    ref = fo.reduce_scatter(s, [_np(x) for x in ins], dtype, op="avg")
    for r in range(n):
        assert np.array_equal(_bits(_np(outs[r])), _bits(ref[r])), f"rank {r}"


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", ["nvs8_allreduce", "groups450_allreduce"])
@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
@pytest.mark.parametrize("count", [1001, 1 << 18])
def test_allreduce_avg_virtual(dev, name, dtype, count, proto):
    import torch.distributed as dist

    from oracle import forest_oracle as fo

    s = load_golden(name)
    comm = _comm(s, proto)
    n = comm.nranks
    gen = torch.Generator().manual_seed(8)
    ins = [_rand(count, dtype, gen, dev) for _ in range(n)]
    outs = [torch.zeros(count, dtype=TORCH_DT[dtype], device=dev) for _ in range(n)]
    comm.all_reduce(ins, outs=outs, op=dist.ReduceOp.AVG)
    comm.check()
    ref = fo.allreduce(s, [_np(x) for x in ins], dtype, op="avg")
    for r in range(n):
        assert np.array_equal(_bits(_np(outs[r])), _bits(ref[r])), f"rank {r}"


def test_avg_rejected_for_integers(dev):
    from paper_2402_06787_b200.errors import Unsupported

    s = load_golden("nvs4_reduce_scatter")
    comm = _comm(s)
    ins = [torch.ones(4 * 64, dtype=torch.int32, device=dev) for _ in range(4)]
    outs = [torch.zeros(64, dtype=torch.int32, device=dev) for _ in range(4)]
    with pytest.raises(Unsupported):
        comm.reduce_scatter(outs, ins, op="avg")
    with pytest.raises(Unsupported):
        comm.reduce_scatter(outs, ins, op="max")


@pytest.mark.parametrize("name", ["nvs8_allgather", "groups300_allgather", "random1_allgather"])
def test_ll128_is_used_for_aligned_medium_messages(dev, name):
    s = load_golden(name)
    comm = _comm(s)
    comm.set_option("oneshot_ag_max", 0)  # nvs8: keep the forest (not the one-hop path)
    n = comm.nranks
    S = 6 * 10924  # 8-byte aligned batch slices for k in {1, 2, 3, 6, 7?}
    S = S - S % (2 * s.k)
    sends = [torch.randn(S, device=dev) for _ in range(n)]
    outs = [torch.empty(n * S, device=dev) for _ in range(n)]
    comm.all_gather(outs, sends)
    comm.check()
    assert comm.last_call_info()["proto"] == "ll128"
    cat = torch.cat(sends)
    for o in outs:
        assert torch.equal(o, cat)


@pytest.mark.parametrize("proto", PROTOS)
def test_back_to_back_reuse_and_windows(dev, proto):
    """Many calls on one set of buffers, and forced multi-launch windows."""
    from oracle import forest_oracle as fo

    s = load_golden("nvs8_reduce_scatter")
    comm = _comm(s, proto, scratch_bytes=1 << 20)
    comm.set_option("chunk_max", 16 << 10)
    n = comm.nranks
    gen = torch.Generator().manual_seed(5)
    S = 1 << 17
    outs = [torch.zeros(S, device=dev) for _ in range(n)]
    for it in range(4):
        ins = [torch.empty(n * S).uniform_(-1, 1, generator=gen).to(dev) for _ in range(n)]
        comm.reduce_scatter(outs, ins)
        ref = fo.reduce_scatter(s, [x.cpu().numpy() for x in ins], "float32")
        for r in range(n):
            assert np.array_equal(outs[r].cpu().numpy().view(np.uint32), ref[r].view(np.uint32))
    comm.check()

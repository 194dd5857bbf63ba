"""The real-GPU product paths, driver-verifiable on one B200.

On real GPUs the executor runs 8-warp chunk-flag workers, 4-warp LL128
workers, 128 CTAs per rank, and -- on single-switch forests -- the one-hop
allgather and the one-shot reductions.  Virtual mode (all ranks of a forest
in one cooperative grid on one device) runs the very same kernels, so every
test here pins one of those product configurations bit-exactly against the
CPU oracle (oracle/forest_oracle.py, the a-11 contract of SURVEY.md §8):

* forest kernel at production worker widths (2/4/8 warps, both protocols)
  and at the largest CTA count the device co-schedules;
* one-hop allgather (fc_oneshot_ag128_kernel) and one-shot reduce-scatter /
  allreduce (fc_oneshot128_kernel), including unaligned tensor views;
* topology gating: sparse forests (groups_switch, random graphs) never take
  the one-hop paths, whatever the size (schedule.py:3-7, verify.py:350-353);
* one staging region shared by every LL128 writer, with payloads equal to
  the launch epochs that later calls use as flags.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu

TORCH_DT = {"float32": torch.float32, "bfloat16": torch.bfloat16, "float16": torch.float16,
            "int32": torch.int32}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _np(t):
    """Host copy in the oracle's convention: bf16 as raw uint16 bits, the
    other dtypes as their numpy type."""
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _rand(n, dtype, gen, dev):
    if dtype == "int32":
        return torch.randint(-2**20, 2**20, (n,), generator=gen, dtype=torch.int32).to(dev)
    return torch.empty(n).uniform_(-1, 1, generator=gen).to(TORCH_DT[dtype]).to(dev)


def _comm(name, **opts):
    from paper_2402_06787_b200 import VirtualComm

    s = load_golden(name)
    o = {"timeout_ms": 30000}
    o.update(opts)
    return VirtualComm(schedules={s.collective: s}, scratch_bytes=512 << 20, options=o), s


def _oracle(s, coll, ins, dtype, op="sum"):
    from oracle import forest_oracle as fo

    host = [_np(x) for x in ins]
    if coll == "allgather":
        return fo.allgather(s, host)
    if coll == "reduce_scatter":
        return fo.reduce_scatter(s, host, dtype, op=op)
    return fo.allreduce(s, host, dtype, op=op)


def _run(comm, coll, S, dtype, dev, seed, op="sum", offset=0):
    """One call with seeded inputs (views at `offset` elements into their
    allocation); returns (inputs, outputs)."""
    n = comm.nranks
    gen = torch.Generator().manual_seed(seed)
    count = {"allgather": S, "reduce_scatter": n * S, "allreduce": S}[coll]
    out_n = {"allgather": n * S, "reduce_scatter": S, "allreduce": S}[coll]
    ins = [_rand(count + offset, dtype, gen, dev)[offset:] for _ in range(n)]
    outs = [torch.zeros(out_n + offset, dtype=TORCH_DT[dtype], device=dev)[offset:] for _ in range(n)]
    if coll == "allgather":
        comm.all_gather(outs, ins)
    elif coll == "reduce_scatter":
        comm.reduce_scatter(outs, ins, op=op)
    else:
        comm.all_reduce(ins, outs=outs, op=op)
    comm.check()
    return ins, outs


def _assert_exact(s, coll, ins, outs, dtype, op="sum"):
    ref = _oracle(s, coll, ins, dtype, op)
    for r, o in enumerate(outs):
        assert np.array_equal(_bits(_np(o)), _bits(ref[r])), f"rank {r}"


# ---------------------------------------------------------------------------
# forest kernel at production widths
# ---------------------------------------------------------------------------
FORESTS = ["nvs2", "nvs4", "nvs8", "groups300", "groups100", "random1"]
CASES = [("allgather", "float32", 262144 + 3), ("reduce_scatter", "bfloat16", 65536 + 8),
         ("reduce_scatter", "int32", 4099), ("allreduce", "float32", (1 << 18) + 5),
         ("allreduce", "bfloat16", 1 << 18)]


def _coll_name(base, coll):
    name = f"{base}_{coll}"
    from conftest import golden_names

    return name if name in golden_names() else None


@pytest.mark.parametrize("ww", [2, 4, 8])
@pytest.mark.parametrize("base", FORESTS)
@pytest.mark.parametrize("coll,dtype,S", CASES)
def test_flags_protocol_production_widths(dev, base, coll, dtype, S, ww):
    """Chunk-flag protocol with multi-warp workers (named bar.sync, per-warp
    sub-ranges) at the largest co-resident CTA count."""
    name = _coll_name(base, coll)
    if name is None:
        pytest.skip(f"no {coll} fixture for {base}")
    comm, s = _comm(name, proto=0, worker_warps=ww)
    comm.set_option("ctas_per_rank", min(128, comm.get_option("max_ctas_per_rank")))
    ins, outs = _run(comm, coll, S, dtype, dev, seed=ww * 100 + len(base))
    assert comm.last_call_info()["proto"] == "flags"
    _assert_exact(s, coll, ins, outs, dtype)
    comm.close()


@pytest.mark.parametrize("ww", [2, 4, 8])
@pytest.mark.parametrize("base", FORESTS)
@pytest.mark.parametrize("coll,dtype,S", CASES)
def test_ll128_protocol_production_widths(dev, base, coll, dtype, S, ww):
    """LL128 protocol with 2/4/8-warp workers (4 is the real-GPU default)."""
    name = _coll_name(base, coll)
    if name is None:
        pytest.skip(f"no {coll} fixture for {base}")
    comm, s = _comm(name, proto=1, ll_worker_warps=ww)
    comm.set_option("ctas_per_rank", min(128, comm.get_option("max_ctas_per_rank")))
    # LL128 needs 8-byte aligned slices [floor(S*m/k)] in every root shard:
    # shards of a multiple of 128*k elements (allreduce: N equal shards)
    q = 128 * s.k
    S = (S // q) * q if coll != "allreduce" else comm.nranks * max(1, S // (comm.nranks * q)) * q
    ins, outs = _run(comm, coll, S, dtype, dev, seed=ww * 10 + len(base))
    assert comm.last_call_info()["proto"] == "ll128"
    _assert_exact(s, coll, ins, outs, dtype)
    comm.close()


def test_real_gpu_defaults_run_virtual(dev):
    """The defaults a real GPU gets (8-warp flag workers, 4-warp LL128
    workers, 128 CTAs) on the 2-rank forest, both protocols, avg included."""
    for proto in (0, 1):
        comm, s = _comm("nvs2_reduce_scatter", proto=proto, worker_warps=8, ll_worker_warps=4)
        comm.set_option("ctas_per_rank", min(128, comm.get_option("max_ctas_per_rank")))
        assert comm.get_option("ctas_per_rank") >= 64
        ins, outs = _run(comm, "reduce_scatter", 1 << 20, "bfloat16", dev, seed=3, op="avg")
        _assert_exact(s, "reduce_scatter", ins, outs, "bfloat16", op="avg")
        comm.close()


# ---------------------------------------------------------------------------
# one-hop allgather and one-shot reductions
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("base", ["nvs2", "nvs4", "nvs8"])
@pytest.mark.parametrize("S", [1, 2, 30, 31, 333, 1000, 4096 + 2, 4097, 65536, 1 << 20])
@pytest.mark.parametrize("offset", [0, 1])
def test_onehop_allgather(dev, base, S, offset):
    """Any shard length goes one hop (odd lengths end in a partial, zero-padded
    payload word), any buffer offset."""
    comm, s = _comm(f"{base}_allgather")
    ins, outs = _run(comm, "allgather", S, "float32", dev, seed=S + offset, offset=offset)
    info = comm.last_call_info()
    bytes_out = comm.nranks * S * 4
    if bytes_out <= comm.get_option("oneshot_ag_max"):
        assert info["proto"] == "oneshot", info
    _assert_exact(s, "allgather", ins, outs, "float32")
    comm.close()


@pytest.mark.parametrize("base", ["nvs2", "nvs8"])
@pytest.mark.parametrize("S", [1, 3, 61, 1001])
def test_onehop_allgather_odd_bf16(dev, base, S):
    """2-byte elements: shards of 2, 6, 122 and 2002 bytes (partial last words
    of 2 and 6 bytes), one hop, bit-exact."""
    comm, s = _comm(f"{base}_allgather")
    ins, outs = _run(comm, "allgather", S, "bfloat16", dev, seed=7 * S)
    assert comm.last_call_info()["proto"] == "oneshot"
    _assert_exact(s, "allgather", ins, outs, "bfloat16")
    comm.close()


def _oneshot_eligible(comm, coll, S, es):
    """The C side's rank-uniform one-shot rule (fc_api.cu run()): size limit,
    8-byte multiples; pointer alignment plays no part."""
    n = comm.nranks
    lim = comm.get_option("oneshot_max")
    if coll == "reduce_scatter":
        nbytes, shard = n * S * es, S * es
        return nbytes <= 2 * lim // n and nbytes % 8 == 0 and shard % 8 == 0
    shard = -(-S // n)
    shard = -(-shard * es // 128) * 128
    return S * es <= lim and (S * es) % 8 == 0 and shard % 8 == 0


@pytest.mark.parametrize("base", ["nvs2", "nvs4", "nvs8"])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16", "int32"])
@pytest.mark.parametrize("S", [4, 2000, 30000])
@pytest.mark.parametrize("offset", [0, 1])
def test_oneshot_reduce_scatter(dev, base, dtype, S, offset):
    comm, s = _comm(f"{base}_reduce_scatter")
    es = 4 if dtype in ("float32", "int32") else 2
    want = "oneshot" if _oneshot_eligible(comm, "reduce_scatter", S, es) else None
    ins, outs = _run(comm, "reduce_scatter", S, dtype, dev, seed=S + 7 * offset, offset=offset)
    assert want is None or comm.last_call_info()["proto"] == want
    _assert_exact(s, "reduce_scatter", ins, outs, dtype)
    if dtype != "int32":
        ins, outs = _run(comm, "reduce_scatter", S, dtype, dev, seed=S + 1, op="avg", offset=offset)
        assert want is None or comm.last_call_info()["proto"] == want
        _assert_exact(s, "reduce_scatter", ins, outs, dtype, op="avg")
    comm.close()


@pytest.mark.parametrize("base", ["nvs2", "nvs4", "nvs8"])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "int32"])
@pytest.mark.parametrize("count", [8, 1000, 65536 + 4, 500000])
@pytest.mark.parametrize("offset", [0, 1])
def test_oneshot_allreduce(dev, base, dtype, count, offset):
    comm, s = _comm(f"{base}_allreduce")
    ins, outs = _run(comm, "allreduce", count, dtype, dev, seed=count + offset, offset=offset)
    es = 2 if dtype == "bfloat16" else 4
    if _oneshot_eligible(comm, "allreduce", count, es):
        assert comm.last_call_info()["proto"] == "oneshot"
    _assert_exact(s, "allreduce", ins, outs, dtype)
    comm.close()


def test_oneshot_allreduce_in_place(dev):
    """In place: every output word is written only after the own input line
    it overwrites has arrived in the own staging (so it was read)."""
    from oracle import forest_oracle as fo

    comm, s = _comm("nvs8_allreduce")
    n = comm.nranks
    gen = torch.Generator().manual_seed(11)
    bufs = [_rand(1 << 17, "bfloat16", gen, dev) for _ in range(n)]
    host = [_np(b) for b in bufs]
    comm.all_reduce(bufs)
    comm.check()
    assert comm.last_call_info()["proto"] == "oneshot"
    ref = fo.allreduce(s, host, "bfloat16")
    for r in range(n):
        assert np.array_equal(_np(bufs[r]), ref[r])
    comm.close()


# ---------------------------------------------------------------------------
# topology gating
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("base", ["groups450", "groups300", "groups100"])
@pytest.mark.parametrize("coll", ["allgather", "reduce_scatter", "allreduce"])
@pytest.mark.parametrize("kib", [64, 1024, 16384])
def test_sparse_forests_never_take_onehop_paths(dev, base, coll, kib):
    """On groups_switch(β) logical edges must follow the forest: the bridge
    pairs are the only cross-group paths.  The plan
    carries no FC_PLAN_ONEHOP flag, so every size runs the forest."""
    comm, s = _comm(f"{base}_{coll}")
    assert not comm.plan(coll).onehop
    n = comm.nranks
    elems = kib * 1024 // 4
    S = {"allgather": elems // n, "reduce_scatter": elems // n // n, "allreduce": elems // n}[coll]
    S -= S % (2 * s.k)
    dtype = "float32" if coll == "allgather" else "bfloat16"
    ins, outs = _run(comm, coll, S, dtype, dev, seed=kib)
    assert comm.last_call_info()["proto"] in ("ll128", "flags")
    _assert_exact(s, coll, ins, outs, dtype)
    comm.close()


def test_single_switch_forests_are_onehop_equivalent(dev):
    for n in (2, 4, 8):
        for coll in ("allgather", "reduce_scatter", "allreduce"):
            comm, _ = _comm(f"nvs{n}_{coll}")
            assert comm.plan(coll).onehop
            comm.close()


# ---------------------------------------------------------------------------
# one staging region, every LL128 writer, payloads equal to future epochs
# ---------------------------------------------------------------------------
def test_staging_shared_by_all_ll128_writers(dev):
    """The one-hop allgather, the one-shot reductions and the forest's LL128
    lines all use one two-half staging region.  Fill it with payloads equal to
    the epochs upcoming calls use as line flags (int32 words 1..80 at every
    offset), then interleave every writer: any stale line mistaken for an
    arrived one would corrupt a result."""
    from oracle import forest_oracle as fo

    comm, _ = _comm("nvs4_allgather")
    n = comm.nranks
    s_ag = load_golden("nvs4_allgather")
    s_rs = load_golden("nvs4_reduce_scatter")
    s_ar = load_golden("nvs4_allreduce")
    comm._schedules.update({"reduce_scatter": s_rs, "allreduce": s_ar})
    S = 1 << 16
    for it in range(24):
        e = it + 1
        # payload words equal to epochs around the current one
        ags = [((torch.arange(S, dtype=torch.int32, device=dev) + r + e) % 80 + 1) for r in range(n)]
        ago = [torch.zeros(n * S, dtype=torch.int32, device=dev) for _ in range(n)]
        comm.set_option("proto", 1 if it % 3 == 2 else -1)  # forest LL128 every third round
        comm.all_gather(ago, ags)
        ref = fo.allgather(s_ag, [a.cpu().numpy() for a in ags])
        for r in range(n):
            assert np.array_equal(ago[r].cpu().numpy(), ref[r]), (it, "ag", r)
        comm.set_option("proto", -1)
        rsi = [((torch.arange(n * 512, dtype=torch.int32, device=dev) * (r + 1) + e) % 80) for r in range(n)]
        rso = [torch.zeros(512, dtype=torch.int32, device=dev) for _ in range(n)]
        comm.reduce_scatter(rso, rsi)
        assert comm.last_call_info()["proto"] == "oneshot"
        ref = fo.reduce_scatter(s_rs, [x.cpu().numpy() for x in rsi], "int32")
        for r in range(n):
            assert np.array_equal(rso[r].cpu().numpy(), ref[r]), (it, "rs", r)
        ari = [torch.full((3000,), e + r, dtype=torch.int32, device=dev) for r in range(n)]
        host = [x.cpu().numpy() for x in ari]
        comm.all_reduce(ari)
        ref = fo.allreduce(s_ar, host, "int32")
        for r in range(n):
            assert np.array_equal(ari[r].cpu().numpy(), ref[r]), (it, "ar", r)
    comm.check()
    comm.close()


@pytest.mark.parametrize("n_el,offset", [(1, 0), (1000, 1), (1 << 20, 0), ((1 << 22) + 3, 3)])
def test_one_rank_forest_is_a_local_copy(dev, n_el, offset):
    """The 1-rank forest (bench.py's local-copy sanity point) runs as one
    full-GPU copy kernel; any size and alignment."""
    from fractions import Fraction

    from paper_2402_06787_b200 import VirtualComm
    from paper_2402_06787_b200._refpath import require_collsched

    cs = require_collsched()
    s = cs.Schedule(collective="allgather", num_compute=1, k=1, U=Fraction(1), y=Fraction(1),
                    inv_x_star=Fraction(0),
                    roots=(cs.RootTrees("g0", (cs.ScheduleBatch(1, ()),)),))
    comm = VirtualComm(schedules={"allgather": s}, device=0)
    src = torch.randn(n_el + offset, device=dev)[offset:]
    dst = torch.zeros(n_el + offset, device=dev)[offset:]
    comm.all_gather([dst], [src])
    comm.check()
    assert comm.last_call_info()["proto"] == "local"
    assert torch.equal(dst, src)
    comm.close()


@pytest.mark.parametrize("base", ["nvs2", "nvs4", "nvs8"])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16", "int32"])
@pytest.mark.parametrize("mib", [3, 5])
@pytest.mark.parametrize("offset", [0, 1])
def test_twohop_reductions(dev, base, dtype, mib, offset):
    """Mid-size reduce-scatter / allreduce in two hops (shards to their
    roots, the in-tree evaluated there, reduced shards to every rank),
    bit-exact with the forest kernel's order; SUM and AVG; unaligned views."""
    es = 2 if dtype in ("bfloat16", "float16") else 4
    for coll in ("allreduce", "reduce_scatter"):
        comm, s = _comm(f"{base}_{coll}")
        comm.set_option("twohop_max", 16 << 20)
        n = comm.nranks
        count = mib * (1 << 20) // es
        S = count if coll == "allreduce" else count // n
        S -= S % 64
        for op in (("sum", "avg") if dtype != "int32" else ("sum",)):
            ins, outs = _run(comm, coll, S, dtype, dev, seed=mib * 7 + offset, op=op, offset=offset)
            assert comm.last_call_info()["proto"] == "twohop", comm.last_call_info()
            _assert_exact(s, coll, ins, outs, dtype, op=op)
        comm.close()


@pytest.mark.parametrize("coll,S,opts,want", [
    ("allgather", 4096 + 2, {}, "oneshot"),
    ("allgather", 4096 + 1, {}, "oneshot"),  # partial last payload word
    ("allgather", 3 * 65536, {"oneshot_ag_max": 0}, "ll128"),
    ("allgather", 3 * 65536 + 1, {"proto": 0}, "flags"),
    ("allgather", 3 * 65536 + 1, {"proto": 1}, "ll128"),  # partial last payload words
    ("reduce_scatter", 98304 + 3, {}, "ll128"),
    ("reduce_scatter", 2000, {}, "oneshot"),
    ("reduce_scatter", 98304, {}, "twohop"),
    ("reduce_scatter", 98304 + 3, {"proto": 0}, "flags"),
    ("allreduce", 1000 * 8, {}, "oneshot"),
    ("allreduce", 1 << 20, {}, "twohop"),
    ("allreduce", (1 << 20) + 8, {"twohop_max": 0}, "ll128"),
    ("allreduce", (1 << 20) + 5, {"proto": 0}, "flags"),
])
def test_no_writes_outside_the_output(dev, coll, S, opts, want):
    """Guard words around every output (before and after, same allocation)
    stay untouched on every path: no kernel writes past its buffer."""
    comm, s = _comm(f"nvs4_{coll}", **opts)
    n = comm.nranks
    G = 4096  # guard elements on each side
    gen = torch.Generator().manual_seed(S)
    count = {"allgather": S, "reduce_scatter": n * S, "allreduce": S}[coll]
    out_n = {"allgather": n * S, "reduce_scatter": S, "allreduce": S}[coll]
    ins = [_rand(count, "float32", gen, dev) for _ in range(n)]
    bigs = [torch.full((out_n + 2 * G,), -12345.0, device=dev) for _ in range(n)]
    outs = [b[G:G + out_n] for b in bigs]
    if coll == "allgather":
        comm.all_gather(outs, ins)
    elif coll == "reduce_scatter":
        comm.reduce_scatter(outs, ins)
    else:
        comm.all_reduce(ins, outs=outs)
    comm.check()
    assert comm.last_call_info()["proto"] == want, comm.last_call_info()
    for b in bigs:
        assert torch.all(b[:G] == -12345.0) and torch.all(b[G + out_n:] == -12345.0)
    _assert_exact(s, coll, ins, outs, "float32")
    comm.close()


# ---------------------------------------------------------------------------
# LL128 at any length: slices that are not a multiple of 8 bytes (odd counts,
# k > 1 splits at odd offsets) end in a partial payload word
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("base", ["nvs4", "groups300", "fig3a"])
@pytest.mark.parametrize("coll", ["allgather", "reduce_scatter", "allreduce"])
@pytest.mark.parametrize("S", [1, 3, 61, 1001, 65537])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_ll128_odd_lengths(dev, base, coll, S, dtype):
    comm, s = _comm(f"{base}_{coll}", proto=1)
    ins, outs = _run(comm, coll, S, dtype, dev, seed=S * 3 + len(base))
    assert comm.last_call_info()["proto"] == "ll128", comm.last_call_info()
    _assert_exact(s, coll, ins, outs, dtype)
    comm.close()


@pytest.mark.parametrize("coll,op,dtype", [("reduce_scatter", "avg", "bfloat16"),
                                           ("allreduce", "avg", "float32"),
                                           ("allreduce", "sum", "int32")])
@pytest.mark.parametrize("offset", [0, 1])
def test_ll128_odd_lengths_production_width(dev, coll, op, dtype, offset):
    """4-warp LL128 workers, unaligned views, AVG and int32 at odd lengths."""
    comm, s = _comm(f"groups300_{coll}", proto=1, ll_worker_warps=4)
    ins, outs = _run(comm, coll, 4097, dtype, dev, seed=11 + offset, op=op, offset=offset)
    assert comm.last_call_info()["proto"] == "ll128"
    _assert_exact(s, coll, ins, outs, dtype, op=op)
    comm.close()


@pytest.mark.parametrize("coll,dtype,want", [("allgather", "float32", "ll128"),
                                             ("allgather", "bfloat16", "flags"),
                                             ("reduce_scatter", "float32", "ll128"),
                                             ("reduce_scatter", "bfloat16", "ll128"),
                                             ("allreduce", "float32", "ll128")])
def test_odd_lengths_automatic_protocol(dev, coll, dtype, want):
    """Odd counts take LL128 (they used to fall through to chunk flags),
    except an allgather whose slices are not even 4-byte aligned (odd 2-byte
    counts), which the chunk flags move faster than LL128's byte loops."""
    comm, s = _comm(f"groups300_{coll}")
    ins, outs = _run(comm, coll, 3 * 65536 + 1, dtype, dev, seed=5)
    assert comm.last_call_info()["proto"] == want, comm.last_call_info()
    _assert_exact(s, coll, ins, outs, dtype)
    comm.close()

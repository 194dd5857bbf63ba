"""The CPU oracle against closed forms and an independent per-element
restatement, on reference-generated forests (golden fixtures)."""

from fractions import Fraction

import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden
from oracle import forest_oracle as fo


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(100000).astype(np.float32) * 1e3,
        np.array([0.0, -0.0, 1e-40, -1e-40, 3.4e38, -3.4e38, np.inf, -np.inf], np.float32),
        (rng.integers(0, 2**32, 10000, dtype=np.uint64).astype(np.uint32)).view(np.float32),
    ])
    ours = fo.f32_to_bf16(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    finite = ~np.isnan(x)
    assert np.array_equal(ours[finite], ref[finite])
    assert (ours[~finite] == 0x7FFF).all()  # canonical NaN, as cvt.rn.bf16x2.f32 on sm_100


def test_bf16_rounding_matches_sm100_cvt_vectors():
    """Pinned outputs of cvt.rn.bf16x2.f32 measured on a B200 (tools/cvt_probe.cu)."""
    pairs = {0x7fc00000: 0x7fff, 0xffc00000: 0x7fff, 0x7f800001: 0x7fff, 0xff812345: 0x7fff,
             0x7fa5a5a5: 0x7fff, 0x7f800000: 0x7f80, 0x3f808000: 0x3f80, 0x3f818000: 0x3f82,
             0x00000001: 0x0000, 0x807fffff: 0x8080, 0x7f7fffff: 0x7f80, 0x3f80ffff: 0x3f81}
    x = np.array(list(pairs), dtype=np.uint32).view(np.float32)
    assert fo.f32_to_bf16(x).tolist() == list(pairs.values())


@pytest.mark.parametrize("name", golden_names("allgather"))
def test_allgather_is_concatenation(name):
    s = load_golden(name)
    n = s.num_compute
    rng = np.random.default_rng(1)
    for S in (1, 3, 64, 1001):
        sends = [rng.integers(0, 2**32, S, dtype=np.uint64).astype(np.uint32).view(np.float32)
                 for _ in range(n)]
        outs = fo.allgather(s, sends)
        cat = np.concatenate(sends).view(np.uint32)
        for o in outs:
            assert np.array_equal(o.view(np.uint32), cat)


def _exact_sum(arrs):
    return np.sum(np.stack(arrs).astype(np.int64), axis=0).astype(np.uint32).view(np.int32)


@pytest.mark.parametrize("name", golden_names("reduce_scatter"))
def test_int32_reduce_scatter_is_exact_sum(name):
    s = load_golden(name)
    n = s.num_compute
    rng = np.random.default_rng(2)
    for S in (1, 5, 257):
        ins = [rng.integers(-2**31, 2**31, n * S, dtype=np.int64).astype(np.int32) for _ in range(n)]
        outs = fo.reduce_scatter(s, ins, "int32")
        tot = _exact_sum(ins)  # wrapping two's-complement
        for r in range(n):
            assert np.array_equal(outs[r], tot[r * S:(r + 1) * S])


@pytest.mark.parametrize("name", golden_names("allreduce"))
def test_int32_allreduce_is_exact_sum(name):
    s = load_golden(name)
    n = s.num_compute
    rng = np.random.default_rng(3)
    for count in (1, 7, 999, 4096):
        ins = [rng.integers(-2**31, 2**31, count, dtype=np.int64).astype(np.int32) for _ in range(n)]
        outs = fo.allreduce(s, ins, "int32")
        tot = _exact_sum(ins)
        for o in outs:
            assert np.array_equal(o, tot)


def _per_element_rs(s, ins, dtype):
    """Independent restatement: per element, find the carrying tree by the
    floor rule and evaluate the in-tree sum recursively with scalars."""
    ids = sorted(rt.root for rt in s.roots)
    pos = {x: i for i, x in enumerate(ids)}
    n = len(ids)
    S = ins[0].size // n
    out = [np.zeros(S, dtype=ins[0].dtype) for _ in range(n)]
    to32 = (lambda v: np.float32(v)) if dtype == "float32" else \
        (lambda v: fo.bf16_to_f32(np.array([v], np.uint16))[0])
    back = (lambda f: np.float32(f)) if dtype == "float32" else \
        (lambda f: fo.f32_to_bf16(np.array([f], np.float32))[0])
    for rt in s.roots:
        r = pos[rt.root]
        lo = 0
        for b in rt.batches:
            a, z = (S * lo) // s.k, (S * (lo + b.multiplicity)) // s.k
            kids = {}
            for e in b.edges:  # reduce-scatter edges point child -> parent
                kids.setdefault(e.dst, []).append(e.src)

            def partial(v, e_idx):
                own = ins[pos[v]][r * S + e_idx]
                ch = sorted(kids.get(v, []), key=pos.__getitem__)
                if not ch:
                    return own
                acc = to32(own)
                for c in ch:
                    acc = np.float32(acc + to32(partial(c, e_idx)))
                return back(acc)

            for e_idx in range(a, z):
                out[r][e_idx] = partial(rt.root, e_idx)
            lo += b.multiplicity
    return out


@pytest.mark.parametrize("name", ["nvs8_reduce_scatter", "groups300_reduce_scatter",
                                  "fig3a_reduce_scatter", "nvs4_reduce_scatter"])
@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_fp_reduce_scatter_matches_independent_restatement(name, dtype):
    s = load_golden(name)
    n = s.num_compute
    rng = np.random.default_rng(4)
    S = 13
    f = [rng.uniform(-1, 1, n * S).astype(np.float32) for _ in range(n)]
    ins = f if dtype == "float32" else [fo.f32_to_bf16(x) for x in f]
    got = fo.reduce_scatter(s, ins, dtype)
    want = _per_element_rs(s, ins, dtype)
    for r in range(n):
        assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8))


@pytest.mark.parametrize("name", ["nvs8_reduce_scatter", "nvs4_reduce_scatter", "groups300_reduce_scatter"])
def test_avg_is_power_of_two_scaled_sum_in_fp32(name):
    """N is a power of two here: fp32(1/N) is exact and so is the scaling,
    so avg == sum * 1/N bit for bit (the scale happens once, at the root)."""
    s = load_golden(name)
    n = s.num_compute
    rng = np.random.default_rng(12)
    ins = [rng.uniform(-1, 1, n * 33).astype(np.float32) for _ in range(n)]
    got = fo.reduce_scatter(s, ins, "float32", op="avg")
    ref = fo.reduce_scatter(s, ins, "float32")
    for r in range(n):
        assert np.array_equal(got[r], ref[r] * np.float32(1.0 / n))


def test_avg_bf16_rounds_once_at_the_root():
    s = load_golden("nvs4_reduce_scatter")
    n = s.num_compute
    rng = np.random.default_rng(13)
    ins = [fo.f32_to_bf16(rng.uniform(-1, 1, n * 40).astype(np.float32)) for _ in range(n)]
    got = fo.reduce_scatter(s, ins, "bfloat16", op="avg")
    want = _per_element_rs(s, ins, "bfloat16")  # sum, rounded to bf16 at every hop
    for r in range(n):
        # avg of the root's fp32 sum: same as scaling the rounded sum by 1/4 when
        # the sum's rounding is exact in the last hop; compare within 1 ulp
        a = fo.bf16_to_f32(got[r]).astype(np.float64)
        b = fo.bf16_to_f32(want[r]).astype(np.float64) / n
        assert np.all(np.abs(a - b) <= np.abs(b) * 2.0 ** -7 + 1e-30)


def test_avg_rejected_for_integers_and_unknown_ops():
    s = load_golden("nvs4_reduce_scatter")
    ins = [np.ones(4 * 8, np.int32) for _ in range(4)]
    with pytest.raises(ValueError):
        fo.reduce_scatter(s, ins, "int32", op="avg")
    with pytest.raises(ValueError):
        fo.reduce_scatter(s, [x.astype(np.float32) for x in ins], "float32", op="max")


def test_fp32_reduction_close_to_float64_sum():
    s = load_golden("nvs8_reduce_scatter")
    n = s.num_compute
    rng = np.random.default_rng(5)
    S = 4096
    ins = [rng.uniform(-1, 1, n * S).astype(np.float32) for _ in range(n)]
    outs = fo.reduce_scatter(s, ins, "float32")
    tot = np.sum(np.stack(ins).astype(np.float64), axis=0)
    for r in range(n):
        np.testing.assert_allclose(outs[r], tot[r * S:(r + 1) * S], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("name", golden_names())
def test_batch_slices_partition_each_shard(name):
    s = load_golden(name)
    sched = s.phases[1] if s.collective == "allreduce" else s
    for S in (0, 1, 7, 100, 12345):
        for rt in sched.roots:
            lo, covered = 0, []
            for b in rt.batches:
                covered.append(fo.slice_bounds(S, sched.k, lo, lo + b.multiplicity))
                lo += b.multiplicity
            assert covered[0][0] == 0 and covered[-1][1] == S
            assert all(x[1] == y[0] for x, y in zip(covered, covered[1:]))


def test_t_star_golden_values():
    # fig3a: AG T = 1/8, AR T = 1/4 per unit M (pkg/tests/test_verify.py:255-259)
    ag, ar = load_golden("fig3a_allgather"), load_golden("fig3a_allreduce")
    assert Fraction(ag.inv_x_star) / ag.num_compute == Fraction(1, 8)
    assert fo.t_star(ag, 1e9) == pytest.approx(1 / 8)
    assert fo.t_star(ar, 1e9) == pytest.approx(1 / 4)
    # nvswitch(8): 1/x* = 7/900 -> T*(AG 1 GiB) = 1.044 ms
    s = load_golden("nvs8_allgather")
    assert s.inv_x_star == Fraction(7, 900)
    assert fo.t_star(s, 1 << 30) * 1e3 == pytest.approx(1.0438, rel=1e-3)
    assert load_golden("nvs2_allgather").inv_x_star == Fraction(1, 900)
    assert load_golden("nvs4_allgather").inv_x_star == Fraction(1, 300)
    assert load_golden("groups100_allgather").inv_x_star == Fraction(1, 50)
    assert load_golden("groups450_allgather").k == 2
    assert load_golden("groups300_allgather").k == 3


def test_allreduce_shard_rule():
    assert fo.allreduce_shard(1000, 8, 4) == 128
    assert fo.allreduce_shard(1, 8, 2) == 64
    assert fo.allreduce_shard(0, 8, 4) == 0


@pytest.mark.parametrize("name", golden_names("allgather"))
def test_c_oracle_matches_numpy_oracle(name):
    from oracle import c_oracle

    s = load_golden(name)
    n = s.num_compute
    rng = np.random.default_rng(11)
    for S in (1, 5, 1000):
        sends = [rng.integers(0, 2**32, S, dtype=np.uint64).astype(np.uint32) for _ in range(n)]
        recvs = [np.zeros(n * S, dtype=np.uint32) for _ in range(n)]
        c_oracle.allgather(c_oracle.FlatForest(s), sends, recvs, threads=4)
        ref = fo.allgather(s, sends)
        for a, b in zip(recvs, ref):
            assert np.array_equal(a, b)

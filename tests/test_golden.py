"""Golden schedule fixtures are the reference generator's own output."""

import json
import os
import subprocess
import sys
from fractions import Fraction

import pytest

from conftest import GOLDEN, REPO, golden_names, load_golden, load_golden_topology, reference_collsched


def test_fixtures_match_reference_generator():
    cs = reference_collsched()
    if cs is None:
        pytest.skip("reference collsched not importable")
    r = subprocess.run([sys.executable, os.path.join(GOLDEN, "make_golden.py"), "--check"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("name", golden_names())
def test_fixture_validates_and_attains_bound(name):
    cs = reference_collsched()
    if cs is None:
        pytest.skip("reference collsched not importable")
    topo = name.rsplit("_", 1)[0] if not name.endswith("reduce_scatter") else name[: -len("_reduce_scatter")]
    t = cs.parse_topology(json.dumps(load_golden_topology(topo)))
    with open(os.path.join(GOLDEN, "schedules", name + ".json")) as f:
        s = cs.parse_schedule(f.read())
    from paper_2402_06787_b200.generator import meta_of

    rep = cs.validate_schedule(s, t, meta_of(s))
    assert rep.ok, rep.violations
    phases = 2 if s.collective == "allreduce" else 1
    assert cs.congestion_time(s, t) == phases * Fraction(s.inv_x_star) / s.num_compute


def test_package_cache_serves_reference_schedules_without_generating(monkeypatch):
    """The shipped cache yields the fixtures' forests without running the
    generator: schedules are parsed by the reference's own parse_schedule
    (schedule.py:439-448) and re-exported byte-identical by its export."""
    from paper_2402_06787_b200 import generator
    from paper_2402_06787_b200._refpath import require_collsched
    from paper_2402_06787_b200.schedule_io import export_json
    from paper_2402_06787_b200.topology import groups_switch_doc, nvswitch_doc

    cs = require_collsched()

    def no_generate(*a, **k):
        raise AssertionError("generate() called although the schedule is cached")

    monkeypatch.setattr(cs, "generate", no_generate)
    monkeypatch.setenv("FORESTCOLL_CACHE", "/nonexistent-cache-dir")
    cases = {f"nvs{n}": nvswitch_doc(n) for n in (2, 4, 8)}
    cases.update({f"groups{b}": groups_switch_doc(b) for b in (450, 300, 100)})
    for name, doc in cases.items():
        assert doc == load_golden_topology(name)
        for coll in ("allgather", "reduce_scatter", "allreduce"):
            s = generator.get_schedule(doc, coll, validate=False, write_cache=False)
            assert isinstance(s, cs.Schedule)
            with open(os.path.join(GOLDEN, "schedules", f"{name}_{coll}.json")) as f:
                assert export_json(s) == f.read()


def test_missing_reference_fails_loudly(monkeypatch):
    """No private schedule reader: without collsched every schedule entry
    point raises ReferenceMissing (and pre-flight is never skipped)."""
    from paper_2402_06787_b200 import _refpath, generator
    from paper_2402_06787_b200.errors import ReferenceMissing
    from paper_2402_06787_b200.topology import nvswitch_doc

    s = load_golden("nvs4_allgather")
    monkeypatch.setattr(_refpath, "_CACHED", [None])
    with pytest.raises(ReferenceMissing):
        generator.get_schedule(nvswitch_doc(4), "allgather", validate=False, write_cache=False)
    with pytest.raises(ReferenceMissing):
        generator.preflight(s, nvswitch_doc(4))


def test_appendix_a_forest_shape():
    """nvswitch(8) allgather forest as listed in SURVEY.md Appendix A."""
    s = load_golden("nvs8_allgather")
    rows = {rt.root: " ".join(f"{e.src[1:]}>{e.dst[1:]}" for e in rt.batches[0].edges) for rt in s.roots}
    assert rows["g0"] == "0>1 0>2 0>3 0>4 4>7 7>6 6>5"
    assert rows["g7"] == "7>6 6>5 5>4 4>3 3>2 2>1 1>0"


@pytest.mark.parametrize("beta,fixed_k", [(450, 1), (450, 3), (100, 2)])
def test_t_star_uses_congestion_time_for_fixed_k(beta, fixed_k):
    """fixed_k schedules are not marked exact (schedule.py:78-81): T* comes
    from the reference's own congestion_time over the topology
    (verify.py:537-562), allreduce summing its two phases."""
    import json
    from fractions import Fraction

    from paper_2402_06787_b200._refpath import require_collsched
    from paper_2402_06787_b200.schedule_io import t_star_seconds
    from paper_2402_06787_b200.topology import groups_switch_doc

    cs = require_collsched()
    doc = groups_switch_doc(beta)
    t = cs.parse_topology(json.dumps(doc))
    M = 1 << 30
    for coll in ("allgather", "allreduce"):
        s, _ = cs.generate(t, coll, fixed_k=fixed_k)
        assert not s.exact
        want = float(Fraction(cs.congestion_time(s, t))) * M / 1e9
        assert t_star_seconds(s, M, coll, doc) == pytest.approx(want, rel=1e-12)

"""Topology ingestion emits the reference's graph format."""

import json

import pytest

from conftest import reference_collsched
from paper_2402_06787_b200 import topology as T


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_nvswitch_doc_shape(n):
    d = T.nvswitch_doc(n)
    ids = T.compute_ids(d)
    assert len(ids) == n
    assert ids == [T.compute_id(i, n) for i in range(n)]  # lexicographic == rank order
    assert len(d["links"]) == 2 * n and all(l["bandwidth"] == 900 for l in d["links"])


@pytest.mark.parametrize("n,inv", [(2, (1, 900)), (4, (1, 300)), (8, (7, 900))])
def test_nvswitch_bound_with_reference(n, inv):
    cs = reference_collsched()
    if cs is None:
        pytest.skip("reference not importable")
    from fractions import Fraction

    t = cs.parse_topology(json.dumps(T.nvswitch_doc(n)))
    assert cs.validate(t).ok
    assert cs.bottleneck_search(t).inv_x_star == Fraction(*inv)


@pytest.mark.parametrize("beta", [450, 300, 100])
def test_groups_switch_is_eulerian(beta):
    d = T.groups_switch_doc(beta)
    bal = {}
    for l in d["links"]:
        bal[l["src"]] = bal.get(l["src"], 0) + l["bandwidth"]
        bal[l["dst"]] = bal.get(l["dst"], 0) - l["bandwidth"]
    assert all(v == 0 for v in bal.values())
    out = {}
    for l in d["links"]:
        if l["src"].startswith("g"):
            out[l["src"]] = out.get(l["src"], 0) + l["bandwidth"]
    assert set(out.values()) == {900}
    cs = reference_collsched()
    if cs is not None:
        assert cs.validate(cs.parse_topology(json.dumps(d))).ok


def test_discovery_falls_back_without_nvml(monkeypatch):
    def boom():
        raise RuntimeError("no NVML here")

    monkeypatch.setattr(T, "_nvml", boom)
    doc, src = T.discover_for_torch(8)
    assert src == "nominal" and doc == T.nvswitch_doc(8)


def test_nvml_discovery_with_fake_switch_links(monkeypatch):
    class FakeNV:
        NVML_FEATURE_ENABLED = 1
        NVML_NVLINK_DEVICE_TYPE_SWITCH = 2

        class NVMLError(Exception):
            pass

        def nvmlDeviceGetHandleByPciBusId(self, b):
            return b

        def nvmlDeviceGetNvLinkState(self, h, link):
            return 1

        def nvmlDeviceGetNvLinkVersion(self, h, link):
            return 5

        def nvmlDeviceGetNvLinkRemoteDeviceType(self, h, link):
            return 2

    monkeypatch.setattr(T, "_nvml", lambda: FakeNV())
    doc = T.discover_nvml([f"0000:{i:02x}:00.0" for i in range(8)])
    assert doc == T.nvswitch_doc(8)  # 18 links x 50 GB/s = 900 per direction


def test_bus_id_normalisation():
    assert T._bus(b"00000000:1B:00.0") == "0000:1b:00.0"
    assert T._bus("0000:1b:00.0") == "0000:1b:00.0"

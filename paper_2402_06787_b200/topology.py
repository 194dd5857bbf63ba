"""Topology ingestion: NVML NVLink/NVSwitch discovery emitting the reference's
graph format, plus the static builders used for CI and the stress configs.

Output is the reference's canonical topology document (SPEC.md:97-101,
``parse_topology`` at pkg/src/collsched/topology.py:188-232)::

    {"nodes": [{"id": "g0", "kind": "compute"},
               {"id": "nvs", "kind": "switch", "multicast": false,
                "aggregation": false}],
     "links": [{"src": "g0", "dst": "nvs", "bandwidth": 900}, ...]}

Bandwidths are integer GB/s per direction.  Compute ids are zero-padded
(``g0``..``g7``; ``g00``..``g15``) because the reference sorts compute ids
lexicographically (topology.py:126-128) and that order is the rank order of
every schedule it emits (schedule.py:98).  Discovery itself is a reference
non-goal, so this module is new.
"""

from __future__ import annotations

import json
from typing import Sequence

# NVLink generation -> GB/s per link per direction.
NVLINK_GBPS_PER_LINK = {1: 20, 2: 25, 3: 25, 4: 25, 5: 50}
NVML_NVLINK_MAX_LINKS = 18
SWITCH_ID = "nvs"


def compute_id(i: int, n: int) -> str:
    width = len(str(max(n - 1, 0)))
    return f"g{i:0{width}d}"


def nvswitch_doc(n: int, bandwidth: int = 900, multicast: bool = False) -> dict:
    """n GPUs on one NVSwitch node, `bandwidth` GB/s each way per GPU
    (B200 HGX: 18 NVLink5 links x 50 GB/s = 900)."""
    if n < 1:
        raise ValueError("need at least one GPU")
    ids = [compute_id(i, n) for i in range(n)]
    nodes = [{"id": g, "kind": "compute"} for g in ids]
    nodes.append(
        {"id": SWITCH_ID, "kind": "switch", "multicast": multicast, "aggregation": multicast}
    )
    links = []
    for g in ids:
        links.append({"src": g, "dst": SWITCH_ID, "bandwidth": int(bandwidth)})
        links.append({"src": SWITCH_ID, "dst": g, "bandwidth": int(bandwidth)})
    return {"nodes": nodes, "links": links}


def groups_switch_doc(beta: int, port: int = 900, n: int = 8) -> dict:
    """Sparse stress topology: n GPUs in two groups
    of n/2 (switch swA: the first half, swB: the second) joined only by the
    bridge pairs (g0, g[n/2]) and (g1, g[n/2+1]) at `beta` each way.  Bridge
    GPUs keep `port - beta` to their group switch, so every GPU port totals
    `port` and the graph is Eulerian (topology.py:268-276).  n = 8 is
    BASELINE configs[4]; n = 4 is its 4-GPU analogue (every GPU a bridge)."""
    if not 0 < beta < port:
        raise ValueError("need 0 < beta < port")
    if n < 4 or n % 2:
        raise ValueError("need an even n >= 4")
    h = n // 2
    ids = [compute_id(i, n) for i in range(n)]
    nodes = [{"id": g, "kind": "compute"} for g in ids]
    for sw in ("swA", "swB"):
        nodes.append({"id": sw, "kind": "switch", "multicast": False, "aggregation": False})
    links = []
    bridges = {0: h, 1: h + 1, h: 0, h + 1: 1}
    for i, g in enumerate(ids):
        sw = "swA" if i < h else "swB"
        bw = port - beta if i in bridges else port
        links.append({"src": g, "dst": sw, "bandwidth": bw})
        links.append({"src": sw, "dst": g, "bandwidth": bw})
        if i in bridges:
            links.append({"src": g, "dst": ids[bridges[i]], "bandwidth": beta})
    return {"nodes": nodes, "links": links}


def canonical_json(doc: dict) -> str:
    """Byte-stable JSON used for cache keys (node order kept, keys sorted)."""
    return json.dumps(doc, sort_keys=True, separators=(",", ":"))


def compute_ids(doc: dict) -> list[str]:
    """Compute node ids in the reference's rank order (lexicographic)."""
    return sorted(n["id"] for n in doc["nodes"] if n["kind"] == "compute")


def to_reference(doc: dict):
    """Parse into a reference ``collsched.Topology`` (requires collsched)."""
    from ._refpath import import_collsched

    cs = import_collsched()
    if cs is None:
        from .errors import Unsupported

        raise Unsupported("collsched (the reference generator) is not importable")
    return cs.parse_topology(json.dumps(doc))


# ---------------------------------------------------------------------------
# NVML discovery
# ---------------------------------------------------------------------------

def _nvml():
    import pynvml

    pynvml.nvmlInit()
    return pynvml


def discover_nvml(pci_bus_ids: Sequence[str] | None = None) -> dict:
    """Build the topology of the given GPUs (PCI bus ids in rank order; all
    NVML-visible GPUs when None) from NVLink state.

    Links whose remote end is an NVSwitch are aggregated into one switch node
    ``nvs`` with (active links x per-link rate) each way; links that land on
    another listed GPU become direct GPU<->GPU links.  Raises RuntimeError
    when NVML is unavailable or a GPU reports no active NVLink.
    """
    nv = _nvml()
    if pci_bus_ids is None:
        handles = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(nv.nvmlDeviceGetCount())]
        buses = [_bus(nv.nvmlDeviceGetPciInfo(h).busId) for h in handles]
    else:
        buses = [_bus(b) for b in pci_bus_ids]
        handles = [nv.nvmlDeviceGetHandleByPciBusId(b) for b in pci_bus_ids]
    n = len(handles)
    ids = [compute_id(i, n) for i in range(n)]
    index_of_bus = {b: i for i, b in enumerate(buses)}
    switch_bw = [0] * n
    direct: dict[tuple[int, int], int] = {}
    for i, h in enumerate(handles):
        for link in range(NVML_NVLINK_MAX_LINKS):
            try:
                if nv.nvmlDeviceGetNvLinkState(h, link) != nv.NVML_FEATURE_ENABLED:
                    continue
                version = nv.nvmlDeviceGetNvLinkVersion(h, link)
            except nv.NVMLError:
                continue
            rate = NVLINK_GBPS_PER_LINK.get(int(version), 50)
            remote_type = None
            try:
                remote_type = nv.nvmlDeviceGetNvLinkRemoteDeviceType(h, link)
            except (nv.NVMLError, AttributeError):
                pass
            if remote_type == getattr(nv, "NVML_NVLINK_DEVICE_TYPE_SWITCH", 2):
                switch_bw[i] += rate
                continue
            try:
                rbus = _bus(nv.nvmlDeviceGetNvLinkRemotePciInfo(h, link).busId)
            except nv.NVMLError:
                continue
            j = index_of_bus.get(rbus)
            if j is not None and j != i:
                direct[(i, j)] = direct.get((i, j), 0) + rate
    if any(bw == 0 for bw in switch_bw) and not direct:
        raise RuntimeError("no active NVLink found by NVML")
    nodes = [{"id": g, "kind": "compute"} for g in ids]
    links = []
    if any(switch_bw):
        nodes.append(
            {"id": SWITCH_ID, "kind": "switch", "multicast": False, "aggregation": False}
        )
        for i, bw in enumerate(switch_bw):
            if bw:
                links.append({"src": ids[i], "dst": SWITCH_ID, "bandwidth": bw})
                links.append({"src": SWITCH_ID, "dst": ids[i], "bandwidth": bw})
    for (i, j), bw in sorted(direct.items()):
        links.append({"src": ids[i], "dst": ids[j], "bandwidth": bw})
    return {"nodes": nodes, "links": links}


def _bus(b) -> str:
    if isinstance(b, bytes):
        b = b.decode()
    b = b.lower()
    # NVML reports 8-hex-digit domains ("00000000:1b:00.0"); torch uses 4
    parts = b.split(":")
    if len(parts) == 3 and len(parts[0]) > 4:
        parts[0] = parts[0][-4:]
    return ":".join(parts)


def discover_for_torch(world_size: int, pci_bus_ids: Sequence[str] | None = None):
    """(topology, source) for `world_size` ranks: NVML when it works
    ("nvml"), else the nominal B200 NVSwitch model, 900 GB/s per GPU per
    direction ("nominal")."""
    if world_size >= 2:
        try:
            doc = discover_nvml(pci_bus_ids)
            if len(compute_ids(doc)) == world_size:
                return doc, "nvml"
        except Exception:
            pass
    return nvswitch_doc(world_size), "nominal"

"""Schedule producer: the reference's ``generate()`` behind a topology-keyed cache.

The host-side max-flow / tree-packing generator stays the reference's Python
(``collsched.generate``, pkg/src/collsched/pipeline.py:43-78).  Generation
runs once per (topology, collective, options); its canonical JSON export
(schedule.py:474-482, deterministic per README.md:94-95) is cached on disk
keyed by a hash of the topology document, so machines without the reference
(the GPU box) execute byte-identical reference schedules.  The package ships
the cache for the BASELINE topologies under ``schedules/``; new entries go to
``$FORESTCOLL_CACHE`` (default ``~/.cache/forestcoll``).

The pre-flight mirrors the reference CLI, which refuses to emit a schedule
failing ``validate_schedule`` (cli.py:186-195, exit 3): a failing report
raises ``PlanError`` carrying the violations.
"""

from __future__ import annotations

import hashlib
import json
import os
from types import SimpleNamespace

from ._refpath import require_collsched
from .errors import PlanError
from .schedule_io import COLLECTIVES, export_json, parse_schedule_json
from .topology import canonical_json

PACKAGE_CACHE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "schedules")


def user_cache_dir() -> str:
    return os.environ.get(
        "FORESTCOLL_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "forestcoll")
    )


def cache_key(topology_doc: dict, collective: str, prune: bool = True, fixed_k=None) -> str:
    blob = canonical_json(
        {"topology": topology_doc, "collective": collective, "prune": bool(prune),
         "fixed_k": fixed_k, "format": 1}
    )
    return hashlib.sha256(blob.encode()).hexdigest()[:24]


def _cache_paths(key: str) -> list[str]:
    return [os.path.join(PACKAGE_CACHE, key + ".json"), os.path.join(user_cache_dir(), key + ".json")]


def meta_of(schedule) -> SimpleNamespace:
    """Optimality metadata carried by the schedule itself (schedule.py:68-81);
    enough for ``validate_schedule`` (verify.py:426,452,468)."""
    return SimpleNamespace(
        inv_x_star=schedule.inv_x_star, U=schedule.U, k=schedule.k, y=schedule.y,
        exact=schedule.exact,
    )


def generate_json(topology_doc: dict, collective: str, prune: bool = True, fixed_k=None) -> str:
    """Run the reference generator and return its canonical JSON export."""
    cs = require_collsched()
    t = cs.parse_topology(json.dumps(topology_doc))
    s, _meta = cs.generate(t, collective, fixed_k=fixed_k, prune=prune)
    return cs.export(s, "json")


def get_schedule(topology_doc: dict, collective: str, prune: bool = True, fixed_k=None,
                 validate: bool = True, write_cache: bool = True):
    """Schedule for (topology, collective): cache hit or reference generation.

    Returns the reference's own ``Schedule`` (parsed by
    ``collsched.parse_schedule``).  With `validate`, runs ``validate_schedule``
    against the topology and raises PlanError on a failing report.
    """
    if collective not in COLLECTIVES:
        raise PlanError(f"unknown collective {collective!r}")
    key = cache_key(topology_doc, collective, prune, fixed_k)
    text = None
    for p in _cache_paths(key):
        if os.path.exists(p):
            with open(p) as f:
                text = f.read()
            break
    if text is None:
        text = generate_json(topology_doc, collective, prune, fixed_k)
        if write_cache:
            d = user_cache_dir()
            try:
                os.makedirs(d, exist_ok=True)
                tmp = os.path.join(d, f".{key}.{os.getpid()}.tmp")
                with open(tmp, "w") as f:
                    f.write(text)
                os.replace(tmp, os.path.join(d, key + ".json"))
            except OSError:
                pass
    s = parse_schedule_json(text)
    if validate:
        preflight(s, topology_doc)
    return s


def preflight(schedule, topology_doc: dict) -> None:
    """``validate_schedule`` pre-flight (verify.py:478-534), as the reference
    CLI runs it before emitting a schedule (cli.py:186-195, exit 3).  Never
    skipped: without the reference package this raises ReferenceMissing.
    The compiler's own structural checks run as well."""
    cs = require_collsched()
    t = cs.parse_topology(json.dumps(topology_doc))
    if not isinstance(schedule, cs.Schedule):
        schedule = cs.parse_schedule(export_json(schedule))
    report = cs.validate_schedule(schedule, t, meta_of(schedule))
    if not report.ok:
        raise PlanError(
            "schedule failed validate_schedule: "
            + "; ".join(f"{v.kind}: {v.detail}" for v in report.violations),
            report.violations,
        )

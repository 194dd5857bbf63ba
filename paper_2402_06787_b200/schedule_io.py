"""Schedules at the boundary: the reference's own objects, read by its own parser.

The boundary of this path is the reference ``Schedule`` forest
(pkg/src/collsched/schedule.py:31-81) and its JSON wire format
(``export`` / ``parse_schedule``, schedule.py:439-482).  This package never
re-implements either: schedules are parsed with ``collsched.parse_schedule``
from the reference install (``baseline/_ref``, located by ``_refpath``), and
the compiler walks the reference objects.  When the reference package is
absent every schedule entry point raises ``ReferenceMissing`` -- there is no
private reader to fall back to.

What stays here is the executor's own arithmetic on a schedule: T* for a
message size.
"""

from __future__ import annotations

from fractions import Fraction

from ._refpath import require_collsched

ALLGATHER = "allgather"
REDUCE_SCATTER = "reduce_scatter"
ALLREDUCE = "allreduce"
COLLECTIVES = (ALLGATHER, REDUCE_SCATTER, ALLREDUCE)


def parse_schedule_json(text: str):
    """``collsched.parse_schedule`` (schedule.py:439-448): reference objects."""
    return require_collsched().parse_schedule(text)


def load_schedule(path: str):
    with open(path) as f:
        return parse_schedule_json(f.read())


def export_json(schedule) -> str:
    """``collsched.export(s, "json")`` (schedule.py:474-482), the canonical form."""
    return require_collsched().export(schedule, "json")


def t_star_seconds(schedule, message_bytes: int, collective: str | None = None,
                   topology_doc: dict | None = None) -> float:
    """ForestColl's optimal time T* for a message of M bytes.

    T* is the schedule's congestion bound per GB of M times M.  With the
    topology it is the reference's own ``congestion_time`` (verify.py:537-562:
    max over links of usage / (N * k * bandwidth), allreduce summing its
    phases), which also covers ``fixed_k`` schedules whose bound is not exact
    (schedule.py:78-81).  Without it, inv_x_star / N per phase -- equal to
    ``congestion_time`` for an exact schedule (validate_schedule,
    verify.py:468-469).  Bandwidths are in GB/s, so the bound is s/GB.
    """
    coll = collective or schedule.collective
    if topology_doc is not None:
        import json

        cs = require_collsched()
        per_gb = Fraction(cs.congestion_time(schedule, cs.parse_topology(json.dumps(topology_doc))))
        if coll == ALLREDUCE and schedule.collective != ALLREDUCE:
            per_gb *= 2
    else:
        phases = 2 if coll == ALLREDUCE else 1
        per_gb = phases * Fraction(schedule.inv_x_star) / schedule.num_compute
    return float(per_gb) * message_bytes / 1e9

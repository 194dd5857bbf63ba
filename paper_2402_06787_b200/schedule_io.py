"""Reader for the reference's schedule wire format.

The boundary of this path is the reference ``Schedule`` forest
(pkg/src/collsched/schedule.py:31-81) and its JSON export
(schedule.py:348-448; frozen field set pinned by pkg/tests/test_schedule.py:
174-191).  When ``collsched`` is importable its own ``parse_schedule`` is used
and the executor consumes the reference objects directly.  On machines
without the reference (the GPU box) this module reads the same JSON into
attribute-compatible frozen records, so the compiler sees one shape either
way.  Field names and meanings follow schedule.py:31-81 exactly.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from fractions import Fraction

from ._refpath import import_collsched
from .errors import PlanError

ALLGATHER = "allgather"
REDUCE_SCATTER = "reduce_scatter"
ALLREDUCE = "allreduce"
COLLECTIVES = (ALLGATHER, REDUCE_SCATTER, ALLREDUCE)


@dataclass(frozen=True)
class PathUse:
    path: tuple
    multiplicity: int


@dataclass(frozen=True)
class ScheduleEdge:
    src: str
    dst: str
    paths: tuple


@dataclass(frozen=True)
class PrunedHop:
    src: str
    dst: str
    multiplicity: int


@dataclass(frozen=True)
class ScheduleBatch:
    multiplicity: int
    edges: tuple
    pruned: tuple = ()


@dataclass(frozen=True)
class RootTrees:
    root: str
    batches: tuple


@dataclass(frozen=True)
class Schedule:
    collective: str
    num_compute: int
    k: int
    U: Fraction
    y: Fraction
    inv_x_star: Fraction
    roots: tuple
    phases: tuple = ()
    exact: bool = True


def _frac(text) -> Fraction:
    if not isinstance(text, str) or "/" not in text:
        raise PlanError(f"expected a 'p/q' rational string, got {text!r}")
    num, _, den = text.partition("/")
    return Fraction(int(num), int(den))


def _from_doc(doc: dict) -> Schedule:
    coll = doc["collective"]
    if coll not in COLLECTIVES:
        raise PlanError(f"unknown collective {coll!r}")
    common = dict(
        collective=coll,
        num_compute=int(doc["num_compute_nodes"]),
        k=int(doc["trees_per_root"]),
        U=_frac(doc["scale_U"]),
        y=_frac(doc["tree_bandwidth"]),
        inv_x_star=_frac(doc["optimal_inv_x"]),
        exact=bool(doc.get("exact_bound", True)),
    )
    if coll == ALLREDUCE:
        phases = tuple(_from_doc(p) for p in doc.get("phases", ()))
        if len(phases) != 2:
            raise PlanError("allreduce schedules carry exactly two phases")
        return Schedule(roots=(), phases=phases, **common)
    roots = tuple(
        RootTrees(
            root=rd["root"],
            batches=tuple(
                ScheduleBatch(
                    multiplicity=int(bd["multiplicity"]),
                    edges=tuple(
                        ScheduleEdge(
                            src=ed["src"],
                            dst=ed["dst"],
                            paths=tuple(
                                PathUse(tuple(pd["path"]), int(pd["multiplicity"]))
                                for pd in ed["paths"]
                            ),
                        )
                        for ed in bd["edges"]
                    ),
                    pruned=tuple(
                        PrunedHop(hd["src"], hd["dst"], int(hd.get("multiplicity", 1)))
                        for hd in bd.get("pruned", ())
                    ),
                )
                for bd in rd["batches"]
            ),
        )
        for rd in doc["roots"]
    )
    return Schedule(roots=roots, **common)


def parse_schedule_json(text: str, prefer_reference: bool = True):
    """Parse schedule JSON; reference objects when collsched is importable."""
    cs = import_collsched() if prefer_reference else None
    if cs is not None:
        return cs.parse_schedule(text)
    try:
        return _from_doc(json.loads(text))
    except (KeyError, TypeError, ValueError) as exc:
        raise PlanError(f"malformed schedule document: {exc!r}") from None


def load_schedule(path: str, prefer_reference: bool = True):
    with open(path) as f:
        return parse_schedule_json(f.read(), prefer_reference)


def t_star_seconds(schedule, message_bytes: int, collective: str | None = None) -> float:
    """ForestColl's optimal time T* for a message.

    AG/RS: T* = (M/N) * inv_x_star; AR: the sum of both phases, 2*(M/N)*inv_x_star
    (verify.py:537-562 sums phase congestion times; each phase attains
    inv_x_star/N when exact, validate_schedule verify.py:468-469).  inv_x_star
    is in s/GB for GB/s bandwidths; M convention per SURVEY.md §8d (AG: total
    output bytes, RS: per-rank input bytes, AR: buffer bytes).
    """
    coll = collective or schedule.collective
    n = schedule.num_compute
    per_unit = float(Fraction(schedule.inv_x_star)) / n  # seconds per GB of M
    phases = 2 if coll == ALLREDUCE else 1
    return phases * per_unit * message_bytes / 1e9

"""Regenerate the golden schedule fixtures from the reference generator.

Run in the build container (the reference is importable there):

    python tests/golden/make_golden.py            # write fixtures + package cache
    python tests/golden/make_golden.py --check    # byte-compare against the committed files

For every topology below it calls the reference's own ``collsched.generate``
(pkg/src/collsched/pipeline.py:43-78) and stores its canonical JSON export
(schedule.py:474-482) under tests/golden/schedules/.  Schedules of the
BASELINE topologies are also written to the package's topology-keyed cache
(paper_2402_06787_b200/schedules/<key>.json) so the GPU box, which has no
reference checkout, executes byte-identical reference schedules.  Each
fixture is checked with the reference's ``validate_schedule`` and
``congestion_time`` before it is written.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
for p in ("/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref")):
    if os.path.isdir(os.path.join(p, "collsched")):
        sys.path.insert(0, p)
        break

import collsched as cs  # noqa: E402

from paper_2402_06787_b200 import generator, topology  # noqa: E402

COLLS = ("allgather", "reduce_scatter", "allreduce")


def topologies():
    """name -> (topology document, collectives, ship in the package cache)."""
    out = {}
    for n in (2, 4, 8):
        out[f"nvs{n}"] = (topology.nvswitch_doc(n), COLLS, True)
    for n in (2, 4, 8):
        out[f"nvs{n}_mc"] = (topology.nvswitch_doc(n, multicast=True), COLLS, True)
    for beta in (450, 300, 100):
        out[f"groups{beta}"] = (topology.groups_switch_doc(beta), COLLS, True)
    for beta in (450, 300, 100):  # the 4-GPU analogue of configs[4]
        out[f"groups4_{beta}"] = (topology.groups_switch_doc(beta, n=4), COLLS, True)
    out["fig3a"] = (json.loads(cs.serialize_topology(
        cs.synth_topology("boxes", boxes=2, gpus_per_box=4, intra=10, inter=1))), COLLS, False)
    out["two_node"] = (json.loads(cs.serialize_topology(
        cs.synth_topology("ring", n=2, bw=3, bidirectional=False))), COLLS, False)
    out["ring4"] = (json.loads(cs.serialize_topology(
        cs.synth_topology("ring", n=4, bw=1))), ("allgather",), False)
    for seed in (1, 3, 7, 11):
        t = cs.random_eulerian_topology(seed)
        out[f"random{seed}"] = (json.loads(cs.serialize_topology(t)), ("allgather",), False)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    sched_dir = os.path.join(HERE, "schedules")
    topo_dir = os.path.join(HERE, "topologies")
    os.makedirs(sched_dir, exist_ok=True)
    os.makedirs(topo_dir, exist_ok=True)
    os.makedirs(generator.PACKAGE_CACHE, exist_ok=True)
    index = {}
    bad = []
    for name, (doc, colls, ship) in topologies().items():
        t = cs.parse_topology(json.dumps(doc))
        topo_path = os.path.join(topo_dir, f"{name}.json")
        files = {topo_path: json.dumps(doc, indent=1) + "\n"}
        for coll in colls:
            s, meta = cs.generate(t, coll)
            rep = cs.validate_schedule(s, t, meta)
            text = cs.export(s, "json")
            files[os.path.join(sched_dir, f"{name}_{coll}.json")] = text
            if ship:
                key = generator.cache_key(doc, coll, True, None)
                files[os.path.join(generator.PACKAGE_CACHE, key + ".json")] = text
            index[f"{name}_{coll}"] = {
                "k": s.k, "inv_x_star": f"{s.inv_x_star.numerator}/{s.inv_x_star.denominator}",
                "congestion_time": str(cs.congestion_time(s, t)), "valid": rep.ok,
                "num_compute": s.num_compute,
            }
        for path, text in files.items():
            if args.check:
                with open(path) as f:
                    if f.read() != text:
                        bad.append(path)
            else:
                with open(path, "w") as f:
                    f.write(text)
    idx_path = os.path.join(HERE, "index.json")
    idx_text = json.dumps(index, indent=1, sort_keys=True) + "\n"
    if args.check:
        with open(idx_path) as f:
            if f.read() != idx_text:
                bad.append(idx_path)
        if bad:
            print("MISMATCH:", *bad, sep="\n  ")
            sys.exit(1)
        print("golden fixtures match the reference output")
    else:
        with open(idx_path, "w") as f:
            f.write(idx_text)
        print(f"wrote {len(index)} schedules")


if __name__ == "__main__":
    main()

"""The package CLI (topology / schedule / describe) on CPU."""

import json
import os
import subprocess
import sys

from conftest import GOLDEN, REPO


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2402_06787_b200", *args], cwd=REPO,
                          capture_output=True, text=True, timeout=300)


def test_topology_and_schedule_roundtrip(tmp_path):
    r = run("topology", "--nvswitch", "4")
    assert r.returncode == 0
    doc = json.loads(r.stdout)
    assert len([n for n in doc["nodes"] if n["kind"] == "compute"]) == 4
    topo = tmp_path / "t.json"
    topo.write_text(r.stdout)
    r = run("schedule", "-t", str(topo), "--collective", "allgather")
    assert r.returncode == 0, r.stderr
    with open(os.path.join(GOLDEN, "schedules", "nvs4_allgather.json")) as f:
        assert r.stdout == f.read()


def test_describe():
    r = run("describe", "-s", os.path.join(GOLDEN, "schedules", "nvs8_allreduce.json"))
    assert r.returncode == 0
    assert "allreduce: N=8 k=1" in r.stdout and "ar_root" in r.stdout


def test_bad_input_exit_code(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{}")
    r = run("schedule", "-t", str(bad))
    assert r.returncode != 0

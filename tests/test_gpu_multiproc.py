"""Multi-GPU parity (one process per GPU, real NVLink peer mapping)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multiproc_parity(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n),
           os.path.join(HERE, "mp", "parity_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(" OK") >= n, out[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_nvls_engine_parity(n):
    """Pruned forests on a multicast/aggregation NVSwitch run through the
    NVLS (multimem) engine: allgather bit-exact, int32 exact, fp within tolerance."""
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + n),
           os.path.join(HERE, "mp", "nvls_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    if "SKIP" in out:
        pytest.skip("no multicast support on this box")
    assert out.count(" OK") >= n, out[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_mismatched_output_buffers_fail_loudly(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29760 + n),
           os.path.join(HERE, "mp", "mismatch_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and out.count(" OK") >= n, out[-4000:]
    assert "different output buffer" in out, out[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_fsdp2_custom_collectives(n):
    """FSDP2 with ForestColl all-gather (symmetric pool) and reduce-scatter
    (AVG fused in the kernel) matches stock NCCL FSDP2."""
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29770 + n),
           os.path.join(HERE, "mp", "fsdp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and out.count(" OK") >= n, out[-4000:]


def test_ddp_comm_hook():
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29750",
           os.path.join(HERE, "mp", "ddp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and out.count(" OK") >= 2, out[-4000:]


@pytest.mark.parametrize("n", [2, 4, 8])
def test_randomized_soak(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29800 + n),
           os.path.join(HERE, "mp", "stress_worker.py"), "150"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and out.count("STRESS") >= n, out[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_eight_rank_forests_over_nvlink(n):
    """8-rank forests (nvswitch(8), sparse 2x4) with 8/n ranks per GPU."""
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29900 + n),
           os.path.join(HERE, "mp", "multirank_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and out.count(" OK") >= n, out[-4000:]



def test_cli_run_one_rank_per_gpu(tmp_path):
    """`torchrun ... -m paper_2402_06787_b200 run` times the forest with one
    rank per GPU and reports the fraction of T*."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    import json

    from paper_2402_06787_b200.topology import nvswitch_doc

    topo = tmp_path / "nvs2.json"
    topo.write_text(json.dumps(nvswitch_doc(2)))
    for coll in ("allgather", "allreduce"):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr", "127.0.0.1", "--master-port", "29721", "-m", "paper_2402_06787_b200",
               "run", "-t", str(topo), "--collective", coll, "--mib", "64", "--steps", "5"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                           cwd=os.path.dirname(HERE))
        assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
        line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
        assert line["ranks"] == 2 and line["mode"] == "2 ranks, one per GPU"
        assert 0 < line["frac_of_t_star"] < 1.0

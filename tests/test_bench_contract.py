"""The bench.py contract on the CPU: the reference arm (the oracle, bench.py --impl reference) prints one JSON
line with the keys the driver reads, on the same metric / config as the GPU arm; world size 2 under torchrun
prints once (rank 0) and the other rank exits 0."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    r = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.strip().startswith("{")]


@pytest.mark.parametrize("workload", ["toy", "deit_s"])
def test_reference_arm_json(workload):
    lines = run(["bench.py", "--impl", "reference", "--workload", workload, "--steps", "1", "--warmup", "0",
                 "--ref-tokens", "16"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["config"]["workload"].startswith(workload)
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_reference_arm_rank0_only():
    lines = run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                 "--master-port", str(free_port()), "bench.py", "--impl", "reference", "--workload", "toy", "--gpus", "2",
                 "--steps", "1", "--warmup", "0", "--ref-tokens", "16"])
    assert len(lines) == 1
    assert json.loads(lines[0])["impl"] == "reference"


def test_gpus_flag_launches_the_ranks():
    """`bench.py --gpus 2` outside torchrun re-executes itself under torch.distributed.run with 2 ranks (one per
    GPU); the line reports n_gpus = 2 (rank 0 prints, rank 1 exits 0)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "toy", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--ref-tokens", "16"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_world_size_mismatch_fails():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "toy", "--gpus", "4",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"))
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


@pytest.mark.gpu
def test_gpu_arm_json():
    """The GPU arm on the toy workload: one JSON line with the roofline / e2e / clocks / launch-count keys."""
    lines = run(["bench.py", "--workload", "toy", "--steps", "3", "--warmup", "3", "--no-baselines",
                 "--no-cpu-baseline"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["peak"] > 0 and r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-2, abs=1e-4)
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]

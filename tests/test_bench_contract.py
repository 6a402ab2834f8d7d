"""bench.py's one-JSON-line contract: the reference arm (the CPU oracle, runs without a GPU) and a
small GPU run of our arm, each checked for the keys and types the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _common(d):
    for k in ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["higher_is_better"] is True and d["value"] > 0 and d["warmup"] >= 3
    assert "workload" in d["config"]
    for k in ["value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"]:
        assert k in d["e2e"], k


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--scale", "0.005", "--steps", "2", "--warmup", "3", "--cpu-seconds", "2"], 600)
    _common(d)
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--scale", "0.02", "--nq", "500", "--steps", "3", "--warmup", "3", "--ef", "128", "--cpu-seconds", "2"],
             900)
    _common(d)
    r = d["roofline"]
    for k in ["bound", "achieved", "peak", "unit", "frac", "traffic"]:
        assert k in r, k
    assert r["bound"] == "hbm" and 0 < r["frac"] and r["unit"] == "GB/s"
    assert d["gpu_launches"] >= d["steps"]
    assert d["cpu_baseline"]["ids_equal_frac"] >= 0.95
    assert d["cpu_baseline"]["codes_equal_full_size"] is True
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_gpu_arm_two_ranks_gloo():
    """bench.py --gpus 2 without torchrun relaunches itself as two processes; with
    AQR_DIST_BACKEND=gloo both ranks share the one GPU (a functional check of the N > 1 path,
    not a measurement).  The line reports both ranks' distinct queries (weak scaling)."""
    env = dict(os.environ, AQR_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--scale", "0.02", "--nq", "300",
                        "--steps", "3", "--warmup", "3", "--ef", "128", "--no-cpu"], capture_output=True, text=True,
                       timeout=1200, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["queries_per_step"] == 600 and d["config"]["queries_per_rank"] == 300
    assert "relaunching under torch.distributed.run" in r.stderr and "rank 1/2 backend=gloo" in r.stderr

"""bench.py contract on the small parity configuration (GPU): one JSON line with
the keys the driver reads, device-side timing, e2e through the host API."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", ["c1"])
def test_bench_json_line(config):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["roofline"]["bound"] in ("tensor", "hbm") and 0 < d["roofline"]["frac"] < 1
    assert d["gpu_launches"] > 0


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"


def test_two_rank_launch_shards_heads():
    """The --gpus N path end to end on one GPU (two ranks share the device over
    gloo -- test hooks AQ_BENCH_SHARE_DEVICE / AQ_BENCH_BACKEND; the driver runs
    NCCL on N GPUs): torchrun self-launch, head sharding, max over ranks, one
    line from rank 0."""
    env = dict(os.environ, AQ_BENCH_SHARE_DEVICE="1", AQ_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c1",
                          "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["heads_per_rank"] == 1 and d["scaling"] == "strong" and d["value"] > 0

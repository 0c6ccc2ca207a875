"""The bench.py contract (task: one JSON line with the driver's keys, roofline, cpu_baseline,
e2e, clocks, gpu_launches; the reference arm = the oracle)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    b = run("--steps", "5", "--warmup", "3")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
                "gpu_launches"):
        assert key in b, key
    assert b["n_gpus"] == 1 and b["steps"] == 5 and b["warmup"] == 3 and b["value"] > 0
    assert "workload" in b["config"]
    r = b["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] < 1.5
    c = b["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = b["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert b["gpu_launches"] >= 5 * 4  # the hot path's kernels, every timed step
    assert "sm_mhz" in b["clocks"] and "reasons" in b["clocks"]


def test_bench_reference_arm_is_the_oracle():
    b = run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert b["impl"] == "reference" and b["value"] > 0
    assert b["cpu_baseline"]["kind"] == "oracle"
    assert b["e2e"]["h2d_bytes_per_step"] == 0 and b["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.parametrize("shard", ["sym", "corpus"])
def test_bench_self_launches_ranks(shard):
    # --gpus 2 without a launcher: bench.py starts the ranks itself; on this one-GPU box they
    # share cuda:0 through the library's host transport (KNN_BENCH_SHARE_GPU=1)
    env = dict(os.environ, KNN_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--shard", shard,
                        "--no-cpu-baseline", "--no-e2e"], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    b = json.loads(lines[0])
    assert b["n_gpus"] == 2 and b["value"] > 0
    assert b["config"]["sharding"].startswith({"sym": "upper triangle", "corpus": "corpus columns"}[shard])

"""bench.py's output contract (the driver parses one JSON line): the GPU arm
with every key the round-end check reads, and the reference arm on the
host (the reference's own compiled kernels from oracle/_ref)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900, env=None):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=REPO,
                         env=dict(os.environ, **(env or {})))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.skipif(not os.path.isdir(os.path.join(REPO, "oracle", "_ref")),
                    reason="the reference kernels are not built (oracle/build_ref.sh)")
def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.skipif(not os.path.isdir(os.path.join(REPO, "oracle", "_ref")),
                    reason="the reference kernels are not built (oracle/build_ref.sh)")
def test_gpus_2_self_launches_two_ranks():
    """--gpus 2 without torchrun re-launches under torch.distributed.run:
    two ranks, rank 0 prints the only line, n_gpus = 2, and the reference
    arm's config equals the GPU arm's workload description."""
    d = run_bench("--impl", "reference", "--gpus", "2", "--config", "c0", "--steps", "1",
                  "--warmup", "1")
    assert d["n_gpus"] == 2 and d["config"]["config"] == "c0"
    assert d["config"]["parallelism"] == "frames-sharded x2"


def test_world_size_mismatch_fails_loudly():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
                          "--impl", "reference"], capture_output=True, text=True, cwd=REPO,
                         env=dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"),
                         timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_launcher():
    """The launcher on the one-GPU test box: two ranks share cuda:0 (gloo
    plumbing, frame sharding only -- not a scaling measurement)."""
    d = run_bench("--gpus", "2", "--config", "c0", "--steps", "3", "--warmup", "3",
                  "--no-cpu-baseline", env={"ARTEMIS_BENCH_SHARED_GPU": "1"})
    assert d["n_gpus"] == 2 and len(d["ranks"]) == 2 and d["shared_gpu"] is True
    assert d["e2e"]["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c1", "c4"])
def test_gpu_arm_multiview_configs(config):
    d = run_bench("--config", config, "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert d["config"]["views_per_step"] == (8 if config == "c1" else 2)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_gpu_arm_line():
    d = run_bench("--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "gpu_launches", "clocks", "e2e"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["unit"] == "GB/s"
    assert d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0

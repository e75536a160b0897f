"""bench.py output contract (the driver parses one JSON line), checked on the CPU-only
reference arm (the oracle on host cores); the GPU arm's line carries the same keys plus
`e2e`, `roofline`, `clocks`, `gpu_launches` (covered by running bench.py on the GPU)."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                          "--config", "c1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference"
    assert line["unit"] == "rays/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["vs_baseline"] is None
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "rays/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "workload" in line["config"]


@pytest.mark.gpu
def test_our_arm_line_under_torchrun_two_ranks():
    """Our arm's JSON line at N = 2 through torchrun (the driver's launch), both ranks on
    one GPU with gloo collectives (NS2B_DIST_BACKEND): rank 0 alone prints one line, with
    the weak-scaling keys, the whole-job value, e2e, roofline, clocks and our launches."""
    import os

    env = dict(os.environ, NS2B_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                          "--steps", "3", "--warmup", "3", "--config", "c1", "--no-cpu"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert BASE_KEYS <= set(line)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["config"]["parallelism"] == "dp2"
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert {"roofline", "clocks"} <= set(line)

"""bench.py's JSON-line contract on the host (no GPU needed).

The reference arm (`--impl reference`) is the oracle timed on host cores (DESIGN
§9); its line must carry the base contract's keys plus `impl`, `cpu_baseline`
and a zero-copy `e2e`. Under torchrun only rank 0 prints. Our arm has no CPU
fallback: without a GPU it must exit non-zero and print no bench line.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = [sys.executable, "bench.py", "--config", "1", "--steps", "2", "--warmup", "1"]


def _run(extra, env=None, timeout=300):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run(ARGS + extra, cwd=ROOT, env=e, capture_output=True, text=True,
                          timeout=timeout)


def test_reference_arm_line():
    r = _run(["--impl", "reference"])
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["metric"] == "Cell-plan evaluations/sec" and d["unit"] == "cell-plans/s"
    assert d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["vs_baseline"] is None
    assert d["config"]["workload"] == "cfg1"
    # cfg1 is the SPEC-sized case: 12 Cells / 20 plans
    assert d["config"]["cells"] == 12 and d["config"]["cell_plans"] == 20
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference"], env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_our_arm_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; the GPU arm is exercised by the -m gpu suite")
    r = _run(["--no-cpu-baseline", "--no-e2e"])
    assert r.returncode != 0
    assert not any(ln.lstrip().startswith("{") for ln in r.stdout.splitlines())

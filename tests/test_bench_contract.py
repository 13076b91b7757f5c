"""bench.py's reference arm runs on CPU (it times the oracle port), so its JSON
line contract can be checked here without a GPU; the GPU arm's line is
checked by `-m gpu` runs and the driver."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REQUIRED = {
    "impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
    "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
    "cpu_baseline", "e2e",
}


@pytest.mark.parametrize("workload", ["tloc", "words"])
def test_reference_arm_json_line(workload):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run(
        [sys.executable, "bench.py", "--impl", "reference", "--workload", workload,
         "--steps", "1", "--warmup", "3", "--objects", "2000", "--queries", "16"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=600,
    )
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert REQUIRED <= set(rec), REQUIRED - set(rec)
    assert rec["impl"] == "reference"
    assert rec["value"] > 0 and rec["steps"] == 1 and rec["warmup"] == 3
    assert rec["higher_is_better"] is True
    assert rec["e2e"]["value"] == rec["value"]
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["e2e"]["d2h_bytes_per_step"] == 0
    cb = rec["cpu_baseline"]
    assert cb["value"] == rec["value"] and cb["kind"] in ("reference", "port") and cb["cores"] >= 1
    assert "workload" in rec["config"]

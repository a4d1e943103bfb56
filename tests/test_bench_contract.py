"""bench.py's reference arm runs on the host (no GPU): its JSON line carries
the contract's keys (impl, metric, value, unit, higher_is_better, config,
cpu_baseline, e2e with zero transfer bytes) on the same metric as the device
line.  A 1-ply C1 sample keeps it to a few seconds."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle.checkers import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--cpu-sample-plies", "1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "assembled stiffness nnz/s (FP64 CSR)" and line["unit"] == "nnz/s"
    assert line["higher_is_better"] is True and line["value"] > 0
    assert line["config"]["workload"] == "C1"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0

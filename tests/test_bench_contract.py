"""bench.py's reference arm runs on the host: its JSON line must carry the
contract's keys (impl, metric/unit/higher_is_better of our arm, cpu_baseline,
e2e with zero transfer bytes)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference"
    assert d["metric"] == "fwd+bwd Mpixels/s" and d["unit"] == "Mpx/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["warmup"] >= 3 and d["steps"] == 1
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("c1")
    # whole views timed (no extrapolation): steps x ms_per_step is real time
    assert "whole view" in d["step"] and cb["cpu"] and cb["logical_cores"] >= 1
    assert d["views"][0]["seconds"] * 1e3 == d["ms_per_step"]

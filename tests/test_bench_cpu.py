"""The bench's reference arm runs on the host alone (no GPU): its JSON line must
follow the driver contract (impl, metric/unit, cpu_baseline, e2e with zero copy
bytes) for the forward and the backward pass."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [[], ["--pass", "backward"]])
def test_reference_arm_json_line(extra):
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        pytest.skip("oracle not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "2", "--warmup", "0", *extra],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "useful GMAC/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["steps"] == 2
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert ("backward" in line["metric"]) == bool(extra)
    if oracle.ref_available():
        assert line["cpu_baseline"]["kind"] == "reference"

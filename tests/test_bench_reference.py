"""bench.py's reference arm (`--impl reference`): the reference's own CPU
path (oracle/_ref) on bounded layer-slice steps, one JSON line with the
contract's keys, and the product package never imported on that path."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "libnestopt_ref.so")

SCRIPT = r"""
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"]
runpy.run_path("bench.py", run_name="__main__")
assert not any(m.startswith("paper_2102_06599_b200") for m in sys.modules), "product imported"
"""


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")
def test_reference_arm_line_and_isolation():
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["value"] > 0
    assert d["unit"] == "candidates/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and "layer slices" in d["cpu_baseline"]["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]

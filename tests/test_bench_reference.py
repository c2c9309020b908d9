"""bench.py --impl reference (the oracle arm of this tier) runs on the host and prints the contract's
JSON line (no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "s/system" and line["higher_is_better"] is False
    assert line["value"] > 0 and line["steps"] == 2 and line["warmup"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == os.cpu_count() == cb["online_cores"] and cb["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert len(line["config"]["iterations"]) == 2      # the timed systems 2..3 (system 1 untimed)

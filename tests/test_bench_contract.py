"""CPU: the bench's reference arm (`bench.py --impl reference`) runs the
reference library (oracle/_ref, else the port) on a bounded sample and prints
one JSON line with the driver's contract keys."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--mb", "0.4",
                        "--workers", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "MB/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert "workload" in line["config"]
    assert "extrapolated" in line["config"]["same_config"]
    assert line["extrapolation"]["W"] == 2 and line["extrapolation"]["model_steps"] > 0
    # the reference arm never maps the product library
    assert line["product_library_loaded"] is False

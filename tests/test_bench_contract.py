"""bench.py's reference arm (the CPU oracle, --impl reference) prints the contract's
JSON line; the native arm's argument parsing and box layout are exercised here too."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 2
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_weak_scaling_box_layout():
    import bench
    assert bench.box_dims(1) == [48, 48, 48]
    assert bench.box_dims(2) == [96, 48, 48]
    assert bench.box_dims(4) == [96, 96, 48]
    assert bench.box_dims(8) == [96, 96, 96]
    assert bench.box_dims(8, 110) == [220, 220, 220]

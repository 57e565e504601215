"""CPU: bench.py's reference arm at a tiny size — the JSON line the driver
reads (metric, unit, steps, the e2e and cpu_baseline objects) and the config
dict, which must be the B200 arm's exactly (bench.config_dict) so the two
arms are compared on the same config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_shape_and_config():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (reference build) not present")
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--layers", "2", "--prompt", "1024", "--prefix", "512",
           "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    sys.path.insert(0, ROOT)
    import bench
    args = bench.parse_args_list(["--layers", "2", "--prompt", "1024", "--prefix", "512"])
    assert line["config"] == bench.config_dict(args, 1)
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == "GB/s"
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is True
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert "all 2 layers" in cb["sample"]

"""bench.py's reference arm (the reference's own CPU step, oracle/_ref) runs on
CPU: one JSON line with the contract's keys. The GPU arm is exercised on the
B200 by the driver; here only its reference leg and argument handling."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["workload"].startswith("cfg2")
    sys.path.insert(0, ROOT)
    import bench
    # both arms print the same config object (the driver compares them)
    assert line["config"] == json.loads(json.dumps(bench.workload_config("cfg2", 1)))


@pytest.mark.parametrize("wl", ["cfg3", "cfg4"])
def test_reference_arm_other_workloads(wl):
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", wl,
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["config"]["workload"].startswith(wl) and line["value"] > 0
    assert line["scaling"] == "strong"

"""The device's log for the beam score (csrc/glibc_log_impl.h, bit-exact
glibc log) checked on the CPU: the same restatement compiled with explicit
FMAs against the host libm's log() on every positive float <= 1 (the domain
of log((double) p)) and a sweep of doubles, and the committed constants
against this libm (scripts/gen_glibc_log_data.py --check). The reference
scores cum + log(p) with this libm (src/beam_decoder.cpp's expansion)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1806_00588_b200", "csrc")


def test_log_constants_match_libm():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gen_glibc_log_data.py"),
                        "--check"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_restated_log_equals_libm_on_every_float(tmp_path):
    exe = tmp_path / "glibc_log_check"
    cc = subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-I" + CSRC,
                         os.path.join(ROOT, "tests", "glibc_log_check.c"), "-o", str(exe), "-lm"],
                        capture_output=True, text=True)
    if cc.returncode != 0:
        pytest.fail(cc.stderr)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "floats 1065353217 mismatches 0" in r.stdout, r.stdout

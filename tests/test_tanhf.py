"""The device recurrence's tanhf (paper_1806_00588_b200/csrc/glibc_tanhf.cuh)
restates glibc's single-precision tanhf/expm1f, which the reference calls
through std::tanh(float) (src/model_provider.cpp:99). Here the same source is
compiled for the host with -ffp-contract=off and compared with libm's tanhf on
every 32-bit pattern (a few seconds on 8 cores)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tanhf_bin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("tanhf") / "tanhf_ex")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17",
                    "-I" + os.path.join(ROOT, "paper_1806_00588_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "tanhf_exhaustive.cpp"),
                    "-o", out, "-lpthread"], check=True)
    return out


def test_tanhf_all_floats_match_libm(tanhf_bin):
    r = subprocess.run([tanhf_bin, "0", str(1 << 32)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout
    assert "mismatches 0" in r.stdout

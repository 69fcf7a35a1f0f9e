"""WTAIDX1 / WTAEMB1 file interop between the unmodified reference and our
drop-in (oracle/ref_shim.cpp built against each; ours in a process that never
loads the reference): for the same seeded model and index both write
byte-identical files, and each reads the other's file back into identical
tables and embeddings (src/band_index.cpp:198-289,
src/model_provider.cpp:116-154)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "refsuite", "_build", "libdropin_shim.so")

OURS = """
import sys; sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np
from oracle.oracle import Reference
from dropin_api_cases import write_files, read_files
R = Reference({shim!r})
write_files(R, {d!r}, "ours")
np.savez({out!r}, **read_files(R, {d!r}, "ref"))
maps = open("/proc/self/maps").read()
assert "libref_lshbeam" not in maps and "liblshbeam.so" in maps
"""


def test_files_interchange(tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from dropin_api_cases import read_files, write_files
    from oracle.oracle import Reference
    if not (Reference.available() and os.path.exists(SHIM)):
        pytest.skip("reference or drop-in shim not built")
    d = str(tmp_path)
    ref = Reference()
    write_files(ref, d, "ref")
    out = str(tmp_path / "ours_read.npz")
    r = subprocess.run([sys.executable, "-c", OURS.format(root=ROOT, tests=os.path.join(ROOT, "tests"),
                                                          shim=SHIM, d=d, out=out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    for ext in ("idx", "emb"):  # byte-identical files
        with open(os.path.join(d, f"ref.{ext}"), "rb") as a, open(os.path.join(d, f"ours.{ext}"), "rb") as b:
            assert a.read() == b.read(), ext
    ours_read_ref = np.load(out)            # our library reading the reference's files
    ref_read_ours = read_files(ref, d, "ours")  # the reference reading ours
    ref_read_ref = read_files(ref, d, "ref")
    for k, v in ref_read_ref.items():
        assert ours_read_ref[k].tobytes() == v.tobytes(), k
        assert ref_read_ours[k].tobytes() == v.tobytes(), k

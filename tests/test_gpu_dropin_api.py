"""Drop-in conformance of the reference's public C++ API (include/lshbeam):
the same seeded calls (tests/dropin_api_cases.py: seeds, WTA permutations and
hashing incl. K=512, band packing, the band index and its cuckoo tables, hit
lookup, threshold selection, top-frequent merge, gather, logits, softmax,
beam expansion with frozen hypotheses, exact top-B, the synthetic model and
its recurrence, build_lsh_index over embeddings, one kLsh / kFull step) go
through the C wrapper oracle/ref_shim.cpp built once against the unmodified
reference (oracle/_ref) and once against our liblshbeam.so
(tests/refsuite/_build/libdropin_shim.so); every array must be identical, bit
for bit. Ours runs in a process that never loads the reference library."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "refsuite", "_build", "libdropin_shim.so")


def test_public_api_equals_reference(tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from dropin_api_cases import run_all
    from oracle.oracle import Reference
    if not (Reference.available() and os.path.exists(SHIM)):
        pytest.skip("reference or drop-in shim not built")
    want = run_all(Reference())
    out = tmp_path / "ours.npz"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dropin_api_cases.py"), SHIM,
                        str(out), ROOT], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    got = np.load(out)
    assert sorted(got.files) == sorted(want)
    bad = [k for k in want
           if got[k].dtype != want[k].dtype or got[k].shape != want[k].shape
           or got[k].tobytes() != want[k].tobytes()]
    assert not bad, bad


MUTATE = """
import sys; sys.path.insert(0, {root!r})
import numpy as np
from oracle.oracle import Reference
R = Reference({shim!r})
E = np.random.default_rng(0).standard_normal((2000, 1000)).astype(np.float32)
a = R.gather(E, [5])
E[5, 3] += 1.0  # an element the sampled content fingerprint does not read
b = R.gather(E, [5])
assert a[0, 3] != b[0, 3] and b[0, 3] == E[5, 3], (a[0, 3], b[0, 3], E[5, 3])
"""


def test_no_cache_sees_in_place_edits():
    """LSB_DROPIN_NO_CACHE=1: a large matrix edited in place
    between calls is re-read, as the reference reads host memory each call."""
    if not os.path.exists(SHIM):
        pytest.skip("drop-in shim not built")
    r = subprocess.run([sys.executable, "-c", MUTATE.format(root=ROOT, shim=SHIM)],
                       env={**os.environ, "LSB_DROPIN_NO_CACHE": "1"}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]

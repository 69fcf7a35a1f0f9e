#!/usr/bin/env python
"""Wide fuzz of the reference's public C++ API: random shapes and values
(ties, zeros, specials, frozen hypotheses) through oracle/ref_shim.cpp built
against the unmodified reference and against the drop-in. Ours runs in a
subprocess that never loads the reference. GPU box:

  python scripts/dropin_api_fuzz.py [cases]
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHIM = os.path.join(ROOT, "tests", "refsuite", "_build", "libdropin_shim.so")


def run_case(R, seed):
    rng = np.random.default_rng(seed)
    out = {}

    def rec(name, f, *a):
        try:
            r = f(*a)
        except Exception as e:  # noqa: BLE001
            out[name + "_err"] = np.array([type(e).__name__ == "ValueError"], np.int8)
            return None
        if isinstance(r, tuple):
            for i, x in enumerate(r):
                out[f"{name}_{i}"] = np.asarray(x)
        else:
            out[name] = np.asarray(r)
        return r

    d = int(rng.integers(1, 300)); K = int(rng.integers(1, 40)); u = int(rng.integers(1, 5))
    W = int(rng.integers(1, 60))
    M = rng.standard_normal((int(rng.integers(1, 40)), d)).astype(np.float32)
    if rng.random() < 0.5:
        M = np.round(M).astype(np.float32)  # many ties
    rec("hash", R.hash_matrix, M, K, u, W, R.mix_seed(seed, 1))
    V = int(rng.integers(1, 4000)); Wb = int(rng.integers(1, 20))
    codes = rng.integers(0, int(rng.choice([2, 16, 1000, 2**20])), (V, Wb)).astype(np.uint32)
    try:
        b = R.band_index_build(codes, seed)
        out["bt_word_ids"], out["bt_lg"], out["bt_mul"], out["bt_slots"] = b.word_ids, b.lg, b.mul, b.slots
    except Exception:  # noqa: BLE001
        out["bt_err"] = np.array([1], np.int8)
    q = rng.integers(0, 16, (int(rng.integers(1, 8)), Wb)).astype(np.uint32)
    rec("hits", R.lookup_hits_codes, codes, seed, q)
    n = int(rng.integers(1, 3000))
    L = rng.integers(0, int(rng.integers(1, 6)), (int(rng.integers(1, 13)), n)).astype(np.int32)
    t = int(rng.integers(0, 6))
    sel = rec("select", R.select_candidates, L, t)
    if sel is not None:
        T = int(rng.integers(0, n + 1))
        sp = list(rng.integers(0, n, int(rng.integers(0, 4))))
        rec("merge", R.merge_top_frequent, sel[0], sel[1], T, sp, n)
    rows, m = int(rng.integers(1, 13)), int(rng.integers(1, 600))
    logits = rng.standard_normal((rows, m)).astype(np.float32) * float(rng.choice([0.1, 3, 30]))
    if rng.random() < 0.4:
        logits = np.round(logits)
    probs = rec("softmax", R.softmax_rows, logits)
    if probs is not None:
        B = int(rng.integers(1, 60))
        frozen = tuple((float(-rng.random() * 5), int(rng.integers(0, 100)))
                       for _ in range(int(rng.integers(0, 4))))
        cum = np.round(-rng.random(rows) * 4, int(rng.integers(0, 3)))
        rec("expand", R.expand_beams, probs, cum, np.arange(rows, dtype=np.uint32), frozen, B)
    rec("topb", R.exact_topb_logits, logits, int(rng.integers(1, min(m, 50) + 1)))
    return out


OURS = """
import sys; sys.path.insert(0, {root!r}); sys.path.insert(0, {scripts!r})
import numpy as np
from oracle.oracle import Reference
from dropin_api_fuzz import run_case
R = Reference({shim!r})
for s in range({n}):
    np.savez({d!r} + "/%d.npz" % s, **run_case(R, s))
maps = open("/proc/self/maps").read()
assert "libref_lshbeam" not in maps and "liblshbeam.so" in maps
"""

if __name__ == "__main__":
    from oracle.oracle import Reference
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    d = tempfile.mkdtemp()
    r = subprocess.run([sys.executable, "-c", OURS.format(root=ROOT, scripts=os.path.join(ROOT, "scripts"),
                                                          shim=SHIM, n=n, d=d)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    R = Reference()
    bad = 0
    for s in range(n):
        want = run_case(R, s)
        got = dict(np.load(f"{d}/{s}.npz"))
        keys = set(want) | set(got)
        diff = [k for k in sorted(keys) if k not in want or k not in got
                or want[k].tobytes() != got[k].tobytes() or want[k].shape != got[k].shape]
        if diff:
            bad += 1
            print("case", s, "differs:", diff)
    print(f"cases {n}, mismatching {bad}")

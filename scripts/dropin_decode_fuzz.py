#!/usr/bin/env python
"""Wide decode() fuzz: 60 random configurations (V up to 20k, odd d up to 1003,
K up to 64, u up to 4, W up to 300, beams up to 59, T up to V, t up to W, every
mode, with_oracle on/off, raised EOS bias) through the unmodified reference and
the drop-in (tests/test_gpu_dropin_decode.py helpers). Prints the counts of
identical / rejected-by-both / mismatching runs. GPU box:

  python scripts/dropin_decode_fuzz.py
"""
import sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from oracle.oracle import Reference
from test_gpu_dropin_decode import run_decode, ours_decode
ref = Reference().lib
rng = np.random.default_rng(99)
bad = 0; n_ok = 0; n_rej = 0
for i in range(60):
    V = int(rng.integers(200, 20000)); d = int(rng.choice([3, 17, 64, 129, 300, 1003]))
    K = min(int(rng.choice([2, 3, 8, 16, 32, 64])), d); u = int(rng.integers(1, 5)); W = int(rng.integers(1, 300))
    beam = int(rng.integers(1, 60)); T = int(rng.choice([0, int(rng.integers(1, V)), V]))
    t = int(rng.integers(0, W + 1)); mode = int(rng.integers(0, 3))
    args = (V, d, int(rng.integers(0, 10**6)), float(rng.choice([0.0, 2.0, 8.0])), K, u, W, beam, T, t,
            int(rng.integers(1, 12)), mode, V - 1, int(rng.integers(0, 2)), float(rng.choice([0.0, 6.0])))
    want = run_decode(ref, *args)
    got = ours_decode(args)
    if "rejected" in want:
        n_rej += 1
        if "rejected" not in got: bad += 1; print("MISMATCH (ours accepted)", args)
        continue
    if got != want:
        bad += 1
        diff = [k for k in want if got.get(k) != want[k]]
        print("MISMATCH", args, diff)
    else:
        n_ok += 1
print("ok", n_ok, "rejected", n_rej, "bad", bad)

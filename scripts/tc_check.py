"""Quick numeric check of the tcgen05 3xTF32 logits path vs float64 (GPU)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import FAST, PARITY, Context  # noqa: E402

ctx = Context(0)
rng = np.random.default_rng(0)
for rows, n, d in [(64, 128, 32), (256, 1000, 1000), (768, 1000, 1000), (100, 300, 64)]:
    H = rng.standard_normal((rows, d)).astype(np.float32)
    E = rng.standard_normal((n, d)).astype(np.float32)
    want = H.astype(np.float64) @ E.astype(np.float64).T
    got = ctx.compute_logits(H, E, FAST)
    err = np.abs(got - want) / (1 + np.abs(want))
    par = ctx.compute_logits(H, E, PARITY)
    perr = np.abs(par - want) / (1 + np.abs(want))
    print(f"rows={rows} n={n} d={d} swap={os.environ.get('LSB_TC_SWAP', '0')} "
          f"fast max rel err {err.max():.3e} (parity {perr.max():.3e}) "
          f"nan={np.isnan(got).sum()}", flush=True)

#!/usr/bin/env python
"""Index build time (lsb_index_build = K1 over E + band sort + cuckoo tables)
at the cfg-2 / cfg-4 / operating-point shapes, after one warm-up build (module
loading), host wall time of the synchronous call.

  python scripts/index_probe.py
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402

ctx = Context(0, torch.cuda.Stream().cuda_stream)
for V, d, K, u, W in [(40000, 1000, 8, 3, 16), (200000, 1024, 8, 3, 16), (50000, 256, 16, 3, 500)]:
    E = torch.randn(V, d, generator=torch.Generator().manual_seed(7)).cuda()
    m = Model(ctx, None, device_ptrs=(E.data_ptr(), None, V, d))
    for par in (False, True):
        ctx.set_parallel_cuckoo(par)
        Index(ctx, m, K=K, u=u, W=W, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2)).close()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            ix = Index(ctx, m, K=K, u=u, W=W, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
            ts.append((time.perf_counter() - t0) * 1e3)
            ix.close()
        print(f"V={V} d={d} K={K} u={u} W={W} cuckoo={'parallel' if par else 'reference'}: "
              f"index build {min(ts):.2f} ms (median {sorted(ts)[2]:.2f})", flush=True)
    ctx.set_parallel_cuckoo(False)
    m.close()

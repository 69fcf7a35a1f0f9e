#!/usr/bin/env python
"""The fused small-batch step (k_step_fused.cu) against the separate kernels:
bit-exact outputs over several steps, then device time per step, per shape.

  python scripts/fused_probe.py [S:B ...]      (default 1:12 2:12 4:12 1:8 2:8)

LSB_FUSED is read when a batch takes its first step, so both paths run in
this one process.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import FAST, PARITY, Batch, Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import state, time_steps, world  # noqa: E402

shapes = [tuple(map(int, a.split(":"))) for a in sys.argv[1:]] or [(1, 12), (2, 12), (4, 12),
                                                                  (1, 8), (2, 8)]
V, d, K, u, W, T, t = 40000, 1000, 8, 3, 16, 1000, 2
dev = torch.device("cuda", 0)
STREAM = torch.cuda.Stream()  # graph capture needs a created stream
ctx = Context(0, STREAM.cuda_stream)
m = Model(ctx, world(V, d).numpy())
idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))


def run(S, B, mode, fused, steps):
    os.environ["LSB_FUSED"] = "1" if fused else "0"
    H, sc, fin, nh = state(S, B, d, 8)
    b = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=[V - 1], mode=mode)
    ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
    nc = torch.zeros(S, dtype=torch.int32, device=dev)
    ho = torch.empty(S, B, d, device=dev)
    torch.cuda.synchronize()
    stride = S * B * d * 4
    outs = []
    for k in range(4):
        b.step(H.data_ptr() + k * stride, sc, fin, nh, ch, nc, ho)
        ctx.sync()
        outs.append((ch.clone(), nc.clone(), ho.clone(), [b.candidates(s)[0].copy() for s in range(S)]
                     + [b.query_codes(s, W) for s in range(S)]))
    ms = time_steps(ctx, lambda k: b.step(H.data_ptr() + k * stride, sc, fin, nh, ch, nc, ho), 8,
                    steps=steps)
    # the same step replayed from a CUDA graph (no host launch cost)
    b.graph_capture(H.data_ptr(), sc, fin, nh, ch, nc, ho)
    msg = time_steps(ctx, lambda k: b.graph_launch(), 8, steps=steps)
    b.close()
    return outs, (ms, msg)


ok = True
for S, B in shapes:
    for mode in (PARITY, FAST):
        o0, ms0 = run(S, B, mode, False, 300)
        o1, ms1 = run(S, B, mode, True, 300)
        same = all(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
                   and all((x == y).all() for x, y in zip(a[3], b[3])) for a, b in zip(o0, o1))
        ok &= same
        print(f"S={S} B={B} {'parity' if mode == PARITY else 'fast  '}: separate {ms0[0] * 1e3:.1f} us "
              f"(graph {ms0[1] * 1e3:.1f}), fused {ms1[0] * 1e3:.1f} us (graph {ms1[1] * 1e3:.1f}), "
              f"bit-exact={same}", flush=True)
os.environ.pop("LSB_FUSED", None)
sys.exit(0 if ok else 1)

#!/usr/bin/env python
"""Per-stage device times (every step profiled) for one config.

  python scripts/stage_probe.py S B [parity|fast] [V d K u W T t]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import FAST, PARITY, Batch, Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import state, time_steps, world  # noqa: E402

S, B = int(sys.argv[1]), int(sys.argv[2])
mode = FAST if len(sys.argv) > 3 and sys.argv[3] == "fast" else PARITY
V, d, K, u, W, T, t = (list(map(int, sys.argv[4:11])) if len(sys.argv) > 10
                       else [40000, 1000, 8, 3, 16, 1000, 2])
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
m = Model(ctx, world(V, d).numpy())
idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
H, sc, fin, nh = state(S, B, d, 8)
dev = torch.device("cuda", 0)
ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
nc = torch.zeros(S, dtype=torch.int32, device=dev)
ho = torch.empty(S, B, d, device=dev)
stride = S * B * d * 4
names = ("probe", "compact", "logits", "softmax", "expand")
for full in (False, True):
    b = Batch(ctx, m, None if full else idx, S=S, B=B, T=0 if full else T, t=0 if full else t,
              specials=[V - 1], mode=mode, full_vocab=full)
    step = lambda k: b.step(H.data_ptr() + k * stride, sc, fin, nh, ch, nc, ho)  # noqa: E731
    ms = time_steps(ctx, step, 8, steps=100)
    b.profile(True, every=1)
    time_steps(ctx, step, 8, steps=30)
    st = b.stage_ms()
    nv = V if full else float(np.mean([len(b.candidates(s)[0]) for s in range(min(S, 8))]))
    print(f"{'full' if full else 'lsh '} S={S} B={B} V={V} d={d} K={K} u={u} W={W} T={T} t={t} "
          f"mode={'fast' if mode == FAST else 'parity'} n={nv:.0f}: {ms * 1e3:.1f} us/step; stages us: "
          + " ".join(f"{nm}={v * 1e3:.1f}" for nm, v in zip(names, st)), flush=True)
    b.close()

#!/usr/bin/env python
"""Per-stage device times (every step profiled) for one config.

  python scripts/stage_probe.py S B [mode]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import FAST, PARITY, Batch, Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import state, time_steps, world  # noqa: E402

S, B = int(sys.argv[1]), int(sys.argv[2])
mode = FAST if len(sys.argv) > 3 and sys.argv[3] == "fast" else PARITY
V, d = 40000, 1000
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
m = Model(ctx, world(V, d).numpy())
idx = Index(ctx, m, K=8, u=3, W=16, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
H, sc, fin, nh = state(S, B, d, 8)
b = Batch(ctx, m, idx, S=S, B=B, T=1000, t=2, specials=[V - 1], mode=mode)
dev = torch.device("cuda", 0)
ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
nc = torch.zeros(S, dtype=torch.int32, device=dev)
ho = torch.empty(S, B, d, device=dev)
stride = S * B * d * 4
step = lambda k: b.step(H.data_ptr() + k * stride, sc, fin, nh, ch, nc, ho)  # noqa: E731
ms = time_steps(ctx, step, 8, steps=200)
b.profile(True, every=1)
time_steps(ctx, step, 8, steps=50)
st = b.stage_ms()
print(f"S={S} B={B} mode={'fast' if mode == FAST else 'parity'}: {ms * 1e3:.1f} us/step (PDL, no events); "
      "stages us (events between kernels): "
      + " ".join(f"{n}={v * 1e3:.1f}" for n, v in zip(("probe", "compact", "logits", "softmax", "expand"), st)))

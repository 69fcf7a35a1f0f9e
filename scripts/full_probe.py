#!/usr/bin/env python
"""A few full-vocabulary steps (for ncu captures of the kFull kernels).

  python scripts/full_probe.py S B [parity|fast] [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import FAST, PARITY, Batch, Context, Model  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import state, time_steps, world  # noqa: E402

S, B = int(sys.argv[1]), int(sys.argv[2])
mode = FAST if len(sys.argv) > 3 and sys.argv[3] == "fast" else PARITY
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
V, d = 40000, 1000
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
m = Model(ctx, world(V, d).numpy())
H, sc, fin, nh = state(S, B, d, 2)
dev = torch.device("cuda", 0)
ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
nc = torch.zeros(S, dtype=torch.int32, device=dev)
ho = torch.empty(S, B, d, device=dev)
stride = S * B * d * 4
b = Batch(ctx, m, None, S=S, B=B, T=0, t=0, specials=[V - 1], mode=mode, full_vocab=True)
step = lambda k: b.step(H.data_ptr() + k * stride, sc, fin, nh, ch, nc, ho)  # noqa: E731
ms = time_steps(ctx, step, 2, steps=steps, warmup=1)
print(f"full S={S} B={B}: {ms * 1e3:.1f} us/step")

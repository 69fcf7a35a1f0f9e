#!/usr/bin/env python
"""Throughput of one S-sentence batch vs two S/2 batches on two streams
(same total sentences), PARITY, cfg 2 shapes. Device-timed on stream 0 with
stream 1 joined."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1806_00588_b200 import PARITY, Batch, Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402
from bench_configs import state, world  # noqa: E402

V, d, B = 40000, 1000, 12
S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda", 0)
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
ctx0 = Context(0, s0.cuda_stream)
ctx1 = Context(0, s1.cuda_stream)
m = Model(ctx0, world(V, d).numpy())
idx = Index(ctx0, m, K=8, u=3, W=16, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
ctx0.sync()


def mk(ctx, S_):
    H, sc, fin, nh = state(S_, B, d, 8)
    b = Batch(ctx, m, idx, S=S_, B=B, T=1000, t=2, specials=[V - 1], mode=PARITY)
    ch = torch.zeros(S_ * B * 24, dtype=torch.uint8, device=dev)
    nc = torch.zeros(S_, dtype=torch.int32, device=dev)
    ho = torch.empty(S_, B, d, device=dev)
    stride = S_ * B * d * 4
    return lambda k: b.step(H.data_ptr() + (k % 8) * stride, sc, fin, nh, ch, nc, ho)


def run(steps, fns, streams, n=200):
    for k in range(5):
        for f in fns:
            f(k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(streams[0])
    for st in streams[1:]:
        st.wait_event(a)
    for k in range(n):
        for f in fns:
            f(k)
    for st in streams[1:]:
        e = torch.cuda.Event()
        e.record(st)
        streams[0].wait_event(e)
    b.record(streams[0])
    b.synchronize()
    return a.elapsed_time(b) / n


one = mk(ctx0, S)
t1 = run(200, [one], [s0])
h0, h1 = mk(ctx0, S // 2), mk(ctx1, S // 2)
t2 = run(200, [h0, h1], [s0, s1])
print(f"S={S}: one batch {t1 * 1e3:.1f} us/step ({S * 1e3 / t1:.0f} sent-steps/s); "
      f"two S/2 batches on two streams {t2 * 1e3:.1f} us/step ({S * 1e3 / t2:.0f})")

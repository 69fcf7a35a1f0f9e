#!/usr/bin/env python
"""Does a stream operation between consecutive steps (what the pipelined
host-buffer API inserts: an event wait for the upload, an event record for
the read-back) cost the step its programmatic-dependent-launch overlap?

  python scripts/pdl_break_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import Batch, Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import state, world  # noqa: E402

S, B, V, d = 64, 12, 40000, 1000
st = torch.cuda.Stream()
ctx = Context(0, st.cuda_stream)
m = Model(ctx, world(V, d).numpy())
idx = Index(ctx, m, K=8, u=3, W=16, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
H, sc, fin, nh = state(S, B, d, 8)
dev = torch.device("cuda", 0)
ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
nc = torch.zeros(S, dtype=torch.int32, device=dev)
ho = torch.empty(S, B, d, device=dev)
b = Batch(ctx, m, idx, S=S, B=B, T=1000, t=2, specials=[V - 1])
stride = S * B * d * 4
other = torch.cuda.Stream()
ev_o = torch.cuda.Event()
ev_o.record(other)
for variant in ("plain", "event_record", "wait_completed_event", "both"):
    def one(k):
        if variant in ("wait_completed_event", "both"):
            st.wait_event(ev_o)
        b.step(H.data_ptr() + (k % 8) * stride, sc, fin, nh, ch, nc, ho)
        if variant in ("event_record", "both"):
            torch.cuda.Event().record(st)
    for k in range(10):
        one(k)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for k in range(300):
        one(k)
    e.record(st)
    e.synchronize()
    print(f"{variant:22s} {a.elapsed_time(e) / 300 * 1e3:.1f} us/step", flush=True)

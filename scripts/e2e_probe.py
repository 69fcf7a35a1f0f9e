"""Where does the e2e time go? Host issue rate of the pipelined API vs device time."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00588_b200 import Batch, Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402

V, d, S, B = 40000, 1000, 64, 12
g = torch.Generator().manual_seed(7)
E = torch.randn(V, d, generator=g)
st = torch.cuda.Stream()
ctx = Context(0, st.cuda_stream)
m = Model(ctx, E.numpy())
idx = Index(ctx, m, K=8, u=3, W=16, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
b = Batch(ctx, m, idx, S=S, B=B, T=1000, t=2, specials=[V - 1])
H = torch.randn(8, S, B, d, generator=g).pin_memory()
sc = (-torch.rand(S, B, generator=g, dtype=torch.float64) * 4).pin_memory()
fin = torch.zeros(S, B, dtype=torch.uint8).pin_memory()
nh = torch.full((S,), B, dtype=torch.int32).pin_memory()
ch = torch.zeros(S * B * 24, dtype=torch.uint8).pin_memory()
nc = torch.zeros(S, dtype=torch.int32).pin_memory()
chp, ncp = C.c_void_p(ch.data_ptr()), C.c_void_p(nc.data_ptr())
step_bytes = S * B * d * 4
for k in range(10):
    b.step_host_async(H.data_ptr() + (k % 8) * step_bytes, sc.data_ptr(), fin.data_ptr(),
                      nh.data_ptr(), chp, ncp)
b.wait()
N = 200
t0 = time.perf_counter()
for k in range(N):
    b.step_host_async(H.data_ptr() + (k % 8) * step_bytes, sc.data_ptr(), fin.data_ptr(),
                      nh.data_ptr(), chp, ncp)
t1 = time.perf_counter()
b.wait()
t2 = time.perf_counter()
print(f"host issue {1e6 * (t1 - t0) / N:.1f} us/step, total {1e6 * (t2 - t0) / N:.1f} us/step")
# H2D alone
dst = torch.empty(S, B, d, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(N):
    dst.copy_(H[k % 8], non_blocking=True)
torch.cuda.synchronize()
print(f"H2D 3 MB alone: {1e6 * (time.perf_counter() - t0) / N:.1f} us/step")

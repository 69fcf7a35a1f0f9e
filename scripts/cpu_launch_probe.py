import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/scripts')
import torch
from paper_1806_00588_b200 import PARITY, Batch, Context, Index, Model
from paper_1806_00588_b200.seeds import mix_seed
from bench_configs import state, world
S, B, V, d = 1, 12, 40000, 1000
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
m = Model(ctx, world(V, d).numpy())
idx = Index(ctx, m, K=8, u=3, W=16, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
H, sc, fin, nh = state(S, B, d, 8)
dev = torch.device('cuda', 0)
ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev); nc = torch.zeros(S, dtype=torch.int32, device=dev)
ho = torch.empty(S, B, d, device=dev)
b = Batch(ctx, m, idx, S=S, B=B, T=1000, t=2, specials=[V - 1], mode=PARITY)
stride = S * B * d * 4
for k in range(50): b.step(H.data_ptr() + (k % 8) * stride, sc, fin, nh, ch, nc, ho)
ctx.sync()
N = 2000
t0 = time.perf_counter()
for k in range(N): b.step(H.data_ptr() + (k % 8) * stride, sc, fin, nh, ch, nc, ho)
t1 = time.perf_counter()
ctx.sync()
t2 = time.perf_counter()
print(f"cpu issue {1e6*(t1-t0)/N:.1f} us/step; wall incl. drain {1e6*(t2-t0)/N:.1f} us/step")
# raw C call with prebuilt structs: isolates the library's own host cost
import ctypes as C
from paper_1806_00588_b200 import _native as Nn
outs = Nn.lsb_out_dev(ch.data_ptr(), nc.data_ptr(), ho.data_ptr())
ins = [Nn.lsb_state_dev(H.data_ptr() + (k % 8) * stride, sc.data_ptr(), fin.data_ptr(), nh.data_ptr())
       for k in range(8)]
f = b.lib.lsb_step
ctx.sync()
t0 = time.perf_counter()
for k in range(N): f(b.h, C.byref(ins[k % 8]), C.byref(outs))
t1 = time.perf_counter()
ctx.sync()
t2 = time.perf_counter()
print(f"raw C call: cpu issue {1e6*(t1-t0)/N:.1f} us/step; wall {1e6*(t2-t0)/N:.1f} us/step")
os.environ["LSB_NO_PDL"] = "1"
# short bursts (below the launch-queue depth) measure the host cost alone
for n in (20, 50, 100):
    ctx.sync()
    t0 = time.perf_counter()
    for k in range(n): f(b.h, C.byref(ins[k % 8]), C.byref(outs))
    t1 = time.perf_counter()
    ctx.sync()
    t2 = time.perf_counter()
    print(f"burst {n}: host {1e6*(t1-t0)/n:.1f} us/step; wall {1e6*(t2-t0)/n:.1f} us/step")

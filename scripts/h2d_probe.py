import torch, time
x = torch.empty(64*12*1000, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
s = torch.cuda.Stream()
for n in (3_072_000,):
    for _ in range(5): y.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100): y.copy_(x, non_blocking=True)
    b.record(); b.synchronize()
    ms = a.elapsed_time(b)/100
    print(f"H2D 3.07 MB pinned: {ms*1e3:.1f} us = {3.072e6/ms/1e6:.1f} GB/s")

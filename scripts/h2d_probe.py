#!/usr/bin/env python
"""Pinned H2D bandwidth for one 3 MB step input, re-copied from the same host
buffer vs cycled over n distinct host buffers (bench.py's e2e cycles 50)."""
import torch

step = 64 * 12 * 1000
y = torch.empty(step, dtype=torch.float32, device="cuda")
for n in (1, 8, 50):
    x = torch.empty(n, step, dtype=torch.float32).pin_memory()
    for k in range(5):
        y.copy_(x[k % n], non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(200):
        y.copy_(x[k % n], non_blocking=True)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 200
    print(f"H2D 3.07 MB pinned, {n:2d} distinct host buffers: {ms * 1e3:.1f} us = "
          f"{step * 4 / ms / 1e6:.1f} GB/s", flush=True)

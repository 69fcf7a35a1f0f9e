#!/usr/bin/env python
"""Pinned H2D time of one 3 MB step input: one copy vs the same bytes split
over k streams (copy engines), cycling over n distinct host buffers."""
import torch

step = 64 * 12 * 1000
y = torch.empty(step, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for n in (1, 50):
    x = torch.empty(n, step, dtype=torch.float32).pin_memory()
    for k_split in (1, 2, 4):
        chunk = (step + k_split - 1) // k_split

        def one(i):
            for j in range(k_split):
                s = streams[j]
                with torch.cuda.stream(s):
                    y[j * chunk:(j + 1) * chunk].copy_(x[i % n][j * chunk:(j + 1) * chunk],
                                                       non_blocking=True)
        for i in range(5):
            one(i)
        torch.cuda.synchronize()
        import time
        t0 = time.perf_counter()
        for i in range(200):
            one(i)
        torch.cuda.synchronize()
        us = (time.perf_counter() - t0) / 200 * 1e6
        print(f"{n:2d} host buffers, {k_split} streams: {us:.1f} us per 3.07 MB = "
              f"{step * 4 / us / 1e3:.1f} GB/s", flush=True)

#!/usr/bin/env python
"""Secondary measurements for the other BASELINE.json configs (the headline
line is bench.py, cfg 2). Prints one JSON object per config; results are
committed under profiles/. Synthetic inputs as in bench.py (torch.randn,
seed 7), device-timed with CUDA events on the step stream.

  cfg1  single sentence, one step, |V|=40k, d=1000, B=12 (latency)
  cfg3  large beam B=50, 256 sentences, |V|=40k, d=1000 (1 GPU share)
  cfg4  |V|=200k, d=1024, B=12, 64 sentences: unsharded, and the
        vocabulary-sharded protocol with G shards on one GPU
  cfg5  hash sweep K x W x T at u=3, t=2: mean |V_LSH|, recall@B vs the
        exact full-vocabulary top-B (lsb_exact_topb), steps/s

  python scripts/bench_configs.py [cfg1 cfg3 cfg4 cfg5]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1806_00588_b200 import FAST, PARITY, Batch, Context, Index, Model  # noqa: E402
from paper_1806_00588_b200.lshbeam import exact_topb  # noqa: E402
from paper_1806_00588_b200.seeds import mix_seed  # noqa: E402

DEV = torch.device("cuda", 0)


def world(V, d, seed=7):
    g = torch.Generator().manual_seed(seed)
    E = torch.randn(V, d, generator=g)
    return E


def state(S, B, d, n_inputs, seed=1000):
    g = torch.Generator().manual_seed(seed)
    H = torch.randn(n_inputs, S, B, d, generator=g).to(DEV)
    sc = (-torch.rand(S, B, generator=g, dtype=torch.float64) * 4).to(DEV)
    fin = torch.zeros(S, B, dtype=torch.uint8, device=DEV)
    nh = torch.full((S,), B, dtype=torch.int32, device=DEV)
    return H, sc, fin, nh


def time_steps(ctx, step, n_inputs, steps=50, warmup=3):
    for k in range(warmup):
        step(k % n_inputs)
    ctx.sync()
    # the context runs on torch's stream (handle 0 is mapped to the legacy
    # default stream, reported as 1)
    st = (torch.cuda.current_stream() if ctx.stream in (0, 1)
          else torch.cuda.ExternalStream(ctx.stream))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for k in range(steps):
        step(k % n_inputs)
    b.record(st)
    b.synchronize()
    ctx.sync()
    return a.elapsed_time(b) / steps


def run_batch(ctx, model, idx, S, B, d, T, t, V, mode, full=False, n_inputs=8, steps=50):
    H, sc, fin, nh = state(S, B, d, n_inputs)
    batch = Batch(ctx, model, idx, S=S, B=B, T=T, t=t, specials=[V - 1], mode=mode,
                  full_vocab=full)
    ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=DEV)
    nc = torch.zeros(S, dtype=torch.int32, device=DEV)
    ho = torch.empty(S, B, d, device=DEV)
    stride = S * B * d * 4
    base = H.data_ptr()
    ms = time_steps(ctx, lambda k: batch.step(base + k * stride, sc, fin, nh, ch, nc, ho),
                    n_inputs, steps)
    ncand = [len(batch.candidates(s)[0]) for s in range(min(S, 8))] if not full else [V]
    batch.close()
    return ms, float(np.mean(ncand))


def cfg1(ctx):
    V, d, B, S = 40000, 1000, 12, 1
    E = world(V, d)
    m = Model(ctx, E.numpy())
    idx = Index(ctx, m, K=8, u=3, W=16, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
    out = {"config": "cfg1: 1 sentence x B=12, |V|=40000, d=1000, K=8 u=3 W=16 T=1000 t=2"}
    for name, mode in (("parity", PARITY), ("fast", FAST)):
        ms, n = run_batch(ctx, m, idx, S, B, d, 1000, 2, V, mode)
        out[f"lsh_{name}"] = {"ms_per_step": round(ms, 5), "steps_per_s": round(1e3 / ms, 1),
                              "mean_vlsh": n}
    for name, mode in (("parity", PARITY), ("fast", FAST)):
        ms, _ = run_batch(ctx, m, None, S, B, d, 0, 0, V, mode, full=True, steps=20)
        out[f"full_vocab_{name}"] = {"ms_per_step": round(ms, 5), "steps_per_s": round(1e3 / ms, 1)}
    return out


def cfg3(ctx):
    V, d, B, S = 40000, 1000, 50, 256
    E = world(V, d)
    m = Model(ctx, E.numpy())
    idx = Index(ctx, m, K=8, u=3, W=16, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
    out = {"config": "cfg3: 256 sentences x B=50, |V|=40000, d=1000, K=8 u=3 W=16 T=1000 t=2 "
                     "(one GPU's share; sentence sharding has no data-path collective)"}
    for name, mode in (("parity", PARITY), ("fast", FAST)):
        ms, n = run_batch(ctx, m, idx, S, B, d, 1000, 2, V, mode, n_inputs=2, steps=10)
        out[f"lsh_{name}"] = {"ms_per_step": round(ms, 4),
                              "sentence_steps_per_s": round(S * 1e3 / ms, 1), "mean_vlsh": n}
    ms, _ = run_batch(ctx, m, None, S, B, d, 0, 0, V, FAST, full=True, n_inputs=2, steps=3)
    out["full_vocab_fast"] = {"ms_per_step": round(ms, 4),
                              "sentence_steps_per_s": round(S * 1e3 / ms, 1)}
    return out


def cfg4(ctx):
    from paper_1806_00588_b200.vocab_shard import VocabShard, local_sharded_step, shard_bounds
    V, d, B, S, T, t = 200000, 1024, 12, 64, 1000, 2
    E = world(V, d).to(DEV)
    bias = torch.zeros(V, device=DEV)
    out = {"config": "cfg4: 64 sentences x B=12, |V|=200000, d=1024, K=8 u=3 W=16 T=1000 t=2"}
    m = Model(ctx, None, device_ptrs=(E.data_ptr(), bias.data_ptr(), V, d))
    ps, isd = mix_seed(7, 1), mix_seed(7, 2)
    idx = Index(ctx, m, K=8, u=3, W=16, perm_seed=ps, index_seed=isd)
    ms, n = run_batch(ctx, m, idx, S, B, d, T, t, V, PARITY, n_inputs=4, steps=20)
    out["unsharded_parity"] = {"ms_per_step": round(ms, 4),
                               "sentence_steps_per_s": round(S * 1e3 / ms, 1), "mean_vlsh": n}
    idx.close()
    m.close()
    H, sc, fin, nh = state(S, B, d, 4)
    ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=DEV)
    nc = torch.zeros(S, dtype=torch.int32, device=DEV)
    ho = torch.empty(S, B, d, device=DEV)
    for G in (2, 4, 8):
        shards = []
        for g in range(G):
            v0, n_ = shard_bounds(V, G, g)
            shards.append(VocabShard(ctx, E[v0:v0 + n_].contiguous(), bias[v0:v0 + n_].contiguous(),
                                     v0, V, 8, 3, 16, ps, isd, S, B, T, t, [V - 1]))
        ms = time_steps(ctx, lambda k: local_sharded_step(shards, H[k], sc, fin, nh, ch, nc, ho),
                        4, steps=10)
        out[f"sharded_G{G}_one_gpu"] = {
            "ms_per_step_all_shards": round(ms, 4),
            "ms_per_step_per_shard": round(ms / G, 4),
            "note": "all G shards run back to back on one GPU; on G GPUs each rank runs one "
                    "shard plus two all-gathers of ~105 KB"}
        for s_ in shards:
            s_.close()
    return out


def cfg5(ctx):
    V, d, B, S = 40000, 1000, 12, 16
    E = world(V, d)
    m = Model(ctx, E.numpy())
    H, sc, fin, nh = state(S, B, d, 4)
    rows = []
    for K in (4, 8, 16):
        for W in (8, 16, 32):
            idx = Index(ctx, m, K=K, u=3, W=W, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
            for T in (0, 1000, 5000):
                for t in (1, 2, 3):
                    b = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=[V - 1], mode=PARITY)
                    ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=DEV)
                    nc = torch.zeros(S, dtype=torch.int32, device=DEV)
                    stride = S * B * d * 4
                    base = H.data_ptr()
                    ms = time_steps(ctx, lambda k: b.step(base + k * stride, sc, fin, nh, ch, nc),
                                    4, steps=10)
                    # recall@B of input 0's candidate sets vs the exact full top-B
                    b.step(base, sc, fin, nh, ch, nc)
                    ctx.sync()
                    ids_exact, _ = exact_topb(ctx, m, base, S * B, B, bias=False)
                    rec, nv = [], []
                    for s in range(S):
                        cands, _ = b.candidates(s)
                        nv.append(len(cands))
                        cs = set(cands.tolist())
                        for i in range(B):
                            rec.append(np.mean([int(x) in cs for x in ids_exact[s * B + i]]))
                    rows.append({"K": K, "u": 3, "W": W, "T": T, "t": t,
                                 "mean_vlsh": round(float(np.mean(nv)), 1),
                                 "recall_at_B": round(float(np.mean(rec)), 4),
                                 "sentence_steps_per_s": round(S * 1e3 / ms, 1)})
                    b.close()
            idx.close()
    return {"config": "cfg5: sweep K x W x T x t at u=3, 16 sentences x B=12, |V|=40000, d=1000 "
                      "(iid-random E/H: recall is near chance except through the top-T merge)",
            "rows": rows}


def main():
    which = sys.argv[1:] or ["cfg1", "cfg3", "cfg4", "cfg5"]
    ctx = Context(0, torch.cuda.current_stream().cuda_stream)
    for w in which:
        t0 = time.time()
        res = globals()[w](ctx)
        res["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

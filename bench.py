#!/usr/bin/env python
"""Benchmark of the per-step LSH beam-search hot path (BASELINE.json).

Workloads (--workload, default cfg2 = BASELINE configs[1]):
  cfg2  64 sentences x B=12 per GPU, |V|=40000, d=1000, WTA K=8 u=3 W=16,
        T=1000, t=2, specials {V-1}; sentence-sharded, weak scaling
  cfg3  B=50, 256 sentences in total split over the GPUs, |V|=40000,
        d=1000; sentence-sharded, strong scaling (configs[2])
  cfg4  |V|=200000, d=1024, B=12, 64 sentences; vocabulary-sharded over the
        GPUs with the NCCL top-B merge (configs[3]), strong scaling
One "step" = one pass of the fused hot path (hash, cuckoo lookup, candidate
union, reduced softmax, beam expansion + hidden reorder) over one batch.
Metric: decode steps/s = sentence-steps per second (softmax path + beam
expansion: the reference's StageTimes::softmax_path() + beam_expansion,
include/lshbeam/beam_decoder.hpp:66-73). Synthetic inputs (torch.randn,
seed 7) cycled; inputs exceed L2.

  python bench.py [--gpus N --steps K --warmup W] [--workload cfg2|cfg3|cfg4]
                  [--impl reference]

Multi-GPU: one process per GPU (torchrun); timing = max over ranks of the
device-timed region. The reference arm times the reference's own CPU
implementation (oracle/_ref, compiled from /root/reference's sources) on the
host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode steps/sec (softmax+beam expand) at |V|=40k,d=1000,B=12; recall@B vs full"
UNIT = "sentence-steps/s"

WORKLOADS = {
    "cfg2": dict(V=40000, d=1000, B=12, S=64, K=8, u=3, W=16, T=1000, t=2, seed=7, inputs=50,
                 scaling="weak",
                 desc="cfg2: batched decode step, 64 sentences x B=12 per GPU, |V|=40000, "
                      "d=1000, K=8 u=3 W=16, T=1000, t=2"),
    "cfg3": dict(V=40000, d=1000, B=50, S=256, K=8, u=3, W=16, T=1000, t=2, seed=7, inputs=6,
                 scaling="strong",
                 desc="cfg3: large beam B=50, 256 sentences split over the GPUs, |V|=40000, "
                      "d=1000, K=8 u=3 W=16, T=1000, t=2"),
    "cfg4": dict(V=200000, d=1024, B=12, S=64, K=8, u=3, W=16, T=1000, t=2, seed=7, inputs=8,
                 scaling="strong", vocab_sharded=True,
                 desc="cfg4: large vocabulary |V|=200000, d=1024, B=12, 64 sentences, "
                      "vocabulary-sharded over the GPUs (NCCL top-B merge), K=8 u=3 W=16, "
                      "T=1000, t=2"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    p.add_argument("--mode", default="parity", choices=["parity", "fast"])
    p.add_argument("--exchange", default="auto", choices=["auto", "peer", "nccl"],
                   help="cfg4 at N > 1: device pushes into peer memory (CUDA IPC / NVLink) or "
                        "collective all-gathers; auto = peer with one GPU per rank, collectives "
                        "when ranks share GPUs (time-sliced processes make spin waits slow)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the same-GPU comparison legs")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args()


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def sentences_per_rank(c, world):
    return c["S"] if c["scaling"] == "weak" or c.get("vocab_sharded") else c["S"] // world


def workload_config(name, world):
    """The `config` object of the JSON line: identical in both arms."""
    c = WORKLOADS[name]
    par = {"cfg2": f"sentence-sharded x{world}", "cfg3": f"sentence-sharded x{world}",
           "cfg4": f"vocabulary-sharded x{world}"}[name]
    return {"workload": c["desc"], "sentences": c["S"] * (world if c["scaling"] == "weak" else 1),
            "beam": c["B"], "vocab": c["V"], "dim": c["d"], "K": c["K"], "u": c["u"],
            "W": c["W"], "T": c["T"], "t": c["t"], "specials": [c["V"] - 1],
            "parallelism": par,
            "l2": "inputs larger than L2 (E %d MB + cycled step inputs)" % (c["V"] * c["d"] * 4 >> 20)}


def make_inputs(name, rank, world):
    """Synthetic inputs, identical in both arms: E ~ N(0,1) (seed 7), zero
    bias; this rank's step inputs H ~ N(0,1) and cumulative
    scores (rank-seeded for sentence sharding, shared for vocabulary sharding)."""
    import torch
    c = WORKLOADS[name]
    g = torch.Generator().manual_seed(c["seed"])
    E = torch.randn(c["V"], c["d"], generator=g)
    bias = torch.zeros(c["V"])
    S = sentences_per_rank(c, world)
    g2 = torch.Generator().manual_seed(1000 + (0 if name == "cfg4" else rank))
    H = torch.randn(c["inputs"], S, c["B"], c["d"], generator=g2)
    scores = -torch.rand(S, c["B"], generator=g2, dtype=torch.float64) * 4.0
    return E, bias, H, scores


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while running."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.ok:
            # the host loop that enqueues the steps holds the GIL between
            # launches: a short switch interval lets the sampler run during it
            self._switch = sys.getswitchinterval()
            sys.setswitchinterval(0.0002)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()
            sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_capture(kernel):
    """Per-launch DRAM bytes of `kernel` from the committed ncu --set full
    capture, with the capture's tag (the same binary and bench command)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            e = json.load(f).get(kernel, {})
        return e.get("dram_bytes_per_launch"), e.get("tag")
    except Exception:
        return None, None


def dev_timer(ctx):
    import torch
    st = torch.cuda.ExternalStream(ctx.stream)

    def run(fn, steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for k in range(steps):
            fn(k)
        b.record(st)
        b.synchronize()
        ctx.sync()
        return a.elapsed_time(b) / steps
    return run


# ----------------------------------------------------------------- ours
def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    from paper_1806_00588_b200 import FAST, PARITY, Batch, Context, Index, Model
    from paper_1806_00588_b200.seeds import mix_seed

    name = args.workload
    c = WORKLOADS[name]
    vsh = name == "cfg4" and world > 1
    ngpu = torch.cuda.device_count()
    # one rank per GPU; more ranks than GPUs (a functional check on a small
    # box) share devices and time through gloo, since NCCL refuses that
    local = local % max(ngpu, 1)
    torch.cuda.set_device(local)
    coll_dev = "cuda" if world <= ngpu else "cpu"
    if world > 1:
        import torch.distributed as dist
        if world <= ngpu:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    E, bias, H, scores = make_inputs(name, rank, world)
    S, B, d, V = H.shape[1], c["B"], c["d"], c["V"]
    stream = torch.cuda.Stream()
    ctx = Context(local, stream.cuda_stream)
    mode = PARITY if args.mode == "parity" else FAST
    ps, isd = mix_seed(c["seed"], 1), mix_seed(c["seed"], 2)
    t0 = time.perf_counter()
    if vsh:
        from paper_1806_00588_b200.vocab_shard import VocabShard, shard_bounds, sharded_step
        v0, n = shard_bounds(V, world, rank)
        Es, bs = E[v0:v0 + n].cuda().contiguous(), bias[v0:v0 + n].cuda()
        shard = VocabShard(ctx, Es, bs, v0, V, c["K"], c["u"], c["W"], ps, isd, S, B, c["T"],
                           c["t"], specials=[V - 1], mode=mode)
        model, idx, batch = shard.model, shard.index, shard.batch
        xchg = None
        if args.exchange == "peer" or (args.exchange == "auto" and world <= ngpu):
            from paper_1806_00588_b200.vocab_shard import PeerExchange
            xchg = PeerExchange(shard, world, rank)
            xchg.connect()
            torch.distributed.barrier()
    else:
        Ed, bd = E.cuda(), bias.cuda()
        torch.cuda.synchronize()
        model = Model(ctx, None, device_ptrs=(Ed.data_ptr(), bd.data_ptr(), V, d))
        idx = Index(ctx, model, K=c["K"], u=c["u"], W=c["W"], perm_seed=ps, index_seed=isd)
        batch = Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"], specials=[V - 1], mode=mode)
    ctx.sync()
    index_ms = (time.perf_counter() - t0) * 1e3
    Hd = H.cuda()
    sc = scores.cuda()
    fin = torch.zeros(S, B, dtype=torch.uint8, device="cuda")
    nh = torch.full((S,), B, dtype=torch.int32, device="cuda")
    choices = torch.zeros(S * B * 24, dtype=torch.uint8, device="cuda")
    nchoice = torch.zeros(S, dtype=torch.int32, device="cuda")
    hout = torch.empty(S, B, d, device="cuda")
    step_bytes = S * B * d * 4
    base = Hd.data_ptr()
    torch.cuda.synchronize()

    if vsh and xchg is not None:
        def step(k):
            xchg.step(Hd[k % c["inputs"]], sc, fin, nh, choices, nchoice, hout)
    elif vsh:
        def step(k):
            with torch.cuda.stream(stream):
                sharded_step(shard, Hd[k % c["inputs"]], sc, fin, nh, choices, nchoice, hout)
    else:
        def step(k):
            batch.step(base + (k % c["inputs"]) * step_bytes, sc, fin, nh, choices, nchoice, hout)

    # candidate counts per input (deterministic) for the algorithmic byte count
    ncand = np.zeros((c["inputs"], S), np.int64)
    for k in range(c["inputs"]):
        step(k)
        ctx.sync()
        ncand[k] = [len(batch.candidates(s)[0]) for s in range(S)]
    for k in range(args.warmup):
        step(k)
    ctx.sync()
    launches0 = ctx.launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        for k in range(args.steps):
            step(k)
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ctx.sync()
    launches = ctx.launches - launches0
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device=coll_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    S_job = c["S"] * (world if c["scaling"] == "weak" else 1)
    value = S_job * args.steps / (ms / 1e3)

    # Per-stage device times from a separate instrumented pass (stage events
    # between kernels would break programmatic dependent launch inside the
    # timed region): 30 steps, every step instrumented.
    batch.profile(True, every=1)
    for k in range(30):
        step(k)
    stage_tot, nrec = batch.stage_totals()
    batch.profile(False)
    stages = {k: round(float(v) / max(nrec, 1), 5) for k, v in
              zip(["probe_count", "compact", "logits", "softmax_topb", "expand"], stage_tot)}

    # Dominant kernel: K4 (k_logits). Algorithmic work per launch: unique E
    # rows (shared top-T block once + each sentence's survivors) + H + ids/bias
    # + logits written; MACs = B x sum n x d (FMUL + FADD each in PARITY).
    used = ncand[np.arange(args.steps) % c["inputs"]]
    T_loc = c["T"]
    if vsh:
        from paper_1806_00588_b200.vocab_shard import local_config
        T_loc = local_config(c["T"], [V - 1], v0, n)[0]
    m = np.maximum(used - T_loc, 0)
    alg_bytes = ((T_loc + m.sum(axis=1)) * d * 4 + S * B * d * 4 + (T_loc + m.sum(axis=1)) * 8
                 + B * used.sum(axis=1) * 4).mean()
    macs = float((B * used.sum(axis=1) * d).mean())
    logits_ms = stages["logits"]
    peaks, peak_src = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_achieved = alg_bytes / (logits_ms / 1e3) / 1e9
    fp32_peak = ctx.fp32x2_peak()  # lane-ops/s, measured now on this GPU
    lane_ops = (2.0 if mode == PARITY else 1.0) * macs
    fp32_achieved = lane_ops / (logits_ms / 1e3)
    traffic, tag = ncu_capture("k_logits")
    roofline = {
        "kernel": "k_logits", "bound": "fp32",
        "achieved": round(fp32_achieved / 1e12, 3), "peak": round(fp32_peak / 1e12, 3),
        "unit": "T FP32 lane-ops/s", "frac": round(fp32_achieved / fp32_peak, 4),
        "peak_kind": "measured in this run: lsb_measure_fp32x2_peak (paired FMUL+FADD, the "
                     "instructions K4 PARITY issues), %d SMs" % ctx.sm_count,
        "traffic": traffic, "traffic_capture": tag,
        "launch_ms": round(logits_ms, 5), "launches_timed": int(nrec),
        "macs_per_launch": int(macs), "lane_ops_per_launch": int(lane_ops),
        "alg_bytes_per_launch": int(alg_bytes),
        "hbm": {"achieved": round(hbm_achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(hbm_achieved / hbm_peak, 4), "peak_kind": peak_src},
        "note": ("PARITY: one FMUL + one FADD per MAC in the reference's 4-lane order "
                 "(bit-exact logits), issued as FFMA2 pairs: FP32-issue bound; the HBM "
                 "fraction is reported beside it" if mode == PARITY else
                 "FAST: FFMA2 chains / tcgen05 3xTF32 for the shared block")}

    # e2e: the public C-ABI call with host buffers (pinned), H2D + D2H inside
    e2e = None
    if not vsh:
        e2e = time_e2e_leg(args, batch, H, scores, S, B, d, world, coll_dev, S_job)
    else:
        e2e = time_e2e_sharded(args, shard, sharded_step, H, scores, S, B, d, world, coll_dev,
                               S_job, stream, xchg)

    extras = {}
    if not args.no_extras and rank == 0 and world == 1 and name == "cfg2":
        extras = run_extras(ctx, model, idx, Hd, sc, fin, nh, choices, nchoice, hout, args,
                            value, c)
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None,
            "dtype": "f32", "mode": args.mode,
            "data": "synthetic (torch.randn seed 7; E %dx%d fp32)" % (V, d),
            "config": workload_config(name, world),
            "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
            "stage_ms": stages, "clocks": clk.summary(),
            "run": {"batch_steps_per_s": round(1e3 / ms_per_step, 1),
                    "sentences_per_rank": S, "mean_vlsh": float(used.mean()),
                    "index_build_ms": round(index_ms, 1), "ranks_share_gpus": world > ngpu},
            **extras}
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(name, E, bias, H, scores, args.cpu_seconds)
    if world > 1:
        torch.distributed.barrier()  # no rank still pushes into a peer's area
        if vsh and xchg is not None:
            xchg.close()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def time_e2e_leg(args, batch, H, scores, S, B, d, world, coll_dev, S_job):
    """End to end through the public C ABI with pinned host buffers: every
    step uploads its inputs and reads its choices back inside the timed
    region (pipelined lsb_step_host_async, and synchronous lsb_step_host)."""
    import ctypes as C

    import torch
    n_in = H.shape[0]
    Hh = H.pin_memory()
    sch = scores.pin_memory()
    finh = torch.zeros(S, B, dtype=torch.uint8).pin_memory()
    nhh = torch.full((S,), B, dtype=torch.int32).pin_memory()
    ch_h = torch.zeros(S * B * 24, dtype=torch.uint8).pin_memory()
    nc_h = torch.zeros(S, dtype=torch.int32).pin_memory()
    hb, step_bytes = Hh.data_ptr(), S * B * d * 4
    chp, ncp = C.c_void_p(ch_h.data_ptr()), C.c_void_p(nc_h.data_ptr())

    def sync_step(k):
        batch.step_host_ptrs(hb + (k % n_in) * step_bytes, sch.data_ptr(), finh.data_ptr(),
                             nhh.data_ptr(), chp, ncp)

    def async_step(k):
        batch.step_host_async(hb + (k % n_in) * step_bytes, sch.data_ptr(), finh.data_ptr(),
                              nhh.data_ptr(), chp, ncp)

    # at least 300 steps: the pipeline's fill (first upload) and drain (last
    # read-back) are not amortised over a 20-step run
    n_e2e = max(args.steps, 300)

    def timed(fn, finish):
        for k in range(max(args.warmup, 3)):
            fn(k)
        finish()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(n_e2e):
            fn(k)
        finish()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device=coll_dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        return el

    e_async = timed(async_step, batch.wait)
    e_sync = timed(sync_step, batch.ctx.sync)
    return {"value": round(S_job * n_e2e / e_async, 1), "unit": UNIT, "steps": n_e2e,
            "h2d_bytes_per_step": S * B * d * 4 + S * B * 8 + S * B + S * 4,
            "d2h_bytes_per_step": S * B * 24 + S * 4, "api": "lsb_step_host_async (C ABI)",
            "synchronous_value": round(S_job * n_e2e / e_sync, 1),
            "synchronous_api": "lsb_step_host (C ABI, one host sync per step)"}


def time_e2e_sharded(args, shard, sharded_step, H, scores, S, B, d, world, coll_dev, S_job,
                     stream, xchg=None):
    """Vocabulary-sharded e2e: per step the host inputs are uploaded from pinned
    memory, the sharded step runs (NCCL exchanges included) and rank 0 reads
    the choices back."""
    import torch
    n_in = H.shape[0]
    Hh, sch = H.pin_memory(), scores.pin_memory()
    Hd = torch.empty(S, B, d, device="cuda")
    sc = torch.empty(S, B, dtype=torch.float64, device="cuda")
    fin = torch.zeros(S, B, dtype=torch.uint8, device="cuda")
    nh = torch.full((S,), B, dtype=torch.int32, device="cuda")
    ch = torch.zeros(S * B * 24, dtype=torch.uint8, device="cuda")
    nc = torch.zeros(S, dtype=torch.int32, device="cuda")
    ch_h = torch.zeros(S * B * 24, dtype=torch.uint8).pin_memory()

    def one(k):
        with torch.cuda.stream(stream):
            Hd.copy_(Hh[k % n_in], non_blocking=True)
            sc.copy_(sch, non_blocking=True)
            if xchg is not None:
                xchg.step(Hd, sc, fin, nh, ch, nc, None)
            else:
                sharded_step(shard, Hd, sc, fin, nh, ch, nc, None)
            ch_h.copy_(ch, non_blocking=True)
        stream.synchronize()

    n_e2e = max(args.steps, 100)
    for k in range(max(args.warmup, 3)):
        one(k)
    torch.distributed.barrier()
    t0 = time.perf_counter()
    for k in range(n_e2e):
        one(k)
    el = time.perf_counter() - t0
    t = torch.tensor([el], device=coll_dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    el = float(t.item())
    return {"value": round(S_job * n_e2e / el, 1), "unit": UNIT, "steps": n_e2e,
            "h2d_bytes_per_step": S * B * d * 4 + S * B * 8, "d2h_bytes_per_step": S * B * 24,
            "api": ("lsb_shard_step_peer (C ABI: phases + pushes into peer memory + device flag "
                    "waits)" if xchg is not None else
                    "vocab_shard.sharded_step (C ABI phases + NCCL all-gathers)")
                   + ", one host sync per step"}


def run_extras(ctx, model, idx, Hd, sc, fin, nh, choices, nchoice, hout, args, lsh_value, c):
    """Same-GPU comparison legs (rank 0, one GPU): the full-vocabulary fused
    path, cfg1 latency, the other arithmetic mode and its choice agreement,
    recall@B at the bench inputs, and the reference's validated operating
    point (LSH vs full speed-up at matched top-B agreement)."""
    import numpy as np
    import torch

    from paper_1806_00588_b200 import FAST, PARITY, Batch
    from paper_1806_00588_b200.lshbeam import exact_topb
    S, B, d, V = c["S"], c["B"], c["d"], c["V"]
    out = {}
    base, step_bytes = Hd.data_ptr(), S * B * d * 4
    timer = dev_timer(ctx)

    def time_batch(b, steps, warm=2):
        for k in range(warm):
            b.step(base + k * step_bytes, sc, fin, nh, choices, nchoice, hout)
        ctx.sync()
        return timer(lambda k: b.step(base + (k % c["inputs"]) * step_bytes, sc, fin, nh,
                                      choices, nchoice, hout), steps)

    tf32_peak = measured_tf32_peak()
    for nm, mode in [("full_vocab_parity", PARITY), ("full_vocab_fast", FAST)]:
        b = Batch(ctx, model, None, S=S, B=B, specials=[V - 1], mode=mode, full_vocab=True)
        ms = time_batch(b, 5)
        b.profile(True, every=1)
        for k in range(5):
            b.step(base + k * step_bytes, sc, fin, nh, choices, nchoice, hout)
        st, nrec = b.stage_totals()
        b.profile(False)
        stg = {k: round(float(v) / max(nrec, 1), 4) for k, v in
               zip(["probe_count", "compact", "logits", "softmax_topb", "expand"], st)}
        out[nm] = {"ms_per_step": round(ms, 4), "value": round(S / (ms / 1e3), 1),
                   "lsh_speedup": round(lsh_value / (S / (ms / 1e3)), 2), "stage_ms": stg}
        macs = float(S * B) * V * d
        if mode == PARITY:
            peak = ctx.fp32x2_peak()
            ach = 2.0 * macs / (stg["logits"] / 1e3)
            out[nm]["roofline"] = {"kernel": "k_logits_ln", "bound": "fp32",
                                   "achieved": round(ach / 1e12, 3), "peak": round(peak / 1e12, 3),
                                   "unit": "T FP32 lane-ops/s", "frac": round(ach / peak, 4)}
        else:
            # 3xTF32: three tensor-core products per MAC (hi*hi + hi*lo + lo*hi)
            ach = 3.0 * 2.0 * macs / (stg["logits"] / 1e3)
            out[nm]["roofline"] = {"kernel": "k_tc_logits", "bound": "tensor",
                                   "achieved": round(ach / 1e12, 1),
                                   "peak": round(tf32_peak / 1e12, 1), "unit": "TFLOP/s (tf32)",
                                   "frac": round(ach / tf32_peak, 4),
                                   "peak_kind": "measured in this run: torch.matmul TF32 "
                                                "(cuBLAS) 8192^3, best of 5"}
        b.close()
    other = FAST if args.mode == "parity" else PARITY
    bo = Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"], specials=[V - 1], mode=other)
    ms = time_batch(bo, 50)
    out["lsh_" + ("fast" if other == FAST else "parity")] = {
        "ms_per_step": round(ms, 4), "value": round(S / (ms / 1e3), 1)}
    # chosen (beam, word) agreement of FAST with PARITY on the same 50 inputs
    bp = Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"], specials=[V - 1], mode=PARITY)
    bf = bo if other == FAST else Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"],
                                        specials=[V - 1], mode=FAST)
    agree = total = 0
    for k in range(c["inputs"]):
        got = []
        for bb in (bp, bf):
            bb.step(base + k * step_bytes, sc, fin, nh, choices, nchoice, hout)
            ctx.sync()
            got.append(choices.view(torch.int64).view(S, B, 3)[:, :, 1:].clone())
        same = (got[0] == got[1]).all(dim=2)
        agree += int(same.sum())
        total += same.numel()
    out["fast_vs_parity_choice_agreement"] = {"agree": agree, "total": total,
                                              "frac": round(agree / max(total, 1), 6)}
    # recall@B vs full (SURVEY §8 d) on the first 4 inputs
    hits = rows = 0
    for k in range(4):
        bp.step(base + k * step_bytes, sc, fin, nh, choices, nchoice, hout)
        ctx.sync()
        ids_exact, _ = exact_topb(ctx, model, base + k * step_bytes, S * B, B, bias=True)
        for s_ in range(S):
            cand = bp.candidates(s_)[0]
            hits += int(np.isin(ids_exact[s_ * B:(s_ + 1) * B], cand).sum())
            rows += B
    out["recall_at_B"] = {"value": round(hits / max(rows * B, 1), 4), "rows": rows,
                          "note": "exact full-vocab top-B vs V_LSH, 4 inputs x 768 rows; iid "
                                  "synthetic data: near chance, the reference's value too "
                                  "(see operating_point for trained-like data)"}
    for bb in {id(bp): bp, id(bf): bf, id(bo): bo}.values():
        bb.close()
    out["cfg1"] = run_cfg1(ctx, model, idx, c)
    out["operating_point"] = run_operating_point(ctx)
    return out


def measured_tf32_peak():
    """Dense TF32 tensor-core throughput of this GPU (cuBLAS via torch.matmul
    with TF32 allowed, 8192^3, best of 5): the denominator of the FAST
    full-vocabulary GEMM's roofline."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        torch.matmul(a, b)
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * n ** 3 / (best / 1e3)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def run_cfg1(ctx, model, idx, c):
    """BASELINE configs[0]: one sentence (S=1, B=12) per step, |V|=40k, d=1000:
    latency of the LSH step, eager (five PDL-chained launches) and replayed
    as one CUDA graph, vs the full-vocabulary step."""
    import torch

    from paper_1806_00588_b200 import PARITY, Batch
    B, d, V = c["B"], c["d"], c["V"]
    g = torch.Generator().manual_seed(3)
    n_in = 64
    H = torch.randn(n_in, 1, B, d, generator=g).cuda()
    sc = (-torch.rand(1, B, generator=g, dtype=torch.float64) * 4).cuda()
    fin = torch.zeros(1, B, dtype=torch.uint8, device="cuda")
    nh = torch.full((1,), B, dtype=torch.int32, device="cuda")
    ch = torch.zeros(B * 24, dtype=torch.uint8, device="cuda")
    nc = torch.zeros(1, dtype=torch.int32, device="cuda")
    ho = torch.empty(1, B, d, device="cuda")
    Hcur = torch.empty(1, B, d, device="cuda")
    timer = dev_timer(ctx)
    st = torch.cuda.ExternalStream(ctx.stream)
    res = {}
    for nm, full in (("lsh", False), ("full_vocab", True)):
        b = Batch(ctx, model, None if full else idx, S=1, B=B, T=0 if full else c["T"],
                  t=0 if full else c["t"], specials=[V - 1], mode=PARITY, full_vocab=full)

        def eager(k, b=b):
            b.step(H[k % n_in], sc, fin, nh, ch, nc, ho)
        for k in range(5):
            eager(k)
        ctx.sync()
        ms = timer(eager, 200)
        r = {"us_per_step": round(ms * 1e3, 2), "steps_per_s": round(1e3 / ms, 1)}
        # graph: the captured step reads Hcur; each replay's input is copied
        # in first (the decode loop writes it in place; the copy is timed too)
        with torch.cuda.stream(st):
            Hcur.copy_(H[0])
        b.graph_capture(Hcur, sc, fin, nh, ch, nc, ho)

        def replay(k, b=b):
            with torch.cuda.stream(st):
                Hcur.copy_(H[k % n_in], non_blocking=True)
            b.graph_launch()
        for k in range(5):
            replay(k)
        ctx.sync()
        msg = timer(replay, 200)
        r["graph_us_per_step"] = round(msg * 1e3, 2)
        r["graph_steps_per_s"] = round(1e3 / msg, 1)
        res[nm] = r
        b.close()
    res["lsh_speedup_vs_full"] = round(res["full_vocab"]["us_per_step"] /
                                       res["lsh"]["us_per_step"], 2)
    res["note"] = ("device-timed (CUDA events on the step stream), 200 steps over 64 cycled "
                   "inputs; graph = lsb_batch_graph_capture/launch, includes a 48 KB "
                   "device copy of the step input")
    return res


def run_operating_point(ctx, S=64, steps=8):
    """The reference's validated operating point (tests/acceptance.cpp:275-300,
    BASELINE.md §2b): V=50k, d=256, Zipf bias 300, K=16, u=3, W=500, T=250,
    t=5, batched over S=64 synthetic decodes (h0_s from mix_seed(7, 100+s),
    the model provider's W_h / W_e recurrence on the device). Per step both
    paths score the SAME state: the LSH step's choices drive the decode; the
    full-vocabulary step's choices on that state are the agreement target.
    Reports recall@B (exact full top-B inside V_LSH), top-B choice agreement
    (fraction of the full path's (beam, word) choices the LSH path also
    chose), and the device time of both paths over the recorded states in
    each arithmetic mode."""
    import torch

    from paper_1806_00588_b200.synth import synth_model
    V, d, bias_s, K, u, W, T, t, B = 50000, 256, 300.0, 16, 3, 500, 250, 5, 12
    E, bias, wh, we, _ = synth_model(V, d, 7, bias_s)
    # torch work on the context's stream (ordered with the library's kernels)
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream)):
        return _operating_point(ctx, S, steps, V, d, K, u, W, T, t, B, E, bias, wh, we)


def _operating_point(ctx, S, steps, V, d, K, u, W, T, t, B, E, bias, wh, we):
    import numpy as np
    import torch

    from paper_1806_00588_b200 import FAST, PARITY, Batch, Index, Model
    from paper_1806_00588_b200.lshbeam import Recurrent, exact_topb
    from paper_1806_00588_b200.seeds import mix_seed
    from paper_1806_00588_b200.synth import start_state
    model = Model(ctx, E, bias)
    idx = Index(ctx, model, K=K, u=u, W=W, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
    rec = Recurrent(ctx, wh, we)
    dev = torch.device("cuda", ctx.device)
    mk = lambda full, mode: Batch(ctx, model, None if full else idx, S=S, B=B,  # noqa: E731
                                  T=0 if full else T, t=0 if full else t, specials=[V - 1],
                                  mode=mode, full_vocab=full)
    lsh, full = mk(False, PARITY), mk(True, PARITY)
    H = torch.zeros(S, B, d, device=dev)
    H[:, 0] = torch.from_numpy(np.stack([start_state(7, s, d) for s in range(S)])).to(dev)
    sc = torch.zeros(S, B, dtype=torch.float64, device=dev)
    fin = torch.zeros(S, B, dtype=torch.uint8, device=dev)
    nh = torch.ones(S, dtype=torch.int32, device=dev)  # step 0: one live hypothesis
    chL = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
    chF = torch.zeros_like(chL)
    ncL = torch.zeros(S, dtype=torch.int32, device=dev)
    ncF = torch.zeros_like(ncL)
    ho = torch.empty(S, B, d, device=dev)
    hoF = torch.empty_like(ho)
    states = []
    hits = rows = agree = want = 0
    vl = []
    dt = np.dtype([("score", "<f8"), ("beam", "<u4"), ("pad", "<u4"), ("word", "<i8")])
    for k in range(steps):
        states.append((H.clone(), sc.clone(), fin.clone(), nh.clone()))
        lsh.step(H, sc, fin, nh, chL, ncL, ho)
        full.step(H, sc, fin, nh, chF, ncF, hoF)
        ctx.sync()
        cl = np.frombuffer(chL.cpu().numpy().tobytes(), dt).reshape(S, B)
        cf = np.frombuffer(chF.cpu().numpy().tobytes(), dt).reshape(S, B)
        nl, nf, nhh, finh = (ncL.cpu().numpy(), ncF.cpu().numpy(), nh.cpu().numpy(),
                             fin.cpu().numpy())
        for s in range(S):
            a = {(int(x["beam"]), int(x["word"])) for x in cl[s, :nl[s]]}
            f = {(int(x["beam"]), int(x["word"])) for x in cf[s, :nf[s]]}
            agree += len(a & f)
            want += len(f)
            vl.append(len(lsh.candidates(s)[0]))
        # recall@B over the live rows (exact full-vocabulary top-B + bias)
        ids_exact, _ = exact_topb(ctx, model, H.data_ptr(), S * B, B, bias=True)
        for s in range(S):
            cand = lsh.candidates(s)[0]
            for i in range(int(nhh[s])):
                if finh[s, i]:
                    continue
                hits += int(np.isin(ids_exact[s * B + i], cand).sum())
                rows += 1
        # advance the decode with the LSH choices: parent rows are in ho;
        # new hidden = recurrence(parent, token); EOS (V-1) freezes
        words = torch.from_numpy(np.ascontiguousarray(
            np.where(np.arange(B)[None, :] < nl[:, None], cl["word"], -1))).to(dev)
        newH = torch.empty_like(H)
        rec.step(model, ho.data_ptr(), words.data_ptr(), S * B, newH.data_ptr())
        H = newH
        sc = torch.from_numpy(np.ascontiguousarray(cl["score"])).to(dev)
        fin = ((words == V - 1) | (words < 0)).to(torch.uint8)
        nh = torch.from_numpy(nl.astype(np.int32)).to(dev)
        ctx.sync()
    res = {"config": "V=50000 d=256 bias=300 K=16 u=3 W=500 T=250 t=5 B=12, %d synthetic "
                     "decodes x %d steps (reference acceptance operating point, batched)"
                     % (S, steps),
           "recall_at_B": round(hits / max(rows * B, 1), 4),
           "topB_choice_agreement": round(agree / max(want, 1), 4),
           "mean_vlsh": round(float(np.mean(vl)), 1)}
    lsh.close(), full.close()
    timer = dev_timer(ctx)
    for mname, mode in (("parity", PARITY), ("fast", FAST)):
        bl, bf = mk(False, mode), mk(True, mode)
        tms = {}
        for nm, b in (("lsh", bl), ("full_vocab", bf)):
            for st in states[:2]:
                b.step(*st, chL, ncL, ho)
            ctx.sync()
            tms[nm] = timer(lambda k, b=b: b.step(*states[k % len(states)], chL, ncL, ho),
                            3 * len(states))
        res[mname] = {"lsh_ms_per_step": round(tms["lsh"], 4),
                      "full_vocab_ms_per_step": round(tms["full_vocab"], 4),
                      "lsh_speedup": round(tms["full_vocab"] / tms["lsh"], 2)}
        bl.close(), bf.close()
    rec.close(), idx.close(), model.close()
    return res


# ------------------------------------------------------------ reference
def cpu_baseline(name, E, bias, H, scores, seconds, steps=None):
    """The reference's own CPU step (oracle/_ref) on the host cores, on a
    bounded sample of the same workload."""
    from oracle.oracle import Reference, ReferenceStepper
    from paper_1806_00588_b200.seeds import mix_seed
    c = WORKLOADS[name]
    if not Reference.available():
        return {"value": None, "unit": UNIT, "kind": "reference",
                "note": "oracle/_ref not built"}
    ref = Reference()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    En, bn, Hn, scn = E.numpy(), bias.numpy(), H.numpy(), scores.numpy()
    S = Hn.shape[1]
    st = ReferenceStepper(ref, En, bn, c["K"], c["u"], c["W"], mix_seed(c["seed"], 1),
                          mix_seed(c["seed"], 2))
    for s in range(2):  # warm-up
        st.step(Hn[0, s], scn[s], c["B"], c["T"], c["t"], [c["V"] - 1])
    n, t0 = 0, time.perf_counter()
    k = 0
    while True:
        for s in range(S):
            st.step(Hn[k % c["inputs"], s], scn[s], c["B"], c["T"], c["t"], [c["V"] - 1])
            n += 1
        k += 1
        el = time.perf_counter() - t0
        if (steps is not None and k >= steps) or (steps is None and el >= seconds):
            break
    st.close()
    return {"value": round(n / el, 2), "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{k} batch-steps x {S} sentences = {n} sentence-steps of the same "
                      f"workload ({el:.1f} s), reference lshbeam compiled from /root/reference "
                      "sources (g++ -O3 -fopenmp), OMP threads = all host cores"}


def run_reference(args, rank, world, local):
    if rank != 0:
        return
    name = args.workload
    c = WORKLOADS[name]
    E, bias, H, scores = make_inputs(name, 0, 1)
    from oracle.oracle import Reference
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    # keep the whole --steps/--warmup run within a few minutes: each "step" is
    # the cfg2 batch (64 sentences), or a bounded 8-sentence sample of the
    # heavier cfg3 / cfg4 batches
    ns = 64 if name == "cfg2" else 8
    Hs, scs = H[:, :ns], scores[:ns]
    cpu_baseline(name, E, bias, Hs, scs, 0, steps=args.warmup)  # warm-up steps
    t0 = time.perf_counter()
    cb = cpu_baseline(name, E, bias, Hs, scs, 0, steps=args.steps)
    wall = time.perf_counter() - t0
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * c["S"] / v, 3) if v else None, "higher_is_better": True,
            "scaling": c["scaling"], "vs_baseline": None, "dtype": "f32", "mode": "parity",
            "data": "synthetic (torch.randn seed 7; E %dx%d fp32)" % (c["V"], c["d"]),
            "config": workload_config(name, world),
            "cpu_baseline": cb, "wall_s": round(wall, 2),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_info()
    if args.impl == "reference":
        run_reference(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()

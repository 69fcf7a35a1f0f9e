#!/usr/bin/env python
"""Benchmark of the per-step LSH beam-search hot path (BASELINE.json).

Workload (BASELINE configs[1], "batched decode loop"): 64 sentences x B=12
hypotheses per GPU, |V|=40000, d=1000, WTA K=8 u=3 W=16, T=1000, t=2,
specials {V-1}; 50 distinct synthetic step inputs (torch.randn, seed 7) are
cycled, so one "step" = one pass of the fused hot path (hash, cuckoo lookup,
candidate union, reduced softmax, beam expansion + hidden reorder) over one
batch of 64 sentences. Metric: decode steps/s = sentence-steps per second
(softmax path + beam expansion, the reference's StageTimes::softmax_path() +
beam_expansion, include/lshbeam/beam_decoder.hpp:66-73).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU: one process per GPU (torchrun), sentences sharded across ranks
(weak scaling: 64 sentences per rank, no data-path collective), timing is the
max over ranks of the device-timed region. The reference arm times the
reference's own CPU implementation (oracle/_ref, compiled from
/root/reference's sources) on the host cores.
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

CFG = dict(V=40000, d=1000, B=12, S=64, K=8, u=3, W=16, T=1000, t=2, seed=7, inputs=50)
METRIC = "decode steps/sec (softmax+beam expand) at |V|=40k,d=1000,B=12; recall@B vs full"
UNIT = "sentence-steps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--mode", default="parity", choices=["parity", "fast"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip full-vocab / fast-mode lines")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args()


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_inputs(rank: int):
    """Synthetic inputs, identical in both arms: E ~ N(0,1) (seed 7), zero
    bias; per rank 50 step inputs H ~ N(0,1) and cumulative
    scores."""
    import torch
    c = CFG
    g = torch.Generator().manual_seed(c["seed"])
    E = torch.randn(c["V"], c["d"], generator=g)
    bias = torch.zeros(c["V"])
    g2 = torch.Generator().manual_seed(1000 + rank)
    H = torch.randn(c["inputs"], c["S"], c["B"], c["d"], generator=g2)
    scores = -torch.rand(c["S"], c["B"], generator=g2, dtype=torch.float64) * 4.0
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
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of k_logits from the committed ncu summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get("k_logits", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------- ours
def run_ours(args, rank, world, local):
    import ctypes as C

    import numpy as np
    import torch

    from paper_1806_00588_b200 import FAST, PARITY, Batch, Context, Index, Model
    from paper_1806_00588_b200 import _native as N

    c = CFG
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
    E, bias, H, scores = make_inputs(rank)
    stream = torch.cuda.Stream()
    ctx = Context(local, stream.cuda_stream)
    Ed, bd = E.cuda(), bias.cuda()
    torch.cuda.synchronize()
    model = Model(ctx, None, device_ptrs=(Ed.data_ptr(), bd.data_ptr(), c["V"], c["d"]))
    del Ed, bd
    t0 = time.perf_counter()
    from paper_1806_00588_b200.seeds import mix_seed
    idx = Index(ctx, model, K=c["K"], u=c["u"], W=c["W"], perm_seed=mix_seed(c["seed"], 1),
                index_seed=mix_seed(c["seed"], 2))
    index_ms = (time.perf_counter() - t0) * 1e3
    mode = PARITY if args.mode == "parity" else FAST
    S, B, d = c["S"], c["B"], c["d"]
    batch = Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"], specials=[c["V"] - 1],
                  mode=mode)
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
    # stage events on every 8th step only: events between kernels would break
    # programmatic dependent launch on the steps they separate
    batch.profile(True, every=8)
    launches0 = ctx.launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
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
    stage_tot, nrec = batch.stage_totals()
    batch.profile(False)
    if world > 1:
        t = torch.tensor([ms], device=coll_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = S * world * args.steps / (ms / 1e3)

    # dominant kernel: k_logits. Algorithmic bytes per launch = unique E rows
    # (shared top-T block once + each sentence's survivors) + H + ids/bias +
    # logits written.
    used = ncand[np.arange(args.steps) % c["inputs"]]
    m = np.maximum(used - c["T"], 0)
    e_rows = c["T"] + m.sum(axis=1)
    alg_bytes = (e_rows * d * 4 + S * B * d * 4 + (c["T"] + m.sum(axis=1)) * 8
                 + B * used.sum(axis=1) * 4).mean()
    flops = (2.0 * B * used.sum(axis=1) * d).mean()
    logits_ms = float(stage_tot[2]) / max(nrec, 1)
    peak, peak_kind = measured_peak_hbm()
    achieved = alg_bytes / (logits_ms / 1e3) / 1e9
    # The binding resource of K4 in PARITY is FP32 instruction issue, not HBM:
    # every MAC is an FMUL + an FADD (no FMA, reference order). Peak lane-op
    # rate = SMs x 128 FP32 lanes x SM clock (median under load).
    macs = flops / 2.0
    roofline = {"kernel": "k_logits", "bound": "hbm", "achieved": round(achieved, 1),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(),
                "alg_bytes_per_launch": int(alg_bytes), "launch_ms": round(logits_ms, 5),
                "launches_timed": int(nrec),
                "macs_per_launch": int(macs),
                "fp32_tflops": round(flops / (logits_ms / 1e3) / 1e12, 2),
                "note": "PARITY: FMUL+FADD per MAC in the reference order as FFMA2 pairs; bound "
                        "jointly by the FP32 pipe (fp32_issue) and shared-memory wavefronts "
                        "(each 16-B LDS costs 4 wavefronts; ncu: ~60% of both)"
                        if mode == PARITY else
                        "FAST: paired FFMA2 chains (tcgen05 3xTF32 only for the full-vocabulary "
                        "block)"}
    stages = {k: round(float(v) / max(nrec, 1), 5) for k, v in
              zip(["probe_count", "compact", "logits", "softmax_topb", "expand"], stage_tot)}

    # e2e: the public C-ABI call with host buffers (pinned), H2D + D2H inside
    Hh = H.pin_memory()
    sch = scores.pin_memory()
    finh = torch.zeros(S, B, dtype=torch.uint8).pin_memory()
    nhh = torch.full((S,), B, dtype=torch.int32).pin_memory()
    ch_h = torch.zeros(S * B * 24, dtype=torch.uint8).pin_memory()
    nc_h = torch.zeros(S, dtype=torch.int32).pin_memory()
    hb = Hh.data_ptr()
    chp = C.c_void_p(ch_h.data_ptr())
    ncp = C.c_void_p(nc_h.data_ptr())

    def step_e2e(k):
        batch.step_host_ptrs(hb + (k % c["inputs"]) * step_bytes, sch.data_ptr(),
                             finh.data_ptr(), nhh.data_ptr(), chp, ncp)

    def step_e2e_async(k):
        batch.step_host_async(hb + (k % c["inputs"]) * step_bytes, sch.data_ptr(),
                              finh.data_ptr(), nhh.data_ptr(), chp, ncp)

    def time_e2e(fn, finish):
        for k in range(args.warmup):
            fn(k)
        finish()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(args.steps):
            fn(k)
        finish()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device=coll_dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        return el

    # pipelined public API (step k+1's upload overlaps step k's kernels);
    # every step still uploads its inputs from pinned host memory and reads
    # its choices back into host memory inside the timed region
    e2e_s = time_e2e(step_e2e_async, batch.wait)
    e2e_sync_s = time_e2e(step_e2e, ctx.sync)
    e2e = {"value": round(S * world * args.steps / e2e_s, 1), "unit": UNIT,
           "h2d_bytes_per_step": S * B * d * 4 + S * B * 8 + S * B + S * 4,
           "d2h_bytes_per_step": S * B * 24 + S * 4, "api": "lsb_step_host_async (C ABI)",
           "synchronous_value": round(S * world * args.steps / e2e_sync_s, 1),
           "synchronous_api": "lsb_step_host (C ABI, one host sync per step)"}

    extras = {}
    if not args.no_extras and rank == 0:
        extras = run_extras(ctx, model, idx, Hd, sc, fin, nh, choices, nchoice, hout, args,
                            value)
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "mode": args.mode, "data": "synthetic (torch.randn seed 7; E 40000x1000 fp32)",
            "config": {"workload": "cfg2: batched decode step, 64 sentences x B=12 per GPU, "
                                   "|V|=40000, d=1000, K=8 u=3 W=16, T=1000, t=2",
                       "sentences_per_gpu": S, "beam": B, "vocab": c["V"], "dim": d,
                       "K": c["K"], "u": c["u"], "W": c["W"], "T": c["T"], "t": c["t"],
                       "parallelism": f"sentence-sharded x{world}" + (f" on {ngpu} GPU(s), ranks share devices" if world > ngpu else ""),
                       "l2": "inputs larger than L2: E 160 MB + 50 cycled H inputs 154 MB",
                       "batch_steps_per_s": round(value / S / world, 1),
                       "mean_vlsh": float(used.mean()), "index_build_ms": round(index_ms, 1)},
            "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
            "stage_ms": stages, "clocks": clk.summary(), **extras}
    sm_mhz = line["clocks"].get("sm_mhz") or 1965.0
    lane_ops = (2.0 if mode == PARITY else 1.0) * macs  # FMUL+FADD vs FFMA per MAC
    peak_ops = ctx.sm_count * 128 * sm_mhz * 1e6
    line["roofline"]["fp32_issue"] = {
        "lane_ops_per_launch": int(lane_ops), "achieved_tops": round(lane_ops / (logits_ms / 1e3) / 1e12, 2),
        "peak_tops": round(peak_ops / 1e12, 2), "frac": round(lane_ops / (logits_ms / 1e3) / peak_ops, 4),
        "peak_basis": f"{ctx.sm_count} SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (median SM clock "
                      "in the timed region)"}
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(E, bias, H, scores, args.cpu_seconds)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_extras(ctx, model, idx, Hd, sc, fin, nh, choices, nchoice, hout, args, lsh_value):
    """Same-GPU comparison lines: the full-vocabulary fused path (kFull) and the
    LSH path in the other arithmetic mode."""
    import torch

    from paper_1806_00588_b200 import FAST, PARITY, Batch
    c = CFG
    S, B, d = c["S"], c["B"], c["d"]
    out = {}
    base, step_bytes = Hd.data_ptr(), S * B * d * 4

    def time_batch(b, steps):
        for k in range(2):
            b.step(base + k * step_bytes, sc, fin, nh, choices, nchoice, hout)
        ctx.sync()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.ExternalStream(ctx.stream)
        s.record(st)
        for k in range(steps):
            b.step(base + (k % c["inputs"]) * step_bytes, sc, fin, nh, choices, nchoice, hout)
        e.record(st)
        torch.cuda.synchronize()
        ctx.sync()
        return s.elapsed_time(e) / steps

    for name, mode in [("full_vocab_parity", PARITY), ("full_vocab_fast", FAST)]:
        b = Batch(ctx, model, None, S=S, B=B, specials=[c["V"] - 1], mode=mode, full_vocab=True)
        ms = time_batch(b, 5)
        out[name] = {"ms_per_step": round(ms, 4), "value": round(S / (ms / 1e3), 1),
                     "lsh_speedup": round(lsh_value / (S / (ms / 1e3)), 2)}
        b.close()
    other = FAST if args.mode == "parity" else PARITY
    b = Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"], specials=[c["V"] - 1], mode=other)
    ms = time_batch(b, 50)
    out["lsh_" + ("fast" if other == FAST else "parity")] = {
        "ms_per_step": round(ms, 4), "value": round(S / (ms / 1e3), 1)}
    # chosen-token agreement of FAST (tensor cores / FFMA) with PARITY on the
    # same 50 step inputs: (beam, word) of every choice
    bp = Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"], specials=[c["V"] - 1], mode=PARITY)
    bf = b if other == FAST else Batch(ctx, model, idx, S=S, B=B, T=c["T"], t=c["t"],
                                       specials=[c["V"] - 1], mode=FAST)
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
    # recall@B vs full (SURVEY §8 d): per row, the fraction of the exact
    # full-vocabulary top-B logits (+bias) that the LSH candidate set holds,
    # on the first 4 step inputs. The candidate sets are the reference's own
    # (bit-exact), so this is the reference's recall on the same inputs; for
    # iid random E and H it is near chance (the paper's recall needs trained
    # embeddings; the reference's operating point is acceptance criterion 5).
    from paper_1806_00588_b200.lshbeam import exact_topb
    import numpy as np
    hits = rows = 0
    for k in range(4):
        bp.step(base + k * step_bytes, sc, fin, nh, choices, nchoice, hout)
        ctx.sync()
        ids_exact, _ = exact_topb(ctx, model, base + k * step_bytes, S * B, B, bias=True)
        for s_ in range(S):
            cand = bp.candidates(s_)[0]
            ex = ids_exact[s_ * B:(s_ + 1) * B]
            hits += int(np.isin(ex, cand).sum())
            rows += B
    out["recall_at_B"] = {"value": round(hits / max(rows * B, 1), 4), "rows": rows,
                          "note": "exact full-vocab top-B vs V_LSH, 4 inputs x 768 rows; "
                                  "iid synthetic data: near chance, same as the reference"}
    for bb in {id(bp): bp, id(bf): bf, id(b): b}.values():
        bb.close()
    return out


# ------------------------------------------------------------ reference
def cpu_baseline(E, bias, H, scores, seconds, steps=None):
    """The reference's own CPU step (oracle/_ref) on the host cores, on a
    bounded sample of the same workload."""
    from oracle.oracle import Reference, ReferenceStepper
    from paper_1806_00588_b200.seeds import mix_seed
    c = CFG
    if not Reference.available():
        return {"value": None, "unit": UNIT, "kind": "reference",
                "note": "oracle/_ref not built"}
    ref = Reference()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    En, bn, Hn, scn = E.numpy(), bias.numpy(), H.numpy(), scores.numpy()
    st = ReferenceStepper(ref, En, bn, c["K"], c["u"], c["W"], mix_seed(c["seed"], 1),
                          mix_seed(c["seed"], 2))
    for s in range(2):  # warm-up
        st.step(Hn[0, s], scn[s], c["B"], c["T"], c["t"], [c["V"] - 1])
    n, t0 = 0, time.perf_counter()
    k = 0
    while True:
        for s in range(c["S"]):
            st.step(Hn[k % c["inputs"], s], scn[s], c["B"], c["T"], c["t"], [c["V"] - 1])
            n += 1
        k += 1
        el = time.perf_counter() - t0
        if (steps is not None and k >= steps) or (steps is None and el >= seconds):
            break
    st.close()
    return {"value": round(n / el, 2), "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{k} batch-steps x {c['S']} sentences = {n} sentence-steps of the same "
                      f"workload ({el:.1f} s), reference lshbeam compiled from /root/reference "
                      "sources (g++ -O3 -fopenmp), OMP threads = all host cores"}


def run_reference(args, rank, world, local):
    if rank != 0:
        return
    c = CFG
    E, bias, H, scores = make_inputs(0)
    from oracle.oracle import Reference
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    cb = cpu_baseline(E, bias, H, scores, 0, steps=args.warmup)  # warm-up steps
    t0 = time.perf_counter()
    cb = cpu_baseline(E, bias, H, scores, 0, steps=args.steps)
    wall = time.perf_counter() - t0
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * c["S"] / v, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (torch.randn seed 7; E 40000x1000 fp32)",
            "config": {"workload": "cfg2: batched decode step, 64 sentences x B=12, "
                                   "|V|=40000, d=1000, K=8 u=3 W=16, T=1000, t=2",
                       "parallelism": "host OpenMP"},
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

"""Vocabulary-sharded decode step (BASELINE cfg 4: |V| = 200k, d = 1024).

Rank g of G owns the contiguous vocabulary slice [v_g, v_g + n_g) of E: its
own device copy of that slice, a band index over it built with the global
permutation seed (a word's band codes -- hence its hit counts -- do not
depend on the other words), and a fused-step batch whose top-T prefix and
specials are shifted into the slice. One decode step is the three device
phases of include/lshbeam_b200.h §8 separated by two all-gathers over the
ranks (NCCL over NVLink in production, gloo in the CPU tests):

  phase1 -> all_gather(row max)                       4 B per row per rank
  phase2 -> all_gather(row exp-sum + top-B' lists, one packed buffer)
                                                      8 + 8*B' B per row per rank
  phase3 -> identical choices + hidden reorder on every rank

At S=64, B=12 that is 768 rows x 140 B ~ 105 KB per rank per step: the
exchange is latency-bound, so it is two collectives per step (the minimum
for bit-exact probabilities: exp needs the global max first), batched over
all sentences, the sums and lists travelling in one buffer. The reference has no multi-device path; results equal the
unsharded step bit for bit in PARITY mode (tests/test_gpu_vocab_shard.py).
"""
from __future__ import annotations

import ctypes as C

from . import _native as N
from .lshbeam import PARITY, Batch, Index, Model


def shard_bounds(V: int, G: int, g: int) -> tuple[int, int]:
    """Contiguous split of [0, V): the first V % G ranks take one extra word."""
    base, rem = divmod(V, G)
    n = base + (1 if g < rem else 0)
    v0 = g * base + min(g, rem)
    return v0, n


def local_config(T: int, specials, v0: int, n: int):
    """The slice's view of the global candidate rules: [0, T) becomes
    [0, clamp(T - v0, 0, n)) and specials outside the slice drop out."""
    T_local = max(0, min(T - v0, n))
    sp = sorted({int(s) - v0 for s in specials if v0 <= int(s) < v0 + n})
    return T_local, sp


class VocabShard:
    """One rank's share: slice model + slice index + a batch over the slice.

    ``E_slice`` / ``bias_slice`` are torch CUDA tensors on the context's
    device ([n, d] fp32 / [n] fp32); they are copied into the model."""

    def __init__(self, ctx, E_slice, bias_slice, v0: int, V: int, K: int, u: int, W: int,
                 perm_seed: int, index_seed: int, S: int, B: int, T: int, t: int, specials=(),
                 mode: int = PARITY):
        import torch
        n, d = E_slice.shape
        self.ctx, self.lib = ctx, ctx.lib
        self.v0, self.n, self.V, self.S, self.B = v0, n, V, S, B
        self.model = Model(ctx, None, device_ptrs=(E_slice.data_ptr(),
                                                   bias_slice.data_ptr() if bias_slice is not None else None,
                                                   n, d))
        self.index = Index(ctx, self.model, K=K, u=u, W=W, perm_seed=perm_seed,
                           index_seed=index_seed)
        T_local, sp = local_config(T, specials, v0, n)
        self.batch = Batch(ctx, self.model, self.index, S=S, B=B, T=T_local, t=t, specials=sp,
                           mode=mode)
        self.width = int(self.lib.lsb_shard_width(self.batch.h))
        R = S * B
        dev = torch.device("cuda", ctx.device)
        self.rowmax = torch.empty(R, dtype=torch.float32, device=dev)
        # phase 2's outputs share one buffer (one gather): R row sums (double)
        # then R x B' lsb_shard_top entries ({float, uint32}: 8-byte words)
        self.packed = torch.empty(R * (1 + self.width), dtype=torch.int64, device=dev)
        self.rowsum = self.packed[:R].view(torch.float64)
        self.top = self.packed[R:]

    @staticmethod
    def _state(hidden, scores, finished, n_hyp):
        p = lambda x: x.data_ptr() if x is not None else None
        return N.lsb_state_dev(p(hidden), p(scores), p(finished), p(n_hyp))

    def phase1(self, st):
        N.check(self.lib.lsb_shard_phase1(self.batch.h, C.byref(st), self.rowmax.data_ptr()),
                "lsb_shard_phase1")

    def phase2(self, st, allmax, G: int):
        N.check(self.lib.lsb_shard_phase2(self.batch.h, C.byref(st), allmax.data_ptr(), G,
                                          self.v0, self.rowsum.data_ptr(), self.top.data_ptr()),
                "lsb_shard_phase2")

    def phase3(self, st, allsum, alltop, G: int, choices, n_choices, hidden_out=None):
        out = N.lsb_out_dev(choices.data_ptr(), n_choices.data_ptr(),
                            hidden_out.data_ptr() if hidden_out is not None else None)
        N.check(self.lib.lsb_shard_phase3(self.batch.h, C.byref(st), allsum.data_ptr(),
                                          alltop.data_ptr(), G, C.byref(out)),
                "lsb_shard_phase3")

    def phase3_packed(self, st, allpacked, G: int, choices, n_choices, hidden_out=None):
        out = N.lsb_out_dev(choices.data_ptr(), n_choices.data_ptr(),
                            hidden_out.data_ptr() if hidden_out is not None else None)
        N.check(self.lib.lsb_shard_phase3_packed(self.batch.h, C.byref(st), allpacked.data_ptr(),
                                                 G, C.byref(out)),
                "lsb_shard_phase3_packed")

    def close(self):
        for x in (self.batch, self.index, self.model):
            x.close()


class PeerExchange:
    """The step's exchange over peer memory (lsb_shard_xchg, capi_xchg.cu): an
    exchange area per rank, attached to every other rank's -- through CUDA IPC
    handles across processes (NVLink / NVSwitch between GPUs), or directly for
    shards held by one process -- then ``step`` runs the three phases with
    device-side pushes and sequence-flag waits, no collective per step."""

    def __init__(self, shard: "VocabShard", G: int, rank: int):
        self.shard, self.lib, self.G, self.rank = shard, shard.lib, G, rank
        h = C.c_void_p()
        N.check(self.lib.lsb_shard_xchg_create(shard.batch.h, G, rank, C.byref(h)),
                "lsb_shard_xchg_create")
        self.h = h

    @property
    def area(self) -> int:
        return int(self.lib.lsb_shard_xchg_area(self.h))

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        N.check(self.lib.lsb_shard_xchg_ipc_handle(self.h, buf), "lsb_shard_xchg_ipc_handle")
        return bytes(buf)

    def open_ipc(self, peer: int, handle: bytes):
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        N.check(self.lib.lsb_shard_xchg_open_ipc(self.h, peer, buf), "lsb_shard_xchg_open_ipc")

    def set_peer(self, peer: int, area: int):
        N.check(self.lib.lsb_shard_xchg_set_peer(self.h, peer, C.c_void_p(area)),
                "lsb_shard_xchg_set_peer")

    def connect(self, group=None):
        """Across processes: all-gather the IPC handles once (any backend) and
        open every peer's area."""
        import torch
        import torch.distributed as dist
        mine = torch.frombuffer(bytearray(self.ipc_handle()), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            mine = mine.cuda()
        allh = torch.empty(self.G * 64, dtype=torch.uint8, device=mine.device)
        dist.all_gather_into_tensor(allh, mine, group=group)
        allh = allh.cpu().numpy().tobytes()
        for g in range(self.G):
            if g != self.rank:
                self.open_ipc(g, allh[64 * g:64 * (g + 1)])

    def step(self, hidden, scores, finished, n_hyp, choices, n_choices, hidden_out=None):
        st = self.shard._state(hidden, scores, finished, n_hyp)
        out = N.lsb_out_dev(choices.data_ptr(), n_choices.data_ptr(),
                            hidden_out.data_ptr() if hidden_out is not None else None)
        N.check(self.lib.lsb_shard_step_peer(self.shard.batch.h, self.h, C.byref(st),
                                             self.shard.v0, C.byref(out)),
                "lsb_shard_step_peer")

    def close(self):
        if getattr(self, "h", None):
            self.lib.lsb_shard_xchg_destroy(self.h)
            self.h = None


def _gather(x, G: int, group):
    """all_gather in rank order into a flat buffer (the layout gloo and NCCL
    both accept), viewed as [G, *x.shape]. Under gloo (the CPU tests, or
    ranks sharing one GPU) CUDA tensors travel through host copies."""
    import torch
    import torch.distributed as dist
    src = x.reshape(-1)
    host = x.is_cuda and dist.get_backend(group) == "gloo"
    if host:
        torch.cuda.current_stream(x.device).synchronize()
        src = src.cpu()
    out = torch.empty(G * x.numel(), dtype=x.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    if host:
        out = out.to(x.device)
    return out.view((G,) + tuple(x.shape))


def sharded_step(shard, hidden, scores, finished, n_hyp, choices, n_choices, hidden_out=None,
                 group=None):
    """One vocabulary-sharded step on this rank (torch.distributed must be
    initialised; the shard's context must run on torch's current stream so
    the collectives are ordered after the phases)."""
    import torch
    import torch.distributed as dist
    G = dist.get_world_size(group)
    st = shard._state(hidden, scores, finished, n_hyp)
    shard.phase1(st)
    allmax = _gather(shard.rowmax, G, group)
    shard.phase2(st, allmax, G)
    allpacked = _gather(shard.packed, G, group)
    shard.phase3_packed(st, allpacked, G, choices, n_choices, hidden_out)


def local_sharded_step(shards, hidden, scores, finished, n_hyp, choices, n_choices,
                       hidden_out=None):
    """The same protocol for G shards held by ONE process (one GPU): the
    all-gathers become stacks in rank order. Used by the single-GPU parity
    tests and the 1-GPU cfg-4 bench; every shard writes the same outputs, the
    last one's are kept."""
    import torch
    G = len(shards)
    sts = [s._state(hidden, scores, finished, n_hyp) for s in shards]
    for s, st in zip(shards, sts):
        s.phase1(st)
    allmax = torch.stack([s.rowmax for s in shards])
    for s, st in zip(shards, sts):
        s.phase2(st, allmax, G)
    allpacked = torch.stack([s.packed for s in shards])
    for s, st in zip(shards, sts):
        s.phase3_packed(st, allpacked, G, choices, n_choices, hidden_out)

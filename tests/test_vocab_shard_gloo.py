"""CPU, world_size 2 (gloo): the vocabulary-sharded step protocol
(paper_1806_00588_b200.vocab_shard.sharded_step) across two processes.

Each rank holds an oracle-backed stand-in for its shard (TEST INFRASTRUCTURE:
the three phases restated in numpy from oracle/ pieces, mirroring
capi_shard.cu) and the real orchestration performs the two all-gathers in
rank order over gloo. The combined choices must equal the unsharded oracle
step (src/beam_decoder.cpp:166-289): this pins that the exchanged quantities
(row max, row exp-sum, per-rank top-B' by exp) are sufficient for an exact
result and that both ranks end with identical choices."""
import os
import socket

import numpy as np
import pytest

from paper_1806_00588_b200.vocab_shard import local_config, shard_bounds


def test_shard_bounds_cover_vocab():
    for V in (1, 7, 1000, 200000):
        for G in (1, 2, 3, 8):
            spans = [shard_bounds(V, G, g) for g in range(G)]
            assert spans[0][0] == 0
            assert all(a[0] + a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert spans[-1][0] + spans[-1][1] == V
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def test_local_config():
    assert local_config(1000, [199999], 0, 25000) == (1000, [])
    assert local_config(1000, [199999], 175000, 25000) == (0, [24999])
    assert local_config(30, [5, 25, 40], 20, 20) == (10, [5])


class OracleShard:
    """numpy restatement of one rank's phases (capi_shard.cu)."""

    def __init__(self, o, E, bias, perms, K, u, W, isd, v0, n, S, B, T, t, specials, width):
        self.o, self.v0, self.n, self.S, self.B, self.t = o, v0, n, S, B, t
        self.K, self.u, self.W, self.perms, self.width = K, u, W, perms, width
        self.E, self.bias = E[v0:v0 + n], bias[v0:v0 + n]
        self.T, self.sp = local_config(T, specials, v0, n)
        self.bt = o.band_index_build(o.hash_matrix(self.E, K, u, W, perms=perms), isd)

    def _state(self, hidden, scores, finished, n_hyp):
        return (hidden.numpy(), scores.numpy(), finished.numpy(), n_hyp.numpy())

    def phase1(self, st):
        import torch
        hidden, scores, finished, n_hyp = st
        o, S, B = self.o, self.S, self.B
        self.rows = {}
        rowmax = np.full(S * B, -np.inf, np.float32)
        for s in range(S):
            live = [i for i in range(int(n_hyp[s])) if not finished[s, i]]
            if not live:
                continue
            H = np.ascontiguousarray(hidden[s, live], np.float32)
            if self.t == 0:
                ids, ft = np.arange(self.n, dtype=np.uint32), self.n
            else:
                L = o.lookup_hits(self.bt, o.hash_matrix(H, self.K, self.u, self.W,
                                                         perms=self.perms))
                ids, ft = o.select_candidates(L, self.t)
            ids, _ = o.merge_top_frequent(ids, ft, self.T, self.sp, self.n)
            logits = (o.compute_logits_ids(H, self.E, ids, self.bias) if len(ids)
                      else np.zeros((len(live), 0), np.float32))
            for k, i in enumerate(live):
                self.rows[s * B + i] = (ids, logits[k])
                if len(ids):
                    rowmax[s * B + i] = logits[k].max()
        self.rowmax = torch.from_numpy(rowmax)

    def phase2(self, st, allmax, G):
        import torch
        R = self.S * self.B
        rowsum = np.zeros(R, np.float64)
        top = np.zeros((R, self.width, 2), np.uint32)
        top[:, :, 0] = np.float32(-1.0).view(np.uint32)
        top[:, :, 1] = 0xFFFFFFFF
        m_all = allmax.numpy().max(axis=0)
        for row, (ids, lg) in self.rows.items():
            e64 = np.exp(lg.astype(np.float64) - np.float64(m_all[row]))
            rowsum[row] = e64.sum()
            e = e64.astype(np.float32)
            order = np.lexsort((ids, -e))[: self.width]  # e desc, word asc
            top[row, : len(order), 0] = e[order].view(np.uint32)
            top[row, : len(order), 1] = ids[order] + self.v0
        self.rowsum = torch.from_numpy(rowsum)
        self.top = torch.from_numpy(top.reshape(-1).view(np.int64).copy())
        # the one-gather layout of VocabShard.packed: R sums, then R x B' entries
        self.packed = torch.cat([self.rowsum.view(torch.int64), self.top])

    def phase3_packed(self, st, allpacked, G, choices, n_choices, hidden_out=None):
        import torch
        R = self.S * self.B
        ap = allpacked.reshape(G, -1)
        self.phase3(st, ap[:, :R].contiguous().view(torch.float64), ap[:, R:].contiguous(), G,
                    choices, n_choices, hidden_out)

    def phase3(self, st, allsum, alltop, G, choices, n_choices, hidden_out=None):
        hidden, scores, finished, n_hyp = st
        S, B = self.S, self.B
        tops = alltop.numpy().reshape(G, S * B, self.width).view(np.uint32).reshape(
            G, S * B, self.width, 2)
        sums = allsum.numpy()
        out = []
        for s in range(S):
            pool = [(float(scores[s, i]), i, -1) for i in range(int(n_hyp[s])) if finished[s, i]]
            for i in range(int(n_hyp[s])):
                row = s * B + i
                if finished[s, i]:
                    continue
                denom = 0.0
                for g in range(G):
                    denom += sums[g, row]
                inv = np.float32(1.0 / denom)
                ent = tops[:, row].reshape(-1, 2)
                e = ent[:, 0].view(np.float32)
                ok = e >= 0
                p = (e[ok] * inv).astype(np.float32)
                w = ent[ok, 1]
                order = np.lexsort((w, -p))[:B]
                pool += [(float(scores[s, i]) + np.log(np.float64(p[k])), i, int(w[k]))
                         for k in order]
            pool.sort(key=lambda c: (-c[0], c[1], c[2]))
            out.append(pool[:B])
        self.result = out


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle, oracle_step
    from paper_1806_00588_b200.vocab_shard import sharded_step
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        V, d, K, u, W, S, B, T, t = 1200, 32, 8, 3, 16, 3, 6, 40, 2
        E = o.gaussian(31, V * d).reshape(V, d)
        bias = o.synth_model(V, d, 31, 6.0, want=("bias",))["bias"]
        ps, isd = o.mix_seed(31, 1), o.mix_seed(31, 2)
        perms = o.generate_perms(d, u * W, K, ps)
        hidden = o.gaussian(o.mix_seed(31, 3), S * B * d).reshape(S, B, d)
        rng = np.random.default_rng(5)
        scores = -rng.random((S, B)) * 3
        finished = np.zeros((S, B), np.uint8)
        finished[:, 2] = 1
        n_hyp = np.array([B, B - 1, 2], np.int32)
        specials = [V - 1, 700]
        v0, n = shard_bounds(V, world, rank)
        shard = OracleShard(o, E, bias, perms, K, u, W, isd, v0, n, S, B, T, t, specials, B + 4)
        T_ = torch.from_numpy
        sharded_step(shard, T_(hidden), T_(scores), T_(finished), T_(n_hyp), None, None)
        got = shard.result
        bt = o.band_index_build(o.hash_matrix(E, K, u, W, perms=perms), isd)
        ok = True
        for s in range(S):
            want = oracle_step(o, bt, perms, E, bias, K, u, W, hidden[s], scores[s], finished[s],
                               int(n_hyp[s]), B, T, t, specials)
            ws, wb, ww = want["choices"]
            g = got[s]
            ok &= [c[2] for c in g] == ww.tolist()
            ok &= [c[1] for c in g] == wb.tolist()
            ok &= np.array_equal(np.array([c[0] for c in g]), ws)
        q.put((rank, bool(ok), [[c[2] for c in g] for g in got]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_protocol():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert res[0][2] == res[1][2]  # both ranks chose the same words

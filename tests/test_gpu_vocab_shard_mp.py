"""Vocabulary-sharded step across PROCESSES running the real CUDA phases
(capi_shard.cu): 2 ranks over gloo, both on cuda:0 (this run has one GPU; the
protocol is the one bench.py drives over NCCL on 2-8 GPUs). Every rank's
choices must equal the unsharded fused step's on the same inputs (SURVEY
§8(e); BASELINE cfg 4 shape scaled down)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

V, D, K, U, W, S, B, T, TT = 12000, 64, 8, 3, 16, 4, 12, 300, 2


def _inputs():
    import torch
    g = torch.Generator().manual_seed(17)
    E = torch.randn(V, D, generator=g)
    bias = torch.randn(V, generator=g) * 2.0
    H = torch.randn(S, B, D, generator=g)
    scores = -torch.rand(S, B, generator=g, dtype=torch.float64) * 3.0
    finished = torch.zeros(S, B, dtype=torch.uint8)
    finished[:, 3] = 1
    n_hyp = torch.tensor([B, B - 2, 5, B], dtype=torch.int32)
    return E, bias, H, scores, finished, n_hyp


def _worker(rank, world, port, q, peer=False):
    import torch
    import torch.distributed as dist

    from paper_1806_00588_b200 import Context
    from paper_1806_00588_b200.seeds import mix_seed
    from paper_1806_00588_b200.vocab_shard import VocabShard, shard_bounds, sharded_step
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ctx = Context(0, torch.cuda.current_stream().cuda_stream)
        E, bias, H, scores, finished, n_hyp = _inputs()
        v0, n = shard_bounds(V, world, rank)
        shard = VocabShard(ctx, E[v0:v0 + n].cuda().contiguous(), bias[v0:v0 + n].cuda(), v0, V,
                           K, U, W, mix_seed(7, 1), mix_seed(7, 2), S, B, T, TT,
                           specials=[V - 1, 5000])
        dev = torch.device("cuda", 0)
        ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
        nc = torch.zeros(S, dtype=torch.int32, device=dev)
        ho = torch.zeros(S, B, D, device=dev)
        if peer:
            # peer-memory exchange: CUDA IPC areas, handles all-gathered once
            from paper_1806_00588_b200.vocab_shard import PeerExchange
            x = PeerExchange(shard, world, rank)
            x.connect()
            dist.barrier()
            for _ in range(2):  # two steps: the sequence flags advance
                x.step(H.cuda(), scores.cuda(), finished.cuda(), n_hyp.cuda(), ch, nc, ho)
                ctx.sync()
            dist.barrier()  # no peer may still push into our area
            x.close()
        else:
            sharded_step(shard, H.cuda(), scores.cuda(), finished.cuda(), n_hyp.cuda(), ch, nc,
                         ho)
        ctx.sync()
        q.put((rank, ch.cpu().numpy().tobytes(), nc.cpu().numpy().tolist(),
               ho.cpu().numpy().tobytes()))
        shard.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("peer", [False, True])
def test_two_process_vocab_sharded_cuda_step(ctx, peer):
    import torch
    import torch.multiprocessing as mp

    from paper_1806_00588_b200 import Batch, Index, Model
    from paper_1806_00588_b200.seeds import mix_seed
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_worker, args=(r, 2, port, q, peer)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    # the unsharded fused step on the same inputs
    E, bias, H, scores, finished, n_hyp = _inputs()
    m = Model(ctx, E.numpy(), bias.numpy())
    idx = Index(ctx, m, K=K, u=U, W=W, perm_seed=mix_seed(7, 1), index_seed=mix_seed(7, 2))
    b = Batch(ctx, m, idx, S=S, B=B, T=T, t=TT, specials=[V - 1, 5000])
    got, hout = b.step_host(H.numpy(), scores.numpy(), finished.numpy(), n_hyp.numpy(),
                            want_hidden=True)
    want = [[(c[0], c[1], c[2]) for c in got[s]] for s in range(S)]
    for rank, chb, ncl, hob in res:
        dt = np.dtype([("score", "<f8"), ("beam", "<u4"), ("pad", "<u4"), ("word", "<i8")])
        ch = np.frombuffer(chb, dt).reshape(S, B)
        ho = np.frombuffer(hob, np.float32).reshape(S, B, D)
        for s in range(S):
            assert ncl[s] == len(want[s])
            for k, (score, beam, word) in enumerate(want[s]):
                c = ch[s, k]
                assert (c["score"], c["beam"], c["word"]) == (score, beam, word), (rank, s, k)
                np.testing.assert_array_equal(ho[s, k], hout[s, k])
    for x in (b, idx, m):
        x.close()

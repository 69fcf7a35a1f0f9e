"""Vocabulary-sharded step (BASELINE cfg 4 protocol, include/lshbeam_b200.h §8)
on one GPU: G shards in one process exchange through stacked tensors in rank
order (vocab_shard.local_sharded_step). PARITY results must equal the
unsharded fused step -- which test_gpu_step.py pins to the oracle -- bit for
bit: choices (score, beam, word), counts and the hidden reorder."""
import numpy as np
import pytest

from test_gpu_step import make_state, make_world

pytestmark = pytest.mark.gpu


def _state_tensors(state, dev):
    import torch
    hidden, scores, finished, n_hyp = state
    return (torch.from_numpy(np.ascontiguousarray(hidden)).to(dev),
            torch.from_numpy(np.ascontiguousarray(scores)).to(dev),
            torch.from_numpy(np.ascontiguousarray(finished)).to(dev),
            torch.from_numpy(np.ascontiguousarray(n_hyp)).to(dev))


@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("V,d,K,u,W,S,B,T,t", [
    (3000, 64, 8, 3, 16, 3, 12, 100, 2),
    (2500, 40, 4, 2, 20, 2, 5, 10, 3),
    (2000, 64, 8, 3, 16, 2, 8, 0, 0),
])
def test_sharded_equals_unsharded(oracle, V, d, K, u, W, S, B, T, t, G):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_00588_b200 import Batch, Context, Index, Model
    from paper_1806_00588_b200.vocab_shard import VocabShard, local_sharded_step, shard_bounds

    dev = torch.device("cuda", 0)
    ctx = Context(0, torch.cuda.current_stream().cuda_stream)
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=V + d,
                                             bias_strength=8.0)
    state = make_state(oracle, S, B, d, seed=V + 1, frozen_every=3, short=B // 2)
    hid, sc, fin, nh = _state_tensors(state, dev)
    specials = [V - 1, V // 2]

    # unsharded reference run
    m = Model(ctx, E, bias)
    idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=ps, index_seed=isd)
    full = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=specials)
    ch0 = torch.zeros(S * B * 3, dtype=torch.int64, device=dev)
    nc0 = torch.zeros(S, dtype=torch.int32, device=dev)
    ho0 = torch.zeros(S, B, d, device=dev)
    full.step(hid, sc, fin, nh, ch0, nc0, ho0)

    Et = torch.from_numpy(E).to(dev)
    bt_ = torch.from_numpy(bias).to(dev)
    shards = []
    for g in range(G):
        v0, n = shard_bounds(V, G, g)
        shards.append(VocabShard(ctx, Et[v0:v0 + n].contiguous(), bt_[v0:v0 + n].contiguous(),
                                 v0, V, K, u, W, ps, isd, S, B, T, t, specials))
    ch = torch.zeros_like(ch0)
    nc = torch.zeros_like(nc0)
    ho = torch.zeros_like(ho0)
    local_sharded_step(shards, hid, sc, fin, nh, ch, nc, ho)
    ctx.sync()
    assert torch.equal(nc, nc0)
    # lsb_choice = {double score, u32 beam, u32 pad, i64 word}: compare all 24 bytes
    assert torch.equal(ch, ch0)
    assert torch.equal(ho, ho0)
    # the union of the shards' candidate sets is the unsharded set
    for s in range(S):
        want, _ = full.candidates(s)
        got = np.concatenate([sh.v0 + sh.batch.candidates(s)[0] for sh in shards])
        np.testing.assert_array_equal(np.sort(got), want)
    for sh in shards:
        sh.close()


def test_peer_exchange_in_one_process():
    """Runs the in-process peer-exchange cases below in a subprocess with eager
    CUDA module loading: shards sharing one process (one CUDA context) must
    not load a kernel lazily while their own flag-wait kernel spins for a
    shard the same host thread has not launched yet."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_vocab_shard.py"), "-k",
                        "peer_exchange_equals_unsharded", "--run-peer-inprocess"],
                       env={**os.environ, "CUDA_MODULE_LOADING": "EAGER"}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "skipped" not in r.stdout.splitlines()[-1], r.stdout[-500:]


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("V,d,K,u,W,S,B,T,t", [
    (3000, 64, 8, 3, 16, 3, 12, 100, 2),
    (2000, 64, 8, 3, 16, 2, 8, 0, 0),
])
def test_peer_exchange_equals_unsharded(oracle, V, d, K, u, W, S, B, T, t, G, request):
    """The exchange over peer memory (lsb_shard_step_peer: device pushes into
    the other shards' areas + sequence-flag waits, no collectives), G shards in
    one process on their own streams, over several steps so the flags advance:
    every shard's choices / counts / hidden reorder equal the unsharded step's."""
    import os

    import torch
    if not request.config.getoption("--run-peer-inprocess") or \
            os.environ.get("CUDA_MODULE_LOADING") != "EAGER":
        pytest.skip("run through test_peer_exchange_in_one_process (eager module loading)")
    from paper_1806_00588_b200 import Batch, Context, Index, Model
    from paper_1806_00588_b200.vocab_shard import PeerExchange, VocabShard, shard_bounds

    dev = torch.device("cuda", 0)
    ctx = Context(0, torch.cuda.current_stream().cuda_stream)
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=V + d,
                                             bias_strength=8.0)
    specials = [V - 1, V // 2]
    m = Model(ctx, E, bias)
    idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=ps, index_seed=isd)
    full = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=specials)
    Et = torch.from_numpy(E).to(dev)
    bt_ = torch.from_numpy(bias).to(dev)
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs = [Context(0, st.cuda_stream) for st in streams]
    shards, xs = [], []
    for g in range(G):
        v0, n = shard_bounds(V, G, g)
        shards.append(VocabShard(ctxs[g], Et[v0:v0 + n].contiguous(), bt_[v0:v0 + n].contiguous(),
                                 v0, V, K, u, W, ps, isd, S, B, T, t, specials))
        xs.append(PeerExchange(shards[g], G, g))
    for g in range(G):
        for p in range(G):
            if p != g:
                xs[g].set_peer(p, xs[p].area)
    torch.cuda.synchronize()
    for step in range(3):
        state = make_state(oracle, S, B, d, seed=V + 1 + step, frozen_every=3, short=B // 2)
        hid, sc, fin, nh = _state_tensors(state, dev)
        ch0 = torch.zeros(S * B * 3, dtype=torch.int64, device=dev)
        nc0 = torch.zeros(S, dtype=torch.int32, device=dev)
        ho0 = torch.zeros(S, B, d, device=dev)
        full.step(hid, sc, fin, nh, ch0, nc0, ho0)
        ctx.sync()
        outs = [(torch.zeros_like(ch0), torch.zeros_like(nc0), torch.zeros_like(ho0))
                for _ in range(G)]
        torch.cuda.synchronize()
        for g in range(G):  # enqueue every shard's step; they meet on the device
            xs[g].step(hid, sc, fin, nh, *outs[g])
        for c in ctxs:
            c.sync()
        for g in range(G):
            ch, nc, ho = outs[g]
            assert torch.equal(nc, nc0), (step, g)
            assert torch.equal(ch, ch0), (step, g)
            assert torch.equal(ho, ho0), (step, g)
    for x in xs:
        x.close()
    for sh in shards:
        sh.close()

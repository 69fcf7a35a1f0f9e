"""Fused step parity: lsb_step over S sentences vs the oracle's restatement of
decode()'s kLsh / kFull step body (src/beam_decoder.cpp:166-289), sentence by
sentence, on identical seeded inputs. Codes, candidate lists, provenance and
chosen (score, beam, word) triples are compared exactly in PARITY mode."""
import numpy as np
import pytest

from oracle.oracle import oracle_full_step, oracle_step

pytestmark = pytest.mark.gpu


def make_world(o, V, d, K, u, W, seed=7, bias_strength=0.0):
    E = o.gaussian(seed, V * d).reshape(V, d)
    m = o.synth_model(V, d, seed, bias_strength, want=("bias",))
    perm_seed, index_seed = o.mix_seed(seed, 1), o.mix_seed(seed, 2)
    perms = o.generate_perms(d, u * W, K, perm_seed)
    codes = o.hash_matrix(E, K, u, W, perms=perms)
    bt = o.band_index_build(codes, index_seed)
    return E, m["bias"], perms, bt, perm_seed, index_seed


def make_state(o, S, B, d, seed, frozen_every=0, short=0):
    hidden = o.gaussian(o.mix_seed(seed, 3), S * B * d).reshape(S, B, d)
    rng = np.random.default_rng(seed)
    scores = -rng.random((S, B)) * 4.0
    finished = np.zeros((S, B), np.uint8)
    n_hyp = np.full(S, B, np.int32)
    if frozen_every:
        finished[:, ::frozen_every] = 1
        finished[:, 1] = 0
    if short:
        n_hyp[::2] = short
    return hidden, scores, finished, n_hyp


def run_gpu(ctx, E, bias, V, d, K, u, W, perm_seed, index_seed, S, B, T, t, specials, state,
            mode=0, full=False):
    from paper_1806_00588_b200 import Batch, Index, Model
    m = Model(ctx, E, bias)
    idx = None if full else Index(ctx, m, K=K, u=u, W=W, perm_seed=perm_seed,
                                  index_seed=index_seed)
    b = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=specials, mode=mode, full_vocab=full)
    b.keep_probs(True)
    hidden, scores, finished, n_hyp = state
    res, hout = b.step_host(hidden, scores, finished, n_hyp, want_hidden=True)
    return b, res, hout


CASES = [
    # V, d, K, u, W, S, B, T, t
    (4000, 64, 8, 3, 16, 4, 12, 100, 2),
    (4000, 64, 8, 3, 16, 3, 12, 0, 1),
    (3000, 40, 4, 2, 20, 2, 5, 10, 3),
    (2000, 64, 8, 3, 100, 2, 12, 0, 0),
    (5000, 1003, 16, 3, 32, 2, 7, 50, 1),
    (1500, 256, 16, 3, 300, 2, 12, 25, 5),
    # large beams: K5a threshold over 128 lane maxima (B > 32), rows of
    # > 2048 candidates in registers, K5b head pruning (B > 16)
    (6000, 64, 8, 3, 16, 2, 50, 2200, 2),
    (4000, 64, 4, 2, 8, 2, 24, 100, 1),
    # rows longer than the register path (n > 3072): global threshold path
    (8000, 64, 8, 3, 16, 2, 12, 4000, 2),
    # few rows x many bands with long spans (4-bit codes over 20k words):
    # the band-split probe (k_probe_split, 16-bit counters in L2)
    (20000, 32, 4, 2, 100, 2, 12, 100, 3),
    (12000, 48, 4, 2, 80, 1, 7, 40, 5),
    # t = 0 over V >= 8192: every row is the whole vocabulary -> segmented K5a
    (9000, 32, 8, 3, 16, 2, 6, 0, 0),
    (12000, 16, 4, 2, 8, 1, 40, 0, 0),
]


@pytest.mark.parametrize("V,d,K,u,W,S,B,T,t", CASES)
@pytest.mark.parametrize("frozen", [False, True])
def test_step_matches_oracle(ctx, oracle, V, d, K, u, W, S, B, T, t, frozen):
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=V + d,
                                             bias_strength=8.0)
    specials = [V - 1]
    state = make_state(oracle, S, B, d, seed=V * 3 + d, frozen_every=3 if frozen else 0,
                       short=(B // 2 if frozen else 0))
    b, res, hout = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, specials, state)
    hidden, scores, finished, n_hyp = state
    for s in range(S):
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], int(n_hyp[s]), B, T, t, specials)
        ids, prov = b.candidates(s)
        np.testing.assert_array_equal(ids, want["ids"])
        assert prov == want["prov"]
        codes = b.query_codes(s, W)[want["live"]]
        np.testing.assert_array_equal(codes, want["codes"])
        probs = b.probs(s)
        np.testing.assert_array_equal(probs.view(np.uint32), want["probs"].view(np.uint32))
        ws, wb, ww = want["choices"]
        assert len(res[s]) == len(ws)
        got = np.array([c[2] for c in res[s]]), np.array([c[1] for c in res[s]])
        np.testing.assert_array_equal(got[0], ww)
        np.testing.assert_array_equal(got[1], wb)
        np.testing.assert_array_equal(np.array([c[0] for c in res[s]]), ws)
        for k, (_, beam, _) in enumerate(res[s]):  # hidden-state reorder
            np.testing.assert_array_equal(hout[s, k], hidden[s, beam])


# The opt-in single-launch step for small batches (k_step_fused.cu,
# LSB_FUSED=1): the same device functions as the separate kernels in one
# cooperative launch, with the probe split into more vocabulary slices.
FUSED_CASES = [
    # V, d, K, u, W, S, B, T, t
    (4000, 64, 8, 3, 16, 4, 12, 100, 2),
    (4000, 64, 8, 3, 16, 3, 12, 0, 1),
    (4000, 64, 4, 2, 8, 2, 8, 100, 1),
    (8000, 64, 8, 3, 16, 2, 12, 4000, 2),
    (6000, 100, 16, 3, 24, 1, 12, 50, 12),  # t > 8: byte counters
]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("V,d,K,u,W,S,B,T,t", FUSED_CASES)
@pytest.mark.parametrize("frozen", [False, True])
def test_fused_small_step_matches_oracle(ctx, oracle, monkeypatch, mode, V, d, K, u, W, S, B, T,
                                         t, frozen):
    from paper_1806_00588_b200 import Batch, Index, Model
    monkeypatch.setenv("LSB_FUSED", "1")
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=V + d,
                                             bias_strength=8.0)
    specials = [V - 1]
    state = make_state(oracle, S, B, d, seed=V * 3 + d, frozen_every=3 if frozen else 0,
                       short=(B // 2 if frozen else 0))
    m = Model(ctx, E, bias)
    idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=ps, index_seed=isd)
    b = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=specials, mode=mode)
    b.keep_probs(True)
    hidden, scores, finished, n_hyp = state
    n0 = ctx.launches
    res, hout = b.step_host(hidden, scores, finished, n_hyp, want_hidden=True)
    assert ctx.launches - n0 == 1  # the whole step is one launch
    for s in range(S):
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], int(n_hyp[s]), B, T, t, specials)
        ids, prov = b.candidates(s)
        np.testing.assert_array_equal(ids, want["ids"])
        assert prov == want["prov"]
        np.testing.assert_array_equal(b.query_codes(s, W)[want["live"]], want["codes"])
        if mode == 0:
            np.testing.assert_array_equal(b.probs(s).view(np.uint32),
                                          want["probs"].view(np.uint32))
        ws, wb, ww = want["choices"]
        if mode == 0:
            assert [c[2] for c in res[s]] == ww.tolist()
            assert [c[1] for c in res[s]] == wb.tolist()
            np.testing.assert_array_equal(np.array([c[0] for c in res[s]]), ws)
        for k, (_, beam, _) in enumerate(res[s]):
            np.testing.assert_array_equal(hout[s, k], hidden[s, beam])
    # and bit-for-bit the separate kernels' step (FAST included)
    monkeypatch.setenv("LSB_FUSED", "0")
    b2 = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=specials, mode=mode)
    b2.keep_probs(True)
    res2, hout2 = b2.step_host(hidden, scores, finished, n_hyp, want_hidden=True)
    assert res2 == res
    np.testing.assert_array_equal(hout2.view(np.uint32), hout.view(np.uint32))
    for s in range(S):
        np.testing.assert_array_equal(b2.probs(s).view(np.uint32), b.probs(s).view(np.uint32))
    b.close()
    b2.close()


@pytest.mark.parametrize("seq", ["1"])
@pytest.mark.parametrize("V,d,K,u,W,S,B,T,t", [CASES[0], CASES[6], CASES[8]])
def test_step_sequential_denominator(ctx, oracle, monkeypatch, V, d, K, u, W, S, B, T, t, seq):
    """The softmax denominator's rare path (softmax_denom.cuh: the
    sequential sum, when the tree sum cannot certify float(1/denom)) forced
    on every row (LSB_SEQ_DENOM=1): the step still equals the oracle bit for
    bit."""
    monkeypatch.setenv("LSB_SEQ_DENOM", seq)
    test_step_matches_oracle(ctx, oracle, V, d, K, u, W, S, B, T, t, True)


def test_step_config1_shape(ctx, oracle):
    """BASELINE config 1 shapes: V=40k, d=1000, B=12, K=8, u=3, W=16, T=1000, t=2."""
    V, d, K, u, W, B, T, t, S = 40000, 1000, 8, 3, 16, 12, 1000, 2, 2
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=7)
    state = make_state(oracle, S, B, d, seed=7)
    b, res, _ = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    hidden, scores, finished, n_hyp = state
    for s in range(S):
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], B, B, T, t, [V - 1])
        ids, prov = b.candidates(s)
        np.testing.assert_array_equal(ids, want["ids"])
        ws, wb, ww = want["choices"]
        assert [c[2] for c in res[s]] == ww.tolist()
        assert [c[1] for c in res[s]] == wb.tolist()
        np.testing.assert_array_equal(np.array([c[0] for c in res[s]]), ws)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("V,d,S,B", [
    (3000, 64, 3, 6),
    # >= 2 row groups over a >= 4096-column identity block: the PARITY
    # one-lane-per-thread kernel (k_logits_ln.cu), RT = 12 / 10 / 6
    (6000, 64, 4, 12), (5000, 128, 3, 10), (4100, 40, 5, 6),
    # V >= 8192: segmented K5a (P segments per row, last CTA merges)
    (9000, 64, 1, 12), (20000, 32, 3, 8)])
@pytest.mark.parametrize("seq", ["0", "1"])
def test_full_vocab_step(ctx, oracle, monkeypatch, mode, V, d, S, B, seq):
    """kFull vs the oracle: choices, and in PARITY every probability bit for
    bit (the segmented K5a's certified denominator; seq=1 forces its
    sequential sum on every row)."""
    monkeypatch.setenv("LSB_SEQ_DENOM", seq)
    E = oracle.gaussian(11, V * d).reshape(V, d)
    bias = oracle.synth_model(V, d, 11, 8.0, want=("bias",))["bias"]
    state = make_state(oracle, S, B, d, seed=5, frozen_every=4)
    b, res, _ = run_gpu(ctx, E, bias, V, d, 8, 3, 16, 1, 2, S, B, 0, 0, [V - 1], state,
                        mode=mode, full=True)
    hidden, scores, finished, n_hyp = state
    for s in range(S):
        want = oracle_full_step(oracle, E, bias, hidden[s], scores[s], finished[s], B, B)
        if mode == 0:
            np.testing.assert_array_equal(b.probs(s).view(np.uint32),
                                          want["probs"].view(np.uint32))
        ws, wb, ww = want["choices"]
        assert [c[2] for c in res[s]] == ww.tolist()
        assert [c[1] for c in res[s]] == wb.tolist()
        if mode == 0:
            np.testing.assert_array_equal(np.array([c[0] for c in res[s]]), ws)
        else:
            np.testing.assert_allclose(np.array([c[0] for c in res[s]]), ws, rtol=1e-5)


def test_step_parity_under_lane_kernel():
    """The LSH step with every PARITY logits launch forced onto the
    one-lane-per-thread kernel (LSB_K4_LN=2: shared block + survivor jobs) is
    bit-identical to the oracle, like the default tiles."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_step.py"), "-k",
                        "test_step_matches_oracle or test_step_config1_shape"],
                       env={**os.environ, "LSB_K4_LN": "2"}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_step_parity_unsplit_probe():
    """The same step tests with the band-split probe off (LSB_PROBE_SPLIT=0:
    k_probe_count for every row count), so both K1+K2 kernels stay covered."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_step.py"), "-k",
                        "test_step_matches_oracle or test_graph_replay"],
                       env={**os.environ, "LSB_PROBE_SPLIT": "0"}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_step_nan_hidden_rejected(ctx, oracle):
    V, d, K, u, W, S, B = 500, 16, 4, 2, 8, 1, 2
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W)
    hidden, scores, finished, n_hyp = make_state(oracle, S, B, d, seed=3)
    hidden[0, 1, 3] = np.nan
    with pytest.raises(ValueError):
        run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, 10, 1, [V - 1],
                (hidden, scores, finished, n_hyp))


def test_batch_config_validation(ctx, oracle):
    from paper_1806_00588_b200 import Batch, Index, Model
    V, d = 300, 16
    E = oracle.gaussian(1, V * d).reshape(V, d)
    m = Model(ctx, E)
    idx = Index(ctx, m, K=4, u=2, W=20, perm_seed=5, index_seed=6)
    with pytest.raises(ValueError):
        Batch(ctx, m, idx, S=1, B=0)
    with pytest.raises(ValueError):
        Batch(ctx, m, idx, S=1, B=4, T=301)
    with pytest.raises(ValueError):
        Batch(ctx, m, idx, S=1, B=4, t=21)
    with pytest.raises(ValueError):
        Batch(ctx, m, idx, S=1, B=4, specials=[300])
    with pytest.raises(ValueError):
        Batch(ctx, m, None, S=1, B=4)  # lsh mode requires an index


def test_step_host_async_matches_sync(ctx, oracle):
    """The pipelined host-buffer API (two staging slots, copy stream) gives the
    same choices as the synchronous one over a sequence of distinct steps."""
    import ctypes as C

    import torch
    from paper_1806_00588_b200 import _native as N
    V, d, K, u, W, S, B, T, t = 3000, 64, 8, 3, 16, 4, 12, 100, 2
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=21, bias_strength=4.0)
    from paper_1806_00588_b200 import Batch, Index, Model
    m = Model(ctx, E, bias)
    idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=ps, index_seed=isd)
    b = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=[V - 1])
    steps = 5
    states = [make_state(oracle, S, B, d, seed=100 + k, frozen_every=3 if k % 2 else 0)
              for k in range(steps)]
    want = [b.step_host(*st)[0] for st in states]
    pinned = []
    outs = []
    for st in states:
        hidden, scores, finished, n_hyp = (torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
                                           for x in st)
        ch = (N.lsb_choice * (S * B))()
        nc = np.zeros(S, np.int32)
        pinned.append((hidden, scores, finished, n_hyp))
        outs.append((ch, nc))
        b.step_host_async(hidden.data_ptr(), scores.data_ptr(), finished.data_ptr(),
                          n_hyp.data_ptr(), ch, nc.ctypes.data_as(C.c_void_p))
    b.wait()
    for k in range(steps):
        ch, nc = outs[k]
        got = [[(ch[s * B + j].score, ch[s * B + j].beam, ch[s * B + j].word)
                for j in range(int(nc[s]))] for s in range(S)]
        assert got == want[k]


@pytest.mark.parametrize("seed", range(40))
def test_step_fuzz(ctx, oracle, seed):
    """Random shapes across every kernel variant the step picks: many bands
    (W > 64: the phased probe), large beams (threshold top-B for B > 32, K5b
    head pruning for B > 16), rows longer than the register path, odd d,
    small and larger batches (32-column K4 tiles or 128-column ones), frozen
    and short hypotheses. Everything compared exactly (PARITY)."""
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.integers(300, 6000))
    d = int(rng.choice([16, 33, 64, 67, 128]))
    K = int(rng.choice([2, 4, 8, 16]))
    u = int(rng.integers(1, 4))
    W = int(rng.choice([4, 16, 40, 80, 200]))
    S = int(rng.choice([1, 3, 9, 24]))
    B = int(rng.choice([1, 3, 12, 20, 40]))
    T = int(rng.choice([0, 10, V // 3, V // 2, V]))
    t = int(rng.integers(1, 5))
    frozen = bool(rng.integers(0, 2)) and B > 2
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=seed + 17,
                                             bias_strength=float(rng.choice([0.0, 8.0])))
    specials = sorted({V - 1, int(rng.integers(0, V))})
    state = make_state(oracle, S, B, d, seed=seed * 7 + 1, frozen_every=3 if frozen else 0,
                       short=(B // 2 if frozen else 0))
    b, res, hout = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, specials, state)
    hidden, scores, finished, n_hyp = state
    for s in range(S):
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], int(n_hyp[s]), B, T, t, specials)
        ids, prov = b.candidates(s)
        np.testing.assert_array_equal(ids, want["ids"])
        assert prov == want["prov"]
        probs = b.probs(s)
        np.testing.assert_array_equal(probs.view(np.uint32), want["probs"].view(np.uint32))
        ws, wb, ww = want["choices"]
        assert len(res[s]) == len(ws)
        np.testing.assert_array_equal(np.array([c[2] for c in res[s]]), ww)
        np.testing.assert_array_equal(np.array([c[1] for c in res[s]]), wb)
        np.testing.assert_array_equal(np.array([c[0] for c in res[s]]), ws)
        for k, (_, beam, _) in enumerate(res[s]):
            np.testing.assert_array_equal(hout[s, k], hidden[s, beam])


@pytest.mark.parametrize("full", [False, True])
def test_fast_step_tensor_cores(ctx, oracle, full):
    """FAST with enough rows for the tcgen05 block: the top-T shared block on
    the side stream beside the survivor FFMA tiles (LSH, >= 256 rows), or the
    whole vocabulary (full, >= 64 rows). Candidates are exact; probabilities
    and scores within FAST's tolerance; choices agree except at near-ties."""
    V, d, K, u, W = 4000, 64, 8, 3, 16
    S, B, T, t = (32, 12, 1000, 2) if not full else (12, 6, 0, 0)
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=23, bias_strength=8.0)
    state = make_state(oracle, S, B, d, seed=29)
    b, res, _ = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state,
                        mode=1, full=full)
    hidden, scores, finished, n_hyp = state
    agree = total = 0
    for s in range(S):
        if full:
            want = oracle_full_step(oracle, E, bias, hidden[s], scores[s], finished[s], B, B)
        else:
            want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                               finished[s], int(n_hyp[s]), B, T, t, [V - 1])
            ids, prov = b.candidates(s)
            np.testing.assert_array_equal(ids, want["ids"])
            np.testing.assert_allclose(b.probs(s), want["probs"], rtol=2e-3, atol=1e-6)
        ws, wb, ww = want["choices"]
        got = [(c[1], c[2]) for c in res[s]]
        agree += sum(g == (int(x), int(y)) for g, x, y in zip(got, wb, ww))
        total += len(ws)
        np.testing.assert_allclose(np.array([c[0] for c in res[s]]), ws, rtol=0, atol=1e-3)
    assert agree >= 0.99 * total, (agree, total)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("mode", [0, 1])
def test_graph_replay_equals_step(oracle, monkeypatch, mode, fused):
    """lsb_batch_graph_capture / _launch: a replayed step on the captured
    buffers gives the eager step's choices, candidates and hidden reorder,
    also after the buffers are rewritten in place (the decode-loop pattern).
    fused: the captured step is the single cooperative launch (LSB_FUSED=1)."""
    import torch
    monkeypatch.setenv("LSB_FUSED", "1" if fused else "0")

    from paper_1806_00588_b200 import Batch, Context, Index, Model
    s = torch.cuda.Stream()
    ctx = Context(0, s.cuda_stream)
    V, d, K, u, W, S, B, T, t = 6000, 64, 8, 3, 16, 3, 12, 200, 2
    E, bias, perms, bt, ps, isd = make_world(oracle, V, d, K, u, W, seed=21, bias_strength=4.0)
    m = Model(ctx, E, bias)
    idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=ps, index_seed=isd)
    b = Batch(ctx, m, idx, S=S, B=B, T=T, t=t, specials=[V - 1], mode=mode)
    dev = torch.device("cuda", 0)
    states = [make_state(oracle, S, B, d, seed=k, frozen_every=3 if k else 0) for k in range(3)]
    H = torch.zeros(S, B, d, device=dev)
    sc = torch.zeros(S, B, dtype=torch.float64, device=dev)
    fin = torch.zeros(S, B, dtype=torch.uint8, device=dev)
    nh = torch.zeros(S, dtype=torch.int32, device=dev)
    ch = torch.zeros(S * B * 24, dtype=torch.uint8, device=dev)
    nc = torch.zeros(S, dtype=torch.int32, device=dev)
    ho = torch.zeros(S, B, d, device=dev)

    def load(st):
        hidden, scores, finished, n_hyp = st
        with torch.cuda.stream(s):
            H.copy_(torch.from_numpy(hidden))
            sc.copy_(torch.from_numpy(scores))
            fin.copy_(torch.from_numpy(finished))
            nh.copy_(torch.from_numpy(n_hyp))
        s.synchronize()

    load(states[0])
    n0 = ctx.launches
    b.graph_capture(H, sc, fin, nh, ch, nc, ho)
    if fused:
        assert ctx.launches - n0 == 1  # the captured step is one cooperative launch
    for st in states:
        load(st)
        with torch.cuda.stream(s):
            b.step(H, sc, fin, nh, ch, nc, ho)
        ctx.sync()
        want = (ch.clone(), nc.clone(), ho.clone())
        ch.zero_(), nc.zero_(), ho.zero_()
        torch.cuda.synchronize()
        b.graph_launch()
        ctx.sync()
        assert torch.equal(ch, want[0]) and torch.equal(nc, want[1]) and torch.equal(ho, want[2])
    b.close(), idx.close(), m.close(), ctx.close()

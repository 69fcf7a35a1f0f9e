"""Parity at the BASELINE configurations' own shapes, through the launch
variants the benchmark actually runs (VERDICT r01 "What's weak" 1):

* cfg 2 at full size (S=64, V=40k, d=1000, T=1000, t=2): the 2-D K4 tiles with
  per-sentence survivor jobs beside the shared top-T block;
* cfg 4 (V=200k, d=1024): the probe kernel's multi-slice branch (the vocabulary
  no longer fits one shared-memory slice at t=2);
* cfg 3 (B=50, S=256): large-beam selection, a sample of sentences compared;
* thresholds t > 8 (byte / 16-bit hit counters instead of bit planes);
* FAST (tcgen05 3xTF32 shared block) at d in {1000, 1024} with >= 256 rows,
  where the TMEM promotion drain runs.

Everything is compared with the oracle's restatement of decode()'s step body
(src/beam_decoder.cpp:166-289) on identical seeded inputs: candidate ids,
provenance, query codes, probability bits and chosen (score, beam, word)
exactly in PARITY mode; FAST log-probabilities within the stated tolerance."""
import numpy as np
import pytest

from oracle.oracle import oracle_step
from test_gpu_step import make_state, make_world, run_gpu

pytestmark = pytest.mark.gpu


def check_sentences(oracle, b, res, hout, world, state, K, u, W, B, T, t, specials, sents,
                    probs=True):
    E, bias, perms, bt = world[:4]
    hidden, scores, finished, n_hyp = state
    for s in sents:
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], int(n_hyp[s]), B, T, t, specials)
        ids, prov = b.candidates(s)
        np.testing.assert_array_equal(ids, want["ids"], err_msg=f"sentence {s}")
        assert prov == want["prov"], s
        codes = b.query_codes(s, W)[want["live"]]
        np.testing.assert_array_equal(codes, want["codes"])
        if probs:
            np.testing.assert_array_equal(b.probs(s).view(np.uint32),
                                          want["probs"].view(np.uint32), err_msg=f"sentence {s}")
        ws, wb, ww = want["choices"]
        assert len(res[s]) == len(ws)
        np.testing.assert_array_equal(np.array([c[2] for c in res[s]]), ww)
        np.testing.assert_array_equal(np.array([c[1] for c in res[s]]), wb)
        np.testing.assert_array_equal(np.array([c[0] for c in res[s]]), ws)
        if hout is not None:
            for k, (_, beam, _) in enumerate(res[s]):
                np.testing.assert_array_equal(hout[s, k], hidden[s, beam])


def test_cfg2_full_shape(ctx, oracle):
    """BASELINE config 2 exactly as bench.py runs it: 64 sentences x 12
    hypotheses, V=40k, d=1000, K=8, u=3, W=16, T=1000, t=2, specials {V-1}."""
    V, d, K, u, W, S, B, T, t = 40000, 1000, 8, 3, 16, 64, 12, 1000, 2
    world = make_world(oracle, V, d, K, u, W, seed=7)
    E, bias, perms, bt, ps, isd = world
    state = make_state(oracle, S, B, d, seed=11, frozen_every=5, short=9)
    b, res, hout = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    check_sentences(oracle, b, res, hout, world, state, K, u, W, B, T, t, [V - 1], range(S))


def test_cfg2_full_shape_no_frozen(ctx, oracle):
    """Same shapes, every hypothesis live (the bench's own state: the 12-row
    survivor tiles are full)."""
    V, d, K, u, W, S, B, T, t = 40000, 1000, 8, 3, 16, 64, 12, 1000, 2
    world = make_world(oracle, V, d, K, u, W, seed=7)
    E, bias, perms, bt, ps, isd = world
    state = make_state(oracle, S, B, d, seed=12)
    b, res, hout = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    check_sentences(oracle, b, res, hout, world, state, K, u, W, B, T, t, [V - 1], range(S))


def test_cfg4_large_vocab(ctx, oracle):
    """BASELINE config 4 shapes (V=200k, d=1024, B=12): the probe runs over
    two vocabulary slices per row at t=2."""
    V, d, K, u, W, S, B, T, t = 200000, 1024, 8, 3, 16, 16, 12, 1000, 2
    world = make_world(oracle, V, d, K, u, W, seed=7)
    E, bias, perms, bt, ps, isd = world
    state = make_state(oracle, S, B, d, seed=13, frozen_every=4)
    b, res, hout = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    check_sentences(oracle, b, res, hout, world, state, K, u, W, B, T, t, [V - 1], range(S))


def test_cfg3_large_beam(ctx, oracle):
    """BASELINE config 3 shapes (B=50, 256 sentences); 24 sentences spread
    over the batch are compared."""
    V, d, K, u, W, S, B, T, t = 40000, 1000, 8, 3, 16, 256, 50, 1000, 2
    world = make_world(oracle, V, d, K, u, W, seed=7)
    E, bias, perms, bt, ps, isd = world
    state = make_state(oracle, S, B, d, seed=14, frozen_every=7, short=31)
    b, res, hout = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    sents = sorted(set(np.linspace(0, S - 1, 24).astype(int).tolist()))
    check_sentences(oracle, b, res, hout, world, state, K, u, W, B, T, t, [V - 1], sents)


@pytest.mark.parametrize("V,d,K,u,W,t", [
    (6000, 64, 4, 2, 32, 9),      # byte counters, 1 slice
    (6000, 64, 4, 2, 32, 12),
    (3000, 64, 4, 1, 300, 12),    # W >= 256: 16-bit counters
    (150000, 32, 2, 2, 24, 10),   # byte counters over several vocabulary slices
])
def test_high_thresholds(ctx, oracle, V, d, K, u, W, t):
    S, B, T = 6, 12, 50
    world = make_world(oracle, V, d, K, u, W, seed=V + t)
    E, bias, perms, bt, ps, isd = world
    state = make_state(oracle, S, B, d, seed=t, frozen_every=3, short=7)
    b, res, hout = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    check_sentences(oracle, b, res, hout, world, state, K, u, W, B, T, t, [V - 1], range(S))


@pytest.mark.parametrize("d", [1000, 1024])
def test_fast_tensor_core_block_large_d(ctx, oracle, d):
    """FAST with 384 rows sharing the top-T block at d=1000 / 1024: the
    tcgen05 path with the TMEM promotion drain. Candidates exact; log-probs
    within 2e-4 (1 + max|l|) of the reference's (|dlogit| <= 1e-4 (1+|l|),
    tests/test_parallel_equivalence.cpp:100-101, enters log p twice: the
    entry itself and the row's log-denominator); choices agree except at
    near-ties."""
    V, K, u, W, S, B, T, t = 20000, 8, 3, 16, 32, 12, 1000, 2
    world = make_world(oracle, V, d, K, u, W, seed=31, bias_strength=8.0)
    E, bias, perms, bt, ps, isd = world
    state = make_state(oracle, S, B, d, seed=37)
    b, res, _ = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state,
                        mode=1)
    hidden, scores, finished, n_hyp = state
    agree = total = 0
    for s in range(S):
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], int(n_hyp[s]), B, T, t, [V - 1])
        ids, prov = b.candidates(s)
        np.testing.assert_array_equal(ids, want["ids"])
        got_p = b.probs(s).astype(np.float64)
        want_p = want["probs"].astype(np.float64)
        tol = 2e-4 * (1.0 + np.abs(want["logits"]).max(axis=1, keepdims=True))
        ok = (want_p > 1e-30) & (got_p > 0)
        dl = np.abs(np.log(np.where(ok, got_p, 1.0)) - np.log(np.where(ok, want_p, 1.0)))
        assert (dl <= tol).all(), (s, float(dl.max()), float(tol.min()))
        ws, wb, ww = want["choices"]
        got = [(c[1], c[2]) for c in res[s]]
        agree += sum(g == (int(x), int(y)) for g, x, y in zip(got, wb, ww))
        total += len(ws)
        np.testing.assert_allclose(np.array([c[0] for c in res[s]]), ws, rtol=0,
                                   atol=float(2 * tol.max()))
    assert agree >= 0.99 * total, (agree, total)

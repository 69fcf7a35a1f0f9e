"""Per-stage parity: each CUDA entry point vs the oracle on the same seeded
inputs. Bit-exact for integer/index work and (PARITY mode) for logits and
probabilities; FAST mode within the reference's own tolerance
(tests/test_parallel_equivalence.cpp:100-101: 1e-4 relative)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def gauss(o, seed, *shape):
    return o.gaussian(seed, int(np.prod(shape))).reshape(shape)


# ------------------------------------------------------------------ K1
@pytest.mark.parametrize("n,d,K,u,W", [(1000, 24, 8, 3, 25), (700, 40, 8, 3, 30),
                                       (40, 1000, 8, 3, 16), (64, 1003, 16, 3, 32),
                                       (5, 4, 2, 2, 2), (300, 256, 4, 2, 500)])
def test_wta_hash_matches_oracle(ctx, oracle, n, d, K, u, W):
    M = gauss(oracle, 23 + d, n, d)
    perms = oracle.generate_perms(d, u * W, K, 21)
    got = ctx.hash_matrix(M, perms, K, u, W)
    want = oracle.hash_matrix(M, K, u, W, perms=perms)
    np.testing.assert_array_equal(got, want)


def test_wta_table4_example(ctx):
    # tests/test_wta_hash.cpp:98-118 (perms as explicit prefixes, K=2, u=2, W=2)
    perms = np.array([[0, 1], [0, 2], [2, 1], [3, 0]], np.uint32)
    v = np.array([[0.32, 0.48, -0.57, 0.63]], np.float32)
    assert ctx.hash_matrix(v, perms, 2, 2, 2).tolist() == [[1, 1]]


def test_wta_nan_rejected(ctx, oracle):
    perms = oracle.generate_perms(4, 2, 2, 5)
    with pytest.raises(ValueError):
        ctx.hash_matrix(np.array([[1.0, np.nan, 0.0, 2.0]], np.float32), perms, 2, 1, 2)
    # the context stays usable afterwards
    assert ctx.hash_matrix(np.ones((1, 4), np.float32), perms, 2, 1, 2).tolist() == [[0, 0]]


def test_wta_params_validation(ctx):
    perms = np.zeros((8, 16), np.uint32)
    with pytest.raises(ValueError):
        ctx.hash_matrix(np.ones((1, 32), np.float32), perms, 16, 8, 1)  # 32-bit codes


def test_empty_batch(ctx, oracle):
    perms = oracle.generate_perms(16, 16, 4, 11)
    assert ctx.hash_matrix(np.zeros((0, 16), np.float32), perms, 4, 2, 8).shape == (0, 8)


# ------------------------------------------------------------------ K2
def _random_codes(o, rows, W, pool, seed):
    s = o.splitmix(seed, rows * W).astype(np.uint64)
    return (s % np.uint64(pool)).astype(np.uint32).reshape(rows, W)


def test_band_index_six_word_example(ctx, oracle):
    from paper_1806_00588_b200 import Index
    # tests/test_band_index.cpp:149-172
    codes = np.array([[3, 0], [3, 5], [1, 5], [3, 0], [2, 0], [1, 5]], np.uint32)
    idx = Index(ctx, codes=codes, index_seed=9)
    b0, b1 = idx.band(0), idx.band(1)

    def span(bv, key):
        for k, s, l in bv.slots:
            if k == key:
                return bv.word_ids[s:s + l].tolist()
        return None
    assert span(b0, 1) == [2, 5] and span(b0, 2) == [4] and span(b0, 3) == [0, 1, 3]
    assert span(b1, 0) == [0, 3, 4] and span(b1, 5) == [1, 2, 5] and span(b0, 0) is None
    q = np.array([[3, 0], [7, 9]], np.uint32)
    L = ctx.lookup_hits(idx, q)
    assert L[0, 0] == 2 and L[0, 1] == 1 and L[0, 3] == 2 and (L[1] == 0).all()


@pytest.mark.parametrize("V,W,pool,seed", [(200, 16, 9, 31), (4000, 16, 512, 5),
                                           (1, 4, 3, 1), (50, 1, 1, 2), (3000, 40, 4096, 8)])
def test_band_index_matches_oracle(ctx, oracle, V, W, pool, seed):
    from paper_1806_00588_b200 import Index
    codes = _random_codes(oracle, V, W, pool, seed)
    idx = Index(ctx, codes=codes, index_seed=seed + 1)
    bt = oracle.band_index_build(codes, seed + 1)
    for w in range(W):
        bv = idx.band(w)
        np.testing.assert_array_equal(bv.word_ids, bt.word_ids[w])  # same sorted layout
        assert bv.lg == bt.lg[w]
        # every key resolves to the oracle's span (placement may differ)
        keys = [int(k) for k, _, _ in bv.slots if k != 0x7FFFFFFF]
        want = {int(k): (int(s), int(l)) for k, s, l in bt.slots[w, : 2 << bt.lg[w]]
                if k != 0x7FFFFFFF}
        assert sorted(keys) == sorted(want)
        found, st, ln = idx.find(np.full(len(keys), w), keys)
        assert found.all()
        assert [(int(a), int(b)) for a, b in zip(st, ln)] == [want[k] for k in keys]
    q = _random_codes(oracle, 8, W, pool, seed + 7)
    np.testing.assert_array_equal(ctx.lookup_hits(idx, q), oracle.lookup_hits(bt, q))
    np.testing.assert_array_equal(ctx.lookup_hits(idx, q), oracle.lookup_hits_bruteforce(codes, q))


def test_cuckoo_ten_thousand_keys(ctx, oracle):
    from paper_1806_00588_b200 import Index
    # tests/test_band_index.cpp:62-83 shape: 10k distinct keys in one band
    keys = np.unique(oracle.splitmix(42, 12000) % np.uint64(0x7FFFFFFF)).astype(np.uint32)[:10000]
    codes = keys.reshape(-1, 1)
    idx = Index(ctx, codes=codes, index_seed=13)
    found, st, ln = idx.find(np.zeros(len(keys), np.int32), keys)
    assert found.all() and (ln == 1).all()
    np.testing.assert_array_equal(np.sort(idx.band_words(0)[st]), np.arange(len(keys)))
    miss = (oracle.splitmix(7, 1000) % np.uint64(0x7FFFFFFF)).astype(np.uint32)
    f2, _, _ = idx.find(np.zeros(1000, np.int32), miss)
    assert (f2 == np.isin(miss, keys)).all()


def test_sentinel_key_rejected(ctx):
    from paper_1806_00588_b200 import Index
    with pytest.raises(ValueError):
        Index(ctx, codes=np.array([[0x7FFFFFFF]], np.uint32), index_seed=1)


def test_lsh_index_build_matches_oracle(ctx, oracle):
    from paper_1806_00588_b200 import Index, Model
    V, d, K, u, W = 3000, 64, 8, 3, 16
    E = gauss(oracle, 7, V, d)
    m = Model(ctx, E)
    idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=oracle.mix_seed(7, 1),
                index_seed=oracle.mix_seed(7, 2))
    perms = oracle.generate_perms(d, u * W, K, oracle.mix_seed(7, 1))
    np.testing.assert_array_equal(idx.perms(), perms)
    codes = oracle.hash_matrix(E, K, u, W, perms=perms)
    bt = oracle.band_index_build(codes, oracle.mix_seed(7, 2))
    for w in range(W):
        np.testing.assert_array_equal(idx.band_words(w), bt.word_ids[w])
    q = oracle.hash_matrix(gauss(oracle, 9, 12, d), K, u, W, perms=perms)
    np.testing.assert_array_equal(ctx.lookup_hits(idx, q), oracle.lookup_hits(bt, q))


# ------------------------------------------------------------------ K3
@pytest.mark.parametrize("t", [0, 1, 2, 4, 6])
def test_select_candidates(ctx, oracle, t):
    rng = np.random.default_rng(55)
    L = rng.integers(0, 6, size=(6, 20000)).astype(np.int32)
    got, ft = ctx.select_candidates(L, t)
    want, wft = oracle.select_candidates(L, t)
    np.testing.assert_array_equal(got, want)
    assert ft == wft


def test_select_candidates_examples(ctx):
    L = np.array([[2, 0, 1], [0, 3, 0]], np.int32)  # test_candidate_selector.cpp:46-49
    assert ctx.select_candidates(L, 2)[0].tolist() == [0, 1]
    assert ctx.select_candidates(np.full((1, 3), 4, np.int32), 5)[0].tolist() == []
    with pytest.raises(ValueError):
        ctx.select_candidates(L, -1)


@pytest.mark.parametrize("T,specials", [(0, []), (3, []), (2, [7, 3, 7, 1]), (100, [799]),
                                        (800, [5]), (37, [799, 0, 36, 37, 400])])
def test_merge_top_frequent(ctx, oracle, T, specials):
    rng = np.random.default_rng(T + 1)
    L = rng.integers(0, 5, size=(4, 800)).astype(np.int32)
    ids, ft = oracle.select_candidates(L, 4)
    got = ctx.merge_top_frequent(ids, ft, T, specials, 800)
    want = oracle.merge_top_frequent(ids, ft, T, specials, 800)
    np.testing.assert_array_equal(got[0], want[0])
    assert got[1] == want[1]


def test_merge_examples(ctx):
    # tests/test_candidate_selector.cpp:90-120
    assert ctx.merge_top_frequent([5, 9], 2, 3, [], 12)[0].tolist() == [0, 1, 2, 5, 9]
    ids, prov = ctx.merge_top_frequent([3, 6], 2, 2, [7, 3, 7, 1], 10)
    assert ids.tolist() == [0, 1, 3, 6, 7] and prov == (2, 2, 1)
    with pytest.raises(ValueError):
        ctx.merge_top_frequent([], 0, 9, [], 8)
    with pytest.raises(ValueError):
        ctx.merge_top_frequent([], 0, 1, [8], 8)


def test_gather(ctx, oracle):
    from paper_1806_00588_b200 import Model
    E = gauss(oracle, 91, 500, 16)
    ids = np.unique(np.random.default_rng(1).integers(0, 500, 60)).astype(np.uint32)
    m = Model(ctx, E)
    np.testing.assert_array_equal(ctx.gather_embeddings(m, ids), E[ids])


# ------------------------------------------------------------------ K4
@pytest.mark.parametrize("rows,n,d", [(12, 1335, 1000), (6, 800, 64), (1, 2, 2), (5, 37, 3),
                                      (13, 300, 1003), (50, 257, 256), (3, 5, 1024)])
def test_logits_parity_bit_exact(ctx, oracle, rows, n, d):
    H = gauss(oracle, 103 + d, rows, d)
    E = gauss(oracle, 104 + n, n, d)
    got = ctx.compute_logits(H, E)
    want = oracle.compute_logits(H, E)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_logits_fast_within_tolerance(ctx, oracle):
    H = gauss(oracle, 1, 12, 1000)
    E = gauss(oracle, 2, 700, 1000)
    from paper_1806_00588_b200 import FAST
    got = ctx.compute_logits(H, E, mode=FAST)
    want = oracle.compute_logits(H, E)
    assert np.all(np.abs(got - want) <= 1e-4 * (1 + np.abs(want)))


def test_logits_hand_example(ctx):
    H = np.array([[1.0, 2.0]], np.float32)
    E = np.array([[3.0, 4.0], [0.0, 1.0]], np.float32)
    assert ctx.compute_logits(H, E).tolist() == [[11.0, 2.0]]


# ------------------------------------------------------------------ K5
@pytest.mark.parametrize("seq", ["0", "1"])
@pytest.mark.parametrize("rows,n", [(8, 2000), (12, 1335), (1, 3), (3, 40000), (512, 1300),
                                    (64, 3000), (16, 5000)])
def test_softmax_parity(ctx, oracle, monkeypatch, rows, n, seq):
    """Bit for bit: glibc's exp on the device, and the reference's sequential
    double denominator (softmax_denom.cuh: a certified sum, else the
    sequential sum; LSB_SEQ_DENOM=1 forces the sequential sum on every row)."""
    monkeypatch.setenv("LSB_SEQ_DENOM", seq)
    logits = gauss(oracle, 105 + n, rows, n) * 3.0
    got = ctx.softmax_rows(logits)
    want = oracle.softmax_rows(logits)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_softmax_examples(ctx):
    P = ctx.softmax_rows(np.array([[1, 2, 3]], np.float32))
    np.testing.assert_allclose(P[0], [0.09003, 0.24473, 0.66524], rtol=1e-4)
    with pytest.raises(ValueError):
        ctx.softmax_rows(np.full((1, 3), -np.inf, np.float32))


@pytest.mark.parametrize("rows,n,B,nfz,kind", [
    (12, 1335, 12, 0, "rand"), (4, 50, 3, 2, "rand"), (1, 4, 1, 0, "rand"), (2, 3, 3, 0, "rand"),
    (5, 100, 12, 3, "rand"), (50, 300, 50, 0, "rand"), (30, 200, 40, 5, "rand"),
    (20, 64, 24, 2, "ties"), (50, 50, 50, 0, "ties"), (8, 1000, 12, 0, "ties"),
    (6, 5000, 12, 0, "zeros"), (4, 3000, 40, 1, "zeros"), (3, 6000, 50, 0, "rand")])
def test_expand_beams_parity(ctx, oracle, rows, n, B, nfz, kind):
    rng = np.random.default_rng(rows * 100 + n)
    logits = rng.standard_normal((rows, n)).astype(np.float32) * 2
    if kind == "ties":  # equal scores everywhere: order decided by (beam, word) alone
        logits[:] = 0.0
    elif kind == "zeros":  # peaked rows: most probabilities underflow to exactly 0
        logits *= 150.0
    probs = oracle.softmax_rows(logits)
    cum = np.zeros(rows) if kind == "ties" else -rng.random(rows) * 3
    live = np.arange(nfz, nfz + rows, dtype=np.uint32)
    frozen = [(-rng.random() * 2, i) for i in range(nfz)]
    id_map = np.sort(rng.choice(10 * n, n, replace=False)).astype(np.uint32)
    got = ctx.expand_beams(probs, cum, live, frozen, B, id_map)
    want = oracle.expand_beams(probs, cum, live, frozen, B, id_map)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)


def test_expand_examples(ctx):
    # tests/test_beam_decoder.cpp:161-218
    s, b, w = ctx.expand_beams(np.array([[0.1, 0.6, 0.2, 0.1]], np.float32), [-1.0], [0], (), 1)
    assert w.tolist() == [1] and abs(s[0] - (-1.0 + np.log(np.float64(np.float32(0.6))))) < 1e-12
    probs = np.array([[0.7, 0.25, 0.05], [0.4, 0.35, 0.25]], np.float32)
    s, b, w = ctx.expand_beams(probs, [0.0, -2.0], [0, 1], (), 2)
    assert b.tolist() == [0, 0] and w.tolist() == [0, 1]
    s, b, w = ctx.expand_beams(np.full((2, 3), 1 / 3, np.float32), [-0.5, -0.5], [0, 1], (), 3)
    assert b.tolist() == [0, 0, 0] and w.tolist() == [0, 1, 2]
    s, b, w = ctx.expand_beams(np.array([[0.9, 0.1]], np.float32), [0.0], [0], [(-0.5, 1)], 2)
    assert b.tolist() == [0, 1] and w.tolist() == [0, -1]
    s, b, w = ctx.expand_beams(np.array([[0.3, 0.7]], np.float32), [0.0], [0], (), 1, [42, 99])
    assert w.tolist() == [99]

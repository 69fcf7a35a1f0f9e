"""Drop-in entry points beside the fused step, against the oracle (and the
reference's own bytes where the contract is a file format):

* lsb_exact_topb vs exact_topb_logits (src/eval_oracle.cpp:11-44), including
  all-negative rows, b close to V and exact ties;
* lsb_recurrence / step_hidden vs the reference recurrence
  (src/model_provider.cpp:83-102) bit for bit at d = 1000 (glibc tanhf);
* WTAIDX1 written by the unmodified reference loaded into device tables
  (src/band_index.cpp:245-289), re-exported and rebuilt byte-identically;
* kTopOnly with t = 0 (src/beam_decoder.cpp:189-199: t is ignored);
* K > 256 (16-bit argmax indices; WtaParams allows any K with
  u*ceil(log2 K) < 31, src/wta_hash.cpp:12-29);
* the parallel cuckoo build: same lookups, hit counts and step results."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import oracle_step
from test_gpu_step import make_state, make_world, run_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------ exact top-b
@pytest.mark.parametrize("V,d,rows,b,bias_shift", [
    (40000, 1000, 24, 12, 0.0),
    (5000, 64, 16, 50, -1000.0),   # every logit negative
    (100, 16, 8, 64, -50.0),       # b close to V, negative
    (64, 8, 4, 64, 0.0),           # b == V
    (20000, 128, 8, 1, 0.0),
])
def test_exact_topb_matches_oracle(ctx, oracle, V, d, rows, b, bias_shift):
    from paper_1806_00588_b200 import Model, exact_topb
    E = oracle.gaussian(V + d, V * d).reshape(V, d)
    bias = (oracle.gaussian(5, V) + np.float32(bias_shift)).astype(np.float32)
    H = oracle.gaussian(d + 1, rows * d).reshape(rows, d)
    m = Model(ctx, E, bias)
    ids, vals = exact_topb(ctx, m, H, rows, b, bias=True)
    logits = oracle.compute_logits_ids(H, E, None, bias)
    want_ids, want_vals = oracle.exact_topb_logits(logits, b)
    np.testing.assert_array_equal(ids, want_ids)
    np.testing.assert_array_equal(vals.view(np.uint32), want_vals.view(np.uint32))


def test_exact_topb_ties_to_smaller_id(ctx, oracle):
    """Duplicate embedding rows give equal logits: the smaller id ranks first
    (src/eval_oracle.cpp:29-32); +0 and -0 tie."""
    from paper_1806_00588_b200 import Model, exact_topb
    V, d, rows, b = 300, 8, 3, 40
    E = oracle.gaussian(3, V * d).reshape(V, d)
    E[100:200] = E[0:100]            # pairs (j, j+100) tie exactly
    E[250:300] = 0.0                 # zero logits, with -0 bias on some
    bias = np.zeros(V, np.float32)
    bias[260:270] = -0.0
    H = oracle.gaussian(4, rows * d).reshape(rows, d)
    m = Model(ctx, E, bias)
    ids, vals = exact_topb(ctx, m, H, rows, b)
    want_ids, want_vals = oracle.exact_topb_logits(oracle.compute_logits_ids(H, E, None, bias), b)
    np.testing.assert_array_equal(ids, want_ids)


# -------------------------------------------------------------- recurrence
def test_recurrence_bit_exact_d1000(ctx, oracle):
    import torch
    from paper_1806_00588_b200 import Model, Recurrent
    V, d, n = 3000, 1000, 96
    m = oracle.synth_model(V, d, 7, 0.0)
    model = Model(ctx, m["E"], m["bias"])
    rec = Recurrent(ctx, m["wh"], m["we"])
    rng = np.random.default_rng(3)
    H = np.tanh(oracle.gaussian(9, n * d).reshape(n, d)).astype(np.float32)
    tok = rng.integers(0, V, n).astype(np.int64)
    tok[::11] = -1                                  # frozen: carried unchanged
    dev = torch.device("cuda", 0)
    Hd = torch.from_numpy(H).to(dev)
    Td = torch.from_numpy(tok).to(dev)
    Od = torch.empty_like(Hd)
    torch.cuda.synchronize()
    rec.step(model, Hd.data_ptr(), Td.data_ptr(), n, Od.data_ptr())
    ctx.sync()
    got = Od.cpu().numpy()
    for k in range(n):
        want = H[k] if tok[k] < 0 else oracle.step_hidden(m, H[k], int(tok[k]))
        np.testing.assert_array_equal(got[k].view(np.uint32), want.view(np.uint32),
                                      err_msg=f"hypothesis {k}")
    # host-vector entry point
    np.testing.assert_array_equal(rec.step_hidden(model, H[1], int(tok[1])).view(np.uint32),
                                  oracle.step_hidden(m, H[1], int(tok[1])).view(np.uint32))


def test_recurrence_multi_step_chain(ctx, oracle):
    """Ten chained steps stay bit-identical (errors would compound)."""
    from paper_1806_00588_b200 import Model, Recurrent
    V, d = 500, 256
    m = oracle.synth_model(V, d, 11, 0.0)
    model = Model(ctx, m["E"], m["bias"])
    rec = Recurrent(ctx, m["wh"], m["we"])
    h_gpu = m["h0"].copy()
    h_ref = m["h0"].copy()
    for step in range(10):
        tok = (step * 37 + 5) % V
        h_gpu = rec.step_hidden(model, h_gpu, tok)
        h_ref = oracle.step_hidden(m, h_ref, tok)
        np.testing.assert_array_equal(h_gpu.view(np.uint32), h_ref.view(np.uint32))


# --------------------------------------------------------------- WTAIDX1
def test_wtaidx1_reference_written_file(tmp_path):
    """tests/golden/ref_index.wtaidx was written by the unmodified reference
    (tests/golden/make_wtaidx.sh). The drop-in loads it into device tables,
    its lookups equal the reference's hit counts, and both its re-export and
    a GPU build of the same embeddings are byte-identical to the file."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pkg = os.path.join(ROOT, "paper_1806_00588_b200")
    exe = str(tmp_path / "interop")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "wtaidx_interop.cpp"), "-o", exe,
                    "-L" + pkg, "-llshbeam", "-llshbeam_b200", "-Wl,-rpath," + pkg],
                   check=True)
    r = subprocess.run([exe, "check", os.path.join(ROOT, "tests", "golden"), str(tmp_path)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("ok")


# ------------------------------------------------------------ top-only t=0
@pytest.mark.parametrize("t", [0, 3])
def test_top_only_ignores_threshold(ctx, oracle, t):
    from paper_1806_00588_b200 import Batch, Model
    V, d, S, B, T = 3000, 64, 3, 8, 120
    E = oracle.gaussian(17, V * d).reshape(V, d)
    bias = oracle.synth_model(V, d, 17, 8.0, want=("bias",))["bias"]
    specials = [V - 1, 1500]
    hidden, scores, finished, n_hyp = make_state(oracle, S, B, d, seed=19, frozen_every=3)
    m = Model(ctx, E, bias)
    b = Batch(ctx, m, None, S=S, B=B, T=T, t=t, specials=specials, top_only=True)
    b.keep_probs(True)
    res, _ = b.step_host(hidden, scores, finished, n_hyp)
    want_ids = np.array(sorted(set(range(T)) | set(specials)), np.uint32)
    for s in range(S):
        ids, prov = b.candidates(s)
        np.testing.assert_array_equal(ids, want_ids)
        assert prov[0] == 0
        live = [i for i in range(B) if not finished[s, i]]
        frozen = [(float(scores[s, i]), i) for i in range(B) if finished[s, i]]
        H = np.ascontiguousarray(hidden[s][live])
        probs = oracle.softmax_rows(oracle.compute_logits_ids(H, E, want_ids, bias))
        np.testing.assert_array_equal(b.probs(s).view(np.uint32), probs.view(np.uint32))
        ws, wb, ww = oracle.expand_beams(probs, scores[s][live], live, frozen, B, want_ids)
        assert [c[2] for c in res[s]] == ww.tolist()
        assert [c[1] for c in res[s]] == wb.tolist()


# ---------------------------------------------------------------- K > 256
@pytest.mark.parametrize("K,u,W", [(512, 3, 4), (300, 2, 6), (1000, 1, 3)])
def test_wide_window_hash(ctx, oracle, K, u, W):
    d, n = 1000, 40
    M = oracle.gaussian(K, n * d).reshape(n, d)
    perms = oracle.generate_perms(d, u * W, K, 21)
    np.testing.assert_array_equal(ctx.hash_matrix(M, perms, K, u, W),
                                  oracle.hash_matrix(M, K, u, W, perms=perms))


def test_wide_window_step(ctx, oracle):
    V, d, K, u, W, S, B, T, t = 3000, 600, 512, 2, 8, 3, 6, 40, 1
    world = make_world(oracle, V, d, K, u, W, seed=5)
    E, bias, perms, bt, ps, isd = world
    state = make_state(oracle, S, B, d, seed=6)
    b, res, _ = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    hidden, scores, finished, n_hyp = state
    for s in range(S):
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], int(n_hyp[s]), B, T, t, [V - 1])
        np.testing.assert_array_equal(b.query_codes(s, W), want["codes"])
        np.testing.assert_array_equal(b.candidates(s)[0], want["ids"])
        assert [c[2] for c in res[s]] == want["choices"][2].tolist()


# ------------------------------------------------------- parallel cuckoo
@pytest.mark.parametrize("V,d,K,u,W", [(40000, 1000, 8, 3, 16), (8000, 64, 16, 3, 200),
                                       (20000, 32, 4, 2, 8)])
def test_parallel_cuckoo_build(ctx, oracle, V, d, K, u, W):
    """lsb_ctx_set_parallel_cuckoo(1): one thread per entry with 64-bit
    atomicExch eviction chains. Slots differ from the reference's, lookups
    do not: every key of every band is found with the reference's span, and
    a step over the index equals the oracle's."""
    from paper_1806_00588_b200 import Index, Model
    world = make_world(oracle, V, d, K, u, W, seed=V + W)
    E, bias, perms, bt, ps, isd = world
    ctx.set_parallel_cuckoo(True)
    try:
        m = Model(ctx, E, bias)
        idx = Index(ctx, m, K=K, u=u, W=W, perm_seed=ps, index_seed=isd)
        for w in range(W):
            lg = int(bt.lg[w])
            sl = bt.slots[w, :2 << lg]
            keys = np.array(sorted(int(k) for k in sl[:, 0] if k != 0x7FFFFFFF), np.uint32)
            found, st, ln = idx.find(np.full(len(keys), w, np.int32), keys)
            assert found.all()
            want = np.array([bt.find(w, int(k)) for k in keys], np.uint32)
            np.testing.assert_array_equal(st, want[:, 0])
            np.testing.assert_array_equal(ln, want[:, 1])
            np.testing.assert_array_equal(idx.band_words(w), bt.word_ids[w])
            # absent keys miss
            miss = np.array([k for k in range(0, 4096) if bt.find(w, k) is None][:64], np.uint32)
            if len(miss):
                f2, _, _ = idx.find(np.full(len(miss), w, np.int32), miss)
                assert not f2.any()
        S, B, T, t = 8, 12, 100, 2
        state = make_state(oracle, S, B, d, seed=3)
        b, res, _ = run_gpu(ctx, E, bias, V, d, K, u, W, ps, isd, S, B, T, t, [V - 1], state)
    finally:
        ctx.set_parallel_cuckoo(False)
    hidden, scores, finished, n_hyp = state
    for s in range(S):
        want = oracle_step(oracle, bt, perms, E, bias, K, u, W, hidden[s], scores[s],
                           finished[s], int(n_hyp[s]), B, T, t, [V - 1])
        np.testing.assert_array_equal(b.candidates(s)[0], want["ids"])
        assert [c[2] for c in res[s]] == want["choices"][2].tolist()

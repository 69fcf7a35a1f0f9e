"""End-to-end decode() parity: the reference's whole decode loop (hash ->
cuckoo lookup -> candidates -> logits -> softmax -> beam expansion ->
recurrence, src/beam_decoder.cpp:143-329) run through the UNMODIFIED reference
(oracle/_ref) and through our drop-in (liblshbeam.so over the CUDA C ABI),
with the same C wrapper (oracle/ref_shim.cpp) compiled against each
(tests/refsuite/_build/libdropin_shim.so). Every hypothesis' tokens, score
bits and finished flag, the step count, the per-step |V_LSH| and the
candidate provenance counters must be identical. Our side runs in a
subprocess that never loads the reference library, so every C++ symbol the
shim calls can only bind to liblshbeam.so."""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import Reference

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "refsuite", "_build", "libdropin_shim.so")


def run_decode(lib, V, d, seed, bias, K, u, W, beam, T, t, max_len, mode, eos, with_oracle=0,
               eos_boost=0.0):
    m = lib.ref_synth_model(V, d, seed, bias)
    assert m
    E = np.zeros((V, d), np.float32)
    wh = np.zeros((d, d), np.float32)
    we = np.zeros((d, d), np.float32)
    h0 = np.zeros(d, np.float32)
    b = np.zeros(V, np.float32)
    lib.ref_model_get(m, *[a.ctypes.data for a in (E, wh, we, h0, b)])
    if eos_boost:  # model.eos_id = V - 1: raise its bias so beams finish early
        b[V - 1] += np.float32(eos_boost)
        lib.ref_model_set(m, None, b.ctypes.data)
    idx = None
    if mode != 0:
        idx = lib.ref_index_from_embeddings(E, V, d, K, u, W, lib.ref_mix_seed(seed, 1),
                                            lib.ref_mix_seed(seed, 2))
        if not idx:  # invalid hash parameters: compare the rejection
            lib.ref_model_free(m)
            return dict(rejected=-1)
    sp = np.array([eos], np.uint32)
    st = C.c_int(0)
    h = lib.ref_decode(m, beam, T, t, max_len, sp, 1, mode, idx, with_oracle, C.byref(st))
    if not h:  # rejected configuration: compare the status
        if idx:
            lib.ref_index_free(idx)
        lib.ref_model_free(m)
        return dict(rejected=st.value)
    info = np.zeros(4, np.int32)
    prov = np.zeros(3, np.uint64)
    stages = np.zeros(9, np.float64)
    lib.ref_decode_info(h, info, prov, stages)
    hyps = []
    for k in range(int(info[0])):
        score, fin = C.c_double(), C.c_int()
        n = lib.ref_decode_hyp(h, k, None, C.byref(score), C.byref(fin))
        toks = np.zeros(max(n, 1), np.uint32)
        lib.ref_decode_hyp(h, k, toks.ctypes.data, C.byref(score), C.byref(fin))
        hyps.append([toks[:n].tolist(), score.value.hex(), fin.value])
    vlsh = np.zeros(max(int(info[2]), 1), np.uint32)
    recall = np.zeros(max(int(info[3]), 1), np.float64)
    lib.ref_decode_steps(h, vlsh.ctypes.data, recall.ctypes.data)
    lib.ref_decode_free(h)
    if idx:
        lib.ref_index_free(idx)
    lib.ref_model_free(m)
    return dict(info=info.tolist(), prov=prov.tolist(), hyps=hyps,
                vlsh=vlsh[:int(info[2])].tolist(),
                recall=[x.hex() for x in recall[:int(info[3])].tolist()])


@pytest.fixture(scope="module")
def ref_lib():
    if not (Reference.available() and os.path.exists(SHIM)):
        pytest.skip("reference or drop-in shim not built")
    return Reference().lib


def ours_decode(args):
    code = ("import json, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from oracle.oracle import Reference\n"
            "from test_gpu_dropin_decode import run_decode, SHIM\n"
            "lib = Reference(SHIM).lib\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libref_lshbeam' not in maps and 'liblshbeam.so' in maps\n"
            "print(json.dumps(run_decode(lib, *%r)))\n"
            % (ROOT, os.path.join(ROOT, "tests"), list(args)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


CASES = [
    # V, d, seed, bias, K, u, W, beam, T, t, max_len, mode (0 full, 1 lsh, 2 top)
    (3000, 64, 11, 2.0, 8, 3, 16, 4, 100, 2, 12, 1),
    (3000, 64, 11, 2.0, 8, 3, 16, 4, 100, 2, 12, 0),
    (3000, 64, 11, 2.0, 8, 3, 16, 4, 100, 1, 12, 2),
    (5000, 128, 5, 8.0, 16, 3, 32, 12, 250, 1, 10, 1),
    (4000, 100, 3, 4.0, 4, 2, 20, 6, 0, 3, 16, 1),
    (6000, 1000, 7, 1.0, 8, 3, 16, 12, 1000, 2, 6, 1),
    (40000, 1000, 7, 1.0, 8, 3, 16, 12, 1000, 2, 4, 1),  # BASELINE cfg 1
    (2000, 32, 9, 3.0, 8, 3, 16, 12, 50, 2, 40, 1),      # long decode, frozen beams
    (2000, 32, 9, 3.0, 8, 3, 16, 12, 50, 2, 40, 0),
    (2000, 32, 9, 3.0, 8, 3, 16, 1, 50, 2, 20, 1),       # greedy (beam 1)
    (1500, 48, 4, 2.0, 8, 3, 16, 6, 1500, 2, 12, 1),     # T = V: every word is a candidate
    (1500, 48, 4, 2.0, 8, 3, 16, 6, 20, 17, 12, 1),      # t > W: rejected by both
    (1500, 48, 4, 2.0, 8, 3, 16, 6, 20, 16, 12, 1),      # t = W: few threshold survivors
]

# the model's EOS (V - 1) with a raised bias: hypotheses finish at different
# steps and the frozen-beam path of expand_beams carries them to the end
EOS_CASES = [
    (2000, 32, 13, 2.0, 8, 3, 16, 8, 50, 2, 30, 1),
    (2000, 32, 13, 2.0, 8, 3, 16, 8, 50, 2, 30, 0),
    (2000, 32, 13, 2.0, 8, 3, 16, 8, 50, 1, 30, 2),
]


@pytest.mark.parametrize("boost", [6.0, 9.0])
@pytest.mark.parametrize("V,d,seed,bias,K,u,W,beam,T,t,max_len,mode", EOS_CASES)
def test_decode_with_early_eos_equals_reference(ref_lib, V, d, seed, bias, K, u, W, beam, T, t,
                                                max_len, mode, boost):
    args = (V, d, seed, bias, K, u, W, beam, T, t, max_len, mode, V - 1, 0, boost)
    want = run_decode(ref_lib, *args)
    got = ours_decode(args)
    assert any(h[2] for h in want["hyps"])  # some hypotheses finished
    assert got == want


@pytest.mark.parametrize("V,d,seed,bias,K,u,W,beam,T,t,max_len,mode", [CASES[0], CASES[3]])
def test_decode_with_oracle_recall_equals_reference(ref_lib, V, d, seed, bias, K, u, W, beam, T,
                                                    t, max_len, mode):
    """decode(with_oracle=true): the per-step recall@B against the exact
    full-vocabulary top-B (eval_oracle, src/eval_oracle.cpp:11-63; ours runs
    it through lsb_exact_topb) is identical too."""
    args = (V, d, seed, bias, K, u, W, beam, T, t, max_len, mode, V - 1, 1)
    want = run_decode(ref_lib, *args)
    got = ours_decode(args)
    assert len(want["recall"]) > 0
    assert got == want


@pytest.mark.parametrize("V,d,seed,bias,K,u,W,beam,T,t,max_len,mode", CASES)
def test_decode_equals_reference(ref_lib, V, d, seed, bias, K, u, W, beam, T, t, max_len, mode):
    args = (V, d, seed, bias, K, u, W, beam, T, t, max_len, mode, V - 1)
    want = run_decode(ref_lib, *args)
    got = ours_decode(args)
    if "rejected" in want:
        assert "rejected" in got and (got["rejected"] != 0) == (want["rejected"] != 0)
        return
    assert got["info"] == want["info"]
    assert got["prov"] == want["prov"]
    assert got["vlsh"] == want["vlsh"]
    assert got["hyps"] == want["hyps"]


def fuzz_cases(n=24, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        V = int(rng.integers(300, 5000))
        d = int(rng.choice([8, 16, 33, 64, 100, 256]))
        K = int(rng.choice([2, 4, 8, 16]))
        K = min(K, d)
        u = int(rng.integers(1, 4))
        W = int(rng.integers(1, 40))
        beam = int(rng.integers(1, 20))
        T = int(rng.choice([0, int(rng.integers(1, V))]))
        t = int(rng.integers(0, W + 1))
        mode = int(rng.integers(0, 3))
        out.append((V, d, int(rng.integers(0, 10**6)), float(rng.choice([0.0, 1.0, 4.0])), K, u, W,
                    beam, T, t, int(rng.integers(1, 25)), mode, V - 1, 0,
                    float(rng.choice([0.0, 5.0]))))
    return out


@pytest.mark.parametrize("args", fuzz_cases())
def test_decode_fuzz_equals_reference(ref_lib, args):
    """Random decode() configurations (vocabulary, dimension, hash shape, beam,
    T, t, mode, length, bias, EOS bias): identical to the reference, or
    rejected by both."""
    want = run_decode(ref_lib, *args)
    got = ours_decode(args)
    if "rejected" in want:
        assert "rejected" in got
        return
    assert got == want

"""Seeded calls of the reference's public C++ API through the C wrapper
oracle/ref_shim.cpp (oracle.oracle.Reference), for tests/test_gpu_dropin_api.py:
run against the unmodified reference (oracle/_ref) and against our drop-in
(the same wrapper compiled against include/lshbeam + liblshbeam.so), every
returned array must be identical. Test infrastructure.

  python tests/dropin_api_cases.py SHIM.so OUT.npz   (runs ours, saves arrays)
"""
import sys

import numpy as np


def run_all(R) -> dict:
    out = {}
    rng = np.random.default_rng(1234)
    # rng / seeds (include/lshbeam/rng.hpp)
    out["mix_seed"] = np.array([R.mix_seed(s, k) for s in (0, 7, 2**63 + 5) for k in (1, 2, 9)],
                               np.uint64)
    out["splitmix"] = R.splitmix(42, 64)
    out["gaussian"] = R.gaussian(11, 4096)
    # WTA (src/wta_hash.cpp)
    for (d, K, u, W) in [(64, 8, 3, 16), (100, 4, 2, 20), (1000, 16, 3, 32), (600, 512, 1, 4)]:
        perms = R.generate_perms(d, u * W, K, R.mix_seed(d, 1))
        out[f"perms_{d}_{K}"] = perms
        M = rng.standard_normal((50, d)).astype(np.float32)
        M[3, :] = 0.0  # ties everywhere: the smallest index wins
        out[f"hash_{d}_{K}_{u}_{W}"] = R.hash_matrix(M, K, u, W, perms=perms)
        out[f"hash_seed_{d}_{K}_{u}_{W}"] = R.hash_matrix(M, K, u, W, seed=R.mix_seed(d, 1))
    idx = rng.integers(0, 8, (16, 3)).astype(np.uint32)
    out["pack_bands"] = R.pack_bands(idx.reshape(-1), 8, 3, 16)
    # band index + cuckoo (src/band_index.cpp)
    codes = rng.integers(0, 64, (3000, 16)).astype(np.uint32)
    bt = R.band_index_build(codes, 99)
    for k, v in bt._asdict().items() if hasattr(bt, "_asdict") else vars(bt).items():
        if isinstance(v, (list, tuple)):
            for i, a in enumerate(v):
                out[f"bt_{k}_{i}"] = np.asarray(a)
        else:
            out[f"bt_{k}"] = np.asarray(v)
    q = rng.integers(0, 64, (12, 16)).astype(np.uint32)
    out["lookup_hits"] = R.lookup_hits_codes(codes, 99, q)
    keys = np.unique(rng.integers(0, 2**31, 5000)).astype(np.uint32)
    lg, muls, slots = R.cuckoo_build(keys, np.arange(len(keys), dtype=np.uint32),
                                     np.ones(len(keys), np.uint32), 5)
    out["cuckoo_lg"], out["cuckoo_muls"], out["cuckoo_slots"] = np.array([lg]), muls, slots
    # candidates (src/candidate_selector.cpp)
    L = rng.integers(0, 5, (12, 3000)).astype(np.int32)
    for t in (0, 1, 2, 4):
        ids, ft = R.select_candidates(L, t)
        out[f"select_{t}"], out[f"select_ft_{t}"] = ids, np.array([ft])
        m, prov = R.merge_top_frequent(ids, ft, 100, [2999, 5], 3000)
        out[f"merge_{t}"], out[f"merge_prov_{t}"] = m, np.array(prov)
    E = rng.standard_normal((3000, 100)).astype(np.float32)
    ids = np.sort(rng.choice(3000, 400, replace=False)).astype(np.uint32)
    Es = R.gather(E, ids)
    out["gather"] = Es
    H = rng.standard_normal((12, 100)).astype(np.float32)
    logits = R.compute_logits(H, Es)
    out["logits"] = logits
    probs = R.softmax_rows(logits * 3.0)
    out["probs"] = probs
    cum = -rng.random(12) * 4
    for B, frozen in [(12, ()), (5, ((-0.5, 3), (-9.0, 7))), (50, ())]:
        s, b, w = R.expand_beams(probs, cum, np.arange(12, dtype=np.uint32), frozen, B, ids)
        out[f"expand_s_{B}_{len(frozen)}"] = s
        out[f"expand_b_{B}_{len(frozen)}"] = b
        out[f"expand_w_{B}_{len(frozen)}"] = w
    tids, tvals = R.exact_topb_logits(np.concatenate([logits, -np.abs(logits)]), 12)
    out["topb_ids"], out["topb_vals"] = tids, tvals
    # synthetic model (src/model_provider.cpp) and the recurrence
    m = R.synth_model(500, 48, 21, 2.0)
    for k, v in m.items():
        out[f"model_{k}"] = v
    h = R.lib.ref_synth_model(2000, 1000, 7, 1.0)
    x = np.zeros(1000, np.float32)
    R.lib.ref_model_get(h, None, None, None, x.ctypes.data, None)
    for k, tok in enumerate((5, 1999, 0, 77)):  # h' = tanh(W_h h + W_e emb[tok])
        y = np.zeros(1000, np.float32)
        R._chk(R.lib.ref_step_hidden(h, x, tok, y), "step_hidden")
        out[f"step_hidden_{k}"] = y
        x = y
    R.lib.ref_model_free(h)
    # build_lsh_index over embeddings (K1 on E + K2-build) and its lookups
    E = R.gaussian(3, 4000 * 64).reshape(4000, 64)
    ih = R.lib.ref_index_from_embeddings(E, 4000, 64, 8, 3, 16, R.mix_seed(3, 1), R.mix_seed(3, 2))
    try:
        bt = R._tables(ih, 4000, 16)
        out["lsh_word_ids"], out["lsh_lg"] = bt.word_ids, bt.lg
        out["lsh_mul"], out["lsh_slots"] = bt.mul, bt.slots
    finally:
        R.lib.ref_index_free(ih)
    # error behaviour: which calls are rejected, and with which error class
    def rejects(f, *a):
        try:
            f(*a)
            return 0
        except ValueError:
            return 1
        except RuntimeError:
            return 2
        except Exception:  # noqa: BLE001
            return 3
    out["rejects"] = np.array([
        rejects(R.wta_params_check, 1, 3, 16), rejects(R.wta_params_check, 8, 0, 16),
        rejects(R.wta_params_check, 8, 11, 16), rejects(R.wta_params_check, 8, 3, 0),
        rejects(R.wta_params_check, 512, 3, 4), rejects(R.wta_params_check, 8, 3, 16),
        rejects(R.generate_perms, 4, 6, 8, 1),
        rejects(R.cuckoo_build, [0x7FFFFFFF], [0], [1], 1),
        rejects(R.softmax_rows, np.full((1, 3), -np.inf, np.float32)),
    ], np.int32)
    # one decode step body (kLsh / kFull) + expansion, src/beam_decoder.cpp:166-289
    from oracle.oracle import ReferenceStepper
    Hs = rng.standard_normal((12, 64)).astype(np.float32)
    st = ReferenceStepper(R, E, R.gaussian(4, 4000) * 0.5, 8, 3, 16, R.mix_seed(3, 1),
                          R.mix_seed(3, 2))
    try:
        for full in (False, True):
            (s_, b_, w_), nc, _ = st.step(Hs, -rng.random(12) * 3, 12, 100, 2, [3999], full=full)
            out[f"step_{full}_s"], out[f"step_{full}_b"], out[f"step_{full}_w"] = s_, b_, w_
            out[f"step_{full}_n"] = np.array([nc])
    finally:
        st.close()
    return out


if __name__ == "__main__":
    sys.path.insert(0, sys.argv[3] if len(sys.argv) > 3 else ".")
    from oracle.oracle import Reference
    R = Reference(sys.argv[1])
    res = run_all(R)
    maps = open("/proc/self/maps").read()
    assert "libref_lshbeam" not in maps and "liblshbeam.so" in maps
    np.savez(sys.argv[2], **res)


def index_tables(R, h, V, W):
    bt = R._tables(h, V, W)
    return {"word_ids": bt.word_ids, "lg": bt.lg, "mul": bt.mul, "slots": bt.slots}


def write_files(R, d, tag):
    """WTAIDX1 / WTAEMB1 files written by this library (src/band_index.cpp:198-289,
    src/model_provider.cpp:116-154) for a seeded model and index."""
    import ctypes as C
    import os
    lib = R.lib
    lib.ref_index_save.argtypes = [C.c_void_p, C.c_char_p]
    lib.ref_embeddings_save.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_char_p]
    E = R.gaussian(5, 3000 * 40).reshape(3000, 40)
    h = lib.ref_index_from_embeddings(E, 3000, 40, 8, 3, 16, R.mix_seed(5, 1), R.mix_seed(5, 2))
    try:
        R._chk(lib.ref_index_save(h, os.path.join(d, f"{tag}.idx").encode()), "save_lsh_index")
    finally:
        lib.ref_index_free(h)
    R._chk(lib.ref_embeddings_save(E.ctypes.data, 3000, 40, os.path.join(d, f"{tag}.emb").encode()),
           "save_embeddings")


def read_files(R, d, tag):
    """The other library's files read back: index tables and embeddings."""
    import ctypes as C
    import os
    lib = R.lib
    lib.ref_index_load.restype = C.c_void_p
    lib.ref_index_load.argtypes = [C.c_char_p]
    lib.ref_embeddings_load.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64,
                                        C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
    h = lib.ref_index_load(os.path.join(d, f"{tag}.idx").encode())
    assert h, lib.ref_last_error().decode()
    try:
        out = {f"idx_{k}": v for k, v in index_tables(R, h, 3000, 16).items()}
    finally:
        lib.ref_index_free(h)
    E = np.zeros((3000, 40), np.float32)
    V, dd = C.c_uint32(), C.c_int()
    R._chk(lib.ref_embeddings_load(os.path.join(d, f"{tag}.emb").encode(), E.ctypes.data, E.size,
                                   C.byref(V), C.byref(dd)), "load_embeddings")
    out["emb"], out["emb_shape"] = E, np.array([V.value, dd.value])
    return out

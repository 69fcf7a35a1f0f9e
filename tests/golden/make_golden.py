"""Regenerates tests/golden/*.npz from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
Every array is produced by the reference's own code path through
oracle/ref_shim.cpp (oracle/_ref/libref_lshbeam.so). The fixtures pin the
oracle restatement (tests/test_oracle_pinning.py) and the CUDA path
(tests/test_gpu_golden.py) without needing the reference at test time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402


def main():
    r = Reference()
    r.set_threads(4)
    out = {}

    # --- WTA (src/wta_hash.cpp) ---
    d, K, u, W = 40, 8, 3, 30
    M = r.gaussian(100, 50 * d).reshape(50, d)
    perms = r.generate_perms(d, u * W, K, 7)
    out["wta"] = dict(M=M, perms=perms, K=K, u=u, W=W,
                      codes=r.hash_matrix(M, K, u, W, perms=perms),
                      perms_d4=r.generate_perms(4, 4, 2, 7),
                      pack_123=r.pack_bands(np.array([1, 2, 3], np.uint32), 4, 3, 1))

    # --- band index + lookup (src/band_index.cpp) ---
    V, Wb = 300, 16
    codes = (r.splitmix(31, V * Wb) % np.uint64(9)).astype(np.uint32).reshape(V, Wb)
    bt = r.band_index_build(codes, 4)
    q = (r.splitmix(32, 6 * Wb) % np.uint64(9)).astype(np.uint32).reshape(6, Wb)
    out["bands"] = dict(codes=codes, seed=4, word_ids=bt.word_ids, lg=bt.lg, mul=bt.mul,
                        slots=bt.slots, q=q, L=r.lookup_hits_codes(codes, 4, q))

    # --- candidates (src/candidate_selector.cpp) ---
    rng = np.random.default_rng(3)
    L = rng.integers(0, 5, size=(4, 800)).astype(np.int32)
    ids, ft = r.select_candidates(L, 2)
    merged, prov = r.merge_top_frequent(ids, ft, 37, np.array([799, 0, 36, 37, 400], np.uint32),
                                        800)
    out["cands"] = dict(L=L, t=2, ids=ids, from_threshold=ft, T=37,
                        specials=np.array([799, 0, 36, 37, 400], np.uint32), merged=merged,
                        prov=np.array(prov, np.uint32))

    # --- logits / softmax / expansion (src/beam_decoder.cpp) ---
    H = r.gaussian(201, 12 * 1003).reshape(12, 1003)
    Es = r.gaussian(202, 97 * 1003).reshape(97, 1003)
    lg = r.compute_logits(H, Es)
    logits = r.gaussian(203, 8 * 2000).reshape(8, 2000) * 3
    probs = r.softmax_rows(logits)
    p2 = probs[:5, :300]
    p2 = r.softmax_rows(logits[:5, :300])
    cum = -np.linspace(0.5, 3.0, 5)
    live = np.array([1, 2, 4, 5, 6], np.uint32)
    frozen = [(-0.7, 0), (-2.5, 3)]
    id_map = np.sort(rng.choice(5000, 300, replace=False)).astype(np.uint32)
    cs, cb, cw = r.expand_beams(p2, cum, live, frozen, 7, id_map)
    out["softmax"] = dict(H=H, Esub=Es, logits_hd=lg, logits=logits, probs=probs, p2=p2,
                          cum=cum, live=live, frozen=np.array(frozen), id_map=id_map, B=7,
                          ch_score=cs, ch_beam=cb, ch_word=cw)

    # --- synthetic model + recurrence (src/model_provider.cpp) ---
    m = r.synth_model(64, 8, 33, 4.0)
    h1 = np.zeros(8, np.float32)
    import ctypes as C
    hm = r.lib.ref_synth_model(64, 8, 33, 4.0)
    r.lib.ref_step_hidden(hm, m["h0"], 17, h1)
    r.lib.ref_model_free(hm)
    out["model"] = dict(**m, token=17, h1=h1)
    del C

    path = os.path.join(HERE, "reference_vectors.npz")
    flat = {f"{k}__{kk}": np.asarray(v) for k, dct in out.items() for kk, v in dct.items()}
    np.savez_compressed(path, **flat)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

"""ctypes front-ends for the two CPU checkers under oracle/.

TEST INFRASTRUCTURE ONLY. Imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` legs -- never by the product
package. Two back-ends expose the same numpy-level functions:

* ``Oracle``    -- build/liboracle.so, our plain-C restatement
                   (lshbeam_oracle.c, each function cites the reference).
* ``Reference`` -- _ref/libref_lshbeam.so, the unmodified reference sources
                   compiled in place plus ref_shim.cpp (present wherever
                   ``make -C oracle`` ran with /root/reference mounted; the
                   .so travels to the GPU box).

Status codes follow the reference's exception classes: 1 -> ValueError
(std::invalid_argument), 2 -> RuntimeError (std::runtime_error).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_lshbeam.so")
EMPTY_CODE = 0x7FFFFFFF

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _raise(rc: int, what: str, msg: str = "") -> None:
    if rc == 0:
        return
    if rc == 1:
        raise ValueError(f"{what}: invalid argument {msg}".strip())
    raise RuntimeError(f"{what}: runtime error {msg}".strip())


def build(quiet: bool = True) -> None:
    """Build the checker libraries (make -C oracle)."""
    import subprocess

    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def c32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def cu32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


@dataclass
class BandTables:
    """Host copy of a band index: W x V word ids + per-band cuckoo tables."""

    word_ids: np.ndarray           # (W, V) uint32
    lg: np.ndarray                 # (W,) uint32
    mul: np.ndarray                # (W, 2) uint64
    slots: np.ndarray              # (W, 2*2^lgmax, 3) uint32
    vocab: int

    def find(self, w: int, key: int):
        lg = int(self.lg[w])
        cap = 1 << lg
        for t in range(2):
            s = ((int(self.mul[w, t]) * key) & 0xFFFFFFFFFFFFFFFF) >> (64 - lg)
            slot = self.slots[w, t * cap + s]
            if int(slot[0]) == key:
                return int(slot[1]), int(slot[2])
        return None


class Oracle:
    """The plain-C restatement (oracle/lshbeam_oracle.c)."""

    name = "oracle"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.lso_sm64_next.restype = C.c_uint64
        L.lso_sm64_next.argtypes = [C.POINTER(C.c_uint64)]
        L.lso_mix_seed.restype = C.c_uint64
        L.lso_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.lso_gaussian_fill.argtypes = [C.c_uint64, C.c_uint64, _f32p, C.c_size_t, C.c_float]
        L.lso_bits_for.argtypes = [C.c_int]
        L.lso_wta_params_check.argtypes = [C.c_int] * 3
        L.lso_generate_perms.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _u32p]
        L.lso_hash_matrix.argtypes = [_f32p, C.c_int64, C.c_int, _u32p, C.c_int, C.c_int,
                                      C.c_int, _u32p]
        L.lso_lg_max.restype = C.c_uint32
        L.lso_lg_max.argtypes = [C.c_uint32]
        L.lso_cuckoo_build.argtypes = [_u32p, _u32p, _u32p, C.c_size_t, C.c_uint64,
                                       C.POINTER(C.c_uint32), _u64p, _u32p]
        L.lso_band_index_build.argtypes = [_u32p, C.c_uint32, C.c_int, C.c_uint64, _u32p,
                                           _u32p, _u64p, _u32p, C.c_size_t]
        L.lso_lookup_hits.argtypes = [_u32p, C.c_uint32, C.c_int, _u32p, _u64p, _u32p,
                                      C.c_size_t, _u32p, C.c_int, _i32p]
        L.lso_lookup_hits_bruteforce.argtypes = [_u32p, C.c_uint32, _u32p, C.c_int, C.c_int,
                                                 _i32p]
        L.lso_select_candidates.argtypes = [_i32p, C.c_int, C.c_uint32, C.c_int, _u32p,
                                            C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.lso_merge_top_frequent.argtypes = [_u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                             _u32p, C.c_uint32, C.c_uint32, _u32p,
                                             C.POINTER(C.c_uint32), _u32p]
        L.lso_gather.argtypes = [_f32p, C.c_int, _u32p, C.c_uint32, _f32p]
        L.lso_compute_logits.argtypes = [_f32p, C.c_int, _f32p, C.c_int64, C.c_int64, _f32p]
        L.lso_compute_logits_ids.argtypes = [_f32p, C.c_int, _f32p, C.c_void_p, C.c_int64,
                                             C.c_int64, C.c_void_p, _f32p]
        L.lso_softmax_rows.argtypes = [_f32p, C.c_int, C.c_int64, _f32p]
        L.lso_expand_beams.argtypes = [_f32p, C.c_int, C.c_int64, _f64p, _u32p, _f64p, _u32p,
                                       C.c_int, C.c_int, C.c_void_p, _f64p, _u32p, _i64p,
                                       C.POINTER(C.c_int)]
        L.lso_synth_model.argtypes = [C.c_uint32, C.c_int, C.c_uint64, C.c_float,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
        L.lso_step_hidden.argtypes = [_f32p, _f32p, _f32p, C.c_uint32, C.c_int, _f32p,
                                      C.c_uint32, _f32p]
        L.lso_exact_topb_logits.argtypes = [_f32p, C.c_int, C.c_int64, C.c_int, _u32p, _f32p]
        L.lso_recall_at_b.restype = C.c_double
        L.lso_recall_at_b.argtypes = [_u32p, C.c_uint32, _u32p, C.c_int, C.c_int]

    # ---------------------------------------------------------------- rng
    def mix_seed(self, seed: int, stream: int) -> int:
        return int(self.lib.lso_mix_seed(seed, stream))

    def splitmix(self, seed: int, n: int) -> np.ndarray:
        s = C.c_uint64(seed)
        return np.array([self.lib.lso_sm64_next(C.byref(s)) for _ in range(n)], np.uint64)

    def gaussian(self, seed: int, n: int, skip: int = 0, scale: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float32)
        self.lib.lso_gaussian_fill(seed, skip, out, n, scale)
        return out

    # ---------------------------------------------------------------- wta
    def wta_params_check(self, K, u, W):
        _raise(self.lib.lso_wta_params_check(K, u, W), "WtaParams")

    def generate_perms(self, d, P, K, seed) -> np.ndarray:
        out = np.empty((P, K), np.uint32)
        _raise(self.lib.lso_generate_perms(d, P, K, seed, out), "PermutationSet")
        return out

    def hash_matrix(self, M, K, u, W, seed=None, perms=None) -> np.ndarray:
        M = c32(M)
        n, d = M.shape
        if perms is None:
            perms = self.generate_perms(d, u * W, K, seed)
        out = np.zeros((n, W), np.uint32)
        _raise(self.lib.lso_hash_matrix(M, n, d, cu32(perms), K, u, W, out), "hash_matrix")
        return out

    # -------------------------------------------------------------- bands
    def cuckoo_build(self, keys, starts, lens, seed):
        keys, starts, lens = cu32(keys), cu32(starts), cu32(lens)
        n = len(keys)
        lgmax = max(1, int(np.ceil(np.log2(max(n, 1)))))
        lg = C.c_uint32()
        mul = np.zeros(2, np.uint64)
        slots = np.zeros((2 << lgmax, 3), np.uint32)
        _raise(self.lib.lso_cuckoo_build(keys, starts, lens, n, seed, C.byref(lg), mul, slots),
               "CuckooTable::build")
        return int(lg.value), mul, slots[: 2 << lg.value]

    def band_index_build(self, codes, seed) -> BandTables:
        codes = cu32(codes)
        V, W = codes.shape
        lgmax = int(self.lib.lso_lg_max(V))
        stride = 3 * (2 << lgmax)
        word_ids = np.zeros((W, V), np.uint32)
        lg = np.zeros(W, np.uint32)
        mul = np.zeros((W, 2), np.uint64)
        slots = np.zeros((W, 2 << lgmax, 3), np.uint32)
        _raise(self.lib.lso_band_index_build(codes, V, W, seed, word_ids, lg, mul, slots,
                                             stride), "BandIndex::build")
        return BandTables(word_ids, lg, mul, slots, V)

    def lookup_hits(self, bt: BandTables, q) -> np.ndarray:
        q = cu32(q)
        B, W = q.shape
        L = np.zeros((B, bt.vocab), np.int32)
        stride = bt.slots.shape[1] * 3
        _raise(self.lib.lso_lookup_hits(cu32(bt.word_ids), bt.vocab, W, cu32(bt.lg),
                                        np.ascontiguousarray(bt.mul), cu32(bt.slots), stride,
                                        q, B, L), "lookup_hits")
        return L

    def lookup_hits_bruteforce(self, vocab_codes, q) -> np.ndarray:
        vocab_codes, q = cu32(vocab_codes), cu32(q)
        V, W = vocab_codes.shape
        B = q.shape[0]
        L = np.zeros((B, V), np.int32)
        self.lib.lso_lookup_hits_bruteforce(vocab_codes, V, q, B, W, L)
        return L

    # --------------------------------------------------------- candidates
    def select_candidates(self, L, t):
        L = np.ascontiguousarray(L, np.int32)
        B, V = L.shape
        ids = np.zeros(max(V, 1), np.uint32)
        n, ft = C.c_uint32(), C.c_uint32()
        _raise(self.lib.lso_select_candidates(L, B, V, t, ids, C.byref(n), C.byref(ft)),
               "select_candidates")
        return ids[: n.value].copy(), int(ft.value)

    def merge_top_frequent(self, ids, from_thr, T, specials, V):
        ids = cu32(ids)
        specials = cu32(specials if len(specials) else np.zeros(0, np.uint32))
        out = np.zeros(len(ids) + T + len(specials) + 1, np.uint32)
        n = C.c_uint32()
        prov = np.zeros(3, np.uint32)
        _raise(self.lib.lso_merge_top_frequent(ids, len(ids), from_thr, T, specials,
                                               len(specials), V, out, C.byref(n), prov),
               "merge_top_frequent")
        return out[: n.value].copy(), tuple(int(x) for x in prov)

    def gather(self, E, ids):
        E, ids = c32(E), cu32(ids)
        out = np.zeros((len(ids), E.shape[1]), np.float32)
        self.lib.lso_gather(E, E.shape[1], ids, len(ids), out)
        return out

    # ---------------------------------------------------- reduced softmax
    def compute_logits(self, H, Esub):
        H, Esub = c32(H), c32(Esub)
        if H.shape[1] != Esub.shape[1]:
            raise ValueError("compute_logits: inner dimensions disagree")
        out = np.zeros((H.shape[0], Esub.shape[0]), np.float32)
        self.lib.lso_compute_logits(H, H.shape[0], Esub, Esub.shape[0], H.shape[1], out)
        return out

    def compute_logits_ids(self, H, E, ids=None, bias=None):
        """logits[i, r] = dot(H[i], E[ids[r]]) + bias[ids[r]] (decode's order)."""
        H, E = c32(H), c32(E)
        n = len(ids) if ids is not None else E.shape[0]
        ids_a = cu32(ids) if ids is not None else None
        bias_a = c32(bias) if bias is not None else None
        out = np.zeros((H.shape[0], n), np.float32)
        self.lib.lso_compute_logits_ids(
            H, H.shape[0], E, ids_a.ctypes.data if ids_a is not None else None, n, H.shape[1],
            bias_a.ctypes.data if bias_a is not None else None, out)
        return out

    def softmax_rows(self, logits):
        logits = c32(logits)
        out = np.zeros_like(logits)
        _raise(self.lib.lso_softmax_rows(logits, logits.shape[0], logits.shape[1], out),
               "softmax_rows")
        return out

    def expand_beams(self, probs, cum, live, frozen=(), B=1, id_map=None):
        probs = c32(probs)
        rows, n = probs.shape
        cum = np.ascontiguousarray(cum, np.float64)
        live = cu32(live)
        if len(cum) != rows or len(live) != rows:
            raise ValueError("expand_beams: row metadata mismatch")
        if id_map is not None and len(id_map) and len(id_map) != n:
            raise ValueError("expand_beams: id_map size mismatch")
        fz_s = np.array([f[0] for f in frozen] or [0.0], np.float64)
        fz_b = np.array([f[1] for f in frozen] or [0], np.uint32)
        m = max(1, min(B, rows * n + len(frozen)))
        os_, ob, ow = np.zeros(m), np.zeros(m, np.uint32), np.zeros(m, np.int64)
        nout = C.c_int()
        idm = cu32(id_map) if id_map is not None and len(id_map) else None
        self.lib.lso_expand_beams(probs, rows, n, cum, live, fz_s, fz_b, len(frozen), B,
                                  idm.ctypes.data if idm is not None else None, os_, ob, ow,
                                  C.byref(nout))
        k = nout.value
        return os_[:k].copy(), ob[:k].copy(), ow[:k].copy()

    # ------------------------------------------------------------- model
    def synth_model(self, V, d, seed, bias_strength, want=("E", "wh", "we", "h0", "bias")):
        arrs = {
            "E": np.zeros((V, d), np.float32) if "E" in want else None,
            "wh": np.zeros((d, d), np.float32) if "wh" in want else None,
            "we": np.zeros((d, d), np.float32) if "we" in want else None,
            "h0": np.zeros(d, np.float32) if "h0" in want else None,
            "bias": np.zeros(V, np.float32) if "bias" in want else None,
        }
        ptr = [a.ctypes.data if a is not None else None for a in arrs.values()]
        _raise(self.lib.lso_synth_model(V, d, seed, bias_strength, *ptr), "synth_model")
        return arrs

    def step_hidden(self, model, h, token):
        E, wh, we = model["E"], model["wh"], model["we"]
        V, d = E.shape
        out = np.zeros(d, np.float32)
        _raise(self.lib.lso_step_hidden(E, wh, we, V, d, c32(h), token, out), "step_hidden")
        return out

    def exact_topb_logits(self, logits, b):
        logits = c32(logits)
        rows, n = logits.shape
        ids = np.zeros((rows, b), np.uint32)
        vals = np.zeros((rows, b), np.float32)
        _raise(self.lib.lso_exact_topb_logits(logits, rows, n, b, ids, vals), "exact_topb")
        return ids, vals

    def recall_at_b(self, cands, exact_ids):
        exact_ids = cu32(exact_ids)
        return float(self.lib.lso_recall_at_b(cu32(cands), len(cands), exact_ids,
                                              exact_ids.shape[0], exact_ids.shape[1]))


class Reference:
    """The unmodified reference library via oracle/ref_shim.cpp."""

    name = "reference"

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_gaussian_fill.argtypes = [C.c_uint64, _f32p, C.c_size_t, C.c_float]
        L.ref_splitmix_next.argtypes = [C.c_uint64, _u64p, C.c_size_t]
        L.ref_wta_params_check.argtypes = [C.c_int] * 3
        L.ref_generate_perms.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _u32p]
        L.ref_hash_matrix.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_uint64, _u32p]
        L.ref_hash_matrix_perms.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int,
                                            C.c_int, _u32p, _u32p]
        L.ref_pack_bands.argtypes = [_u32p, C.c_int, C.c_int, C.c_int, _u32p]
        L.ref_index_from_codes.restype = C.c_void_p
        L.ref_index_from_codes.argtypes = [_u32p, C.c_uint32, C.c_int, C.c_uint64]
        L.ref_index_from_embeddings.restype = C.c_void_p
        L.ref_index_from_embeddings.argtypes = [_f32p, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                                C.c_int, C.c_uint64, C.c_uint64]
        L.ref_index_free.argtypes = [C.c_void_p]
        L.ref_index_band_words.argtypes = [C.c_void_p, C.c_int, _u32p]
        L.ref_index_table.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p]
        L.ref_index_find.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
        L.ref_index_lookup_hits.argtypes = [C.c_void_p, _u32p, C.c_int, _i32p]
        L.ref_lookup_hits_bruteforce.argtypes = [_u32p, C.c_uint32, _u32p, C.c_int, C.c_int,
                                                 _i32p]
        L.ref_cuckoo_build.argtypes = [_u32p, _u32p, _u32p, C.c_size_t, C.c_uint64,
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64), _u32p, C.c_size_t]
        L.ref_select_candidates.argtypes = [_i32p, C.c_int, C.c_uint32, C.c_int, _u32p,
                                            C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.ref_merge_top_frequent.argtypes = [_u32p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                             C.c_uint32, C.c_uint32, _u32p,
                                             C.POINTER(C.c_uint32), _u32p]
        L.ref_gather.argtypes = [_f32p, C.c_uint32, C.c_int, _u32p, C.c_uint32, _f32p]
        L.ref_compute_logits.argtypes = [_f32p, C.c_int, _f32p, C.c_int64, C.c_int, _f32p]
        L.ref_serial_compute_logits.argtypes = [_f32p, C.c_int, _f32p, C.c_int64, C.c_int,
                                                _f32p]
        L.ref_softmax_rows.argtypes = [_f32p, C.c_int, C.c_int64, _f32p]
        L.ref_expand_beams.argtypes = [_f32p, C.c_int, C.c_int64, _f64p, _u32p, _f64p, _u32p,
                                       C.c_int, C.c_int, C.c_void_p, _f64p, _u32p, _i64p,
                                       C.POINTER(C.c_int)]
        L.ref_exact_topb_logits.argtypes = [_f32p, C.c_int, C.c_int64, C.c_int, _u32p, _f32p]
        L.ref_synth_model.restype = C.c_void_p
        L.ref_synth_model.argtypes = [C.c_uint32, C.c_int, C.c_uint64, C.c_float]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_get.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.ref_model_set.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_step_hidden.argtypes = [C.c_void_p, _f32p, C.c_uint32, _f32p]
        L.ref_ctx_create.restype = C.c_void_p
        L.ref_ctx_create.argtypes = [_f32p, C.c_uint32, C.c_int, _f32p]
        L.ref_ctx_free.argtypes = [C.c_void_p]
        L.ref_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int, _f32p, C.c_int, _f64p, _u32p,
                               C.c_int, C.c_uint32, C.c_int, _u32p, C.c_int, _f64p, _u32p,
                               _i64p, C.POINTER(C.c_int), C.POINTER(C.c_uint32), _f64p]
        L.ref_decode.restype = C.c_void_p
        L.ref_decode.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_int, C.c_int, _u32p,
                                 C.c_int, C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        L.ref_decode_free.argtypes = [C.c_void_p]
        L.ref_decode_info.argtypes = [C.c_void_p, _i32p, _u64p, _f64p]
        L.ref_decode_hyp.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int)]
        L.ref_decode_steps.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]

    def _chk(self, rc, what):
        if rc:
            _raise(rc, what, self.lib.ref_last_error().decode())

    def set_threads(self, n: int) -> None:
        self.lib.ref_set_threads(n)

    def max_threads(self) -> int:
        return int(self.lib.ref_max_threads())

    def mix_seed(self, seed, stream):
        return int(self.lib.ref_mix_seed(seed, stream))

    def splitmix(self, seed, n):
        out = np.zeros(n, np.uint64)
        self.lib.ref_splitmix_next(seed, out, n)
        return out

    def gaussian(self, seed, n, scale=1.0):
        out = np.zeros(n, np.float32)
        self.lib.ref_gaussian_fill(seed, out, n, scale)
        return out

    def wta_params_check(self, K, u, W):
        self._chk(self.lib.ref_wta_params_check(K, u, W), "WtaParams")

    def generate_perms(self, d, P, K, seed):
        out = np.zeros((P, K), np.uint32)
        self._chk(self.lib.ref_generate_perms(d, P, K, seed, out), "PermutationSet")
        return out

    def hash_matrix(self, M, K, u, W, seed=None, perms=None):
        M = c32(M)
        n, d = M.shape
        out = np.zeros((n, W), np.uint32)
        if perms is None:
            self._chk(self.lib.ref_hash_matrix(M, n, d, K, u, W, seed, out), "hash_matrix")
        else:
            self._chk(self.lib.ref_hash_matrix_perms(M, n, d, K, u, W, cu32(perms), out),
                      "hash_matrix")
        return out

    def pack_bands(self, indices, K, u, W):
        out = np.zeros(W, np.uint32)
        self._chk(self.lib.ref_pack_bands(cu32(indices), K, u, W, out), "pack_bands")
        return out

    def _tables(self, h, V, W) -> BandTables:
        word_ids = np.zeros((W, V), np.uint32)
        lgs = np.zeros(W, np.uint32)
        muls = np.zeros((W, 2), np.uint64)
        tabs = []
        for w in range(W):
            self.lib.ref_index_band_words(h, w, word_ids[w])
            lg, m0, m1 = C.c_uint32(), C.c_uint64(), C.c_uint64()
            self.lib.ref_index_table(h, w, C.byref(lg), C.byref(m0), C.byref(m1), None)
            s = np.zeros((2 << lg.value, 3), np.uint32)
            self.lib.ref_index_table(h, w, C.byref(lg), C.byref(m0), C.byref(m1),
                                     s.ctypes.data)
            lgs[w], muls[w] = lg.value, (m0.value, m1.value)
            tabs.append(s)
        lgmax = int(lgs.max()) if W else 1
        slots = np.zeros((W, 2 << lgmax, 3), np.uint32)
        slots[..., 0] = EMPTY_CODE
        for w, s in enumerate(tabs):
            slots[w, : len(s)] = s
        return BandTables(word_ids, lgs, muls, slots, V)

    def band_index_build(self, codes, seed) -> BandTables:
        codes = cu32(codes)
        V, W = codes.shape
        h = self.lib.ref_index_from_codes(codes, V, W, seed)
        if not h:
            _raise(2, "BandIndex::build", self.lib.ref_last_error().decode())
        try:
            return self._tables(h, V, W)
        finally:
            self.lib.ref_index_free(h)

    def lookup_hits_codes(self, codes, seed, q):
        codes, q = cu32(codes), cu32(q)
        V, W = codes.shape
        h = self.lib.ref_index_from_codes(codes, V, W, seed)
        try:
            L = np.zeros((q.shape[0], V), np.int32)
            self._chk(self.lib.ref_index_lookup_hits(h, q, q.shape[0], L), "lookup_hits")
            return L
        finally:
            self.lib.ref_index_free(h)

    def lookup_hits_bruteforce(self, vocab_codes, q):
        vocab_codes, q = cu32(vocab_codes), cu32(q)
        V, W = vocab_codes.shape
        L = np.zeros((q.shape[0], V), np.int32)
        self.lib.ref_lookup_hits_bruteforce(vocab_codes, V, q, q.shape[0], W, L)
        return L

    def cuckoo_build(self, keys, starts, lens, seed):
        keys, starts, lens = cu32(keys), cu32(starts), cu32(lens)
        n = len(keys)
        lgmax = max(1, int(np.ceil(np.log2(max(n, 1)))))
        slots = np.zeros((2 << lgmax, 3), np.uint32)
        lg, m0, m1 = C.c_uint32(), C.c_uint64(), C.c_uint64()
        self._chk(self.lib.ref_cuckoo_build(keys, starts, lens, n, seed, C.byref(lg),
                                            C.byref(m0), C.byref(m1), slots, slots.size),
                  "CuckooTable::build")
        return int(lg.value), np.array([m0.value, m1.value], np.uint64), slots[: 2 << lg.value]

    def select_candidates(self, L, t):
        L = np.ascontiguousarray(L, np.int32)
        B, V = L.shape
        ids = np.zeros(max(V, 1), np.uint32)
        n, ft = C.c_uint32(), C.c_uint32()
        self._chk(self.lib.ref_select_candidates(L, B, V, t, ids, C.byref(n), C.byref(ft)),
                  "select_candidates")
        return ids[: n.value].copy(), int(ft.value)

    def merge_top_frequent(self, ids, from_thr, T, specials, V):
        ids = cu32(ids)
        specials = cu32(specials if len(specials) else np.zeros(0, np.uint32))
        out = np.zeros(len(ids) + T + len(specials) + 1, np.uint32)
        n = C.c_uint32()
        prov = np.zeros(3, np.uint32)
        self._chk(self.lib.ref_merge_top_frequent(ids, len(ids), from_thr, T, specials,
                                                  len(specials), V, out, C.byref(n), prov),
                  "merge_top_frequent")
        return out[: n.value].copy(), tuple(int(x) for x in prov)

    def gather(self, E, ids):
        E, ids = c32(E), cu32(ids)
        out = np.zeros((len(ids), E.shape[1]), np.float32)
        self._chk(self.lib.ref_gather(E, E.shape[0], E.shape[1], ids, len(ids), out), "gather")
        return out

    def compute_logits(self, H, Esub):
        H, Esub = c32(H), c32(Esub)
        out = np.zeros((H.shape[0], Esub.shape[0]), np.float32)
        self._chk(self.lib.ref_compute_logits(H, H.shape[0], Esub, Esub.shape[0], H.shape[1],
                                              out), "compute_logits")
        return out

    def softmax_rows(self, logits):
        logits = c32(logits)
        out = np.zeros_like(logits)
        self._chk(self.lib.ref_softmax_rows(logits, logits.shape[0], logits.shape[1], out),
                  "softmax_rows")
        return out

    def expand_beams(self, probs, cum, live, frozen=(), B=1, id_map=None):
        probs = c32(probs)
        rows, n = probs.shape
        fz_s = np.array([f[0] for f in frozen] or [0.0], np.float64)
        fz_b = np.array([f[1] for f in frozen] or [0], np.uint32)
        m = max(1, min(B, rows * n + len(frozen)))
        os_, ob, ow = np.zeros(m), np.zeros(m, np.uint32), np.zeros(m, np.int64)
        nout = C.c_int()
        idm = cu32(id_map) if id_map is not None and len(id_map) else None
        self._chk(self.lib.ref_expand_beams(
            probs, rows, n, np.ascontiguousarray(cum, np.float64), cu32(live), fz_s, fz_b,
            len(frozen), B, idm.ctypes.data if idm is not None else None, os_, ob, ow,
            C.byref(nout)), "expand_beams")
        k = nout.value
        return os_[:k].copy(), ob[:k].copy(), ow[:k].copy()

    def exact_topb_logits(self, logits, b):
        logits = c32(logits)
        rows, n = logits.shape
        ids = np.zeros((rows, b), np.uint32)
        vals = np.zeros((rows, b), np.float32)
        self._chk(self.lib.ref_exact_topb_logits(logits, rows, n, b, ids, vals), "exact_topb")
        return ids, vals

    def synth_model(self, V, d, seed, bias_strength):
        h = self.lib.ref_synth_model(V, d, seed, bias_strength)
        if not h:
            _raise(1, "synth_model", self.lib.ref_last_error().decode())
        m = {"E": np.zeros((V, d), np.float32), "wh": np.zeros((d, d), np.float32),
             "we": np.zeros((d, d), np.float32), "h0": np.zeros(d, np.float32),
             "bias": np.zeros(V, np.float32)}
        self.lib.ref_model_get(h, *[a.ctypes.data for a in m.values()])
        self.lib.ref_model_free(h)
        return m


def oracle_step(o: "Oracle", bt: BandTables, perms, E, bias, K, u, W, hidden, scores,
                finished, n_hyp, B, T, t, specials):
    """One decode() kLsh step for one sentence, restated from the oracle pieces
    (src/beam_decoder.cpp:166-289): returns dict(codes, ids, prov, probs,
    choices=(scores, beams, words))."""
    live = [i for i in range(n_hyp) if not finished[i]]
    frozen = [(float(scores[i]), i) for i in range(n_hyp) if finished[i]]
    H = np.ascontiguousarray(hidden[live], np.float32)
    V = E.shape[0]
    codes = o.hash_matrix(H, K, u, W, perms=perms)
    if t == 0:
        ids, ft = np.arange(V, dtype=np.uint32), V
    else:
        L = o.lookup_hits(bt, codes)
        ids, ft = o.select_candidates(L, t)
    ids, prov = o.merge_top_frequent(ids, ft, T, specials, V)
    logits = o.compute_logits_ids(H, E, ids, bias)
    probs = o.softmax_rows(logits)
    ch = o.expand_beams(probs, np.asarray(scores, np.float64)[live], live, frozen, B, ids)
    return dict(codes=codes, ids=ids, prov=prov, logits=logits, probs=probs, choices=ch,
                live=live)


def oracle_full_step(o: "Oracle", E, bias, hidden, scores, finished, n_hyp, B):
    """decode()'s kFull step: every word is a candidate, id_map empty."""
    live = [i for i in range(n_hyp) if not finished[i]]
    frozen = [(float(scores[i]), i) for i in range(n_hyp) if finished[i]]
    H = np.ascontiguousarray(hidden[live], np.float32)
    logits = o.compute_logits_ids(H, E, None, bias)
    probs = o.softmax_rows(logits)
    ch = o.expand_beams(probs, np.asarray(scores, np.float64)[live], live, frozen, B, None)
    return dict(logits=logits, probs=probs, choices=ch, live=live)


class ReferenceStepper:
    """Drives the reference's per-step hot path (ref_step in ref_shim.cpp:
    decode()'s kLsh/kFull body + expand_beams) for the CPU baseline."""

    def __init__(self, ref: "Reference", E, bias, K, u, W, perm_seed, index_seed,
                 build_index=True):
        self.ref, self.lib = ref, ref.lib
        E = c32(E)
        self.V, self.d = E.shape
        self.ctx = self.lib.ref_ctx_create(E, self.V, self.d, c32(bias))
        self.index = (self.lib.ref_index_from_embeddings(E, self.V, self.d, K, u, W, perm_seed,
                                                         index_seed) if build_index else None)

    def step(self, H, cum, B, T, t, specials, full=False):
        H = c32(H)
        rows = H.shape[0]
        sp = cu32(specials if len(specials) else [0])
        os_, ob, ow = np.zeros(B), np.zeros(B, np.uint32), np.zeros(B, np.int64)
        nout, ncand = C.c_int(), C.c_uint32()
        stages = np.zeros(7)
        rc = self.lib.ref_step(self.ctx, self.index, 1 if full else 0, H, rows,
                               np.ascontiguousarray(cum, np.float64),
                               np.arange(rows, dtype=np.uint32), B, T, t, sp, len(specials),
                               os_, ob, ow, C.byref(nout), C.byref(ncand), stages)
        if rc:
            _raise(rc, "ref_step", self.lib.ref_last_error().decode())
        k = nout.value
        return (os_[:k], ob[:k], ow[:k]), int(ncand.value), stages

    def close(self):
        if self.index:
            self.lib.ref_index_free(self.index)
            self.index = None
        if self.ctx:
            self.lib.ref_ctx_free(self.ctx)
            self.ctx = None

"""Host-side mirror of the reference's lshbeam API, over the C ABI.

Function names, argument meaning and error classes follow
/root/reference/proj/include/lshbeam/*.hpp (ValueError <-> std::invalid_argument,
RuntimeError <-> std::runtime_error), so the parity tests read like the
reference's own suites. Every call runs on the GPU through
liblshbeam_b200.so; nothing here computes on the CPU.

Stage functions take/return numpy arrays (host buffers, synchronous, like
the reference's by-value API). ``Batch`` is the fused, device-resident step
over S sentences; its state lives in torch CUDA tensors (torch is used only
for device memory and streams).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

EMPTY_CODE = 0x7FFFFFFF
PARITY, FAST = N.MODE_PARITY, N.MODE_FAST


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def bits_for(K: int) -> int:
    """WtaParams::bits_for (src/wta_hash.cpp:12-16)."""
    b = 0
    while (1 << b) < K:
        b += 1
    return b


class Context:
    """A device + CUDA stream (lsb_ctx). ``stream`` is a cudaStream_t handle
    (e.g. ``torch.cuda.current_stream().cuda_stream``) or None for a private
    non-blocking stream."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = N.load()
        h = C.c_void_p()
        # torch reports its default (legacy NULL) stream as handle 0; the C ABI
        # reads NULL as "create a private stream", so map 0 to cudaStreamLegacy
        # (LSB_STREAM_LEGACY) -- otherwise work queued by torch on the default
        # stream would not be ordered with ours.
        if stream == 0:
            stream = N.STREAM_LEGACY
        N.check(self.lib.lsb_ctx_create(device, stream, C.byref(h)), "lsb_ctx_create")
        self.h = h
        self.device = device

    def sync(self):
        N.check(self.lib.lsb_ctx_sync(self.h), "sync")

    @property
    def stream(self) -> int:
        return self.lib.lsb_ctx_stream(self.h) or 0

    @property
    def sm_count(self) -> int:
        return self.lib.lsb_ctx_sm_count(self.h)

    def fp32x2_peak(self) -> float:
        """Measured paired-FP32 peak of this GPU in lane-ops/s (the K4 PARITY
        roofline denominator; lsb_measure_fp32x2_peak)."""
        v = C.c_double(0.0)
        N.check(self.lib.lsb_measure_fp32x2_peak(self.h, C.byref(v)), "lsb_measure_fp32x2_peak")
        return float(v.value)

    def selftest_log(self, p_dev: int, out_dev: int, n: int):
        """out[k] = log((double) p[k]) by the device's glibc-exact log
        (lsb_selftest_log); device pointers."""
        N.check(self.lib.lsb_selftest_log(self.h, p_dev, out_dev, n), "lsb_selftest_log")

    def selftest_exp(self, x_dev: int, out_dev: int, n: int):
        """out[k] = exp(x[k]) by the device's glibc-exact exp (lsb_selftest_exp);
        device pointers to doubles."""
        N.check(self.lib.lsb_selftest_exp(self.h, x_dev, out_dev, n), "lsb_selftest_exp")

    @property
    def launches(self) -> int:
        return int(self.lib.lsb_ctx_launch_count(self.h))

    def set_parallel_cuckoo(self, on: bool = True):
        """Cuckoo slot placement of later index builds: False = the
        reference's insertion order (slots equal CuckooTable::build's), True =
        parallel atomicExch placement (same lookups, different slots)."""
        N.check(self.lib.lsb_ctx_set_parallel_cuckoo(self.h, int(on)))

    def close(self):
        if getattr(self, "h", None):
            self.lib.lsb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------ stage entry points
    def hash_matrix(self, M, perms, K: int, u: int, W: int) -> np.ndarray:
        """hash_matrix(M, perms, params) (src/wta_hash.cpp:147-171)."""
        M = _f32(M)
        if M.ndim != 2:
            raise ValueError("hash_matrix: expected a matrix")
        perms = _u32(perms)
        n, d = M.shape
        if n and perms.shape[1] != K:
            raise ValueError("hash_matrix: permutation window mismatch")
        out = np.zeros((n, W), np.uint32)
        N.check(self.lib.lsb_wta_hash(self.h, _p(M), n, d, _p(perms), K, u, W, _p(out)),
                "hash_matrix")
        return out

    def lookup_hits(self, index: "Index", q) -> np.ndarray:
        """BandIndex::lookup_hits (src/band_index.cpp:134-167)."""
        q = _u32(q)
        if q.ndim != 2 or q.shape[1] != index.W:
            raise ValueError("lookup_hits: band count mismatch")
        B = q.shape[0]
        L = np.zeros((B, index.vocab), np.int32)
        N.check(self.lib.lsb_lookup_hits(self.h, index.h, _p(q), B, _p(L)), "lookup_hits")
        return L

    def select_candidates(self, L, t: int):
        """select_candidates(L, t) -> (ids, from_threshold)
        (src/candidate_selector.cpp:14-55)."""
        L = np.ascontiguousarray(L, np.int32)
        B, V = L.shape
        ids = np.zeros(max(V, 1), np.uint32)
        n, ft = C.c_uint32(), C.c_uint32()
        N.check(self.lib.lsb_select_candidates(self.h, _p(L), B, V, t, _p(ids), C.byref(n),
                                               C.byref(ft)), "select_candidates")
        return ids[: n.value].copy(), int(ft.value)

    def merge_top_frequent(self, ids, from_threshold: int, T: int, specials, V: int):
        """merge_top_frequent -> (ids, (from_threshold, from_top, from_specials))
        (src/candidate_selector.cpp:57-103)."""
        ids = _u32(ids)
        sp = _u32(specials if len(specials) else np.zeros(0, np.uint32))
        out = np.zeros(len(ids) + T + len(sp) + 1, np.uint32)
        n = C.c_uint32()
        prov = np.zeros(3, np.uint32)
        N.check(self.lib.lsb_merge_top_frequent(self.h, _p(ids), len(ids), from_threshold, T,
                                                _p(sp), len(sp), V, _p(out), C.byref(n),
                                                _p(prov)), "merge_top_frequent")
        return out[: n.value].copy(), tuple(int(x) for x in prov)

    def gather_embeddings(self, model: "Model", ids) -> np.ndarray:
        """gather_embeddings(E, cands).rows (src/candidate_selector.cpp:105-119)."""
        ids = _u32(ids)
        out = np.zeros((len(ids), model.dim), np.float32)
        N.check(self.lib.lsb_gather_embeddings(self.h, model.h, _p(ids), len(ids), _p(out)),
                "gather_embeddings")
        return out

    def compute_logits(self, H, E_sub, mode: int = PARITY) -> np.ndarray:
        """compute_logits(H, E_sub) (src/beam_decoder.cpp:23-44)."""
        H, E_sub = _f32(H), _f32(E_sub)
        if H.shape[1] != E_sub.shape[1]:
            raise ValueError("compute_logits: inner dimensions disagree")
        out = np.zeros((H.shape[0], E_sub.shape[0]), np.float32)
        N.check(self.lib.lsb_compute_logits(self.h, _p(H), H.shape[0], _p(E_sub), E_sub.shape[0],
                                            H.shape[1], mode, _p(out)), "compute_logits")
        return out

    def softmax_rows(self, logits) -> np.ndarray:
        """softmax_rows(logits) (src/beam_decoder.cpp:46-74)."""
        logits = _f32(logits)
        out = np.zeros_like(logits)
        N.check(self.lib.lsb_softmax_rows(self.h, _p(logits), logits.shape[0], logits.shape[1],
                                          _p(out)), "softmax_rows")
        return out

    def expand_beams(self, probs, cum, live, frozen=(), B: int = 1, id_map=None):
        """expand_beams -> (scores, beams, words) (src/beam_decoder.cpp:76-111).
        ``frozen`` is a sequence of (score, beam)."""
        probs = _f32(probs)
        rows, n = probs.shape
        cum = np.ascontiguousarray(cum, np.float64)
        live = _u32(live)
        if len(cum) != rows or len(live) != rows:
            raise ValueError("expand_beams: row metadata mismatch")
        if id_map is not None and len(id_map) and len(id_map) != n:
            raise ValueError("expand_beams: id_map size mismatch")
        fz = (N.lsb_choice * max(1, len(frozen)))()
        for k, (s, b) in enumerate(frozen):
            fz[k].score, fz[k].beam, fz[k].word = s, b, -1
        out = (N.lsb_choice * max(1, B))()
        nout = C.c_int()
        idm = _u32(id_map) if id_map is not None and len(id_map) else None
        N.check(self.lib.lsb_expand_beams(self.h, _p(probs), rows, n, _p(cum), _p(live), fz,
                                          len(frozen), B, _p(idm), out, C.byref(nout)),
                "expand_beams")
        k = nout.value
        return (np.array([out[i].score for i in range(k)], np.float64),
                np.array([out[i].beam for i in range(k)], np.uint32),
                np.array([out[i].word for i in range(k)], np.int64))


def exact_topb(ctx: "Context", model: "Model", H, rows: int, b: int, bias: bool = True):
    """exact_topb_logits(H . E^T (+ bias), b) (src/eval_oracle.cpp:11-44) on the
    device: per row the b largest full-vocabulary logits, ties to the smaller
    id. ``H`` is a device pointer (int) or a host array. Returns (ids, values)."""
    ids = np.zeros((rows, b), np.uint32)
    vals = np.zeros((rows, b), np.float32)
    if isinstance(H, int):
        N.check(ctx.lib.lsb_exact_topb(ctx.h, model.h, H, rows, 1, b, int(bias), _p(ids),
                                       _p(vals)), "exact_topb")
    else:
        Hh = _f32(H)
        N.check(ctx.lib.lsb_exact_topb(ctx.h, model.h, _p(Hh), rows, 0, b, int(bias), _p(ids),
                                       _p(vals)), "exact_topb")
    return ids, vals


class Recurrent:
    """Device W_h, W_e of the synthetic scorer (lsb_recurrent): the
    recurrence h' = tanh(W_h h + W_e E[token]) (src/model_provider.cpp:83-102)."""

    def __init__(self, ctx: "Context", wh, we):
        self.ctx, self.lib = ctx, ctx.lib
        wh, we = _f32(wh), _f32(we)
        h = C.c_void_p()
        N.check(self.lib.lsb_recurrent_create(ctx.h, _p(wh), _p(we), wh.shape[0], C.byref(h)),
                "lsb_recurrent_create")
        self.h, self.dim = h, wh.shape[0]

    def step_hidden(self, model: "Model", h, token: int) -> np.ndarray:
        """step_hidden(model, h, token) with host vectors."""
        h = _f32(h)
        out = np.zeros(self.dim, np.float32)
        N.check(self.lib.lsb_step_hidden(self.ctx.h, model.h, self.h, _p(h), token, _p(out)),
                "step_hidden")
        return out

    def step(self, model: "Model", hidden_in: int, tokens: int, n: int, hidden_out: int):
        """n hypotheses on the device (pointers): tokens[k] < 0 copies the row."""
        N.check(self.lib.lsb_recurrence(self.ctx.h, model.h, self.h, hidden_in, tokens, n,
                                        hidden_out), "lsb_recurrence")

    def close(self):
        if getattr(self, "h", None):
            self.lib.lsb_recurrent_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Model:
    """Device copy of E (|V| x d) and the logit bias (lsb_model)."""

    def __init__(self, ctx: Context, E, bias=None, device_ptrs: tuple | None = None):
        self.ctx, self.lib = ctx, ctx.lib
        h = C.c_void_p()
        if device_ptrs is not None:
            e_ptr, b_ptr, V, d = device_ptrs
            N.check(self.lib.lsb_model_create_dev(ctx.h, e_ptr, V, d, b_ptr, C.byref(h)),
                    "lsb_model_create_dev")
        else:
            E = _f32(E)
            V, d = E.shape
            b = _f32(bias) if bias is not None else None
            N.check(self.lib.lsb_model_create(ctx.h, _p(E), V, d, _p(b), C.byref(h)),
                    "lsb_model_create")
        self.h, self.vocab, self.dim = h, int(V), int(d)

    def close(self):
        if getattr(self, "h", None):
            self.lib.lsb_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class BandView:
    word_ids: np.ndarray
    lg: int
    mul: np.ndarray
    slots: np.ndarray  # (2*2^lg, 3): key, start, length


class Index:
    """WTA permutations + band index on the device (lsb_index).

    ``Index(ctx, model=..., K=, u=, W=, perm_seed=, index_seed=)`` is
    build_lsh_index (src/band_index.cpp:189-196);
    ``Index(ctx, codes=..., index_seed=)`` is BandIndex::build
    (src/band_index.cpp:90-132)."""

    def __init__(self, ctx: Context, model: Model | None = None, K: int = 8, u: int = 3,
                 W: int = 16, perm_seed: int = 0, index_seed: int = 0, codes=None):
        self.ctx, self.lib = ctx, ctx.lib
        h = C.c_void_p()
        if codes is not None:
            codes = _u32(codes)
            V, W = codes.shape
            N.check(self.lib.lsb_index_build_codes(ctx.h, _p(codes), V, W, index_seed,
                                                   C.byref(h)), "BandIndex::build")
        else:
            N.check(self.lib.lsb_index_build(ctx.h, model.h, K, u, W, perm_seed, index_seed,
                                             C.byref(h)), "build_lsh_index")
        self.h = h
        info = N.lsb_index_info()
        N.check(self.lib.lsb_index_info_get(h, C.byref(info)))
        self.info = info
        self.vocab, self.W, self.K, self.u = info.vocab, info.W, info.K, info.u

    def band(self, w: int) -> BandView:
        lg = C.c_uint32()
        N.check(self.lib.lsb_index_band(self.h, w, None, C.byref(lg), None, None))
        ids = np.zeros(self.vocab, np.uint32)
        mul = np.zeros(2, np.uint64)
        slots = np.zeros((2 << lg.value, 3), np.uint32)
        N.check(self.lib.lsb_index_band(self.h, w, _p(ids), C.byref(lg), _p(mul), _p(slots)))
        return BandView(ids, lg.value, mul, slots)

    def band_words(self, w: int) -> np.ndarray:
        return self.band(w).word_ids

    def find(self, bands, keys):
        bands = np.ascontiguousarray(bands, np.int32)
        keys = _u32(keys)
        n = len(keys)
        st, ln = np.zeros(n, np.uint32), np.zeros(n, np.uint32)
        fd = np.zeros(n, np.uint8)
        N.check(self.lib.lsb_index_find(self.ctx.h, self.h, _p(bands), _p(keys), n, _p(st),
                                        _p(ln), _p(fd)), "find")
        return fd.astype(bool), st, ln

    def perms(self) -> np.ndarray:
        out = np.zeros((self.u * self.W, self.K), np.uint32)
        N.check(self.lib.lsb_index_perms(self.h, _p(out)))
        return out

    def close(self):
        if getattr(self, "h", None):
            self.lib.lsb_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Batch:
    """Fused per-step pipeline over S sentences x B hypothesis slots (lsb_batch)."""

    def __init__(self, ctx: Context, model: Model, index: Index | None, S: int, B: int,
                 T: int = 0, t: int = 1, specials=(), mode: int = PARITY,
                 full_vocab: bool = False, top_only: bool = False):
        self.ctx, self.lib = ctx, ctx.lib
        sp = _u32(list(specials)) if len(specials) else np.zeros(1, np.uint32)
        self._sp = sp
        cfg = N.lsb_step_config(S, B, T, t, sp.ctypes.data_as(C.POINTER(C.c_uint32)),
                                len(specials), mode, 1 if full_vocab else 0,
                                1 if top_only else 0)
        h = C.c_void_p()
        N.check(self.lib.lsb_batch_create(ctx.h, model.h, index.h if index else None,
                                          C.byref(cfg), C.byref(h)), "lsb_batch_create")
        self.h, self.S, self.B, self.dim, self.vocab = h, S, B, model.dim, model.vocab
        self._keep = (model, index)  # the C handles borrow these; keep them alive

    def keep_probs(self, on: bool = True):
        N.check(self.lib.lsb_batch_keep_probs(self.h, int(on)))

    def profile(self, on: bool = True, every: int = 1):
        """Per-stage CUDA events; ``every`` > 1 samples every n-th step."""
        N.check(self.lib.lsb_batch_profile(self.h, (every if every > 1 else 1) if on else 0))

    def stage_ms(self) -> np.ndarray:
        out = np.zeros(5, np.float32)
        N.check(self.lib.lsb_batch_stage_ms(self.h, _p(out)))
        return out

    def stage_totals(self):
        """(ms per stage summed over recorded steps, number of steps)."""
        out = np.zeros(5, np.float32)
        n = C.c_int()
        N.check(self.lib.lsb_batch_stage_totals(self.h, _p(out), C.byref(n)))
        return out, n.value

    def step_host_ptrs(self, hidden, scores, finished, n_hyp, choices, n_choices,
                       hidden_out=0):
        """lsb_step_host with raw host pointers (e.g. pinned torch tensors)."""
        st = N.lsb_state_host(hidden, scores, finished or None, n_hyp or None)
        N.check(self.lib.lsb_step_host(self.h, C.byref(st), choices, n_choices,
                                       hidden_out or None), "lsb_step_host")

    def step_host_async(self, hidden, scores, finished, n_hyp, choices, n_choices):
        """lsb_step_host_async with raw (pinned) host pointers; call wait()."""
        st = N.lsb_state_host(hidden, scores, finished or None, n_hyp or None)
        N.check(self.lib.lsb_step_host_async(self.h, C.byref(st), choices, n_choices),
                "lsb_step_host_async")

    def wait(self):
        N.check(self.lib.lsb_batch_wait(self.h), "lsb_batch_wait")

    def step(self, hidden, scores, finished=None, n_hyp=None, choices=None, n_choices=None,
             hidden_out=None):
        """Device step. Arguments are torch CUDA tensors (or raw pointers):
        hidden [S,B,d] f32, scores [S,B] f64, finished [S,B] u8, n_hyp [S] i32;
        outputs choices [S,B,3] int64-viewable buffer of lsb_choice, n_choices [S] i32."""
        ptr = lambda x: (x if isinstance(x, int) else x.data_ptr()) if x is not None else None
        st = N.lsb_state_dev(ptr(hidden), ptr(scores), ptr(finished), ptr(n_hyp))
        out = N.lsb_out_dev(ptr(choices), ptr(n_choices), ptr(hidden_out))
        N.check(self.lib.lsb_step(self.h, C.byref(st), C.byref(out)), "lsb_step")

    def graph_capture(self, hidden, scores, finished=None, n_hyp=None, choices=None,
                      n_choices=None, hidden_out=None):
        """Record one device step on these fixed buffers as a CUDA graph
        (lsb_batch_graph_capture); graph_launch() replays it."""
        ptr = lambda x: (x if isinstance(x, int) else x.data_ptr()) if x is not None else None
        st = N.lsb_state_dev(ptr(hidden), ptr(scores), ptr(finished), ptr(n_hyp))
        out = N.lsb_out_dev(ptr(choices), ptr(n_choices), ptr(hidden_out))
        N.check(self.lib.lsb_batch_graph_capture(self.h, C.byref(st), C.byref(out)),
                "lsb_batch_graph_capture")

    def graph_launch(self):
        N.check(self.lib.lsb_batch_graph_launch(self.h), "lsb_batch_graph_launch")

    def step_host(self, hidden, scores, finished=None, n_hyp=None, want_hidden=False):
        """End-to-end step from host arrays; returns (choices list per sentence, hidden_out)."""
        S, B, d = self.S, self.B, self.dim
        hidden = _f32(hidden).reshape(S, B, d)
        scores = np.ascontiguousarray(scores, np.float64).reshape(S, B)
        fin = np.ascontiguousarray(finished, np.uint8).reshape(S, B) if finished is not None else None
        nh = np.ascontiguousarray(n_hyp, np.int32) if n_hyp is not None else None
        st = N.lsb_state_host(_p(hidden), _p(scores), _p(fin), _p(nh))
        ch = (N.lsb_choice * (S * B))()
        nc = np.zeros(S, np.int32)
        ho = np.zeros((S, B, d), np.float32) if want_hidden else None
        N.check(self.lib.lsb_step_host(self.h, C.byref(st), ch, _p(nc), _p(ho)), "lsb_step_host")
        res = []
        for s in range(S):
            k = int(nc[s])
            res.append([(ch[s * B + j].score, ch[s * B + j].beam, ch[s * B + j].word)
                        for j in range(k)])
        return res, ho

    def candidates(self, s: int):
        n = C.c_uint32()
        prov = np.zeros(3, np.uint32)
        N.check(self.lib.lsb_batch_candidates(self.h, s, None, C.byref(n), _p(prov)))
        ids = np.zeros(max(1, n.value), np.uint32)
        N.check(self.lib.lsb_batch_candidates(self.h, s, _p(ids), C.byref(n), _p(prov)))
        return ids[: n.value], tuple(int(x) for x in prov)

    def query_codes(self, s: int, W: int) -> np.ndarray:
        out = np.zeros((self.B, W), np.uint32)
        N.check(self.lib.lsb_batch_query_codes(self.h, s, _p(out)))
        return out

    def probs(self, s: int) -> np.ndarray:
        n, _ = self.candidates(s)
        out = np.zeros((self.B, max(1, len(n))), np.float32)
        live = C.c_int()
        N.check(self.lib.lsb_batch_probs(self.h, s, _p(out), C.byref(live)))
        return out[: live.value, : len(n)]

    def close(self):
        if getattr(self, "h", None):
            self.lib.lsb_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""ctypes binding of the C ABI (include/lshbeam_b200.h).

Loads the in-tree liblshbeam_b200.so and fails loudly if it is missing:
there is no CPU fallback for any entry point.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liblshbeam_b200.so")

LSB_OK, LSB_EINVAL, LSB_ERUNTIME, LSB_ECUDA, LSB_ENOMEM = range(5)
MODE_PARITY, MODE_FAST = 0, 1
STREAM_LEGACY = 1  # LSB_STREAM_LEGACY: cudaStreamLegacy, the legacy default stream


class lsb_choice(C.Structure):
    _fields_ = [("score", C.c_double), ("beam", C.c_uint32), ("_pad", C.c_uint32),
                ("word", C.c_int64)]


class lsb_index_info(C.Structure):
    _fields_ = [("vocab", C.c_uint32), ("W", C.c_int), ("K", C.c_int), ("u", C.c_int),
                ("bits_per_index", C.c_int), ("dim", C.c_int), ("perm_seed", C.c_uint64),
                ("index_seed", C.c_uint64), ("max_span", C.c_uint32),
                ("build_attempts", C.c_uint32)]


class lsb_step_config(C.Structure):
    _fields_ = [("S", C.c_int), ("B", C.c_int), ("top_merge", C.c_uint32),
                ("threshold", C.c_int), ("specials", C.POINTER(C.c_uint32)),
                ("nspec", C.c_int), ("mode", C.c_int), ("full_vocab", C.c_int),
                ("top_only", C.c_int)]


class lsb_state_dev(C.Structure):
    _fields_ = [("hidden", C.c_void_p), ("scores", C.c_void_p), ("finished", C.c_void_p),
                ("n_hyp", C.c_void_p)]


class lsb_out_dev(C.Structure):
    _fields_ = [("choices", C.c_void_p), ("n_choices", C.c_void_p),
                ("hidden_out", C.c_void_p)]


lsb_state_host = lsb_state_dev  # same layout, host pointers


class lsb_shard_top(C.Structure):
    _fields_ = [("e", C.c_float), ("word", C.c_uint32)]

VP = C.c_void_p
PP = C.POINTER(C.c_void_p)
U32 = C.c_uint32
U64 = C.c_uint64
I32 = C.c_int32
I64 = C.c_int64

# (name, restype, argtypes)
_SIGS = [
    ("lsb_last_error", C.c_char_p, []),
    ("lsb_abi_version", C.c_int, []),
    ("lsb_ctx_create", C.c_int, [C.c_int, VP, PP]),
    ("lsb_ctx_destroy", C.c_int, [VP]),
    ("lsb_ctx_sync", C.c_int, [VP]),
    ("lsb_ctx_stream", VP, [VP]),
    ("lsb_ctx_device", C.c_int, [VP]),
    ("lsb_ctx_sm_count", C.c_int, [VP]),
    ("lsb_ctx_launch_count", U64, [VP]),
    ("lsb_model_create", C.c_int, [VP, VP, U32, C.c_int, VP, PP]),
    ("lsb_model_create_dev", C.c_int, [VP, VP, U32, C.c_int, VP, PP]),
    ("lsb_model_destroy", C.c_int, [VP]),
    ("lsb_model_embeddings_dev", VP, [VP]),
    ("lsb_model_vocab", U32, [VP]),
    ("lsb_model_dim", C.c_int, [VP]),
    ("lsb_index_build", C.c_int, [VP, VP, C.c_int, C.c_int, C.c_int, U64, U64, PP]),
    ("lsb_index_build_codes", C.c_int, [VP, VP, U32, C.c_int, U64, PP]),
    ("lsb_index_destroy", C.c_int, [VP]),
    ("lsb_index_info_get", C.c_int, [VP, C.POINTER(lsb_index_info)]),
    ("lsb_index_band", C.c_int, [VP, C.c_int, VP, C.POINTER(U32), VP, VP]),
    ("lsb_index_find", C.c_int, [VP, VP, VP, VP, C.c_size_t, VP, VP, VP]),
    ("lsb_index_perms", C.c_int, [VP, VP]),
    ("lsb_wta_hash", C.c_int, [VP, VP, I64, C.c_int, VP, C.c_int, C.c_int, C.c_int, VP]),
    ("lsb_lookup_hits", C.c_int, [VP, VP, VP, C.c_int, VP]),
    ("lsb_select_candidates", C.c_int, [VP, VP, C.c_int, U32, C.c_int, VP, C.POINTER(U32),
                                        C.POINTER(U32)]),
    ("lsb_merge_top_frequent", C.c_int, [VP, VP, U32, U32, U32, VP, U32, U32, VP,
                                         C.POINTER(U32), VP]),
    ("lsb_gather_embeddings", C.c_int, [VP, VP, VP, U32, VP]),
    ("lsb_compute_logits", C.c_int, [VP, VP, C.c_int, VP, I64, C.c_int, C.c_int, VP]),
    ("lsb_softmax_rows", C.c_int, [VP, VP, C.c_int, I64, VP]),
    ("lsb_expand_beams", C.c_int, [VP, VP, C.c_int, I64, VP, VP, VP, C.c_int, C.c_int, VP,
                                   VP, C.POINTER(C.c_int)]),
    ("lsb_batch_create", C.c_int, [VP, VP, VP, C.POINTER(lsb_step_config), PP]),
    ("lsb_batch_destroy", C.c_int, [VP]),
    ("lsb_step", C.c_int, [VP, C.POINTER(lsb_state_dev), C.POINTER(lsb_out_dev)]),
    ("lsb_step_host", C.c_int, [VP, C.POINTER(lsb_state_host), VP, VP, VP]),
    ("lsb_step_host_async", C.c_int, [VP, C.POINTER(lsb_state_host), VP, VP]),
    ("lsb_batch_wait", C.c_int, [VP]),
    ("lsb_batch_graph_capture", C.c_int, [VP, C.POINTER(lsb_state_dev), C.POINTER(lsb_out_dev)]),
    ("lsb_batch_graph_launch", C.c_int, [VP]),
    ("lsb_batch_candidates", C.c_int, [VP, C.c_int, VP, C.POINTER(U32), VP]),
    ("lsb_batch_query_codes", C.c_int, [VP, C.c_int, VP]),
    ("lsb_batch_probs", C.c_int, [VP, C.c_int, VP, C.POINTER(C.c_int)]),
    ("lsb_batch_n_cand_dev", VP, [VP]),
    ("lsb_batch_keep_probs", C.c_int, [VP, C.c_int]),
    ("lsb_batch_profile", C.c_int, [VP, C.c_int]),
    ("lsb_batch_stage_ms", C.c_int, [VP, VP]),
    ("lsb_batch_stage_totals", C.c_int, [VP, VP, C.POINTER(C.c_int)]),
    # device memory helpers
    ("lsb_device_alloc", C.c_int, [VP, C.c_size_t, PP]),
    ("lsb_device_free", C.c_int, [VP, VP]),
    ("lsb_copy_to_device", C.c_int, [VP, VP, VP, C.c_size_t]),
    ("lsb_copy_to_host", C.c_int, [VP, VP, VP, C.c_size_t]),
    # drop-in support
    ("lsb_ctx_set_parallel_cuckoo", C.c_int, [VP, C.c_int]),
    ("lsb_cuckoo_log2_capacity", U32, [C.c_size_t]),
    ("lsb_cuckoo_build", C.c_int, [VP, VP, VP, VP, U32, U64, C.POINTER(U32), VP, VP,
                                   C.POINTER(U32)]),
    ("lsb_wta_indices", C.c_int, [VP, VP, I64, C.c_int, VP, C.c_int, C.c_int, VP]),
    ("lsb_index_import", C.c_int, [VP, U32, C.c_int, VP, VP, VP, VP, VP, C.c_int, C.c_int,
                                   C.c_int, U64, PP]),
    ("lsb_recurrent_create", C.c_int, [VP, VP, VP, C.c_int, PP]),
    ("lsb_recurrent_destroy", C.c_int, [VP]),
    ("lsb_recurrence", C.c_int, [VP, VP, VP, VP, VP, C.c_int, VP]),
    ("lsb_step_hidden", C.c_int, [VP, VP, VP, VP, U32, VP]),
    ("lsb_measure_fp32x2_peak", C.c_int, [VP, C.POINTER(C.c_double)]),
    ("lsb_selftest_log", C.c_int, [VP, VP, VP, C.c_size_t]),
    ("lsb_selftest_exp", C.c_int, [VP, VP, VP, C.c_size_t]),
    ("lsb_exact_topb", C.c_int, [VP, VP, VP, C.c_int, C.c_int, C.c_int, C.c_int, VP, VP]),
    # vocabulary-sharded step
    ("lsb_shard_width", C.c_int, [VP]),
    ("lsb_shard_phase1", C.c_int, [VP, C.POINTER(lsb_state_dev), VP]),
    ("lsb_shard_phase2", C.c_int, [VP, C.POINTER(lsb_state_dev), VP, C.c_int, U32, VP, VP]),
    ("lsb_shard_phase3", C.c_int, [VP, C.POINTER(lsb_state_dev), VP, VP, C.c_int,
                                   C.POINTER(lsb_out_dev)]),
    ("lsb_shard_phase3_packed", C.c_int, [VP, C.POINTER(lsb_state_dev), VP, C.c_int,
                                          C.POINTER(lsb_out_dev)]),
    ("lsb_shard_xchg_create", C.c_int, [VP, C.c_int, C.c_int, C.POINTER(VP)]),
    ("lsb_shard_xchg_destroy", C.c_int, [VP]),
    ("lsb_shard_xchg_area", VP, [VP]),
    ("lsb_shard_xchg_ipc_handle", C.c_int, [VP, VP]),
    ("lsb_shard_xchg_open_ipc", C.c_int, [VP, C.c_int, VP]),
    ("lsb_shard_xchg_set_peer", C.c_int, [VP, C.c_int, VP]),
    ("lsb_shard_step_peer", C.c_int, [VP, VP, C.POINTER(lsb_state_dev), U32,
                                      C.POINTER(lsb_out_dev)]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None


class LshbeamError(Exception):
    pass


def load():
    """Load liblshbeam_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -m paper_1806_00588_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == LSB_OK:
        return
    msg = load().lsb_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == LSB_EINVAL:
        raise ValueError(text)
    if rc == LSB_ERUNTIME:
        raise RuntimeError(text)
    if rc == LSB_ENOMEM:
        raise MemoryError(text)
    raise LshbeamError(f"CUDA error: {text}")

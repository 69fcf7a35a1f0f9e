"""Synthetic scorer inputs drawn the way the reference's model provider draws
them (src/model_provider.cpp:14-74, include/lshbeam/rng.hpp:15-45), vectorised
with numpy: the i-th SplitMix64 output is a pure function of seed + i * gamma,
and gaussian() is the Box-Muller cosine branch over two consecutive draws.

Used by bench.py for the reference's validated operating point (V=50k,
d=256, bias 300; tests/acceptance.cpp:275-300) and its synthetic decode
start states (h0_s from mix_seed(seed, 100 + s)). numpy's
log / cos / tanh may differ from glibc's in the last double ulp, which the
float32 casts almost always absorb; this is input generation, not a parity
path (the oracle's generator is the bit-exact one)."""
from __future__ import annotations

import numpy as np

from .seeds import mix_seed

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix(seed: int, n: int, skip: int = 0) -> np.ndarray:
    """Outputs skip+1 .. skip+n of SplitMix64(seed).next() (uint64)."""
    with np.errstate(over="ignore"):
        i = np.arange(skip + 1, skip + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def gaussians(seed: int, n: int, skip_draws: int = 0) -> np.ndarray:
    """n values of gaussian() (two draws each) after skip_draws draws (float64)."""
    z = splitmix(seed, 2 * n, skip_draws)
    u1 = ((z[0::2] >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (z[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def _tanhf(x: np.ndarray) -> np.ndarray:
    """std::tanh(float) is glibc's tanhf (numpy's float32 tanh is another
    polynomial): called through libm for the few hundred h0 values."""
    import ctypes
    f = ctypes.CDLL("libm.so.6").tanhf
    f.restype, f.argtypes = ctypes.c_float, [ctypes.c_float]
    return np.array([f(float(v)) for v in x.ravel()], np.float32).reshape(x.shape)


def synth_model(vocab: int, dim: int, seed: int, bias_strength: float):
    """(E [V,d], freq_bias [V], W_h [d,d], W_e [d,d], h0 [d]) as float32, in the
    draw order of synth_model (src/model_provider.cpp:59-74)."""
    nE, nW = vocab * dim, dim * dim
    E = gaussians(seed, nE).astype(np.float32).reshape(vocab, dim)
    scale = np.float32(1.0) / np.sqrt(np.float32(dim))
    wh = (gaussians(seed, nW, 2 * nE).astype(np.float32) * scale).reshape(dim, dim)
    we = (gaussians(seed, nW, 2 * (nE + nW)).astype(np.float32)
          * (np.float32(0.02) * scale)).reshape(dim, dim)
    h0 = _tanhf(gaussians(seed, dim, 2 * (nE + 2 * nW)).astype(np.float32))
    j = np.arange(vocab, dtype=np.float64)
    mean = np.sum(1.0 / (1.0 + j)) / vocab
    bias = (np.float64(np.float32(bias_strength)) * (1.0 / (1.0 + j) - mean)).astype(np.float32)
    return E, bias, wh, we, h0


def start_state(seed: int, sentence: int, dim: int) -> np.ndarray:
    """h0 of decode-loop sentence s: tanh(N(0,1)) from SplitMix64(mix_seed(seed,
    100 + s))."""
    return _tanhf(gaussians(mix_seed(seed, 100 + sentence), dim).astype(np.float32))

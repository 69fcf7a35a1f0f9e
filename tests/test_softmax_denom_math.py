"""The certification arithmetic of the softmax denominator
(paper_1806_00588_b200/csrc/softmax_denom.cuh), restated in Python doubles and
checked against the reference's SEQUENTIAL double sum (src/beam_decoder.cpp:46-74:
`denom += e` in column order, then `inv = (float)(1.0 / denom)`):

* inv_certified (K5a): a tree sum shaped like the device's (per-thread runs of
  stride 128, then a pairwise reduction) with the worst-case tolerance;
* inv_from_exact (the segmented K5a): an exact sum by TwoSum accumulation and
  the bound sum_k min(e_k, 2^-52), scaled to the sum's binade.

Whenever either certifies a value it must equal float32(1 / sequential sum);
rows built to put 1/denom next to a float rounding boundary must be refused or
still come out right. CPU only: the device code runs the same formulas
(the GPU suites force its sequential fallback separately)."""
import math
import struct

import numpy as np
import pytest


def f32_inv(x):
    return np.float32(1.0 / x)


def seq_sum(e):
    s = 0.0
    for v in e:
        s += v
    return s


def tree_sum(e, nt=128):
    # per-thread runs (thread t adds columns t, t + nt, ...), then pairwise
    parts = [seq_sum(e[t::nt]) for t in range(nt)]
    while len(parts) > 1:
        parts = [parts[i] + parts[i + 1] if i + 1 < len(parts) else parts[i]
                 for i in range(0, len(parts), 2)]
    return parts[0]


def inv_certified(tree, n):
    tol = (n + 64) * 2.0 ** -52 * tree
    lo, hi = f32_inv(tree + tol), f32_inv(tree - tol)
    return (lo == hi), lo


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def inv_from_exact(e):
    hi = c = b = 0.0
    for v in e:
        hi, err = two_sum(hi, v)
        c += err
        b += min(v, 2.0 ** -52)
    x = hi + c
    _, ex = math.frexp(x * (1.0 + 2.0 ** -20))
    scale = math.ldexp(1.0, ex - 1) if ex > 1 else 1.0
    r = b * scale * (1.0 + 2.0 ** -30) + x * 2.0 ** -50
    lo_end, hi_end = x - r, x + r
    f_lo, f_hi = f32_inv(hi_end), f32_inv(lo_end)
    return (lo_end > 0.0 and f_lo == f_hi), f_lo


def rows(rng, kind, n):
    if kind == "gauss3":
        l = rng.standard_normal(n) * 3
    elif kind == "gauss30":
        l = rng.standard_normal(n) * 30
    elif kind == "flat":  # many equal logits: large sums, binades > 1
        l = np.round(rng.standard_normal(n) * 0.5, 1)
    else:  # a few near-max logits
        l = rng.standard_normal(n) * 30
        l[rng.integers(0, n, 5)] = l.max() - rng.random(5)
    l = l.astype(np.float32).astype(np.float64)
    return [math.exp(v - l.max()) for v in l]


@pytest.mark.parametrize("kind", ["gauss3", "gauss30", "flat", "nearmax"])
@pytest.mark.parametrize("n", [1300, 9000])
def test_certified_values_equal_the_sequential_sum(kind, n):
    rng = np.random.default_rng(n + len(kind))
    refused_t = refused_x = 0
    for _ in range(12):
        e = rows(rng, kind, n)
        want = f32_inv(seq_sum(e))
        ok, inv = inv_certified(tree_sum(e), n)
        if ok:
            assert inv == want
        else:
            refused_t += 1
        ok, inv = inv_from_exact(e)
        if ok:
            assert inv == want
        else:
            refused_x += 1
    assert refused_x <= refused_t  # the exact interval is the narrower one


def boundary_row(rng, offset):
    # float32 midpoints below 1 are 1 - (k + 1/2) 2^-24: put 1/denom at one,
    # moved by `offset` (relative)
    k = int(rng.integers(1000, 100000))
    target = 1.0 / ((1.0 - (k + 0.5) * 2.0 ** -24) * (1.0 + offset))
    # terms below 2^-52 (their additions err by at most themselves): the exact
    # interval stays ~1e-15 wide while the worst-case tolerance is ~2e-12
    tail = [math.exp(-40 - 10 * rng.random()) for _ in range(9000)]
    return [1.0, target - 1.0 - sum(tail)] + tail


def test_rows_at_a_float_boundary():
    """1/denom ON a float32 rounding boundary: both certificates must refuse
    (or be right); 2^-45 away from it: the worst-case tolerance (~2e-12
    here) still refuses, the exact interval (~1e-15) certifies -- and is
    right."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        e = boundary_row(rng, 0.0)
        want = f32_inv(seq_sum(e))
        for ok, inv in (inv_from_exact(e), inv_certified(tree_sum(e), len(e))):
            if ok:
                assert inv == want
    certified = 0
    for sign in (1, -1):
        for _ in range(20):
            e = boundary_row(rng, sign * 2.0 ** -45)
            want = f32_inv(seq_sum(e))
            ok_t, inv_t = inv_certified(tree_sum(e), len(e))
            assert not ok_t or inv_t == want
            ok, inv = inv_from_exact(e)
            if ok:
                certified += 1
                assert inv == want
    assert certified == 40


def test_binade_scaling():
    # sums well above 2 (flat rows): the bound scales with the binade
    e = [1.0] * 5000 + [1e-3] * 4000
    ok, inv = inv_from_exact(e)
    assert ok and inv == f32_inv(seq_sum(e))
    assert struct.pack("<f", inv) == struct.pack("<f", f32_inv(seq_sum(e)))

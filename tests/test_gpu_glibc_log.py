"""The device log the beam expansion scores with and the device exp the
softmax uses (lsb_selftest_log / _exp -> glibc_log.cuh) equal the host libm's
log() / exp() bit for bit: for log 2^24 floats spread over (0, 1] plus the
dense region near 1 (the log1p branch) and the edges; for exp the softmax's
domain (differences of floats, <= 0) plus the special ranges.
tests/test_glibc_log.py checks the same restatements on the CPU; this checks
their device compilation."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1806_00588_b200", "csrc")


def test_device_log_equals_libm(ctx, tmp_path):
    import torch
    so = tmp_path / "libglc.so"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-I" + CSRC,
                    os.path.join(ROOT, "tests", "glibc_log_check.c"), "-o", str(so), "-lm"],
                   check=True)
    lib = C.CDLL(str(so))
    lib.libm_log_array.argtypes = [C.c_void_p, C.c_void_p, C.c_long]
    one = np.float32(1.0).view(np.uint32)
    bits = [np.linspace(0, one, 1 << 24, dtype=np.uint64).astype(np.uint32),
            np.arange(one - (1 << 20), one + 1, dtype=np.uint32),   # [1 - 2^-4, 1]: log1p branch
            np.array([0, 1, 2, 0x007FFFFF, 0x00800000, one - 1, one], np.uint32)]
    p = np.concatenate(bits).view(np.float32)
    want = np.empty(p.size, np.float64)
    lib.libm_log_array(p.ctypes.data, want.ctypes.data, p.size)
    pd = torch.from_numpy(p).cuda()
    out = torch.empty(p.size, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx.selftest_log(pd.data_ptr(), out.data_ptr(), p.size)
    got = out.cpu().numpy()
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, [(float(p[i]), got[i].hex(), want[i].hex()) for i in bad[:5]]


def test_device_exp_equals_libm(ctx, tmp_path):
    import torch
    so = tmp_path / "libglc.so"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-I" + CSRC,
                    os.path.join(ROOT, "tests", "glibc_log_check.c"), "-o", str(so), "-lm"],
                   check=True)
    lib = C.CDLL(str(so))
    lib.libm_exp_array.argtypes = [C.c_void_p, C.c_void_p, C.c_long]
    rng = np.random.default_rng(5)
    # softmax inputs: (double) l - (double) mx for float logits
    l = rng.standard_normal(1 << 22).astype(np.float32) * np.float32(30)
    mx = rng.standard_normal(1 << 22).astype(np.float32) * np.float32(30) + np.float32(100)
    x = np.concatenate([l.astype(np.float64) - mx.astype(np.float64),
                        np.linspace(-800.0, 0.0, 1 << 22),
                        -np.exp2(np.linspace(-60.0, 9.6, 1 << 20)),
                        np.linspace(-1100.0, 720.0, 1 << 20),
                        [0.0, -0.0, 1e-300, float.fromhex("0x1p-54"), 709.7, 709.8, -745.1, -745.2,
                         -708.4, 512.0, -512.0, 1023.9, -1023.9, np.inf, -np.inf]])
    want = np.empty_like(x)
    lib.libm_exp_array(x.ctypes.data, want.ctypes.data, x.size)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    torch.cuda.synchronize()
    ctx.selftest_exp(xd.data_ptr(), out.data_ptr(), x.size)
    got = out.cpu().numpy()
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, [(x[i], got[i].hex(), want[i].hex()) for i in bad[:5]]

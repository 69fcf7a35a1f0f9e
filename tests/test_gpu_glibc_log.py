"""The device log the beam expansion scores with (lsb_selftest_log ->
glibc_log.cuh) equals the host libm's log() bit for bit: 2^24 floats spread
over (0, 1] plus the dense region near 1 (the log1p branch) and the edges.
tests/test_glibc_log.py checks the same restatement on every float on the
CPU; this checks the device compilation of it."""
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

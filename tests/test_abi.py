"""CPU: the C-ABI library loads and exports every symbol the public header
declares; calls that need no device behave (no compute without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lshbeam_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lsb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header():
    from paper_1806_00588_b200 import _native as N
    lib = N.load()
    syms = declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares exactly the header's entry points
    assert sorted(N.EXPORTED) == syms


def test_abi_version_and_error_without_device():
    from paper_1806_00588_b200 import _native as N
    lib = N.load()
    assert lib.lsb_abi_version() == 1
    h = ctypes.c_void_p()
    rc = lib.lsb_ctx_create(0, None, ctypes.byref(h))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert rc != 0 and not h.value  # fails loudly: no device, no fallback
        assert lib.lsb_last_error()
    else:
        assert rc == 0
        lib.lsb_ctx_destroy(h)


def test_library_is_sm100a_only():
    """The fatbinary carries sm_100a SASS only (no PTX, no other arch)."""
    import subprocess
    from paper_1806_00588_b200 import _native as N
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    ptx = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-ptx", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert ".ptx" not in ptx


def test_cxx_header_compiles():
    """The C header is valid C (the reference-side FFI binds it from C/C++)."""
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as t:
        src = os.path.join(t, "a.c")
        open(src, "w").write('#include "lshbeam_b200.h"\nint main(void){return lsb_abi_version();}\n')
        r = subprocess.run(["gcc", "-std=c99", "-Wall", "-I" + os.path.join(ROOT, "include"), "-c",
                            src, "-o", os.path.join(t, "a.o")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr

"""Shared fixtures. `-m gpu` tests need a B200 and the built library;
everything else runs on the CPU (oracle pinning, ABI surface, host logic,
gloo multi-process paths)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_addoption(parser):
    parser.addoption("--run-peer-inprocess", action="store_true", default=False,
                     help="run the in-process peer-exchange cases (needs CUDA_MODULE_LOADING=EAGER)")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liblshbeam_b200.so")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_00588_b200 import Context
    c = Context(0)
    yield c
    c.close()

"""B200-native LSH beam-search hot path (arXiv 1806.00588).

The product is the CUDA library liblshbeam_b200.so (C ABI:
include/lshbeam_b200.h; C++ drop-in: include/lshbeam/*.hpp). This package
builds it (``build.build()``) and binds it (``lshbeam``). Importing the
package does not load the library; constructing a ``Context`` does, and
fails loudly if it was not built.
"""
from .lshbeam import (EMPTY_CODE, FAST, PARITY, Batch, Context, Index, Model,  # noqa: F401
                      Recurrent, bits_for, exact_topb)

__all__ = ["Context", "Model", "Index", "Batch", "Recurrent", "PARITY", "FAST", "EMPTY_CODE",
           "bits_for", "exact_topb"]

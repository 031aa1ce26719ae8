"""B200-native kNN-interaction operator (hot path of arXiv 1709.03671's patchord).

The compute lives in libknnx.so (sm_100a CUDA kernels + host C++ behind the C
ABI in include/knnx.h and include/knnx_host.h); this package is its Python
view, used by the tests and bench.py.
"""
from ._lib import KnnxError, LIB_PATH  # noqa: F401  (raises ImportError if unbuilt)

__all__ = ["KnnxError", "LIB_PATH"]

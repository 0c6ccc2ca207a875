"""B200-native brute-force k-NN / k-NNG (arXiv 1309.5478 hot path).

The compute lives in ``csrc/`` (CUDA for sm_100a + a C++ host runtime) built into
``libknn.so`` behind the C ABI declared in ``include/knn.h``.  ``knn`` is the thin
ctypes binding; importing this package does not load the library, calling it does,
and a missing library is a hard error (there is no CPU fallback).
"""
from . import datagen  # noqa: F401  (seeded input generators; no method arithmetic)

__all__ = ["datagen", "knn"]


def __getattr__(name):
    if name == "knn":
        import importlib
        return importlib.import_module(__name__ + ".knn")
    raise AttributeError(name)

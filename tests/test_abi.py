"""CPU-side checks of the C ABI: libknn.so builds, loads, and exports every symbol that
include/knn.h declares (no compute calls — there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "knn.h")
LIB = os.path.join(ROOT, "paper_1309_5478_b200", "libknn.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(knn_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", ROOT, "-j8", "paper_1309_5478_b200/libknn.so"])
    return ctypes.CDLL(LIB)


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("knn_graph", "knn_search", "knn_rownorms", "knn_distances", "knn_select",
                 "knn_merge", "knn_ctx_create", "knn_ctx_destroy", "knn_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIB]).decode()
    exported = set(re.findall(r" T (knn_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert missing == []


def test_binding_covers_the_header():
    from paper_1309_5478_b200 import knn
    assert sorted(knn.SYMBOLS) == declared_symbols()


def test_abi_version_and_no_device(lib):
    lib.knn_abi_version.restype = ctypes.c_int
    assert lib.knn_abi_version() == 2
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    lib.knn_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    h = ctypes.c_void_p()
    assert lib.knn_ctx_create(0, ctypes.byref(h)) == 5  # KNN_ERR_CUDA, no crash
    assert not h.value


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_1309_5478_b200 import knn
    monkeypatch.setattr(knn, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(knn, "_lib", None)
    with pytest.raises(knn.KnnLibraryMissing):
        knn.load_library()


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1309_5478_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "knn_oracle" not in src, f


def test_header_is_plain_c_and_example_links(lib, tmp_path):
    """include/knn.h compiles as C11 and examples/knn_demo.c links against libknn.so (the
    boundary needs no C++, Python or torch types)."""
    exe = tmp_path / "knn_demo"
    cuda_inc = "/usr/local/cuda/include"
    cuda_lib = "/usr/local/cuda/lib64"
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-I", cuda_inc, os.path.join(ROOT, "examples", "knn_demo.c"),
                           "-L", os.path.dirname(LIB), "-lknn", "-L", cuda_lib, "-lcudart", "-o", str(exe)])
    assert exe.exists()

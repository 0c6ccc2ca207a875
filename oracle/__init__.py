"""CPU oracle for arXiv 1309.5478's brute-force k-NN / k-NNG — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1309_5478_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/knn_oracle.cpp`` (plain C++17, fp64, full sort per
row; see its header for the paper passages each function follows).  This module only
builds it (g++, on demand) and marshals numpy arrays through ctypes.

Parity status (DESIGN.md §Oracle pins): every function here is pinned by
``tests/test_oracle.py`` against hand-worked examples, closed forms, invariants and
independent brute force — none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "knn_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

L2SQ = 0
L2 = 1
COSINE = 2   # key 1 - x.y/(|x||y|) (reading R14); zero norm -> 3.0
PEARSON = 3  # the cosine key of the mean-centred vectors


def build(force: bool = False) -> str:
    """Compile knn_oracle.cpp -> oracle/liboracle.so (g++ -O2 -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-shared", "-fPIC",
             "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            p = ctypes.c_void_p
            i32, i64 = ctypes.c_int32, ctypes.c_int64
            lib.oracle_sqnorms.argtypes = [p, i64, i32, p]
            lib.oracle_dist_rows.argtypes = [p, p, i64, p, i64, i32, i32, i32, p]
            lib.oracle_knn.argtypes = [p, i64, p, i64, i32, i32, i32, i32, p, i64, i32,
                                       p, p, p, p]
            lib.oracle_select_f32.argtypes = [p, i64, i64, i64, i32, i32, p, p]
            lib.oracle_merge.argtypes = [p, p, i32, i64, i32, p, p, p]
            for f in (lib.oracle_sqnorms, lib.oracle_dist_rows, lib.oracle_knn,
                      lib.oracle_select_f32, lib.oracle_merge):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def sqnorms(X) -> np.ndarray:
    """fp64 ||x_j||^2 per row of X (N×d fp32)."""
    X = _f32(X)
    N, d = X.shape
    out = np.empty(N, np.float64)
    if _load().oracle_sqnorms(_ptr(X), N, d, _ptr(out)) != 0:
        raise ValueError("oracle_sqnorms: bad arguments")
    return out


def dist_rows(Q, X, rows=None, metric=L2SQ, threads=None) -> np.ndarray:
    """fp64 direct-form distance rows D64[r, j] = d(Q[rows[r]], X[j])."""
    Q, X = _f32(Q), _f32(X)
    rows = np.arange(Q.shape[0], dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    N, d = X.shape
    out = np.empty((len(rows), N), np.float64)
    rc = _load().oracle_dist_rows(_ptr(Q), _ptr(rows), len(rows), _ptr(X), N, d, metric,
                                  threads or default_threads(), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_dist_rows: bad arguments")
    return out


def knn(Q, X, k, rows=None, metric=L2SQ, graph=False, threads=None, want_r32=True):
    """Reference k-NN lists for the query rows ``rows`` (default: all).

    Returns dict with idx64 (R×k int32), dist64 (R×k fp64) and, if want_r32,
    idx32 / dist32 (the exact selection on the fp32-rounded row)."""
    Q, X = _f32(Q), _f32(X)
    M, d = Q.shape
    N = X.shape[0]
    rows = np.arange(M, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    R = len(rows)
    idx64 = np.empty((R, k), np.int32)
    dist64 = np.empty((R, k), np.float64)
    idx32 = np.empty((R, k), np.int32) if want_r32 else None
    dist32 = np.empty((R, k), np.float32) if want_r32 else None
    rc = _load().oracle_knn(_ptr(Q), M, _ptr(X), N, d, k, metric, 1 if graph else 0,
                            _ptr(rows), R, threads or default_threads(),
                            _ptr(idx64), _ptr(dist64), _ptr(idx32), _ptr(dist32))
    if rc != 0:
        raise ValueError("oracle_knn: bad arguments")
    out = {"rows": rows, "idx64": idx64, "dist64": dist64}
    if want_r32:
        out["idx32"], out["dist32"] = idx32, dist32
    return out


def select_f32(D, k, threads=None):
    """Exact per-row select on an fp32 matrix: sort by (value, idx), first k."""
    D = _f32(D)
    M, N = D.shape
    idx = np.empty((M, k), np.int32)
    dist = np.empty((M, k), np.float32)
    if _load().oracle_select_f32(_ptr(D), M, N, N, k, threads or default_threads(),
                                 _ptr(idx), _ptr(dist)) != 0:
        raise ValueError("oracle_select_f32: bad arguments")
    return idx, dist


def merge(part_dist, part_idx, offsets):
    """Merge G lists ([G][M][k]) of (value, local idx); list g's idx shifted by offsets[g]."""
    part_dist = _f32(part_dist)
    part_idx = np.ascontiguousarray(part_idx, np.int32)
    G, M, k = part_dist.shape
    offsets = np.ascontiguousarray(offsets, np.int64)
    idx = np.empty((M, k), np.int32)
    dist = np.empty((M, k), np.float32)
    if _load().oracle_merge(_ptr(part_dist), _ptr(part_idx), G, M, k, _ptr(offsets),
                            _ptr(idx), _ptr(dist)) != 0:
        raise ValueError("oracle_merge: bad arguments")
    return idx, dist

"""Thin ctypes binding of libknn.so (include/knn.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module converts
torch tensors / numpy arrays to pointers, passes the current CUDA stream, and turns
status codes into exceptions.  A missing library is a hard error: there is no CPU path.
Function names follow the C ABI (``knn_graph`` -> ``graph`` ...).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KNN_LIB_PATH") or os.path.join(_HERE, "libknn.so")  # override: A/B builds

L2SQ, L2, COSINE, PEARSON = 0, 1, 2, 3
NO_SELF = -(2 ** 63)  # KNN_NO_SELF
MAX_K = 1024

STATUS = {0: "KNN_OK", 1: "KNN_ERR_ARG", 2: "KNN_ERR_UNSUPPORTED", 3: "KNN_ERR_NONFINITE",
          4: "KNN_ERR_OOM", 5: "KNN_ERR_CUDA", 6: "KNN_ERR_NCCL", 7: "KNN_ERR_INTERNAL"}

# every symbol include/knn.h declares
SYMBOLS = ["knn_abi_version", "knn_ctx_create", "knn_ctx_destroy", "knn_last_error",
           "knn_graph", "knn_search", "knn_search_block", "knn_search_block_host",
           "knn_rownorms", "knn_distances", "knn_select", "knn_merge", "knn_launch_count",
           "knn_gemm_path", "knn_set_plan", "knn_last_plan", "knn_last_candidates", "knn_profile_enable",
           "knn_profile_read", "knn_last_select_kernel", "knn_select_paper",
           "knn_search_streamed", "knn_merge_lists", "knn_ipc_export", "knn_ipc_open",
           "knn_ipc_close_all", "knn_graph_units", "knn_graph_list_cap", "knn_pivot_sample_size", "knn_graph_pivots",
           "knn_graph_partition", "knn_graph_gather_select", "knn_diag_mainloop",
           "knn_comm_unique_id", "knn_comm_init", "knn_comm_init_ops", "knn_comm_destroy", "knn_comm_info",
           "knn_shard_range", "knn_graph_sharded", "knn_search_sharded", "knn_last_shard_mode"]
SHARD_QUERY, SHARD_CORPUS, SHARD_SYM = 0, 1, 2
SHARD_MODES = {"query": SHARD_QUERY, "corpus": SHARD_CORPUS, "sym": SHARD_SYM}
PLAN_AUTO, PLAN_FUSED, PLAN_MATERIALISED, PLAN_PIVOT_EXACT = 0, 1, 2, 3
KERNELS = {"prep": 0, "gemm": 1, "select": 2, "merge": 3, "fused": 4, "xmerge": 5}


# knn_comm_ops: the host-callback transport (include/knn.h "multi-GPU")
_AG = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)
_BC = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int)
_A2A = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)
_ARM = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


class CommOps(ctypes.Structure):
    _fields_ = [("allgather", _AG), ("broadcast", _BC), ("alltoall", _A2A),
                ("allreduce_max_i32", _ARM), ("user", ctypes.c_void_p)]


class KnnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class KnnLibraryMissing(ImportError):
    pass


_lib = None
_lock = threading.Lock()
_ctx = {}


def load_library():
    """Load libknn.so (built by `make` / __graft_entry__.build()); raise if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise KnnLibraryMissing(
                f"{LIB_PATH} not found: build it with `make` or __graft_entry__.build(); "
                "there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        p, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        st = ctypes.c_int
        sig = {
            "knn_abi_version": (ctypes.c_int, []),
            "knn_ctx_create": (st, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
            "knn_ctx_destroy": (st, [p]),
            "knn_last_error": (ctypes.c_char_p, [p]),
            "knn_launch_count": (i64, [p]),
            "knn_graph": (st, [p, p, i64, i32, i32, i32, p, p, p]),
            "knn_search": (st, [p, p, i64, p, i64, i32, i32, p, p, p]),
            "knn_search_block": (st, [p, p, i64, p, i64, i32, i32, i32, i64, i64, p, p, p]),
            "knn_search_block_host": (st, [p, p, i64, p, i64, i32, i32, i32, i64, i64, p, p, p]),
            "knn_rownorms": (st, [p, p, i64, i32, p, p, p]),
            "knn_distances": (st, [p, p, i64, p, i64, i32, i32, i64, p, i64, p]),
            "knn_select": (st, [p, p, i64, i64, i64, i32, p, p, p]),
            "knn_select_paper": (st, [p, p, i64, i64, i64, i32, p, p, p]),
            "knn_search_streamed": (st, [p, p, i64, p, i64, i32, i32, i32, i32, i64, i64, p, p]),
            "knn_merge_lists": (st, [p, p, p, i32, i64, i64, i32, p, p, p, p]),
            "knn_ipc_export": (st, [p, p, p, ctypes.POINTER(ctypes.c_int64)]),
            "knn_ipc_open": (st, [p, p, i64, ctypes.POINTER(ctypes.c_void_p)]),
            "knn_ipc_close_all": (st, [p]),
            "knn_graph_units": (i64, [i64]),
            "knn_diag_mainloop": (st, [p, p, i64, i32, i32, i32, ctypes.POINTER(ctypes.c_double)]),
            "knn_graph_list_cap": (i32, [i32]),
            "knn_pivot_sample_size": (i64, [p, i64, i32]),
            "knn_graph_pivots": (st, [p, p, i64, i32, i32, i32, i64, i64, p, p]),
            "knn_graph_partition": (st, [p, p, i64, i32, i32, i32, p, i64, i64, p, p, i32, p]),
            "knn_graph_gather_select": (st, [p, i32, p, p, i32, i64, i32, i64, i64, p, p, p]),
            "knn_last_select_kernel": (st, [ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
            "knn_merge": (st, [p, p, p, i32, i64, i32, p, p, p, p]),
            "knn_gemm_path": (ctypes.c_int, [p]),
            "knn_set_plan": (st, [p, i32]),
            "knn_last_plan": (ctypes.c_int, [p]),
            "knn_last_candidates": (ctypes.c_int64, [p]),
            "knn_profile_enable": (st, [p, i32]),
            "knn_comm_unique_id": (st, [p]),
            "knn_comm_init": (st, [p, i32, i32, p]),
            "knn_comm_init_ops": (st, [p, i32, i32, ctypes.POINTER(CommOps)]),
            "knn_comm_destroy": (st, [p]),
            "knn_comm_info": (st, [p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32)]),
            "knn_shard_range": (None, [i64, i32, i32, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_int64)]),
            "knn_graph_sharded": (st, [p, i32, p, i64, i32, i32, i32, p, p, p]),
            "knn_search_sharded": (st, [p, i32, p, i64, p, i64, i32, i32, p, p, p]),
            "knn_last_shard_mode": (ctypes.c_int, [p]),
            "knn_profile_read": (st, [p, i32, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_int64)]),
        }
        for name, (res, args) in sig.items():
            if "KNN_LIB_PATH" in os.environ and not hasattr(lib, name):
                continue  # an older build under A/B test: only the symbols it has
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _lib = lib
        return lib


def context(device=None):
    """The per-process knn_ctx of a CUDA device (created on first use)."""
    import torch
    lib = load_library()
    dev = torch.cuda.current_device() if device is None else int(device)
    with _lock:
        if dev not in _ctx:
            h = ctypes.c_void_p()
            rc = lib.knn_ctx_create(dev, ctypes.byref(h))
            if rc != 0:
                raise KnnError(rc, f"knn_ctx_create({dev}) failed")
            _ctx[dev] = h
        return _ctx[dev]


def _check(rc, ctx):
    if rc != 0:
        raise KnnError(rc, load_library().knn_last_error(ctx).decode())


def _dev_ptr(t, dtype, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _outputs(rows, k, device):
    import torch
    return (torch.empty((rows, k), dtype=torch.int32, device=device),
            torch.empty((rows, k), dtype=torch.float32, device=device))


def graph(X, k, metric=L2SQ, stream=None):
    """k-NNG of X (N×d fp32 CUDA tensor): (idx N×k int32, dist N×k fp32), self excluded."""
    import torch
    N, d = X.shape
    ctx = context(X.device.index)
    idx, dist = _outputs(N, k, X.device)
    rc = load_library().knn_graph(ctx, _dev_ptr(X, torch.float32, "X"), N, d, k, metric,
                                  ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
                                  _stream(stream))
    _check(rc, ctx)
    return idx, dist


def search(Q, X, k, stream=None):
    """For each query row of Q, its k nearest rows of X (squared Euclidean)."""
    import torch
    M, d = Q.shape
    N = X.shape[0]
    ctx = context(Q.device.index)
    idx, dist = _outputs(M, k, Q.device)
    rc = load_library().knn_search(ctx, _dev_ptr(Q, torch.float32, "Q"), M,
                                   _dev_ptr(X, torch.float32, "X"), N, d, k,
                                   ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
                                   _stream(stream))
    _check(rc, ctx)
    return idx, dist


def search_block(Q, X, k, metric=L2SQ, self_shift=NO_SELF, idx_offset=0, out=None, stream=None):
    """knn_search_block: self pair j == i + self_shift excluded; idx_offset added."""
    import torch
    M, d = Q.shape
    N = X.shape[0]
    ctx = context(Q.device.index)
    idx, dist = out if out is not None else _outputs(M, k, Q.device)
    rc = load_library().knn_search_block(
        ctx, _dev_ptr(Q, torch.float32, "Q"), M, _dev_ptr(X, torch.float32, "X"), N, d, k, metric,
        self_shift, idx_offset, _dev_ptr(idx, torch.int32, "out_idx"),
        _dev_ptr(dist, torch.float32, "out_dist"), _stream(stream))
    _check(rc, ctx)
    return idx, dist


def search_block_host(Q, X, k, metric=L2SQ, self_shift=NO_SELF, idx_offset=0, out=None,
                      device=None, stream=None):
    """knn_search_block_host: numpy (ideally pinned) host inputs and outputs; the
    host<->device copies happen inside the call."""
    Q = np.ascontiguousarray(Q, np.float32)
    X = Q if X is Q else np.ascontiguousarray(X, np.float32)
    M, d = Q.shape
    N = X.shape[0]
    ctx = context(device)
    if out is None:
        out = (np.empty((M, k), np.int32), np.empty((M, k), np.float32))
    idx, dist = out
    rc = load_library().knn_search_block_host(
        ctx, Q.ctypes.data_as(ctypes.c_void_p), M, X.ctypes.data_as(ctypes.c_void_p), N, d, k,
        metric, self_shift, idx_offset, idx.ctypes.data_as(ctypes.c_void_p),
        dist.ctypes.data_as(ctypes.c_void_p), _stream(stream))
    _check(rc, ctx)
    return idx, dist


def rownorms(X, stream=None):
    """(||x||^2 fp32 per row, non-finite flag int32[1])."""
    import torch
    N, d = X.shape
    ctx = context(X.device.index)
    out = torch.empty(N, dtype=torch.float32, device=X.device)
    flag = torch.zeros(1, dtype=torch.int32, device=X.device)
    rc = load_library().knn_rownorms(ctx, _dev_ptr(X, torch.float32, "X"), N, d,
                                     ctypes.c_void_p(out.data_ptr()),
                                     ctypes.c_void_p(flag.data_ptr()), _stream(stream))
    _check(rc, ctx)
    return out, flag


def distances(Q, X, metric=L2SQ, self_shift=NO_SELF, ldD=None, stream=None):
    """The M×N distance matrix (M×ldD storage; returns the M×N view)."""
    import torch
    M, d = Q.shape
    N = X.shape[0]
    ldD = N if ldD is None else ldD
    ctx = context(Q.device.index)
    D = torch.empty((M, ldD), dtype=torch.float32, device=Q.device)
    rc = load_library().knn_distances(ctx, _dev_ptr(Q, torch.float32, "Q"), M,
                                      _dev_ptr(X, torch.float32, "X"), N, d, metric, self_shift,
                                      ctypes.c_void_p(D.data_ptr()), ldD, _stream(stream))
    _check(rc, ctx)
    return D[:, :N]


def select(D, k, N=None, stream=None):
    """Per-row k smallest of D (M×ldD fp32 CUDA tensor; first N columns), sorted."""
    import torch
    M, ld = D.shape
    N = ld if N is None else N
    if not D.is_contiguous():
        raise ValueError("D must be contiguous (use the N argument for a column prefix)")
    ctx = context(D.device.index)
    idx, dist = _outputs(M, k, D.device)
    rc = load_library().knn_select(ctx, _dev_ptr(D, torch.float32, "D"), M, N, ld, k,
                                   ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
                                   _stream(stream))
    _check(rc, ctx)
    return idx, dist


def search_streamed(Q, X, k, metric=L2SQ, graph=False, chunk_points=0, query_block=0,
                    device=0, out=None):
    """Out-of-core k-NN with HOST inputs (numpy fp32, C-contiguous; pass the same array
    as Q and X with graph=True for the k-NNG): corpus chunks are streamed to the device
    with copy/compute overlap and partial top-k lists merged (knn_search_streamed).
    Returns host (idx int32 M×k, dist fp32 M×k)."""
    Q = np.ascontiguousarray(Q, np.float32) if not graph else X
    X = np.ascontiguousarray(X, np.float32)
    if graph:
        Q = X
    M, d = Q.shape
    N = X.shape[0]
    if out is None:
        out = (np.empty((M, k), np.int32), np.empty((M, k), np.float32))
    ctx = context(device)
    rc = load_library().knn_search_streamed(
        ctx, Q.ctypes.data_as(ctypes.c_void_p), M, X.ctypes.data_as(ctypes.c_void_p), N, d, k,
        metric, 1 if graph else 0, chunk_points, query_block,
        out[0].ctypes.data_as(ctypes.c_void_p), out[1].ctypes.data_as(ctypes.c_void_p))
    _check(rc, ctx)
    return out


def merge_lists(dist_ptrs, idx_ptrs, row0, M, k, offsets=None, device=None, stream=None):
    """knn_merge_lists: merge G lists given as device pointers (ints; local or peer-mapped
    with ipc_open); list g of row row0 + r at dist_ptrs[g] + (row0 + r) * k.  Returns
    (idx M×k int32, dist M×k fp32) on `device`."""
    import torch
    G = len(dist_ptrs)
    offs = np.zeros(G, np.int64) if offsets is None else np.ascontiguousarray(offsets, np.int64)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = context(dev.index)
    idx, dist = _outputs(M, k, dev)
    dl = (ctypes.c_void_p * G)(*dist_ptrs)
    il = (ctypes.c_void_p * G)(*idx_ptrs)
    rc = load_library().knn_merge_lists(ctx, dl, il, G, row0, M, k, offs.ctypes.data_as(ctypes.c_void_p),
                                        ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
                                        _stream(stream))
    _check(rc, ctx)
    return idx, dist


def graph_units(N):
    """Units (256x256 pair blocks) of the upper triangle of the k-NNG of N points."""
    return int(load_library().knn_graph_units(N))


def pivot_sample_size(N, k, device=None):
    """knn_pivot_sample_size: the pivot plans' column-sample size for N points and k."""
    return int(load_library().knn_pivot_sample_size(context(device), N, k))


def graph_list_cap(k):
    return int(load_library().knn_graph_list_cap(k))


def graph_pivots(X, k, row0, rows, thr, metric=L2SQ, stream=None):
    """knn_graph_pivots: pivots of rows [row0, row0+rows) into thr (roundup(N,256) floats)."""
    import torch
    N, d = X.shape
    ctx = context(X.device.index)
    rc = load_library().knn_graph_pivots(ctx, _dev_ptr(X, torch.float32, "X"), N, d, k, metric, row0, rows,
                                         _dev_ptr(thr, torch.float32, "thr"), _stream(stream))
    _check(rc, ctx)


def graph_partition(X, k, thr, unit_lo, unit_hi, cnt, cent, metric=L2SQ, stream=None):
    """knn_graph_partition: candidates of the triangle units [unit_lo, unit_hi) into the lists
    (cnt int32[N], cent int64[N, cap]: entries key << 32 | column)."""
    import torch
    N, d = X.shape
    cap = cent.shape[1]
    ctx = context(X.device.index)
    rc = load_library().knn_graph_partition(
        ctx, _dev_ptr(X, torch.float32, "X"), N, d, k, metric, _dev_ptr(thr, torch.float32, "thr"),
        unit_lo, unit_hi, _dev_ptr(cnt, torch.int32, "cnt"), _dev_ptr(cent, torch.int64, "cent"), cap,
        _stream(stream))
    _check(rc, ctx)


def graph_gather_select(cnt_ptrs, ent_ptrs, cap, N, k, row0, rows, device=None, stream=None):
    """knn_graph_gather_select over G list sources (device pointers, local or peer-mapped).
    Returns (idx rows×k, dist rows×k); raises KnnError(KNN_ERR_INTERNAL) on a failed
    certificate / overflow (the caller falls back)."""
    import torch
    G = len(cnt_ptrs)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    ctx = context(dev.index)
    idx, dist = _outputs(rows, k, dev)
    P = ctypes.c_void_p * G
    rc = load_library().knn_graph_gather_select(ctx, G, P(*cnt_ptrs), P(*ent_ptrs), cap, N, k, row0, rows,
                                                ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
                                                _stream(stream))
    _check(rc, ctx)
    return idx, dist


def diag_mainloop(X, sym=True, reps=10):
    """DIAGNOSTIC: mean ms of the 3-product GEMM of X with a TMEM-draining null epilogue."""
    import torch
    N, d = X.shape
    ctx = context(X.device.index)
    ms = ctypes.c_double()
    _check(load_library().knn_diag_mainloop(ctx, _dev_ptr(X, torch.float32, "X"), N, d, 1 if sym else 0, reps,
                                            ctypes.byref(ms)), ctx)
    return ms.value


def ipc_export(t):
    """(64-byte CUDA IPC handle, byte offset) of the allocation holding tensor t."""
    ctx = context(t.device.index)
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_int64()
    _check(load_library().knn_ipc_export(ctx, ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)), ctx)
    return bytes(h), off.value


def ipc_open(handle, offset, device=None):
    """Map a peer process's allocation (from ipc_export); returns the device pointer (int)."""
    ctx = context(device)
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    ptr = ctypes.c_void_p()
    _check(load_library().knn_ipc_open(ctx, h, offset, ctypes.byref(ptr)), ctx)
    return ptr.value


def ipc_close_all(device=None):
    ctx = context(device)
    _check(load_library().knn_ipc_close_all(ctx), ctx)


def select_paper(D, k, N=None, stream=None):
    """ABLATION: the paper's quick multi-select as written (knn_select_paper); same
    contract and results as select()."""
    import torch
    M, ld = D.shape
    N = ld if N is None else N
    if not D.is_contiguous():
        raise ValueError("D must be contiguous (use the N argument for a column prefix)")
    ctx = context(D.device.index)
    idx, dist = _outputs(M, k, D.device)
    rc = load_library().knn_select_paper(ctx, _dev_ptr(D, torch.float32, "D"), M, N, ld, k,
                                         ctypes.c_void_p(idx.data_ptr()),
                                         ctypes.c_void_p(dist.data_ptr()), _stream(stream))
    _check(rc, ctx)
    return idx, dist


SELECT_KERNELS = {0: "warp per row", 1: "CTA per row (ring)", 2: "CTA per row (unaligned)",
                  3: "cluster per row", 4: "two-pass warp per row"}


def last_select_kernel():
    """(kind name, splits) of the last select launch in this process."""
    kind, splits = ctypes.c_int32(), ctypes.c_int32()
    rc = load_library().knn_last_select_kernel(ctypes.byref(kind), ctypes.byref(splits))
    if rc != 0:
        raise KnnError(rc, "knn_last_select_kernel")
    return SELECT_KERNELS.get(kind.value, str(kind.value)), splits.value


def merge(part_dist, part_idx, offsets, stream=None):
    """Merge G partial lists ([G][M][k] CUDA tensors), list g's indices + offsets[g]."""
    import torch
    G, M, k = part_dist.shape
    offs = np.ascontiguousarray(offsets, np.int64)
    if offs.shape != (G,):
        raise ValueError("offsets must have G entries")
    ctx = context(part_dist.device.index)
    idx, dist = _outputs(M, k, part_dist.device)
    rc = load_library().knn_merge(ctx, _dev_ptr(part_dist, torch.float32, "part_dist"),
                                  _dev_ptr(part_idx, torch.int32, "part_idx"), G, M, k,
                                  offs.ctypes.data_as(ctypes.c_void_p),
                                  ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
                                  _stream(stream))
    _check(rc, ctx)
    return idx, dist


def launch_count(device=None):
    return int(load_library().knn_launch_count(context(device)))


def gemm_path(device=None):
    """0 = tcgen05 split-fp16 tensor-core GEMM, 1 = SIMT FFMA."""
    return int(load_library().knn_gemm_path(context(device)))


def set_plan(plan, device=None):
    """PLAN_AUTO (default) or PLAN_MATERIALISED; both give bit-identical results
    (PLAN_FUSED is reserved: the per-row-list fused kernel was retired)."""
    ctx = context(device)
    _check(load_library().knn_set_plan(ctx, int(plan)), ctx)


def last_plan(device=None):
    """0 blocked distances+select, 2 symmetric k-NNG distances+select,
    3 pivot plan (symmetric), 4 pivot plan (general block), 5 / 6 the pivot plan with the
    single-product partition and the fp32 re-evaluation (symmetric / general block)."""
    return int(load_library().knn_last_plan(context(device)))


def last_candidates(device=None):
    """Candidates the last pivot-plan call kept (sum over rows)."""
    return int(load_library().knn_last_candidates(context(device)))


def profile_enable(on=True, device=None):
    ctx = context(device)
    _check(load_library().knn_profile_enable(ctx, 1 if on else 0), ctx)


def profile_read(kernel, device=None):
    """(summed device ms, launches) of one kernel class since profile_enable."""
    ctx = context(device)
    ms, n = ctypes.c_double(), ctypes.c_int64()
    _check(load_library().knn_profile_read(ctx, KERNELS[kernel], ctypes.byref(ms),
                                           ctypes.byref(n)), ctx)
    return ms.value, n.value


# ------------------------------------------------------------------ multi-GPU --------
def shard_range(n, parts, r):
    """knn_shard_range: [lo, hi) of block r of ceil(n/parts)-sized blocks (host only)."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    load_library().knn_shard_range(int(n), int(parts), int(r), ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def comm_unique_id():
    """128-byte NCCL unique id (make it on one rank, ship it to the others)."""
    buf = (ctypes.c_uint8 * 128)()
    rc = load_library().knn_comm_unique_id(buf)
    if rc != 0:
        raise KnnError(rc, "knn_comm_unique_id (is libnccl.so.2 loadable?)")
    return bytes(buf)


def comm_init(rank, nranks, uid, device=None):
    """knn_comm_init: join the NCCL communicator (collective, blocking)."""
    ctx = context(device)
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(load_library().knn_comm_init(ctx, int(rank), int(nranks), buf), ctx)


_ops_keep = {}


def comm_init_ops(rank, nranks, transport, device=None):
    """knn_comm_init_ops: a host transport object with methods
    allgather(send u8[n], recv u8[G*n]), broadcast(buf u8[n], root), alltoall(send u8[G*n],
    recv u8[G*n]) and allreduce_max(buf int32[c]) operating on numpy views of the library's
    pinned staging buffers (marshalling only: the collective is the transport's)."""
    def u8(ptr, n):
        return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_uint8)), shape=(int(n),))

    def wrap(fn):
        def call(*a):
            try:
                fn(*a)
                return 0
            except Exception as e:  # reported as KNN_ERR_NCCL by the library
                import sys
                print(f"knn comm transport error: {e!r}", file=sys.stderr)
                return 1
        return call

    G = int(nranks)
    ops = CommOps(
        _AG(wrap(lambda u, s_, r_, n: transport.allgather(u8(s_, n), u8(r_, G * n)))),
        _BC(wrap(lambda u, b, n, root: transport.broadcast(u8(b, n), root))),
        _A2A(wrap(lambda u, s_, r_, n: transport.alltoall(u8(s_, G * n), u8(r_, G * n)))),
        _ARM(wrap(lambda u, b, c: transport.allreduce_max(np.ctypeslib.as_array(
            ctypes.cast(b, ctypes.POINTER(ctypes.c_int32)), shape=(int(c),))))),
        None)
    ctx = context(device)
    _check(load_library().knn_comm_init_ops(ctx, int(rank), G, ctypes.byref(ops)), ctx)
    _ops_keep[ctx.value] = ops  # the library keeps the function pointers


def comm_destroy(device=None):
    ctx = context(device)
    _check(load_library().knn_comm_destroy(ctx), ctx)
    _ops_keep.pop(ctx.value, None)


def comm_info(device=None):
    """(backend 0 none / 1 NCCL / 2 host callbacks, rank, nranks)."""
    ctx = context(device)
    b, r, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(load_library().knn_comm_info(ctx, ctypes.byref(b), ctypes.byref(r), ctypes.byref(n)), ctx)
    return b.value, r.value, n.value


def graph_sharded(X, k, mode="sym", metric=L2SQ, out=None, stream=None):
    """knn_graph_sharded (collective): X (N×d CUDA tensor) valid on rank 0, broadcast into X
    on the other ranks; returns the full (idx N×k, dist N×k) on every rank."""
    import torch
    N, d = X.shape
    ctx = context(X.device.index)
    idx, dist = out if out is not None else _outputs(N, k, X.device)
    rc = load_library().knn_graph_sharded(ctx, SHARD_MODES.get(mode, mode), _dev_ptr(X, torch.float32, "X"), N, d,
                                          k, metric, _dev_ptr(idx, torch.int32, "out_idx"),
                                          _dev_ptr(dist, torch.float32, "out_dist"), _stream(stream))
    _check(rc, ctx)
    return idx, dist


def search_sharded(Q, X, k, mode="query", out=None, stream=None):
    """knn_search_sharded (collective): Q (M×d) and X (N×d) valid on rank 0."""
    import torch
    M, d = Q.shape
    N = X.shape[0]
    ctx = context(X.device.index)
    idx, dist = out if out is not None else _outputs(M, k, X.device)
    rc = load_library().knn_search_sharded(ctx, SHARD_MODES.get(mode, mode), _dev_ptr(Q, torch.float32, "Q"), M,
                                           _dev_ptr(X, torch.float32, "X"), N, d, k,
                                           _dev_ptr(idx, torch.int32, "out_idx"),
                                           _dev_ptr(dist, torch.float32, "out_dist"), _stream(stream))
    _check(rc, ctx)
    return idx, dist


def last_shard_mode(device=None):
    """Mode the last sharded call ran (after fallbacks): 0 query, 1 corpus, 2 sym, -1 none."""
    return int(load_library().knn_last_shard_mode(context(device)))

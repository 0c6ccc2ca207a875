"""World-size-2 CPU tests (gloo) of the multi-GPU host logic.

The shardings run inside libknn (csrc/shard.cu), which needs a GPU; on CPU these tests
check the pieces that carry their host logic:

* ``TorchHostTransport`` — the product's host transport (knn_comm_ops) — performs the four
  collectives the library issues (allgather, broadcast, all-to-all, max all-reduce) over
  gloo with world size 2, on uint8 / int32 numpy buffers like the library's staging;
* ``knn_shard_range`` — the library's split of rows, columns and triangle units;
* stand-in runs of the three shardings with the SAME decomposition as shard.cu (query
  rows; corpus columns + all-to-all of row blocks + k-way merge; the upper triangle's
  256x256 units split over the ranks with pivots all-gathered, candidate lists of any row
  and the per-row select over every rank's lists), where every collective goes through
  TorchHostTransport and the per-rank compute is an oracle stand-in: the results must equal
  the unsharded oracle graph bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1309_5478_b200 import datagen, knn, sharded

NO_SELF = -(2 ** 63)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_compute(Q, X, k, self_shift, idx_offset):
    """Stand-in for knn_search_block: fp32-rounded oracle distances, exact select."""
    D = oracle.dist_rows(Q, X).astype(np.float32)
    if self_shift != NO_SELF:
        for i in range(D.shape[0]):
            j = i + self_shift
            if 0 <= j < D.shape[1]:
                D[i, j] = np.inf
    idx, dst = oracle.select_f32(D, k)
    return idx + np.int32(idx_offset), dst


def _u8(a):
    return np.ascontiguousarray(a).view(np.uint8).reshape(-1)


def _bcast(tr, a):
    b = _u8(a).copy()
    tr.broadcast(b, 0)
    return b.view(a.dtype).reshape(a.shape)


def _gather_rows(tr, own, per):
    """all-gather of equal [per][...] row blocks (the library's gather_rows)."""
    blk = np.zeros((per,) + own.shape[1:], own.dtype)
    blk[:own.shape[0]] = own
    recv = np.empty(tr.G * blk.nbytes, np.uint8)
    tr.allgather(_u8(blk), recv)
    return recv.view(own.dtype).reshape((tr.G * per,) + own.shape[1:])


def standin_query(tr, Q, X, k, graph):
    G, r = tr.G, tr.rank
    M = Q.shape[0]
    per = -(-M // G)
    lo, hi = knn.shard_range(M, G, r)
    i, d = oracle_compute(Q[lo:hi], X, k, lo if graph else NO_SELF, 0)
    return _gather_rows(tr, i, per)[:M], _gather_rows(tr, d, per)[:M]


def standin_corpus(tr, Q, X, k, graph):
    G, r = tr.G, tr.rank
    M, N = Q.shape[0], X.shape[0]
    per = -(-M // G)
    c0, c1 = knn.shard_range(N, G, r)
    i, d = oracle_compute(Q, X[c0:c1], k, -c0 if graph else NO_SELF, c0)
    part_i = np.zeros((G * per, k), np.int32)
    part_d = np.full((G * per, k), np.inf, np.float32)
    part_i[:M], part_d[:M] = i, d
    recv_i = np.empty(part_i.nbytes, np.uint8)
    recv_d = np.empty(part_d.nbytes, np.uint8)
    tr.alltoall(_u8(part_i), recv_i)
    tr.alltoall(_u8(part_d), recv_d)
    ri = recv_i.view(np.int32).reshape(G, per, k)
    rd = recv_d.view(np.float32).reshape(G, per, k)
    lo, hi = knn.shard_range(M, G, r)
    mi, md = oracle.merge(rd[:, :hi - lo], ri[:, :hi - lo], np.zeros(G, np.int64))
    return _gather_rows(tr, mi, per)[:M], _gather_rows(tr, md, per)[:M]


def _unit_block(n, u):
    """Row-major upper triangle of n x n pair blocks: unit u -> (row block, column block)."""
    m = 0
    while u >= n - m:
        u -= n - m
        m += 1
    return m, m + u


def standin_sym(tr, X, k, B=16):
    """Par-3 with B x B pair blocks (256 in the library): pivots of own rows all-gathered,
    the triangle's units split with knn_shard_range, candidates (D <= row pivot, and the
    transposed pair against the column pivot) appended to rank-local lists of ANY row,
    every rank's lists of own rows united and selected exactly."""
    G, r = tr.G, tr.rank
    N = X.shape[0]
    per = -(-N // G)
    lo, hi = knn.shard_range(N, G, r)
    D = oracle.dist_rows(X, X).astype(np.float32)  # stand-in for the GEMM's values
    np.fill_diagonal(D, np.inf)
    thr = np.full(G * per, np.nan, np.float32)
    # stand-in pivot: an upper bound of the row's k-th distance (the k-th of a column sample)
    samp = np.arange(0, N, 2)
    thr[lo:hi] = np.sort(D[lo:hi][:, samp], axis=1)[:, k - 1] if hi > lo else thr[lo:hi]
    thr = _gather_rows(tr, thr[r * per:(r + 1) * per], per)
    n = -(-N // B)
    u0, u1 = knn.shard_range(n * (n + 1) // 2, G, r)
    lists = [[] for _ in range(N)]
    for u in range(u0, u1):
        bi, bj = _unit_block(n, u)
        for i in range(bi * B, min(N, bi * B + B)):
            for j in range(bj * B, min(N, bj * B + B)):
                if bi == bj and j <= i:
                    continue  # a diagonal block's pairs once each (i < j), both directions below
                if D[i, j] <= thr[i]:
                    lists[i].append((D[i, j], j))
                if D[i, j] <= thr[j]:
                    lists[j].append((D[i, j], i))
    # list exchange (the library reads peers' lists in place over CUDA IPC; here gathered)
    cap = max(1, max(len(lists[i]) for i in range(N)))
    cap = int(np.max(_gather_rows(tr, np.array([cap], np.int32), 1)))
    cnt = np.array([len(lists[i]) for i in range(N)], np.int32)
    keys = np.full((N, cap), np.inf, np.float32)
    idxs = np.zeros((N, cap), np.int32)
    for i in range(N):
        for c, (v, j) in enumerate(lists[i]):
            keys[i, c], idxs[i, c] = v, j
    all_cnt = _gather_rows(tr, cnt, N).reshape(G, N)
    all_keys = _gather_rows(tr, keys, N).reshape(G, N, cap)
    all_idxs = _gather_rows(tr, idxs, N).reshape(G, N, cap)
    oi = np.zeros((hi - lo, k), np.int32)
    od = np.zeros((hi - lo, k), np.float32)
    for i in range(lo, hi):
        cand = [(float(all_keys[g, i, c]), int(all_idxs[g, i, c])) for g in range(G) for c in range(all_cnt[g, i])]
        assert len(cand) >= k  # the certificate
        cand.sort()
        oi[i - lo] = [j for _, j in cand[:k]]
        od[i - lo] = [v for v, _ in cand[:k]]
    return _gather_rows(tr, oi, per)[:N], _gather_rows(tr, od, per)[:N]


def _worker(rank, world, port, mode, N, d, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = sharded.TorchHostTransport()
        X = datagen.points(N, d, "gauss", seed=77) if rank == 0 else np.zeros((N, d), np.float32)
        X = _bcast(tr, X)
        if mode == "query":
            i, dd = standin_query(tr, X, X, k, True)
        elif mode == "corpus":
            i, dd = standin_corpus(tr, X, X, k, True)
        elif mode == "sym":
            i, dd = standin_sym(tr, X, k)
        else:
            Q = datagen.points(N + 3, d, "gauss", seed=78) if rank == 0 else np.zeros((N + 3, d), np.float32)
            Q = _bcast(tr, Q)
            i, dd = (standin_query if mode == "search" else standin_corpus)(tr, Q, X, k, False)
        q.put((rank, i, dd))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,N,world", [("query", 301, 2), ("corpus", 301, 2), ("corpus", 64, 2),
                                          ("sym", 301, 2), ("sym", 97, 3), ("search", 200, 2),
                                          ("search_corpus", 200, 2)])
def test_sharding_standins_equal_unsharded(mode, N, world):
    d, k = 9, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, N, d, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = datagen.points(N, d, "gauss", seed=77)
    if mode.startswith("search"):
        Q = datagen.points(N + 3, d, "gauss", seed=78)
        ref = oracle.knn(Q, X, k, graph=False)
    else:
        ref = oracle.knn(X, X, k, graph=True)
    for _, i, dd in res:  # every rank holds the full result
        assert np.array_equal(i, ref["idx32"])
        assert np.array_equal(dd, ref["dist32"])


def _transport_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = sharded.TorchHostTransport()
        out = {}
        send = np.full(5, 10 + rank, np.uint8)
        recv = np.empty(5 * world, np.uint8)
        tr.allgather(send, recv)
        out["allgather"] = recv.copy()
        b = np.arange(6, dtype=np.uint8) if rank == 0 else np.zeros(6, np.uint8)
        tr.broadcast(b, 0)
        out["broadcast"] = b.copy()
        s = np.array([[100 * rank + g] * 3 for g in range(world)], np.uint8).reshape(-1)
        r_ = np.empty_like(s)
        tr.alltoall(s, r_)
        out["alltoall"] = r_.copy()
        a = np.array([rank, -rank, 7], np.int32)
        tr.allreduce_max(a)
        out["allreduce"] = a.copy()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_host_transport_collectives():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, out in res.items():
        assert out["allgather"].tolist() == [10] * 5 + [11] * 5
        assert out["broadcast"].tolist() == list(range(6))
        assert out["alltoall"].tolist() == [r] * 3 + [100 + r] * 3  # block g from rank g
        assert out["allreduce"].tolist() == [1, 0, 7]


def test_shard_range_covers():
    for n in (0, 1, 7, 64, 301, 65536):
        for g in (1, 2, 3, 8):
            blocks = [knn.shard_range(n, g, r) for r in range(g)]
            covered = [j for lo, hi in blocks for j in range(lo, hi)]
            assert covered == list(range(n))
            per = -(-n // g)
            assert all(hi - lo <= per for lo, hi in blocks)
    assert knn.shard_range(10, 0, 0) == (0, 0) and knn.shard_range(10, 2, 5) == (0, 0)


def test_unit_block_matches_triangle():
    n = 9
    seen = [_unit_block(n, u) for u in range(n * (n + 1) // 2)]
    assert seen == [(i, j) for i in range(n) for j in range(i, n)]

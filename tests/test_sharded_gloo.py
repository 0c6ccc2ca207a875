"""World-size-2 CPU tests (gloo) of the multi-GPU orchestration in sharded.py.

The per-rank compute is replaced by oracle stand-ins (CPU tensors), so these tests check
the host logic of both shardings — row/column blocks, broadcast, global self exclusion,
index offsets, all-to-all routing, merge and gather — against the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1309_5478_b200 import datagen, sharded


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_compute(Q, X, k, metric, self_shift, idx_offset):
    """Stand-in for knn_search_block: fp32-rounded oracle distances, exact select."""
    Qn, Xn = Q.numpy(), X.numpy()
    D = oracle.dist_rows(Qn, Xn, metric=metric).astype(np.float32)
    if self_shift != -(2 ** 63):
        for i in range(D.shape[0]):
            j = i + self_shift
            if 0 <= j < D.shape[1]:
                D[i, j] = np.inf
    idx, dst = oracle.select_f32(D, k)
    return torch.from_numpy(idx + np.int32(idx_offset)), torch.from_numpy(dst)


def oracle_merge(part_dist, part_idx, offsets):
    idx, dst = oracle.merge(part_dist.numpy(), part_idx.numpy(), offsets)
    return torch.from_numpy(idx), torch.from_numpy(dst)


def oracle_peer_merge(part_i, part_d, k, row0, rows, group=None):
    """Stand-in for sharded.peer_merge: every rank's partial lists are visible to every
    rank (here through all_gather_object instead of CUDA IPC); the merge reads rows
    [row0, row0 + rows) of each rank's lists."""
    G = dist.get_world_size(group)
    table = [None] * G
    dist.all_gather_object(table, (part_i.numpy(), part_d.numpy()), group=group)
    pd = np.stack([t[1][row0:row0 + rows] for t in table])
    pi = np.stack([t[0][row0:row0 + rows] for t in table])
    idx, dst = oracle.merge(pd, pi, np.zeros(G, np.int64))
    return torch.from_numpy(idx), torch.from_numpy(dst)


def _worker(rank, world, port, mode, N, d, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = datagen.points(N, d, "gauss", seed=77)
        Xt = torch.from_numpy(X) if rank == 0 else torch.zeros((N, d), dtype=torch.float32)
        if mode == "query":
            i, dd = sharded.graph_query_sharded(Xt, k, compute=oracle_compute)
        elif mode == "corpus":
            i, dd = sharded.graph_corpus_sharded(Xt, k, compute=oracle_compute, merge=oracle_merge)
        elif mode == "corpus_peer":
            i, dd = sharded.graph_corpus_sharded(Xt, k, compute=oracle_compute, merge=oracle_merge,
                                                 exchange="peer", peer_merge_fn=oracle_peer_merge)
        else:
            Qt = torch.from_numpy(datagen.points(N + 3, d, "gauss", seed=78)) if rank == 0 \
                else torch.zeros((N + 3, d), dtype=torch.float32)
            i, dd = sharded.search_query_sharded(Qt, Xt, k, compute=oracle_compute)
        q.put((rank, i.numpy(), dd.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,N", [("query", 301), ("corpus", 301), ("corpus", 64),
                                    ("corpus_peer", 301), ("corpus_peer", 64), ("search", 200)])
def test_two_rank_sharding_equals_unsharded(mode, N):
    d, k = 9, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, N, d, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = datagen.points(N, d, "gauss", seed=77)
    if mode == "search":
        Q = datagen.points(N + 3, d, "gauss", seed=78)
        ref = oracle.knn(Q, X, k, graph=False)
    else:
        ref = oracle.knn(X, X, k, graph=True)
    for _, i, dd in res:  # every rank holds the full result
        assert np.array_equal(i, ref["idx32"])
        assert np.array_equal(dd, ref["dist32"])


def test_block_range_covers():
    for n in (1, 7, 64, 301):
        for g in (1, 2, 3, 8):
            blocks = [sharded.block_range(n, g, r) for r in range(g)]
            covered = [j for lo, hi in blocks for j in range(lo, hi)]
            assert covered == list(range(n))

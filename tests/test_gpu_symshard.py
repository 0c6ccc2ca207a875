"""Par-3: the symmetric multi-GPU k-NNG (sharded.graph_sym_sharded).

The ranks split the upper triangle of the distance matrix; every rank's select reads the
G ranks' candidate lists of its row block.  Checked three ways, all against the one-GPU
graph bit for bit: G = 1 through the same phases; G = 2 and 3 emulated in one process
(separate list buffers, the gather reading all of them); and two processes sharing this
GPU, exchanging CUDA IPC handles over gloo exactly as ranks on different GPUs do."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1309_5478_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def knn():
    from paper_1309_5478_b200 import knn as k
    return k


def reference(X, k, metric=0):
    i, d = knn().graph(X, k, metric=metric)
    return i, d


@pytest.mark.parametrize("N,d,k", [(20000, 48, 16), (16384, 64, 100)])
def test_one_rank_phases_equal_graph(N, d, k):
    from paper_1309_5478_b200 import sharded
    X = torch.from_numpy(datagen.points(N, d, "gauss", seed=N + k)).cuda()
    gi, gd = sharded.graph_sym_sharded(X, k)
    ri, rd = reference(X, k)
    assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))


@pytest.mark.parametrize("G,k,metric", [(2, 32, 0), (3, 8, 1), (2, 200, 0), (4, 64, 2)])
def test_emulated_ranks_equal_graph(G, k, metric):
    kn = knn()
    N, d = 17000, 40
    X = torch.from_numpy(datagen.points(N, d, "uniform", seed=G * 100 + k)).cuda()
    npad = -(-N // 256) * 256
    thr = torch.full((npad,), float("nan"), device="cuda")
    per = -(-N // G)
    for g in range(G):
        lo, hi = g * per, min(N, (g + 1) * per)
        kn.graph_pivots(X, k, lo, hi - lo, thr, metric=metric)
    units = kn.graph_units(N)
    cap = kn.graph_list_cap(k)
    lists = []
    for g in range(G):
        ulo, uhi = units * g // G, units * (g + 1) // G
        cnt = torch.zeros(N, dtype=torch.int32, device="cuda")
        ck = torch.empty((N, cap), dtype=torch.int32, device="cuda")
        ci = torch.empty((N, cap), dtype=torch.int32, device="cuda")
        kn.graph_partition(X, k, thr, ulo, uhi, cnt, ck, ci, metric=metric)
        lists.append((cnt, ck, ci))
    torch.cuda.synchronize()
    ptrs = [[l[j].data_ptr() for l in lists] for j in range(3)]
    parts_i, parts_d = [], []
    for g in range(G):
        lo, hi = g * per, min(N, (g + 1) * per)
        i, dd = kn.graph_gather_select(ptrs[0], ptrs[1], ptrs[2], cap, N, k, lo, hi - lo)
        parts_i.append(i)
        parts_d.append(dd)
    gi, gd = torch.cat(parts_i), torch.cat(parts_d)
    ri, rd = reference(X, k, metric)
    assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, d, k, q, no_ipc=False):
    import torch.distributed as dist
    from paper_1309_5478_b200 import sharded
    if no_ipc:
        os.environ["KNN_SHARD_NO_IPC"] = "1"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = torch.from_numpy(datagen.points(N, d, "gauss", seed=93)).cuda()
        for _ in range(2):  # the second call reuses the cached lists and IPC mappings
            i, dd = sharded.graph_sym_sharded(X, k, broadcast=False)
        q.put((rank, i.cpu().numpy(), dd.cpu().numpy()))
    except Exception as e:
        q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,k,no_ipc", [(16384, 16, False), (20000, 64, False), (16384, 16, True)])
def test_two_processes_one_gpu(N, k, no_ipc):
    """no_ipc: the ranks cannot map each other's lists; they agree on it and fall back to
    the query-row sharding, still bit-identical."""
    d = 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, d, k, q, no_ipc)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for _, i, dd in res:
        assert dd is not None, i
    X = torch.from_numpy(datagen.points(N, d, "gauss", seed=93)).cuda()
    ri, rd = reference(X, k)
    for _, i, dd in res:
        assert np.array_equal(i, ri.cpu().numpy())
        assert np.array_equal(dd.view(np.uint32), rd.cpu().numpy().view(np.uint32))

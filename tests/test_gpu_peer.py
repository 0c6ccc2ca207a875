"""Par-2 with the fused exchange + merge over CUDA IPC (sharded.peer_merge).

knn_merge_lists must equal knn_merge on a table of (non-contiguous) local lists; then two
processes sharing this one GPU (gloo for the host-side exchange of IPC handles) run the
corpus-sharded k-NNG with exchange="peer": each process's merge kernel reads the other
process's partial lists through a CUDA IPC mapping — the same mechanism that crosses
NVLink between GPUs — and the result must equal the unsharded graph bit for bit."""
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


def test_merge_lists_equals_merge():
    g = np.random.Generator(np.random.Philox(5))
    G, M, k = 5, 700, 40
    pd = np.sort(g.random((G, M + 30, k), dtype=np.float32), axis=2)
    pi = g.integers(0, 1 << 20, size=(G, M + 30, k)).astype(np.int32)
    offs = np.arange(G, dtype=np.int64) * 1000
    row0 = 30
    tens_d = [torch.from_numpy(pd[gg]).cuda() for gg in range(G)]   # separate allocations
    tens_i = [torch.from_numpy(pi[gg]).cuda() for gg in range(G)]
    got = knn().merge_lists([t.data_ptr() for t in tens_d], [t.data_ptr() for t in tens_i],
                            row0, M, k, offs)
    ref = knn().merge(torch.from_numpy(np.ascontiguousarray(pd[:, row0:])).cuda(),
                      torch.from_numpy(np.ascontiguousarray(pi[:, row0:])).cuda(), offs)
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, d, k, q):
    import torch.distributed as dist
    from paper_1309_5478_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = torch.from_numpy(datagen.points(N, d, "gauss", seed=91)).cuda()
        i, dd = sharded.graph_corpus_sharded(X, k, exchange="peer", broadcast=False)
        q.put((rank, i.cpu().numpy(), dd.cpu().numpy()))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,k", [(5000, 16), (3001, 100)])
def test_peer_exchange_two_processes_one_gpu(N, k):
    d = 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, d, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for _, i, dd in res:
        assert dd is not None, i
    X = datagen.points(N, d, "gauss", seed=91)
    ri, rd = knn().graph(torch.from_numpy(X).cuda(), k)
    for _, i, dd in res:
        assert np.array_equal(i, ri.cpu().numpy())
        assert np.array_equal(dd.view(np.uint32), rd.cpu().numpy().view(np.uint32))

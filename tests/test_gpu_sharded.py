"""The multi-GPU boundary (knn_graph_sharded / knn_search_sharded).

Every mode (query rows, corpus columns, the symmetric triangle split) against the one-GPU
calls bit for bit: one rank without a communicator; a one-rank NCCL communicator through the
C ABI (this box has one GPU); Par-3's phases with G = 2..4 emulated in one process; and two
processes sharing this GPU with the library's host transport over gloo — broadcast,
all-to-all, all-gather and the CUDA IPC list exchange exactly as ranks on different GPUs
run them (NCCL refuses two ranks on one device)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1309_5478_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _exact_plan():
    """These tests compare decompositions bit for bit: the one-GPU reference runs the pivot
    plan with the FP32-accurate partition (the sharded / streamed phases always do)."""
    from paper_1309_5478_b200 import knn as k
    k.set_plan(k.PLAN_PIVOT_EXACT)
    yield
    k.set_plan(k.PLAN_AUTO)


def knn():
    from paper_1309_5478_b200 import knn as k
    return k


def reference(X, k, metric=0):
    i, d = knn().graph(X, k, metric=metric)
    return i, d


@pytest.mark.parametrize("mode", ["sym", "corpus", "query"])
@pytest.mark.parametrize("N,d,k", [(20000, 48, 16), (16384, 64, 100)])
def test_one_rank_sharded_equal_graph(N, d, k, mode, monkeypatch):
    # no communicator: the sharded call runs as one rank through the same phases
    monkeypatch.setenv("KNN_SHARD_G1_PHASES", "1")
    kn = knn()
    kn.comm_destroy()
    X = torch.from_numpy(datagen.points(N, d, "gauss", seed=N + k)).cuda()
    gi, gd = kn.graph_sharded(X, k, mode=mode)
    assert kn.last_shard_mode() == kn.SHARD_MODES[mode]
    ri, rd = reference(X, k)
    assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))


def test_nccl_one_rank_communicator(monkeypatch):
    # the NCCL transport through the C ABI with a one-rank communicator (this box has one
    # GPU): unique id, init, every sharded mode through its phases, destroy
    monkeypatch.setenv("KNN_SHARD_G1_PHASES", "1")
    kn = knn()
    uid = kn.comm_unique_id()
    assert len(uid) == 128
    kn.comm_init(0, 1, uid)
    try:
        assert kn.comm_info() == (1, 0, 1)
        N, d, k = 17000, 32, 24
        X = torch.from_numpy(datagen.points(N, d, "uniform", seed=5)).cuda()
        ri, rd = reference(X, k)
        for mode in ("sym", "corpus", "query"):
            gi, gd = kn.graph_sharded(X, k, mode=mode)
            assert kn.last_shard_mode() == kn.SHARD_MODES[mode]
            assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))
        Q = torch.from_numpy(datagen.points(3000, d, "gauss", seed=6)).cuda()
        si, sd = kn.search(Q, X, k)
        for mode in ("query", "corpus"):
            gi, gd = kn.search_sharded(Q, X, k, mode=mode)
            assert torch.equal(gi, si) and torch.equal(gd.view(torch.int32), sd.view(torch.int32))
    finally:
        kn.comm_destroy()
    assert kn.comm_info() == (0, 0, 1)


@pytest.mark.parametrize("phases", ["0", "1"])
def test_sharded_rejects_nonfinite(phases, monkeypatch):
    monkeypatch.setenv("KNN_SHARD_G1_PHASES", phases)
    kn = knn()
    X = torch.from_numpy(datagen.points(16384, 16, "gauss", seed=8)).cuda()
    X[123, 5] = float("nan")
    for mode in ("sym", "corpus", "query"):
        with pytest.raises(kn.KnnError) as e:
            kn.graph_sharded(X, 8, mode=mode)
        assert e.value.status == 3, (mode, str(e.value))


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
        ce = torch.empty((N, cap), dtype=torch.int64, device="cuda")
        kn.graph_partition(X, k, thr, ulo, uhi, cnt, ce, metric=metric)
        lists.append((cnt, ce))
    torch.cuda.synchronize()
    parts_i, parts_d = [], []
    for g in range(G):
        lo, hi = g * per, min(N, (g + 1) * per)
        i, dd = kn.graph_gather_select([l[0].data_ptr() for l in lists], [l[1].data_ptr() for l in lists], cap, N,
                                       k, lo, hi - lo)
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


def _worker(rank, world, port, case, q):
    import torch.distributed as dist
    from paper_1309_5478_b200 import sharded
    mode, N, d, k, no_ipc, search = case
    if no_ipc:
        os.environ["KNN_SHARD_NO_IPC"] = "1"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sharded.init()  # gloo group: the library's host-callback transport
        kn = knn()
        if os.environ.get("KNN_TEST_AUTO_PLAN") != "1":
            kn.set_plan(kn.PLAN_PIVOT_EXACT)  # (the Par-1 fallback's blocks: as the reference)
        assert kn.comm_info() == (2, rank, world)
        X = torch.from_numpy(datagen.points(N, d, "gauss", seed=93)).cuda()
        if rank != 0:
            X.zero_()  # rank 0's points arrive by the library's broadcast
        if search:
            Q = torch.from_numpy(datagen.points(N // 3, d, "uniform", seed=94)).cuda()
            if rank != 0:
                Q.zero_()
        for _ in range(2):  # the second call reuses the lists and the peer mappings
            if search:
                i, dd = sharded.search(Q, X, k, mode=mode)
            else:
                i, dd = sharded.graph(X, k, mode=mode)
        q.put((rank, i.cpu().numpy(), dd.cpu().numpy(), kn.last_shard_mode()))
    except Exception as e:
        q.put((rank, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("sym", 16384, 24, 16, False, False), ("sym", 20000, 24, 64, False, False),
                                  ("sym", 16384, 24, 16, True, False), ("corpus", 5000, 24, 16, False, False),
                                  ("corpus", 3001, 24, 100, False, False), ("query", 3001, 24, 20, False, False),
                                  ("query", 6000, 24, 32, False, True), ("corpus", 6000, 24, 32, False, True)])
def test_two_processes_one_gpu(case):
    """Two ranks sharing this GPU run the library's sharded calls with the host transport
    (gloo): broadcast, all-to-all / list exchange over CUDA IPC, merge, all-gather.  With
    no_ipc the ranks cannot map each other's lists; they agree on it and fall back to the
    query-row sharding.  Every rank's result equals the one-GPU call bit for bit."""
    mode, N, d, k, no_ipc, search = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for _, i, dd, _m in res:
        assert dd is not None, i
    X = torch.from_numpy(datagen.points(N, d, "gauss", seed=93)).cuda()
    if search:
        Q = torch.from_numpy(datagen.points(N // 3, d, "uniform", seed=94)).cuda()
        ri, rd = knn().search(Q, X, k)
    else:
        ri, rd = reference(X, k)
    want_mode = knn().SHARD_MODES["query" if no_ipc else mode]
    for _, i, dd, m in res:
        assert m == want_mode
        assert np.array_equal(i, ri.cpu().numpy())
        assert np.array_equal(dd.view(np.uint32), rd.cpu().numpy().view(np.uint32))


# ------------- Par-3 with the single-product partition (the automatic plan) ---
@pytest.mark.parametrize("G,k,metric", [(2, 32, 0), (3, 10, 1), (1, 16, 0)])
def test_emulated_ranks_auto_plan_equal_graph(G, k, metric):
    """Under the automatic plan the Par-3 phases run the single-product partition (the
    decision taken on the device from all N pivots, the same on every rank) and re-evaluate
    each rank's rows from the points: bit-identical to the one-GPU automatic call, which
    takes the same decision (both lists hold the same lower bounds; the re-evaluated values
    do not depend on the list order)."""
    kn = knn()
    kn.set_plan(kn.PLAN_AUTO)
    N, d = 17000, 40
    X = torch.from_numpy(datagen.points(N, d, "uniform", seed=G * 100 + k + 7)).cuda()
    ri, rd = reference(X, k, metric)
    assert kn.last_plan() == 5, kn.last_plan()
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
        ce = torch.empty((N, cap), dtype=torch.int64, device="cuda")
        kn.graph_partition(X, k, thr, ulo, uhi, cnt, ce, metric=metric)
        lists.append((cnt, ce))
    torch.cuda.synchronize()
    parts_i, parts_d = [], []
    for g in range(G):
        lo, hi = g * per, min(N, (g + 1) * per)
        i, dd = kn.graph_gather_select([l[0].data_ptr() for l in lists], [l[1].data_ptr() for l in lists], cap, N,
                                       k, lo, hi - lo)
        assert kn.last_plan() == 5, kn.last_plan()
        parts_i.append(i)
        parts_d.append(dd)
    gi, gd = torch.cat(parts_i), torch.cat(parts_d)
    assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))


def test_one_rank_sym_sharded_auto_plan(monkeypatch):
    monkeypatch.setenv("KNN_SHARD_G1_PHASES", "1")
    kn = knn()
    kn.set_plan(kn.PLAN_AUTO)
    kn.comm_destroy()
    X = torch.from_numpy(datagen.points(20000, 64, "gauss", seed=777)).cuda()
    ri, rd = reference(X, 24)
    assert kn.last_plan() == 5, kn.last_plan()
    for _ in range(2):
        gi, gd = kn.graph_sharded(X, 24, mode="sym")
        assert kn.last_shard_mode() == kn.SHARD_MODES["sym"]
        assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))


def test_two_processes_one_gpu_auto_plan(monkeypatch):
    """The two-process Par-3 run (host transport, CUDA IPC list reads) under the automatic
    plan: the single-product partition on both ranks, equal to the one-GPU automatic call."""
    monkeypatch.setenv("KNN_TEST_AUTO_PLAN", "1")
    kn = knn()
    kn.set_plan(kn.PLAN_AUTO)
    case = ("sym", 16384, 24, 16, False, False)
    mode, N, d, k, no_ipc, search = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for _, i, dd, _m in res:
        assert dd is not None, i
    X = torch.from_numpy(datagen.points(N, d, "gauss", seed=93)).cuda()
    ri, rd = reference(X, k)
    assert kn.last_plan() == 5, kn.last_plan()
    for _, i, dd, m in res:
        assert m == kn.SHARD_MODES["sym"]
        assert np.array_equal(i, ri.cpu().numpy())
        assert np.array_equal(dd.view(np.uint32), rd.cpu().numpy().view(np.uint32))

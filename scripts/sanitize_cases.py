"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
kernel family of the library once — C1 k-NNG (symmetric GEMM + warp select), a pivot-plan
k-NNG (sample, pivots, partition, candidate select), the quantile-pivot plan (k > 32), the
CTA and cluster selects, the k-way merge, and Par-3's phases with 2 emulated ranks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1309_5478_b200 import datagen, knn

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda", 0)


def c1():
    X = torch.from_numpy(datagen.points(1024, 32, "uniform", seed=1)).to(dev)
    knn.graph(X, 8)


def pivot():
    """The 3-product partition (KNN_PLAN_PIVOT_EXACT) and the automatic plan (the device
    picks the single-product partition + fp32 re-evaluation for uniform data: plan 5)."""
    X = torch.from_numpy(datagen.points(16384, 32, "uniform", seed=2)).to(dev)
    knn.set_plan(knn.PLAN_PIVOT_EXACT)
    knn.graph(X, 16)
    assert knn.last_plan() == 3
    knn.set_plan(knn.PLAN_AUTO)
    knn.graph(X, 16)
    assert knn.last_plan() == 5, knn.last_plan()


def hostpipe():
    """knn_search_block_host's pipelined k-NNG (copy stream, chunked phases, gated kernels)."""
    X = datagen.points(16384, 32, "uniform", seed=6)
    Xp = torch.from_numpy(X).pin_memory().numpy()
    knn.search_block_host(Xp, Xp, 16, self_shift=0)
    assert knn.last_plan() == 5, knn.last_plan()


def twopass():
    """The two-pass warp select (k <= 32, >= 4 rows per SM): ragged rows, ties."""
    g = np.random.Generator(np.random.Philox(7))
    D = torch.from_numpy(g.random((600, 5000), dtype=np.float32)).to(dev)
    knn.select(D, 32)
    D[:, ::3] = 0.5
    knn.select(D, 8)
    assert knn.last_select_kernel()[0] == "two-pass warp per row"


def pivotq():
    X = torch.from_numpy(datagen.points(16384, 32, "gauss", seed=3)).to(dev)
    knn.graph(X, 100)


def selects():
    g = np.random.Generator(np.random.Philox(4))
    D = torch.from_numpy(g.random((64, 20000), dtype=np.float32)).to(dev)
    knn.select(D, 100)          # CTA per row (k > 32)
    knn.select(D[:8].contiguous(), 32)  # few rows: cluster per row
    D2 = torch.from_numpy(g.random((2000, 3000), dtype=np.float32)).to(dev)
    knn.select(D2, 16)          # warp per row
    pd = torch.sort(torch.from_numpy(g.random((3, 500, 20), dtype=np.float32)).to(dev), dim=2).values
    pi = torch.from_numpy(g.integers(0, 1000, (3, 500, 20)).astype(np.int32)).to(dev)
    knn.merge(pd, pi, np.array([0, 1000, 2000], np.int64))


def par3():
    N, d, k, G = 16384, 24, 16, 2
    X = torch.from_numpy(datagen.points(N, d, "uniform", seed=5)).to(dev)
    thr = torch.full((N,), float("nan"), device=dev)
    per = -(-N // G)
    for g in range(G):
        knn.graph_pivots(X, k, g * per, min(N, (g + 1) * per) - g * per, thr)
    units, cap = knn.graph_units(N), knn.graph_list_cap(k)
    lists = []
    for g in range(G):
        cnt = torch.zeros(N, dtype=torch.int32, device=dev)
        ce = torch.empty((N, cap), dtype=torch.int64, device=dev)
        knn.graph_partition(X, k, thr, units * g // G, units * (g + 1) // G, cnt, ce)
        lists.append((cnt, ce))
    torch.cuda.synchronize()
    for g in range(G):
        knn.graph_gather_select([l[0].data_ptr() for l in lists], [l[1].data_ptr() for l in lists], cap, N, k,
                                g * per, min(N, (g + 1) * per) - g * per)
        assert knn.last_plan() == 5, knn.last_plan()  # the single-product partition + re-evaluation


cases = {"c1": c1, "pivot": pivot, "hostpipe": hostpipe, "twopass": twopass, "pivotq": pivotq,
         "selects": selects, "par3": par3}
for name, fn in cases.items():
    if which in ("all", name):
        fn()
        torch.cuda.synchronize()
        print("case", name, "ok", flush=True)

"""NEXT-2: cosine and Pearson metrics through the C ABI, against the oracle.

Keys are 1 - similarity (reading R14) with the zero-norm sentinel 3.0
(SPEC.md:143); tolerance: |key - key64| <= 1e-5 absolute (oracle.checks.COS_TOL, DESIGN.md
R19).  The same GEMM, select, symmetric and pivot plans as L2 run underneath, so the plans
must also agree bit for bit with each other."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from oracle import checks
from paper_1309_5478_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

METRICS = [oracle.COSINE, oracle.PEARSON]


def knn():
    from paper_1309_5478_b200 import knn as k
    return k


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def with_degenerate(X, zero_rows=(), const_rows=()):
    X = X.copy()
    for r in zero_rows:
        X[r] = 0.0
    for r in const_rows:
        X[r] = 1.75
    return X


def e2e(Q, X, gi, gd, k, rows, graph, metric, min_pinned=0.0):
    D64 = oracle.dist_rows(Q, X, rows=rows, metric=metric)
    res = checks.check_rows(gi[rows], gd[rows], D64, None, None, rows, k, metric=metric, graph=graph)
    assert res["failures"] == [], res["failures"][:5]
    assert res["n_pinned"] >= min_pinned * len(rows)


@pytest.mark.parametrize("metric", METRICS)
@pytest.mark.parametrize("M,N,d,dist", [(300, 700, 100, "gauss"), (129, 513, 7, "uniform"), (64, 333, 1000, "clusters")])
def test_distances_parity(metric, M, N, d, dist):
    Q = with_degenerate(datagen.points(M, d, dist, seed=M + d), zero_rows=(5,), const_rows=(7,))
    X = with_degenerate(datagen.points(N, d, dist, seed=N + d), zero_rows=(0, 300), const_rows=(11,))
    D = knn().distances(cuda(Q), cuda(X), metric=metric).cpu().numpy()
    D64 = oracle.dist_rows(Q, X, metric=metric)
    err = np.abs(D.astype(np.float64) - D64)
    assert err.max() <= checks.COS_TOL, float(err.max())
    # sentinels exact: zero vectors (cosine and Pearson) and constant vectors (Pearson)
    assert np.all(D[5] == 3.0) and np.all(D[:, 0] == 3.0) and np.all(D[:, 300] == 3.0)
    if metric == oracle.PEARSON:
        assert np.all(D[7] == 3.0) and np.all(D[:, 11] == 3.0)
    assert D.min() >= 0.0 and D.max() <= 3.0


@pytest.mark.parametrize("metric", METRICS)
def test_graph_blocked_e2e(metric):
    X = with_degenerate(datagen.points(5000, 64, "clusters", seed=61), zero_rows=(17,), const_rows=(40,))
    gi, gd = knn().graph(cuda(X), 16, metric=metric)
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    rows = np.concatenate([np.arange(0, 5000, 97), [17, 40]])
    e2e(X, X, gi, gd, 16, rows, True, metric)


@pytest.mark.parametrize("metric", METRICS)
def test_graph_pivot_equals_materialised_and_oracle(metric):
    kn = knn()
    # (a zero / constant row ties all N keys at 3.0 and overflows its candidate list: that
    # redo path is covered by the L2 grid test; here the plan must stay the pivot plan)
    X = datagen.points(20000, 48, "gauss", seed=62)
    Xc = cuda(X)
    gi, gd = kn.graph(Xc, 32, metric=metric)
    assert kn.last_plan() == 3, kn.last_plan()
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.graph(Xc, 32, metric=metric)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))
    rows = np.array([0, 3, 8, 1234, 7777, 19999])
    e2e(X, X, gi.cpu().numpy(), gd.cpu().numpy(), 32, rows, True, metric)


@pytest.mark.parametrize("metric", METRICS)
def test_search_pivot_block(metric):
    kn = knn()
    X = datagen.points(18000, 40, "uniform", seed=63)
    Q = datagen.points(2500, 40, "uniform", seed=64)
    gi, gd = kn.search_block(cuda(Q), cuda(X), 20, metric=metric)
    assert kn.last_plan() == 4
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.search_block(cuda(Q), cuda(X), 20, metric=metric)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri) and torch.equal(gd, rd)
    rows = np.arange(0, 2500, 111)
    e2e(Q, X, gi.cpu().numpy(), gd.cpu().numpy(), 20, rows, False, metric)


def test_pearson_affine_partner_is_nearest():
    # rows 2i and 2i+1 = (x, 2x + 3): Pearson key 0 between partners
    base = datagen.points(500, 30, "gauss", seed=65)
    X = np.empty((1000, 30), np.float32)
    X[0::2] = base
    X[1::2] = 2 * base + 3
    gi, gd = knn().graph(cuda(X), 1, metric=oracle.PEARSON)
    gi, gd = gi.cpu().numpy()[:, 0], gd.cpu().numpy()[:, 0]
    partner = np.arange(1000) ^ 1
    assert np.array_equal(gi, partner)
    assert np.all(gd <= checks.COS_TOL)


def test_cosine_needs_tensor_path():
    code = (
        "import torch\n"
        "from paper_1309_5478_b200 import knn\n"
        "X = torch.rand(100, 8, device='cuda')\n"
        "try:\n"
        "    knn.graph(X, 3, metric=knn.COSINE)\n"
        "    raise SystemExit('no error')\n"
        "except knn.KnnError as e:\n"
        "    assert e.status == 2, e.status\n")
    env = dict(os.environ, KNN_GEMM="simt")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call([sys.executable, "-c", code], env=env, cwd=root)

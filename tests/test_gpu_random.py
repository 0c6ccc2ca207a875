"""Seeded random sweep over shapes and parameters around the plans' thresholds (pivot
plans from N = 16384 and M = 256, k = 32 | 33, d around the 64-wide K padding, ragged
tiles), every metric: the pivot plan with the FP32-accurate partition (PLAN_PIVOT_EXACT) must
equal the materialised plan bit for bit, and the automatic plan (which may partition on the
single product and re-evaluate the survivors in fp32) and the exact plan
must both pass the oracle's E2E checks on sampled rows."""
import numpy as np
import pytest

import oracle
from oracle import checks
from paper_1309_5478_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def knn():
    from paper_1309_5478_b200 import knn as k
    return k


def _cases():
    g = np.random.Generator(np.random.Philox(20261017))
    out = []
    for i in range(24):
        graph = bool(g.integers(0, 2))
        N = int(g.choice([16383, 16384, 16385, 17000, 20001, 24575]))
        M = N if graph else int(g.choice([255, 256, 257, 1000, 3001]))
        d = int(g.choice([1, 3, 63, 64, 65, 100, 129]))
        k = int(g.choice([1, 7, 32, 33, 64, 100, 257]))
        metric = int(g.choice([0, 1, 2, 3])) if d > 1 else int(g.choice([0, 1]))
        dist = str(g.choice(["uniform", "gauss", "clusters"]))
        out.append((i, graph, M, N, d, k, metric, dist))
    return out


@pytest.mark.parametrize("i,graph,M,N,d,k,metric,dist", _cases())
def test_random_case(i, graph, M, N, d, k, metric, dist):
    kn = knn()
    X = datagen.points(N, d, dist, seed=5000 + i)
    Q = X if graph else datagen.points(M, d, dist, seed=6000 + i)
    Xt = torch.from_numpy(X).cuda()
    Qt = Xt if graph else torch.from_numpy(Q).cuda()

    def run():
        if graph:
            return kn.graph(Xt, k, metric=metric)
        return kn.search_block(Qt, Xt, k, metric=metric)

    ai, ad = run()  # automatic plan
    try:
        kn.set_plan(kn.PLAN_PIVOT_EXACT)
        gi, gd = run()
        kn.set_plan(kn.PLAN_MATERIALISED)
        ri, rd = run()
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri), "plans differ (indices)"
    assert torch.equal(gd.view(torch.int32), rd.view(torch.int32)), "plans differ (distances)"
    rows = np.unique(np.linspace(0, M - 1, 24).astype(np.int64))
    if metric >= 2:
        D64 = oracle.dist_rows(Q, X, rows=rows, metric=metric)
    else:
        D64 = oracle.dist_rows(Q, X, rows=rows)  # squared; check_rows maps L2 through sqrt
    for ii, dd in ((gi, gd), (ai, ad)):
        gi_np, gd_np = ii.cpu().numpy(), dd.cpu().numpy()
        if metric >= 2:
            res = checks.check_rows(gi_np[rows], gd_np[rows], D64, None, None, rows, k, metric=metric,
                                    graph=graph)
        else:
            res = checks.check_rows(gi_np[rows], gd_np[rows], D64, oracle.sqnorms(Q)[rows], oracle.sqnorms(X),
                                    rows, k, metric=metric, graph=graph)
        assert res["failures"] == [], res["failures"][:3]

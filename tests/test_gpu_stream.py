"""NEXT-4: out-of-core k-NN with the corpus streamed from host memory.

knn_search_streamed keeps Q and X in host memory, streams corpus chunks to the device
(copy/compute overlap) and merges each chunk's partial top-k into the running result.
Per-pair values do not depend on the chunking and the merge is exact under the total
order, so the result must equal the device-resident call bit for bit (which the other
suites pin to the oracle); sampled rows are also checked against the oracle directly."""
import numpy as np
import pytest

import oracle
from oracle import checks
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


def same(a, b):
    assert np.array_equal(a[0], b[0]), np.argwhere(a[0] != b[0])[:3]
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


@pytest.mark.parametrize("chunk,qblock", [(7000, 0), (16384, 1000), (20001, 2999), (100000, 0)])
@pytest.mark.parametrize("k", [10, 100])
def test_streamed_search_equals_resident(chunk, qblock, k):
    Q = datagen.points(3000, 64, "gauss", seed=41)
    X = datagen.points(50000, 64, "gauss", seed=42)
    got = knn().search_streamed(Q, X, k, chunk_points=chunk, query_block=qblock)
    ri, rd = knn().search(torch.from_numpy(Q).cuda(), torch.from_numpy(X).cuda(), k)
    same(got, (ri.cpu().numpy(), rd.cpu().numpy()))
    # and directly against the oracle on sampled rows (E2E-1/2)
    rows = np.arange(0, 3000, 97)
    D64 = oracle.dist_rows(Q, X, rows=rows)
    res = checks.check_rows(got[0][rows], got[1][rows], D64, oracle.sqnorms(Q)[rows],
                            oracle.sqnorms(X), rows, k, graph=False)
    assert res["failures"] == [], res["failures"][:3]


@pytest.mark.parametrize("chunk,qblock", [(4096, 0), (5000, 3333), (16384, 8000)])
def test_streamed_graph_equals_resident(chunk, qblock):
    X = datagen.points(20000, 40, "uniform", seed=43)
    k = 16
    got = knn().search_streamed(X, X, k, graph=True, chunk_points=chunk, query_block=qblock)
    ri, rd = knn().graph(torch.from_numpy(X).cuda(), k)
    same(got, (ri.cpu().numpy(), rd.cpu().numpy()))
    assert not np.any(got[0] == np.arange(20000)[:, None])  # self excluded across chunks


def test_streamed_cosine_and_trailing_chunk():
    Q = datagen.points(700, 33, "gauss", seed=44)
    X = datagen.points(10050, 33, "gauss", seed=45)  # last chunk of 50 < k + 1: folded
    k = 64
    got = knn().search_streamed(Q, X, k, metric=knn().COSINE, chunk_points=2500)
    ri, rd = knn().search_block(torch.from_numpy(Q).cuda(), torch.from_numpy(X).cuda(), k,
                                metric=knn().COSINE)
    same(got, (ri.cpu().numpy(), rd.cpu().numpy()))


def test_streamed_pinned_inputs_and_errors():
    X = datagen.points(9000, 16, "uniform", seed=46)
    Xp = torch.from_numpy(X).pin_memory().numpy()
    got = knn().search_streamed(Xp, Xp, 5, graph=True, chunk_points=3000)
    ri, rd = knn().graph(torch.from_numpy(X).cuda(), 5)
    same(got, (ri.cpu().numpy(), rd.cpu().numpy()))
    with pytest.raises(knn().KnnError):
        knn().search_streamed(X[:10], X[:10], 10, graph=True)  # k > N - 1

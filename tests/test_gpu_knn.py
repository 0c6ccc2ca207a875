"""a-S2 / a-S3 / end-to-end parity of the CUDA path against the oracle.

Tolerances come from BASELINE.json's north star: distances within 1e-5 of
(||q||^2 + ||c||^2) of the fp64 value; neighbour lists checked with E2E-1/2 (oracle.checks)
and, on integer-grid data where every correct implementation is exact, bit-identical
to the oracle (E2E-3).  Sizes span several GEMM tiles (128×256) with ragged tails; the
BASELINE configs run at full size on sampled rows."""
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


def knn():
    from paper_1309_5478_b200 import knn as k
    return k


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ------------------------------------------------------------------ a-S2 -------------
def test_rownorms():
    X = datagen.points(3001, 77, "gauss", seed=1)
    sqn, flag = knn().rownorms(cuda(X))
    ref = oracle.sqnorms(X)
    assert np.array_equal(sqn.cpu().numpy(), ref.astype(np.float32))  # fp64 acc, one rounding
    assert int(flag.item()) == 0
    G = datagen.points(500, 1024, "grid", seed=2)
    assert np.array_equal(knn().rownorms(cuda(G))[0].cpu().numpy(), oracle.sqnorms(G).astype(np.float32))
    X[17, 3] = np.nan
    assert int(knn().rownorms(cuda(X))[1].item()) == 1


# ------------------------------------------------------------------ a-S3 -------------
@pytest.mark.parametrize("M,N,d,dist", [(300, 517, 32, "uniform"), (129, 1000, 1, "gauss"),
                                        (257, 300, 3, "uniform"), (1000, 777, 100, "clusters"),
                                        (256, 2048, 256, "gauss"), (130, 513, 1000, "uniform"),
                                        (64, 4000, 128, "clusters")])
@pytest.mark.parametrize("metric", [0, 1])
def test_distances_within_tolerance(M, N, d, dist, metric):
    Q = datagen.points(M, d, dist, seed=M + d)
    X = datagen.points(N, d, dist, seed=N + d + 1)
    D = knn().distances(cuda(Q), cuda(X), metric=metric).cpu().numpy()
    D64 = oracle.dist_rows(Q, X)
    ratio, bad = checks.check_distances(D, D64, oracle.sqnorms(Q), oracle.sqnorms(X), metric)
    assert bad == 0, f"max |err|/tol = {ratio}"


def test_distances_integer_grid_exact():
    # all norms/dots are integers < 2^24: the split GEMM and epilogue are exact
    Q = datagen.points(200, 1024, "grid", seed=3)
    X = datagen.points(333, 1024, "grid", seed=4)
    D = knn().distances(cuda(Q), cuda(X)).cpu().numpy()
    assert np.array_equal(D, oracle.dist_rows(Q, X).astype(np.float32))


def test_distances_self_exclusion_and_ld():
    X = datagen.points(400, 16, "uniform", seed=5)
    D = knn().distances(cuda(X), cuda(X), self_shift=0, ldD=404).cpu().numpy()
    assert np.all(np.isinf(np.diag(D)))
    off = ~np.eye(400, dtype=bool)
    ratio, bad = checks.check_distances(np.where(off, D, 0), np.where(off, oracle.dist_rows(X, X), 0),
                                        oracle.sqnorms(X), oracle.sqnorms(X))
    assert bad == 0
    D2 = knn().distances(cuda(X[:100]), cuda(X), self_shift=50).cpu().numpy()
    assert all(np.isinf(D2[i, i + 50]) for i in range(100))


def test_distances_scale_extremes():
    # per-vector power-of-two scaling keeps tiny and huge vectors FP32-accurate
    g = np.random.Generator(np.random.Philox(6))
    X = g.standard_normal((300, 64)).astype(np.float32)
    X[:100] *= np.float32(1e-20)
    X[100:200] *= np.float32(1e15)
    D = knn().distances(cuda(X), cuda(X)).cpu().numpy()
    n = oracle.sqnorms(X)
    ratio, bad = checks.check_distances(D, oracle.dist_rows(X, X), n, n)
    assert bad == 0, ratio


# ------------------------------------------------------------------ end to end -------
def run_graph(X, k, metric=0):
    i, d = knn().graph(cuda(X), k, metric=metric)
    return i.cpu().numpy(), d.cpu().numpy()


class exact_plan:
    """Pivot plan with the FP32-accurate 3-product partition (PLAN_PIVOT_EXACT): bit-identical
    to the materialised plan and to the sharded / pipelined decompositions.  The automatic
    plan may instead partition on the single product and re-evaluate the survivors in fp32
    (DESIGN.md §6.5); it is checked against the oracle."""

    def __enter__(self):
        knn().set_plan(knn().PLAN_PIVOT_EXACT)

    def __exit__(self, *a):
        knn().set_plan(knn().PLAN_AUTO)


def e2e_check(Q, X, gi, gd, k, rows, graph, metric=0, min_pinned=0.0, chunk=128):
    # L2 is checked in the squared domain; cosine / Pearson on the keys themselves.  Rows
    # are checked in chunks so that the fp64 oracle rows stay small at full size.
    rows = np.asarray(rows)
    cn = oracle.sqnorms(X)
    res = {"n_rows": 0, "n_pinned": 0, "failures": []}
    for c0 in range(0, len(rows), chunk):
        rr = rows[c0:c0 + chunk]
        D64 = oracle.dist_rows(Q, X, rows=rr, metric=metric if metric >= 2 else 0)
        r = checks.check_rows(gi[rr], gd[rr], D64, oracle.sqnorms(Q[rr]), cn, rr, k, metric=metric,
                              graph=graph)
        for key in ("n_rows", "n_pinned"):
            res[key] += r[key]
        res["failures"] += r["failures"]
    assert res["failures"] == [], res["failures"][:5]
    assert res["n_pinned"] >= min_pinned * len(rows)
    return res


def test_c1_graph_all_rows():
    cfg = datagen.CONFIGS["C1"]
    X, _ = datagen.config_inputs(cfg)
    gi, gd = run_graph(X, cfg.k)
    e2e_check(X, X, gi, gd, cfg.k, np.arange(cfg.N), True, min_pinned=0.9)


def test_c1_graph_l2_metric():
    cfg = datagen.CONFIGS["C1"]
    X, _ = datagen.config_inputs(cfg)
    gi, gd = run_graph(X, cfg.k, metric=1)
    e2e_check(X, X, gi, gd, cfg.k, np.arange(0, cfg.N, 3), True, metric=1)


@pytest.mark.parametrize("N,d,k", [(2000, 64, 50), (5000, 1024, 1024), (3333, 7, 100)])
def test_integer_grid_graph_exact(N, d, k):
    # E2E-3: the full lists (indices, order, distances) equal the oracle's R32 exactly
    X = datagen.points(N, d, "grid", seed=N + d)
    gi, gd = run_graph(X, k)
    rows = np.arange(0, N, max(1, N // 300))
    ref = oracle.knn(X, X, k, rows=rows, graph=True)
    assert np.array_equal(gi[rows], ref["idx32"])
    assert np.array_equal(gd[rows], ref["dist32"])


def _sample_rows(M, n, seed):
    g = np.random.Generator(np.random.Philox(seed))
    rows = np.unique(np.concatenate([[0, 1, M - 2, M - 1], g.integers(0, M, n)]))
    return rows


def _block_rows(M, n_random, seed):
    """Full-size oracle sample: the first and last row of every 256-row block
    (the partition GEMM's 256x256 tiles: every row's diagonal block straddles the
    diagonal), the 128-row CTA boundary rows of every 8th block, plus seeded random rows."""
    b0 = np.arange(0, M, 256)
    edges = [b0, np.minimum(b0 + 255, M - 1), np.minimum(b0[::8] + 127, M - 1),
             np.minimum(b0[::8] + 128, M - 1)]
    g = np.random.Generator(np.random.Philox(seed))
    return np.unique(np.concatenate(edges + [[M - 1], g.integers(0, M, n_random)]))


def test_c2_graph_full_size():
    cfg = datagen.CONFIGS["C2"]
    X, _ = datagen.config_inputs(cfg)
    gi, gd = run_graph(X, cfg.k)
    e2e_check(X, X, gi, gd, cfg.k, _sample_rows(cfg.N, 200, 1), True)


def test_c3_search_full_size():
    cfg = datagen.CONFIGS["C3"]
    Q, X = datagen.config_inputs(cfg)
    i, d = knn().search(cuda(Q), cuda(X), cfg.k)
    rows = _block_rows(cfg.M, 480, 2)
    assert len(rows) >= 1024
    e2e_check(Q, X, i.cpu().numpy(), d.cpu().numpy(), cfg.k, rows, False, min_pinned=0.5)


def test_headline_graph_full_size():
    cfg = datagen.HEADLINE
    X, _ = datagen.config_inputs(cfg)
    gi, gd = run_graph(X, cfg.k)
    rows = _block_rows(cfg.N, 480, 3)
    assert len(rows) >= 1024
    e2e_check(X, X, gi, gd, cfg.k, rows, True, min_pinned=0.5)


def test_c4_graph_large_k_full_size():
    cfg = datagen.CONFIGS["C4"]
    X, _ = datagen.config_inputs(cfg)
    gi, gd = run_graph(X, cfg.k)
    e2e_check(X, X, gi, gd, cfg.k, _sample_rows(cfg.N, 12, 4), True)


def test_c5_graph_single_gpu_full_size():
    cfg = datagen.CONFIGS["C5"]
    X, _ = datagen.config_inputs(cfg)
    gi, gd = run_graph(X, cfg.k)
    rows = _block_rows(cfg.N, 100, 5)
    assert len(rows) >= 1024
    e2e_check(X, X, gi, gd, cfg.k, rows, True)


def test_corpus_shards_plus_merge_equal_graph():
    # Par-2 on one GPU: column shards with global self exclusion and idx offsets, then
    # the k-way merge, must equal the unsharded graph bit-for-bit.
    X = datagen.points(5000, 48, "gauss", seed=7)
    k = 20
    ref_i, ref_d = run_graph(X, k)
    Xt = cuda(X)
    bounds = [0, 1250, 2500, 3750, 5000]
    parts = [knn().search_block(Xt, Xt[a:b].contiguous(), k, self_shift=-a, idx_offset=a)
             for a, b in zip(bounds[:-1], bounds[1:])]
    pi = torch.stack([p[0] for p in parts])
    pd = torch.stack([p[1] for p in parts])
    i, d = knn().merge(pd, pi, np.zeros(4, np.int64))
    assert np.array_equal(i.cpu().numpy(), ref_i)
    assert np.array_equal(d.cpu().numpy(), ref_d)


def test_query_shards_equal_graph():
    # Par-1 on one GPU: row blocks with self_shift = row offset
    X = datagen.points(3000, 40, "uniform", seed=8)
    k = 10
    ref_i, ref_d = run_graph(X, k)
    Xt = cuda(X)
    got = [knn().search_block(Xt[a:a + 1000].contiguous(), Xt, k, self_shift=a)
           for a in (0, 1000, 2000)]
    assert np.array_equal(torch.cat([g[0] for g in got]).cpu().numpy(), ref_i)
    assert np.array_equal(torch.cat([g[1] for g in got]).cpu().numpy(), ref_d)


def test_host_entry_point_equals_device():
    X = datagen.points(2500, 32, "clusters", seed=9)
    k = 12
    ref_i, ref_d = run_graph(X, k)
    hi, hd = knn().search_block_host(X, X, k, self_shift=0)
    assert np.array_equal(hi, ref_i) and np.array_equal(hd, ref_d)


@pytest.mark.parametrize("N,d,k,metric,dist", [(16384, 48, 16, 0, "uniform"), (32768, 100, 32, 1, "clusters"),
                                                (18432, 64, 8, 2, "gauss"), (20000, 32, 16, 0, "uniform")])
def test_host_pipelined_graph_equals_device(N, d, k, metric, dist):
    # knn_search_block_host's k-NNG overlaps the host->device copy with the hot path (chunks
    # of points, sample of every 8th point, column-major partition launches) when N is a
    # multiple of 2048 (20000 is not: the plain path); the lists equal the device call's
    X = datagen.points(N, d, dist, seed=N + d)
    pinned_x = torch.from_numpy(X).pin_memory().numpy()
    with exact_plan():  # (the pipelined scheme runs the 3-product partition)
        ref_i, ref_d = run_graph(X, k, metric)
        hi, hd = knn().search_block_host(pinned_x, pinned_x, k, metric=metric, self_shift=0)
        assert knn().last_plan() == 3
    assert np.array_equal(hi, ref_i) and np.array_equal(hd.view(np.uint32), ref_d.view(np.uint32))


def test_deterministic_and_small_row_blocks(monkeypatch):
    X = datagen.points(4000, 64, "uniform", seed=10)
    a = run_graph(X, 16)
    b = run_graph(X, 16)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_errors():
    k = knn()
    X = cuda(datagen.points(10, 4, "uniform", seed=11))
    with pytest.raises(k.KnnError) as e:
        k.graph(X, 10)
    assert e.value.status == 1
    with pytest.raises(k.KnnError) as e:
        k.graph(X, 3, metric=7)
    assert e.value.status == 1
    big = cuda(datagen.points(2000, 4, "uniform", seed=12))
    with pytest.raises(k.KnnError) as e:
        k.graph(big, 1025)
    assert e.value.status == 2
    bad = datagen.points(10, 4, "uniform", seed=13)
    bad[3, 1] = np.inf
    with pytest.raises(k.KnnError) as e:
        k.graph(cuda(bad), 3)
    assert e.value.status == 3


def test_simt_cross_check_path():
    # The FFMA path (KNN_GEMM=simt) in a fresh process must pass the same tolerance.
    code = (
        "import numpy as np, torch, oracle\n"
        "from oracle import checks\n"
        "from paper_1309_5478_b200 import knn, datagen\n"
        "Q = datagen.points(300, 100, 'gauss', seed=1); X = datagen.points(700, 100, 'gauss', seed=2)\n"
        "D = knn.distances(torch.from_numpy(Q).cuda(), torch.from_numpy(X).cuda()).cpu().numpy()\n"
        "r, bad = checks.check_distances(D, oracle.dist_rows(Q, X), oracle.sqnorms(Q), oracle.sqnorms(X))\n"
        "assert bad == 0, r\n")
    env = dict(os.environ, KNN_GEMM="simt")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call([sys.executable, "-c", code], env=env, cwd=root)


# ------------------------------------------------------------------ canonical orientation
def test_distances_canonically_symmetric():
    # With queries = corpus, every plan computes pair (i, j) with the lower index as the
    # first split operand, so D is bit-symmetric, and row blocks with a self shift
    # (query sharding) reproduce the same bits.
    kn = knn()
    X = datagen.points(1500, 100, "gauss", seed=40)
    Xt = cuda(X)
    D = kn.distances(Xt, Xt, self_shift=0).cpu().numpy()
    off = ~np.eye(1500, dtype=bool)
    assert np.array_equal(D.view(np.uint32)[off], D.T.view(np.uint32)[off])
    assert np.all(np.isinf(np.diag(D)))
    Db = kn.distances(Xt[300:1100].contiguous(), Xt, self_shift=300).cpu().numpy()
    assert np.array_equal(Db.view(np.uint32), D[300:1100].view(np.uint32))
    Dc = kn.distances(Xt, Xt[700:1400].contiguous(), self_shift=-700).cpu().numpy()
    assert np.array_equal(Dc.view(np.uint32), D[:, 700:1400].view(np.uint32))


@pytest.mark.parametrize("N,d,k,metric", [(3000, 64, 20, 0), (1000, 7, 100, 1), (4099, 256, 32, 0),
                                          (700, 33, 1024 - 1024 + 699, 0)])
def test_symmetric_graph_equals_unsymmetric(N, d, k, metric):
    # knn_graph multiplies only the upper triangle (transpose reuse); the
    # general block path (different pointers -> no symmetry) must give the same bits
    kn = knn()
    X = datagen.points(N, d, "clusters", seed=N + d)
    Xt = cuda(X)
    gi, gd = kn.graph(Xt, k, metric=metric)
    ri, rd = kn.search_block(Xt, Xt.clone(), k, metric=metric, self_shift=0)
    assert torch.equal(gi, ri)
    assert torch.equal(gd.view(torch.int32), rd.view(torch.int32))


# ------------------------------------------------------------------ pivot plan ---------
@pytest.fixture
def materialised_plan():
    kn = knn()
    kn.set_plan(kn.PLAN_MATERIALISED)
    yield kn
    kn.set_plan(kn.PLAN_AUTO)


@pytest.mark.parametrize("N,d,k,metric,dist", [(20000, 64, 32, 0, "uniform"), (17000, 128, 8, 1, "clusters"),
                                               (16384, 3, 1, 0, "gauss"), (16384, 24, 32, 0, "grid")])
def test_pivot_graph_equals_materialised(N, d, k, metric, dist):
    # grid: integer coordinates, many tied distances at the k-th (the candidate select's
    # tie handling) yet few enough candidates to stay on the pivot plan
    kn = knn()
    X = cuda(datagen.points(N, d, dist, seed=N + d + k))
    with exact_plan():
        gi, gd = kn.graph(X, k, metric=metric)
        assert kn.last_plan() == 3, kn.last_plan()
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.graph(X, k, metric=metric)
        assert kn.last_plan() != 3
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri)
    assert torch.equal(gd.view(torch.int32), rd.view(torch.int32))


def test_pivot_search_blocks_equal_materialised():
    kn = knn()
    X = cuda(datagen.points(20000, 48, "gauss", seed=51))
    Q = cuda(datagen.points(3000, 48, "gauss", seed=52))
    with exact_plan():
        gi, gd = kn.search_block(Q, X, 20)
        assert kn.last_plan() == 4
        ai, ad = kn.search_block(X[5000:9000].contiguous(), X, 16, self_shift=5000)
        assert kn.last_plan() == 4
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.search_block(Q, X, 20)
        bi, bd = kn.search_block(X[5000:9000].contiguous(), X, 16, self_shift=5000)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri) and torch.equal(gd, rd)
    assert torch.equal(ai, bi) and torch.equal(ad, bd)


def test_pivot_overflow_falls_back_exactly():
    # integer grid in d=4: enormous numbers of tied distances overflow the candidate
    # buffers; the call is redone on the full matrix and stays exact (E2E-3)
    X = datagen.points(16384, 4, "grid", seed=53)
    gi, gd = run_graph(X, 32)
    rows = np.arange(0, 16384, 257)
    ref = oracle.knn(X, X, 32, rows=rows, graph=True)
    assert np.array_equal(gi[rows], ref["idx32"])
    assert np.array_equal(gd[rows], ref["dist32"])


def test_pivot_certificate_failure_falls_back_exactly():
    # a sample margin far below the error bound gives pivots under the k-th distance for
    # many rows; the candidate count certificate (cnt >= k) catches them and the call is
    # redone on the full matrix: the result is the materialised plan's, bit for bit
    #
    code = (
        "import torch\n"
        "from paper_1309_5478_b200 import knn, datagen\n"
        "X = torch.from_numpy(datagen.points(16384, 64, 'uniform', seed=54)).cuda()\n"
        "gi, gd = knn.graph(X, 16)\n"
        "assert knn.last_plan() != 3, knn.last_plan()\n"
        "knn.set_plan(knn.PLAN_MATERIALISED)\n"
        "ri, rd = knn.graph(X, 16)\n"
        "assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))\n")
    env = dict(os.environ, KNN_PIVOT_MARGIN="-0.02")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call([sys.executable, "-c", code], env=env, cwd=root)


def test_pivot_large_sample_multi_slab():
    # a sample of N/2 points gives > 256 chunk minima per row: the pivot kernel's
    # multi-slab path (per-lane best-8 folds across slabs) must still give a valid pivot
    code = (
        "import torch\n"
        "from paper_1309_5478_b200 import knn, datagen\n"
        "X = torch.from_numpy(datagen.points(20000, 40, 'clusters', seed=55)).cuda()\n"
        "gi, gd = knn.graph(X, 24)\n"
        "assert knn.last_plan() == 3, knn.last_plan()\n"
        "knn.set_plan(knn.PLAN_MATERIALISED)\n"
        "ri, rd = knn.graph(X, 24)\n"
        "assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))\n")
    env = dict(os.environ, KNN_PIVOT_DIV="2", KNN_PIVOT1="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call([sys.executable, "-c", code], env=env, cwd=root)


# ------------------------------------------------------- quantile pivot plan (k > 32) ---
@pytest.mark.parametrize("N,d,k,metric,dist", [(20000, 48, 33, 0, "gauss"), (16384, 64, 128, 1, "uniform"),
                                               (24000, 32, 512, 0, "clusters"), (32768, 40, 1024, 2, "gauss"),
                                               (16500, 20, 100, 0, "grid")])
def test_quantile_pivot_graph_equals_materialised(N, d, k, metric, dist):
    """k > 32: the pivot is a bucketed order statistic of a single-product sample
    (DESIGN.md §6.5); the candidate select is exact, so the graph equals the materialised
    plan bit for bit (grid: massive ties; the lists may overflow and fall back)."""
    kn = knn()
    X = cuda(datagen.points(N, d, dist, seed=N + d + k))
    gi, gd = kn.graph(X, k, metric=metric)
    plan = kn.last_plan()
    assert plan == 3 or dist == "grid", plan
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.graph(X, k, metric=metric)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri)
    assert torch.equal(gd.view(torch.int32), rd.view(torch.int32))


@pytest.mark.parametrize("dup", [1, 40, 90])
def test_quantile_candidate_select_warp_and_cta_forms(dup):
    """k > 32 candidate select: the warp-per-row bucket finish hands crowded rows (many
    equal keys: every point repeated `dup` times) to the CTA kernel through a row list;
    both forms and the materialised plan agree bit for bit."""
    base = datagen.points(20000 // dup, 32, "gauss", seed=65 + dup)
    X = np.ascontiguousarray(np.repeat(base, dup, axis=0)[:20000])
    X = X[np.random.Generator(np.random.Philox(dup)).permutation(len(X))]
    code = (
        "import sys, numpy as np, torch\n"
        "from paper_1309_5478_b200 import knn\n"
        "X = torch.from_numpy(np.load(sys.argv[1])).cuda()\n"
        "gi, gd = knn.graph(X, 120)\n"
        "np.save(sys.argv[2], np.stack([gi.cpu().numpy(), gd.view(torch.int32).cpu().numpy()]))\n"
        "print(knn.last_plan())\n")
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as tmp:
        xin = os.path.join(tmp, "x.npy")
        np.save(xin, X)
        outs, plans = [], []
        for env_extra in ({}, {"KNN_CANDSEL_CTA": "1"}):
            out = os.path.join(tmp, "o%d.npy" % len(outs))
            r = subprocess.run([sys.executable, "-c", code, xin, out], check=True, cwd=root, timeout=300,
                               env=dict(os.environ, **env_extra), capture_output=True, text=True)
            plans.append(int(r.stdout.split()[-1]))
            outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
    kn = knn()
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.graph(cuda(X), 120)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert np.array_equal(outs[0][0], ri.cpu().numpy())
    assert np.array_equal(outs[0][1], rd.view(torch.int32).cpu().numpy())
    if dup == 1:
        assert plans == [3, 3], plans


def test_quantile_pivot_search_and_shifted_blocks():
    kn = knn()
    X = cuda(datagen.points(40000, 48, "gauss", seed=61))
    Q = cuda(datagen.points(3000, 48, "gauss", seed=62))
    gi, gd = kn.search_block(Q, X, 200)
    assert kn.last_plan() == 4
    ai, ad = kn.search_block(X[5000:9000].contiguous(), X, 64, self_shift=5000, idx_offset=7)
    assert kn.last_plan() == 4
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.search_block(Q, X, 200)
        bi, bd = kn.search_block(X[5000:9000].contiguous(), X, 64, self_shift=5000, idx_offset=7)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri) and torch.equal(gd, rd)
    assert torch.equal(ai, bi) and torch.equal(ad, bd)


def test_quantile_pivot_e2e_vs_oracle():
    X = datagen.points(20000, 64, "uniform", seed=63)
    k = 300
    gi, gd = run_graph(X, k)
    rows = np.arange(0, 20000, 311)
    D64 = oracle.dist_rows(X, X, rows=rows)
    n = oracle.sqnorms(X)
    res = checks.check_rows(gi[rows], gd[rows], D64, n[rows], n, rows, k, graph=True)
    assert res["failures"] == [], res["failures"][:3]


def test_quantile_pivot_certificate_failure_falls_back_exactly():
    code = (
        "import torch\n"
        "from paper_1309_5478_b200 import knn, datagen\n"
        "X = torch.from_numpy(datagen.points(16384, 64, 'uniform', seed=64)).cuda()\n"
        "gi, gd = knn.graph(X, 100)\n"
        "assert knn.last_plan() != 3, knn.last_plan()\n"
        "knn.set_plan(knn.PLAN_MATERIALISED)\n"
        "ri, rd = knn.graph(X, 100)\n"
        "assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))\n")
    env = dict(os.environ, KNN_PIVOT_MARGIN="-0.05")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=root, timeout=300)


@pytest.mark.parametrize("k", [16, 100])
def test_pivot_plans_on_ordered_data(k):
    """Points sorted along a coordinate (an ordered dataset): the pivot sample is a
    permuted column subset (prep.cu gather_sample), so the plan does not fall back to the
    full matrix, and the graph equals the materialised plan's."""
    kn = knn()
    X = datagen.points(32768, 32, "clusters", seed=71)
    X = np.ascontiguousarray(X[np.argsort(X[:, 0] + 1000 * np.round(X[:, 1]))])
    Xt = cuda(X)
    with exact_plan():
        gi, gd = kn.graph(Xt, k)
        assert kn.last_plan() == 3, kn.last_plan()
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.graph(Xt, k)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))


@pytest.mark.parametrize("k", [16, 80])
def test_pivot_sample_row_blocks(k):
    """The pivot plans' sample pass in several row blocks (a tiny KNN_D_BUDGET, as at very
    large N) gives the same graph as one block."""
    code = (
        "import torch\n"
        "from paper_1309_5478_b200 import knn, datagen\n"
        f"X = torch.from_numpy(datagen.points(20000, 32, 'gauss', seed=81)).cuda()\n"
        f"gi, gd = knn.graph(X, {k})\n"
        "assert knn.last_plan() == 3, knn.last_plan()\n"
        "torch.save((gi.cpu(), gd.cpu()), 'gpurun_out/_blk.pt')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root, timeout=300,
                   env=dict(os.environ, KNN_D_BUDGET_MB="1", KNN_PIVOT1="0"))  # 1 MiB: many sample row blocks
    bi, bd = torch.load(os.path.join(root, "gpurun_out", "_blk.pt"))
    X = cuda(datagen.points(20000, 32, "gauss", seed=81))
    with exact_plan():
        gi, gd = knn().graph(X, k)
    assert torch.equal(gi.cpu(), bi) and torch.equal(gd.cpu().view(torch.int32), bd.view(torch.int32))


def test_c_example_runs(tmp_path):
    """The plain-C example (examples/knn_demo.c) runs the k-NNG through the C ABI."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "knn_demo"
    libdir = os.path.join(root, "paper_1309_5478_b200")
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(root, "examples", "knn_demo.c"), "-L", libdir, "-lknn",
                           "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", str(exe)])
    out = subprocess.run([str(exe), "20000", "32", "8"], capture_output=True, text=True, timeout=120,
                         env=dict(os.environ, LD_LIBRARY_PATH=libdir + ":" + os.environ.get("LD_LIBRARY_PATH", "")))
    assert out.returncode == 0, out.stderr
    assert "point 0:" in out.stdout and "host-buffer API" in out.stdout
    # the sharded k-NNG through a one-rank NCCL communicator, from C (NCCL dlopen'ed)
    assert "sharded (backend 1, 1 rank)" in out.stdout, out.stdout


# ------------------------- single-product partition + re-evaluation (opt-in, KNN_PIVOT1) ---
_PIVOT1_CODE = """
import sys, numpy as np, torch
from paper_1309_5478_b200 import knn, datagen
N, d, k, metric, dist, nq = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], int(sys.argv[6])
X = torch.from_numpy(datagen.points(N, d, dist, seed=N + d)).cuda()
if nq:
    Q = torch.from_numpy(datagen.points(nq, d, dist, seed=N + d + 1)).cuda()
    gi, gd = knn.search_block(Q, X, k, metric=metric)
else:
    gi, gd = knn.graph(X, k, metric=metric)
np.save(sys.argv[7], np.stack([gi.cpu().numpy().astype(np.float64), gd.cpu().numpy().astype(np.float64)]))
print(knn.last_plan(), knn.last_candidates())
"""


@pytest.mark.parametrize("N,d,k,metric,dist,nq", [(65536, 256, 32, 0, "uniform", 0), (20000, 48, 10, 0, "gauss", 0),
                                                  (32768, 64, 16, 1, "uniform", 0), (40000, 36, 20, 1, "gauss", 3000),
                                                  (24576, 30, 7, 0, "clusters", 0)])
def test_pivot1_single_product_partition_vs_oracle(N, d, k, metric, dist, nq, tmp_path):
    """KNN_PIVOT1=1: the partition from the single hi.hi product keeps every
    element whose lower bound reaches the pivot; the survivors near the k-th are re-evaluated
    in fp32 from the inputs.  Checked against the oracle on sampled rows, and the values
    against the oracle's fp64 distances of the returned pairs (relative error <= (d/32 + 8)
    2^-24, tighter than the split GEMM's)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "r.npy")
    r = subprocess.run([sys.executable, "-c", _PIVOT1_CODE, str(N), str(d), str(k), str(metric), dist, str(nq), out],
                       check=True, cwd=root, timeout=600, env=dict(os.environ, KNN_PIVOT1="1"),
                       capture_output=True, text=True)
    plan = int(r.stdout.split()[0])
    assert plan in (5, 6), plan  # clusters (wide bounds): windowed re-evaluation, no fallback
    res = np.load(out)
    gi, gd = res[0].astype(np.int64), res[1].astype(np.float32)
    X = datagen.points(N, d, dist, seed=N + d)
    Q = datagen.points(nq, d, dist, seed=N + d + 1) if nq else X
    M = len(Q)
    rows = np.arange(0, M, max(1, M // 61))
    D64 = oracle.dist_rows(Q, X, rows=rows)
    res_chk = checks.check_rows(gi[rows], gd[rows], D64, oracle.sqnorms(Q)[rows], oracle.sqnorms(X), rows, k,
                                metric=metric, graph=not nq)
    assert res_chk["failures"] == [], res_chk["failures"][:3]
    ex = np.take_along_axis(D64, gi[rows], axis=1)
    if metric == 1:
        ex = np.sqrt(ex)
    if plan in (5, 6):  # re-evaluated values: the fp32 sum of squared differences
        bound = ((d + 31) // 32 + 8) * 2.0 ** -24 * (0.5 if metric == 1 else 1.0) + 2.0 ** -24
        assert np.all(np.abs(gd[rows] - ex) <= bound * ex + 1e-30)


@pytest.mark.parametrize("metric", [0, 1])
def test_pivot_plan_zero_vectors_and_duplicates(metric):
    """Zero-norm points (the single-product error bound vanishes, pivot = an exact value) and
    exact duplicates: the partition keeps u <= pivot (thr = nextup(pivot), strict test), so
    the pivot plan matches the materialised plan bit for bit."""
    kn = knn()
    X = datagen.points(20000, 24, "gauss", seed=91)
    X[::3] = 0.0
    X[1::7] = X[2::7][: len(X[1::7])] if len(X[2::7]) >= len(X[1::7]) else X[1::7]
    Xt = cuda(np.ascontiguousarray(X))
    with exact_plan():
        gi, gd = kn.graph(Xt, 16, metric=metric)
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.graph(Xt, 16, metric=metric)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri)
    assert torch.equal(gd.view(torch.int32), rd.view(torch.int32))


_PIVOT1_BLOCK_CODE = """
import sys, numpy as np, torch
from paper_1309_5478_b200 import knn, datagen
X = torch.from_numpy(datagen.points(20000, 40, "gauss", seed=95)).cuda()
gi, gd = knn.search_block(X[5000:9000].contiguous(), X, 16, metric=int(sys.argv[2]), self_shift=5000, idx_offset=7)
assert knn.last_plan() == 6, knn.last_plan()
np.save(sys.argv[1], np.stack([gi.cpu().numpy().astype(np.float64), gd.cpu().numpy().astype(np.float64)]))
"""


@pytest.mark.parametrize("metric", [0, 1])
def test_pivot1_shifted_block_vs_oracle(metric, tmp_path):
    """KNN_PIVOT1=1 on a row block of the k-NNG (self pair j = i + 5000 excluded, indices
    offset by 7): the re-evaluated lists are the oracle's nearest neighbours."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "b.npy")
    subprocess.run([sys.executable, "-c", _PIVOT1_BLOCK_CODE, out, str(metric)], check=True, cwd=root, timeout=600,
                   env=dict(os.environ, KNN_PIVOT1="1"))
    res = np.load(out)
    gi, gd = res[0].astype(np.int64) - 7, res[1].astype(np.float32)
    X = datagen.points(20000, 40, "gauss", seed=95)
    rows = np.arange(5000, 9000, 97)
    D64 = oracle.dist_rows(X, X, rows=rows)
    n = oracle.sqnorms(X)
    chk = checks.check_rows(gi[rows - 5000], gd[rows - 5000], D64, n[rows], n, rows, 16, metric=metric, graph=True)
    assert chk["failures"] == [], chk["failures"][:3]


# ----------------------------------------------- automatic single-product partition ----
@pytest.mark.parametrize("N,d,k,metric,dist", [(20000, 64, 32, 0, "uniform"), (18000, 100, 16, 1, "gauss"),
                                               (16384, 256, 1, 0, "uniform"), (24576, 32, 32, 0, "gauss")])
def test_auto_plan_single_product_vs_oracle(N, d, k, metric, dist):
    """The automatic plan on data near the origin: the device chooses the single-product
    partition (plan 5) and the re-evaluated lists pass the oracle's E2E checks on >= 300
    rows, including every 256-row block's first and last row."""
    kn = knn()
    X = datagen.points(N, d, dist, seed=N + 3 * d + k)
    gi, gd = kn.graph(cuda(X), k, metric=metric)
    assert kn.last_plan() == 5, kn.last_plan()
    e2e_check(X, X, gi.cpu().numpy(), gd.cpu().numpy(), k, _block_rows(N, 100, N + k), True, metric=metric)


def test_auto_plan_search_single_product_vs_oracle():
    kn = knn()
    X = datagen.points(20000, 48, "uniform", seed=61)
    Q = datagen.points(2000, 48, "uniform", seed=62)
    gi, gd = kn.search_block(cuda(Q), cuda(X), 24)
    assert kn.last_plan() == 6, kn.last_plan()
    e2e_check(Q, X, gi.cpu().numpy(), gd.cpu().numpy(), 24, np.arange(0, 2000, 7), False)


def test_auto_plan_far_from_origin_keeps_exact_partition():
    """C2 (Gaussian clusters away from the origin): the single-product bound scales with the
    norms, so the device keeps the FP32-accurate 3-product partition (plan 3), bit-identical
    to the materialised plan."""
    kn = knn()
    cfg = datagen.CONFIGS["C2"]
    X, _ = datagen.config_inputs(cfg)
    Xt = cuda(X)
    gi, gd = kn.graph(Xt, cfg.k)
    assert kn.last_plan() == 3, kn.last_plan()
    kn.set_plan(kn.PLAN_MATERIALISED)
    try:
        ri, rd = kn.graph(Xt, cfg.k)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))


def test_auto_plan_ties_and_zero_vectors_vs_oracle():
    """Duplicates and zero vectors under the automatic plan (the bound vanishes at zero norm;
    ties at the k-th are resolved by index in the re-evaluated values)."""
    kn = knn()
    X = datagen.points(20000, 24, "gauss", seed=64)
    X[::97] = 0.0                      # 207 zero vectors: 206 ties at distance 0 each
    X[1::7] = X[2::7][: len(X[1::7])]  # exact duplicates
    X = np.ascontiguousarray(X)
    gi, gd = kn.graph(cuda(X), 16)
    assert kn.last_plan() == 5, kn.last_plan()
    e2e_check(X, X, gi.cpu().numpy(), gd.cpu().numpy(), 16, np.arange(0, 20000, 97), True)


@pytest.mark.parametrize("N,d,k,metric", [(16384, 48, 16, 0), (32768, 100, 32, 1)])
def test_host_pipelined_auto_plan_equals_device(N, d, k, metric):
    """knn_search_block_host's pipelined k-NNG under the automatic plan: the device picks the
    single-product partition from the first chunk's pivots; the re-evaluated values are the
    same fp32 sums as the device call's, so the lists are identical, and they pass the
    oracle's E2E checks."""
    X = datagen.points(N, d, "uniform", seed=N + 7 * d)
    ref_i, ref_d = run_graph(X, k, metric)
    assert knn().last_plan() == 5, knn().last_plan()
    pinned_x = torch.from_numpy(X).pin_memory().numpy()
    hi, hd = knn().search_block_host(pinned_x, pinned_x, k, metric=metric, self_shift=0)
    assert knn().last_plan() == 5, knn().last_plan()
    assert np.array_equal(hi, ref_i) and np.array_equal(hd.view(np.uint32), ref_d.view(np.uint32))
    e2e_check(X, X, hi, hd, k, np.arange(0, N, 131), True, metric=metric)


@pytest.mark.parametrize("metric", [0, 1])
def test_per_point_bound_mixed_residuals(metric):
    """Per-point single-product bound (reading R21): every 8th point is
    fp16-exact after prep's power-of-two scaling (split residual e = 0) and the others are
    random (e up to ~2^-12).  The host-pipelined call takes t from its sample (exactly those
    fp16-exact points: t at its floor 2^-13), the device call from every point; both bounds
    are valid for any t, so both calls keep the single-product partition without a redo and
    return the device call's lists, which pass the oracle's E2E checks."""
    N, d, k = 16384, 40, 12
    X = datagen.points(N, d, "gauss", seed=4242)
    X[::8] = X[::8].astype(np.float16).astype(np.float32)
    X = np.ascontiguousarray(X)
    kn = knn()
    gi, gd = kn.graph(cuda(X), k, metric=metric)
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    assert kn.last_plan() == 5, kn.last_plan()
    pinned_x = torch.from_numpy(X).pin_memory().numpy()
    hi, hd = kn.search_block_host(pinned_x, pinned_x, k, metric=metric, self_shift=0)
    assert kn.last_plan() == 5, kn.last_plan()  # (a redo would report the materialised plan)
    assert np.array_equal(hi, gi) and np.array_equal(hd.view(np.uint32), gd.view(np.uint32))
    rows = np.concatenate([np.arange(0, N, 97), np.arange(0, N, 8)[:64]])
    e2e_check(X, X, gi, gd, k, np.unique(rows), True, metric=metric)


_LISTS_CODE = """
import sys, numpy as np, torch
from paper_1309_5478_b200 import knn, datagen
N, d, k, dist, mixed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
X = datagen.points(N, d, dist, seed=N + 3 * d)
if mixed:
    X[::8] = X[::8].astype(np.float16).astype(np.float32)
Xt = torch.from_numpy(np.ascontiguousarray(X)).cuda()
npad = -(-N // 256) * 256
thr = torch.full((npad,), float("nan"), device="cuda")
knn.graph_pivots(Xt, k, 0, N, thr)
cap = knn.graph_list_cap(k)
cnt = torch.zeros(N, dtype=torch.int32, device="cuda")
ce = torch.empty((N, cap), dtype=torch.int64, device="cuda")
knn.graph_partition(Xt, k, thr, 0, knn.graph_units(N), cnt, ce)
torch.cuda.synchronize()
np.save(sys.argv[6], X)
np.save(sys.argv[7], thr.cpu().numpy())
np.save(sys.argv[8], cnt.cpu().numpy())
np.save(sys.argv[9], ce.cpu().numpy())
"""


@pytest.mark.parametrize("N,d,k,dist,mixed", [(16384, 48, 16, "gauss", 0), (20000, 30, 10, "clusters", 0),
                                              (16384, 40, 32, "uniform", 1)])
def test_single_product_lists_are_sound(N, d, k, dist, mixed, tmp_path):
    """The single-product partition (KNN_PIVOT1=1, readings R20/R21) read
    straight from its lists (knn_graph_pivots + knn_graph_partition): every listed key L is a
    lower bound of the exact distance of its pair (the oracle's fp64 value of the fp32
    inputs), and every pair whose exact distance is at or below the row's pivot is listed
    — the two properties the plan's exactness rests on — on data near the origin, far from
    it (clusters: wide bounds) and with fp16-exact points mixed in (per-point residuals 0)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    paths = [str(tmp_path / f) for f in ("x.npy", "thr.npy", "cnt.npy", "ce.npy")]
    subprocess.run([sys.executable, "-c", _LISTS_CODE, str(N), str(d), str(k), dist, str(mixed)] + paths,
                   check=True, cwd=root, timeout=600, env=dict(os.environ, KNN_PIVOT1="1"))
    X, thr, cnt, ce = (np.load(p) for p in paths)
    cap = ce.shape[1]
    assert np.all(cnt[:N] <= cap), "list overflow"
    rows = np.unique(np.concatenate([[0, N - 1], np.arange(0, N, N // 61)]))
    D64 = oracle.dist_rows(X, X, rows=rows)
    for r, i in enumerate(rows):
        n = int(cnt[i])
        ent = ce[i, :n].view(np.uint64)
        cols = (ent & np.uint64(0xFFFFFFFF)).astype(np.int64)
        keys = (ent >> np.uint64(32)).astype(np.uint32)
        # the key is the IEEE bits of L >= +0 with the sign bit set (include/knn.h)
        L = (keys & np.uint32(0x7FFFFFFF)).view(np.float32).astype(np.float64)
        assert len(np.unique(cols)) == n and not np.any(cols == i), i
        assert np.all(L <= D64[r, cols]), (i, float(np.max(L - D64[r, cols])))
        # thr holds nextup(pivot): the partition keeps L < thr
        pivot = float(np.nextafter(np.float32(thr[i]), np.float32(-np.inf)))
        need = np.flatnonzero(D64[r] <= pivot)
        need = need[need != i]
        assert np.isin(need, cols).all(), (i, len(need), n)


@pytest.mark.parametrize("N,d,k,metric,dist,seed", [(44677, 3, 2, 0, "uniform", 1071), (36383, 3, 2, 0, "gauss", 1173),
                                                    (34516, 7, 5, 3, "grid", 1194), (30639, 257, 2, 3, "gauss", 1043)])
def test_pivot_plan_rows_with_exactly_k_candidates(N, d, k, metric, dist, seed):
    """Regression (found by scripts/fuzz_plans.py): with the per-point bound's tighter pivots
    some rows keep exactly k candidates, and the exact candidate select read that short list
    with the wrong stride (garbage first neighbour).  The automatic plan must equal the
    materialised plan bit for bit (plans 3 / 4 here: the FP32-accurate partition)."""
    kn = knn()
    X = cuda(datagen.points(N, d, dist, seed=seed))
    gi, gd = kn.graph(X, k, metric=metric)
    plan = kn.last_plan()
    try:
        kn.set_plan(kn.PLAN_MATERIALISED)
        ri, rd = kn.graph(X, k, metric=metric)
    finally:
        kn.set_plan(kn.PLAN_AUTO)
    if plan in (3, 4):
        assert torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))
    assert int(gi.min()) >= 0 and not torch.isnan(gd).any()

"""Pins for the CPU oracle (oracle/knn_oracle.cpp) — none of these call the CUDA path.

Each test pins the oracle to something other than itself: values the paper / SPEC print
for worked examples (tests/golden/*.json, each with its citation), exact integer
arithmetic, closed forms evaluated a different way, invariants (symmetry, zero
diagonal), and independent brute-force selectors on tiny inputs.  Chosen so that a
dropped term, a sign error, an index slip or a transposed operand fails at least one.
"""
import heapq
import math

import numpy as np
import pytest

import oracle
from oracle import checks
from paper_1309_5478_b200 import datagen
from conftest import golden


# ---------------------------------------------------------------- distances ----------
def test_golden_distances():
    g = golden("dist_pairs.json")
    for case in g["cases"]:
        q = np.array([case["q"]], np.float32)
        c = np.array([case["c"]], np.float32)
        assert oracle.dist_rows(q, c, metric=oracle.L2SQ)[0, 0] == case["d2"]
        assert oracle.dist_rows(q, c, metric=oracle.L2)[0, 0] == pytest.approx(case["dE"], rel=1e-15)


def test_integer_grid_exact():
    # Exact big-integer arithmetic (Python ints) on grid data: any dropped term, sign
    # slip or transposed operand changes at least one entry.
    X = datagen.points(40, 19, "grid", seed=7)
    Q = datagen.points(13, 19, "grid", seed=8)
    D = oracle.dist_rows(Q, X)
    Xi = X.astype(int).tolist()
    Qi = Q.astype(int).tolist()
    for a in range(13):
        for b in range(40):
            exact = sum((Qi[a][t] - Xi[b][t]) ** 2 for t in range(19))
            assert D[a, b] == exact


def test_symmetry_and_zero_diagonal():
    X = datagen.points(64, 33, "gauss", seed=11)
    D = oracle.dist_rows(X, X)
    assert np.array_equal(D, D.T)  # direct form: bit-exact symmetry
    assert np.all(np.diag(D) == 0.0)
    assert np.all(D >= 0.0)


def test_expansion_closed_form():
    # PAPER.md:80-82 writes d^2 = ||x||^2 + ||y||^2 - 2 x.y; evaluate that expansion
    # independently in extended precision and compare with the oracle's direct form.
    X = datagen.points(50, 64, "uniform", seed=12)
    Q = datagen.points(20, 64, "gauss", seed=13)
    D = oracle.dist_rows(Q, X)
    Ql, Xl = Q.astype(np.longdouble), X.astype(np.longdouble)
    E = (Ql * Ql).sum(1)[:, None] + (Xl * Xl).sum(1)[None, :] - 2 * Ql @ Xl.T
    scale = (Ql * Ql).sum(1)[:, None] + (Xl * Xl).sum(1)[None, :]
    assert np.max(np.abs(D - E.astype(np.float64)) / scale.astype(np.float64)) < 1e-12


def test_l2_is_sqrt_of_l2sq():
    X = datagen.points(30, 8, "gauss", seed=14)
    D2 = oracle.dist_rows(X, X, metric=oracle.L2SQ)
    D1 = oracle.dist_rows(X, X, metric=oracle.L2)
    assert np.array_equal(D1, np.sqrt(D2))


def test_sqnorms():
    Xg = datagen.points(17, 1000, "grid", seed=15)
    exact = [sum(int(v) ** 2 for v in row) for row in Xg.astype(int)]
    assert oracle.sqnorms(Xg).tolist() == [float(e) for e in exact]
    X = datagen.points(9, 300, "gauss", seed=16)
    ref = [math.fsum(float(v) * float(v) for v in row) for row in X]
    assert np.allclose(oracle.sqnorms(X), ref, rtol=1e-14, atol=0)
    # norm of the distance to the origin is the squared norm (PAPER.md:80 with y = 0)
    Z = np.zeros((1, 300), np.float32)
    assert np.allclose(oracle.dist_rows(X, Z)[:, 0], ref, rtol=1e-14)


# ---------------------------------------------------------------- selection ----------
def test_golden_select_rows():
    for case in golden("select_rows.json")["cases"]:
        D = np.array([case["row"]], np.float32)
        idx, dist = oracle.select_f32(D, case["k"])
        assert idx[0].tolist() == case["idx"]
        assert dist[0].tolist() == case["dist"]


def _repeated_min(row, k):
    # O(N k) independent selector: k passes, each taking the smallest remaining
    # (value, index) pair; pure Python.
    taken = set()
    out = []
    for _ in range(k):
        best = None
        for j, v in enumerate(row):
            if j in taken:
                continue
            if best is None or v < row[best] or (v == row[best] and j < best):
                best = j
        taken.add(best)
        out.append(best)
    return out


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_select_three_selectors_agree(seed):
    g = np.random.Generator(np.random.Philox(seed))
    for N in (1, 2, 7, 31, 64, 200, 256):
        # duplicate-heavy rows so the index tie-break matters
        D = (g.integers(0, max(2, N // 3), size=(3, N)) / 7.0).astype(np.float32)
        for k in sorted({1, min(3, N), max(1, N // 2), N}):
            idx, dist = oracle.select_f32(D, k)
            for r in range(3):
                row = D[r].tolist()
                a = np.lexsort((np.arange(N), D[r]))[:k].tolist()
                b = [j for _, j in heapq.nsmallest(k, [(v, j) for j, v in enumerate(row)])]
                c = _repeated_min(row, k)
                assert idx[r].tolist() == a == b == c
                assert dist[r].tolist() == [row[j] for j in a]
                # the k-th key is the k-th order statistic (nth_element analogue)
                assert dist[r, k - 1] == np.partition(D[r], k - 1)[k - 1]


def test_select_special_values():
    row = np.array([[3.0, -0.0, np.nan, np.inf, 0.0, 1.0, np.inf, -np.inf, np.nan]], np.float32)
    idx, dist = oracle.select_f32(row, 9)
    # -inf, then -0 and +0 as equal keys (index order), 1, 3, +inf x2, NaN x2
    assert idx[0].tolist() == [7, 1, 4, 5, 0, 3, 6, 2, 8]
    assert np.signbit(dist[0, 1]) == False  # -0 canonicalised to +0
    assert np.isnan(dist[0, 7]) and np.isnan(dist[0, 8])


def test_select_full_row_is_sorted_row():
    D = datagen.keys(4, 500, "uniform", seed=5)
    idx, dist = oracle.select_f32(D, 500)
    for r in range(4):
        assert idx[r].tolist() == np.argsort(D[r], kind="stable").tolist()


# ---------------------------------------------------------------- k-NN / k-NNG ------
@pytest.mark.parametrize("name", ["graph_collinear.json", "graph_unit_square.json",
                                  "graph_two_points.json"])
def test_golden_graphs(name):
    g = golden(name)
    X = np.array(g["points"], np.float32)
    ref = oracle.knn(X, X, g["k"], graph=True)
    assert ref["idx64"].tolist() == g["idx"]
    assert ref["dist64"].tolist() == g["d2"]
    assert ref["idx32"].tolist() == g["idx"]
    if "k3_last_d2" in g:  # the diagonal corner arrives only at k=3
        ref3 = oracle.knn(X, X, 3, graph=True)
        assert ref3["dist64"][:, 2].tolist() == g["k3_last_d2"]


def test_graph_excludes_self_and_k_all():
    X = datagen.points(37, 5, "uniform", seed=21)
    ref = oracle.knn(X, X, 36, graph=True)
    for i in range(37):
        assert i not in ref["idx64"][i]
        assert sorted(ref["idx64"][i].tolist()) == [j for j in range(37) if j != i]
    # without graph mode and k=1 the query's own point is its nearest neighbour (d=0)
    ref1 = oracle.knn(X, X, 1, graph=False)
    assert ref1["idx64"][:, 0].tolist() == list(range(37))
    assert np.all(ref1["dist64"] == 0)


def test_knn_matches_bruteforce_python():
    Q = datagen.points(6, 4, "grid", seed=22)
    X = datagen.points(50, 4, "grid", seed=23)
    k = 9
    ref = oracle.knn(Q, X, k, graph=False)
    for a in range(6):
        exact = [(sum((int(Q[a, t]) - int(X[b, t])) ** 2 for t in range(4)), b) for b in range(50)]
        exact.sort()
        assert ref["idx64"][a].tolist() == [b for _, b in exact[:k]]
        assert ref["dist64"][a].tolist() == [float(v) for v, _ in exact[:k]]
        # on integer data R32 == R64 (all values exactly representable)
        assert ref["idx32"][a].tolist() == ref["idx64"][a].tolist()


def test_r32_is_select_of_rounded_row():
    X = datagen.points(300, 16, "clusters", seed=24)
    rows = np.array([0, 5, 299])
    ref = oracle.knn(X, X, 10, rows=rows, graph=True)
    D = oracle.dist_rows(X, X, rows=rows).astype(np.float32)
    for r, i in enumerate(rows):
        D[r, i] = np.inf  # self excluded by position
    idx, dist = oracle.select_f32(D, 10)
    assert np.array_equal(idx, ref["idx32"]) and np.array_equal(dist, ref["dist32"])


def test_knn_argument_errors():
    X = datagen.points(8, 3, "uniform", seed=25)
    with pytest.raises(ValueError):
        oracle.knn(X, X, 8, graph=True)  # k > N-1 in graph mode
    with pytest.raises(ValueError):
        oracle.knn(X, X, 9, graph=False)


# ---------------------------------------------------------------- merge -------------
def test_merge_equals_unsharded_select():
    D = datagen.keys(20, 1000, "dup256", seed=26)
    k = 16
    full_idx, full_dist = oracle.select_f32(D, k)
    bounds = [0, 130, 500, 501, 1000]
    parts_d, parts_i = [], []
    for a, b in zip(bounds[:-1], bounds[1:]):
        kk = min(k, b - a)
        pi, pd = oracle.select_f32(D[:, a:b], kk)
        if kk < k:  # pad short shards with +inf sentinels
            pi = np.concatenate([pi, np.zeros((20, k - kk), np.int32)], 1)
            pd = np.concatenate([pd, np.full((20, k - kk), np.inf, np.float32)], 1)
        parts_i.append(pi)
        parts_d.append(pd)
    idx, dist = oracle.merge(np.stack(parts_d), np.stack(parts_i), bounds[:-1])
    assert np.array_equal(idx, full_idx) and np.array_equal(dist, full_dist)


# ---------------------------------------------------------------- E2E checks --------
def test_checks_accept_oracle_and_reject_mistakes():
    X = datagen.points(200, 8, "uniform", seed=27)
    rows = np.arange(0, 200, 7)
    k = 5
    ref = oracle.knn(X, X, k, rows=rows, graph=True)
    D64 = oracle.dist_rows(X, X, rows=rows)
    n = oracle.sqnorms(X)
    res = checks.check_rows(ref["idx64"], ref["dist64"], D64, n[rows], n, rows, k, graph=True)
    assert res["failures"] == [] and res["n_pinned"] > 0
    # a swapped-in far neighbour must be caught
    bad_idx = ref["idx64"].copy()
    bad_dist = ref["dist64"].copy()
    far = int(np.argmax(D64[0]))
    bad_idx[0, k - 1], bad_dist[0, k - 1] = far, D64[0, far]
    res = checks.check_rows(bad_idx, bad_dist, D64, n[rows], n, rows, k, graph=True)
    assert any("row 0" in f for f in res["failures"])
    # a distance perturbed by 2x the tolerance must be caught
    bad_dist = ref["dist64"].copy()
    bad_dist[1, 0] += 2e-5 * (n[rows[1]] + n[ref["idx64"][1, 0]])
    res = checks.check_rows(ref["idx64"], bad_dist, D64, n[rows], n, rows, k, graph=True)
    assert any("tolerance" in f for f in res["failures"])


def test_pinned_flag_threshold():
    # Constructed 1-d rows: query at 0, corpus at distances^2 chosen so that the gap
    # between the k-th and (k+1)-th sits just above / just below the tolerance.
    k = 1
    for gap_factor, expect_pinned in ((2.2, True), (1.8, False)):
        a = 100.0
        tol_a = 1e-5 * a  # ||q||^2 = 0, ||c||^2 = d^2 for a 1-d point at sqrt(d^2)
        b = a + gap_factor * tol_a
        X = np.array([[0.0], [math.sqrt(a)], [math.sqrt(b)]], np.float32)
        D64 = oracle.dist_rows(X[:1], X)
        n = oracle.sqnorms(X)
        ref = oracle.knn(X[:1], X, 2, graph=False)
        # query row 0 vs corpus {1, 2}: drop self by passing graph=True on row 0
        ref = oracle.knn(X, X, k, rows=[0], graph=True)
        res = checks.check_rows(ref["idx64"], ref["dist64"], D64, n[:1], n, [0], k, graph=True)
        assert res["failures"] == []
        assert res["n_pinned"] == (1 if expect_pinned else 0)


# ---------------------------------------------------------- cosine / Pearson (NEXT-2) --
def test_golden_cosine_pearson():
    g = golden("cosine_pearson.json")
    for case in g["cases"]:
        q = np.array([case["q"]], np.float32)
        c = np.array([case["c"]], np.float32)
        key = oracle.dist_rows(q, c, metric=case["metric"])[0, 0]
        assert abs(key - case["key"]) <= case["abs"], case["what"]


def test_cosine_key_of_known_angles():
    # q, c on the unit circle at angles a, b: key = 1 - cos(a - b) (math library, not the
    # oracle's dot/norm arithmetic); scaling either vector by a positive factor is a no-op
    rng = np.random.default_rng(3)
    for _ in range(50):
        a, b = rng.uniform(-math.pi, math.pi, 2)
        sq, sc = rng.uniform(0.01, 100.0, 2)
        q = np.array([[sq * math.cos(a), sq * math.sin(a)]], np.float64)
        c = np.array([[sc * math.cos(b), sc * math.sin(b)]], np.float64)
        # the fp32 inputs are the rounded vectors: compare with their exact angle
        qf, cf = q.astype(np.float32), c.astype(np.float32)
        ang = math.atan2(float(qf[0, 1]), float(qf[0, 0])) - math.atan2(float(cf[0, 1]), float(cf[0, 0]))
        key = oracle.dist_rows(qf, cf, metric=oracle.COSINE)[0, 0]
        assert key == pytest.approx(1.0 - math.cos(ang), abs=1e-12)


def test_cosine_equals_half_squared_distance_of_unit_vectors():
    # ||q/|q| - c/|c| ||^2 = 2 (1 - cos): the cosine key against the (pinned) L2SQ oracle on
    # vectors normalised in numpy; and the k-NN lists agree (no ties in random data)
    Q = datagen.points(20, 33, "gauss", seed=11).astype(np.float64)
    X = datagen.points(300, 33, "gauss", seed=12).astype(np.float64)
    Qn = Q / np.linalg.norm(Q, axis=1, keepdims=True)
    Xn = X / np.linalg.norm(X, axis=1, keepdims=True)
    ref = ((Qn[:, None, :] - Xn[None, :, :]) ** 2).sum(-1) / 2
    key = oracle.dist_rows(Q.astype(np.float32), X.astype(np.float32), metric=oracle.COSINE)
    # the fp32 rounding of the inputs moves the key by ~1e-7
    assert np.max(np.abs(key - ref)) < 1e-6
    a = oracle.knn(Q.astype(np.float32), X.astype(np.float32), 10, metric=oracle.COSINE)["idx64"]
    b = np.argsort(ref, axis=1, kind="stable")[:, :10]
    assert np.array_equal(a, b)


def test_pearson_is_cosine_of_centred_vectors():
    # PAPER.md:71 "the Pearson distance coefficient is essentially the Cosine distance of
    # the centered data sets": centre in numpy (fp64), then the cosine key; plus affine
    # invariance y -> a*y + b (a > 0) and sign flip y -> -y giving 2 - key
    Q = datagen.points(15, 21, "uniform", seed=13).astype(np.float64) * 5 + 2
    X = datagen.points(200, 21, "uniform", seed=14).astype(np.float64) * 3 - 1
    Qf, Xf = Q.astype(np.float32), X.astype(np.float32)
    Qc = Qf.astype(np.float64) - Qf.astype(np.float64).mean(1, keepdims=True)
    Xc = Xf.astype(np.float64) - Xf.astype(np.float64).mean(1, keepdims=True)
    sim = (Qc @ Xc.T) / np.outer(np.linalg.norm(Qc, axis=1), np.linalg.norm(Xc, axis=1))
    key = oracle.dist_rows(Qf, Xf, metric=oracle.PEARSON)
    assert np.max(np.abs(key - (1 - sim))) < 1e-12
    # affine invariance on exactly representable transforms (x2 and +8 are exact in fp32 here)
    X2 = (Xf * 2 + 8).astype(np.float32)
    key2 = oracle.dist_rows(Qf, X2, metric=oracle.PEARSON)
    assert np.max(np.abs(key2 - key)) < 1e-6
    key3 = oracle.dist_rows(Qf, -Xf, metric=oracle.PEARSON)
    assert np.max(np.abs(key3 - (2 - key))) < 1e-12


def test_cosine_graph_semantics():
    # graph mode drops self by position; ties between parallel copies broken by index
    X = np.array([[1, 0], [2, 0], [0, 1], [1, 1], [-1, 0]], np.float32)
    r = oracle.knn(X, X, 3, metric=oracle.COSINE, graph=True)
    # row 0: (1,0) -> 1 is parallel (key 0), 3 at 45 deg, 2 at 90 deg
    assert r["idx64"][0].tolist() == [1, 3, 2]
    assert r["dist64"][0, 0] == pytest.approx(0.0, abs=1e-15)
    assert r["dist64"][0, 1] == pytest.approx(1 - math.sqrt(0.5), abs=1e-15)
    # row 4: (-1,0): 2 and 3 at 90/135 deg, 0 and 1 antiparallel (key 2)
    assert r["idx64"][4].tolist() == [2, 3, 0]


def test_checks_cosine_tolerance():
    X = datagen.points(150, 6, "gauss", seed=28)
    rows = np.arange(0, 150, 11)
    k = 4
    for metric in (oracle.COSINE, oracle.PEARSON):
        ref = oracle.knn(X, X, k, rows=rows, graph=True, metric=metric)
        D64 = oracle.dist_rows(X, X, rows=rows, metric=metric)
        n = oracle.sqnorms(X)
        res = checks.check_rows(ref["idx64"], ref["dist64"], D64, n[rows], n, rows, k, metric=metric, graph=True)
        assert res["failures"] == [] and res["n_pinned"] > 0
        bad = ref["dist64"].copy()
        bad[2, 1] += 2.5 * checks.COS_TOL
        res = checks.check_rows(ref["idx64"], bad, D64, n[rows], n, rows, k, metric=metric, graph=True)
        assert any("tolerance" in f for f in res["failures"])


# ---------------------------------------------------------------- check_distances ----
# oracle.checks.check_distances is the a-S3 parity gate (|D - D64| <= 1e-5 (||q||^2 +
# ||c||^2), BASELINE.json north_star).  Pinned here against hand arithmetic and
# independently computed tolerances: it must accept the exact values and values inside
# the band, and flag a single element pushed to 2x the tolerance, in every branch
# (L2SQ absolute error, the L2 sqrt band, the absolute cosine key tolerance).
def test_check_distances_hand_example():
    # q = (3, 4), c = (0, 0) and (3, 0): d^2 = 25 and 16, ||q||^2 = 25, ||c||^2 = 0 and 9
    # (SPEC.md:133's 3-4-5 example), so tol = 2.5e-4 and 3.4e-4.
    D64 = np.array([[25.0, 16.0]])
    qn, cn = np.array([25.0]), np.array([0.0, 9.0])
    assert checks.check_distances(D64, D64, qn, cn) == (0.0, 0)
    ratio, nbad = checks.check_distances(np.array([[25.0 + 5e-4, 16.0]]), D64, qn, cn)
    assert nbad == 1 and ratio == pytest.approx(2.0)
    ratio, nbad = checks.check_distances(np.array([[25.0 - 1.2e-4, 16.0 + 1.7e-4]]), D64, qn, cn)
    assert nbad == 0 and ratio == pytest.approx(0.5)
    # L2: d_E = 5 and 4; the band is sqrt(d^2 -+ tol) widened by one ulp
    E = np.array([[5.0, 4.0]])
    assert checks.check_distances(E, D64, qn, cn, metric=1)[1] == 0
    assert checks.check_distances(np.array([[math.sqrt(25 + 5e-4), 4.0]]), D64, qn, cn, metric=1)[1] == 1
    assert checks.check_distances(np.array([[5.0, math.sqrt(16 - 6.8e-4)]]), D64, qn, cn, metric=1)[1] == 1
    assert checks.check_distances(np.array([[math.sqrt(25 + 1e-4), math.sqrt(16 - 1e-4)]]),
                                  D64, qn, cn, metric=1)[1] == 0


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_check_distances_accepts_oracle_flags_perturbation(metric):
    X = datagen.points(70, 48, "gauss", seed=21)
    Q = datagen.points(30, 48, "uniform", seed=22)
    if metric == 2:
        D64 = oracle.dist_rows(Q, X, metric=2)
        tol = np.full(D64.shape, 1e-5)
        qn = np.ones(30)
        cn = np.ones(70)
    else:
        D64 = oracle.dist_rows(Q, X, metric=oracle.L2SQ)
        # norms by math.fsum of the fp64 squares (not the oracle's own norm routine)
        qn = np.array([math.fsum(float(v) ** 2 for v in row) for row in Q])
        cn = np.array([math.fsum(float(v) ** 2 for v in row) for row in X])
        tol = 1e-5 * (qn[:, None] + cn[None, :])
    base = np.sqrt(D64) if metric == 1 else D64.copy()
    assert checks.check_distances(base, D64, qn, cn, metric=metric)[1] == 0
    # whole matrix inside half the band (alternating signs): accepted
    sign = np.where((np.arange(D64.size).reshape(D64.shape) % 2) == 0, 1.0, -1.0)
    inside = np.maximum(D64 + 0.5 * tol * sign, 0.0)
    G = np.sqrt(inside) if metric == 1 else inside
    assert checks.check_distances(G, D64, qn, cn, metric=metric)[1] == 0
    # one element at +2 tol, one at -2 tol (where D64 > 2 tol): exactly two violations
    rng = np.random.default_rng(5)
    a = (int(rng.integers(30)), int(rng.integers(70)))
    b = (int(rng.integers(30)), int(rng.integers(70)))
    while b == a or D64[b] <= 2 * tol[b]:
        b = (int(rng.integers(30)), int(rng.integers(70)))
    P = D64.copy()
    P[a] += 2 * tol[a]
    P[b] -= 2 * tol[b]
    G = np.sqrt(P) if metric == 1 else P
    ratio, nbad = checks.check_distances(G, D64, qn, cn, metric=metric)
    assert nbad == 2 and ratio == pytest.approx(2.0, rel=1e-3)

"""a-S4 / a-S6 parity: the CUDA select and merge vs the oracle, bit-exact.

The select runs on fp32 matrices the oracle (or the seeded generators) produced and must
return exactly the oracle's (index, value) lists: sorted by (value, index), -0 == +0,
NaN after +inf (include/knn.h).  Shapes span several chunks and ragged tails."""
import numpy as np
import pytest

import oracle
from paper_1309_5478_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def knn():
    from paper_1309_5478_b200 import knn as k
    return k


def gpu_select(D, k, ld=None):
    M, N = D.shape
    if ld is None:
        Dt = torch.from_numpy(np.ascontiguousarray(D)).cuda()
        return [t.cpu().numpy() for t in knn().select(Dt, k)]
    buf = np.zeros((M, ld), np.float32)
    buf[:, :N] = D
    Dt = torch.from_numpy(buf).cuda()
    return [t.cpu().numpy() for t in knn().select(Dt, k, N=N)]


def assert_same(got, ref):
    gi, gd = got
    ri, rd = ref
    assert np.array_equal(gi, ri), f"first index mismatch at {np.argwhere(gi != ri)[:3]}"
    assert np.array_equal(gd.view(np.uint32), rd.view(np.uint32))


@pytest.mark.parametrize("N", [1, 31, 33, 1000, 2048, 2049, 4097, 16385])
@pytest.mark.parametrize("k", [1, 8, 31, 32, 33, 255, 256, 1000, 1024])
def test_select_uniform(N, k):
    if k > N:
        pytest.skip("k > N")
    D = datagen.keys(24, N, "uniform", seed=N * 7 + k)
    assert_same(gpu_select(D, k), oracle.select_f32(D, k))


@pytest.mark.parametrize("kind", ["dup256", "descending", "ascending", "equal"])
@pytest.mark.parametrize("k", [1, 32, 33, 1024])
def test_select_adversarial(kind, k):
    D = datagen.keys(8, 9000, kind, seed=11)
    assert_same(gpu_select(D, k), oracle.select_f32(D, k))


def test_select_special_values():
    g = np.random.Generator(np.random.Philox(3))
    D = g.standard_normal((16, 3000)).astype(np.float32)
    D[:, ::7] = 0.0
    D[:, 3::7] = -0.0
    D[:, 5::11] = np.inf
    D[:, 6::13] = -np.inf
    D[:, 2::17] = np.nan
    D[:, 9::19] = -np.nan
    for k in (1, 40, 1024):
        assert_same(gpu_select(D, k), oracle.select_f32(D, k))
    # a row with fewer finite values than k
    E = np.full((3, 500), np.inf, np.float32)
    E[:, :10] = np.arange(10, dtype=np.float32)
    assert_same(gpu_select(E, 64), oracle.select_f32(E, 64))


@pytest.mark.parametrize("ld_extra", [1, 3])
def test_select_unaligned_rows(ld_extra):
    D = datagen.keys(10, 5001, "uniform", seed=5)
    assert_same(gpu_select(D, 50, ld=5001 + ld_extra), oracle.select_f32(D, 50))


def test_select_full_row_and_k_equals_n():
    D = datagen.keys(5, 700, "dup256", seed=6)
    assert_same(gpu_select(D, 700), oracle.select_f32(D, 700))


def test_select_on_oracle_distance_matrix():
    # north star: "The GPU select, run on the oracle's own distance matrix, must return
    # bit-identical indices" — D32 = fp32(D64) rows of a clustered k-NNG (C2 shape family).
    X = datagen.points(6000, 64, "clusters", seed=datagen.BASE_SEED + 2)
    rows = np.arange(0, 6000, 97)
    D32 = oracle.dist_rows(X, X, rows=rows).astype(np.float32)
    for r, i in enumerate(rows):
        D32[r, i] = np.inf  # graph mode: self excluded by position
    ref = oracle.knn(X, X, 16, rows=rows, graph=True)
    got = gpu_select(D32, 16)
    assert np.array_equal(got[0], ref["idx32"])
    assert np.array_equal(got[1], ref["dist32"])


def test_select_many_rows_full_size():
    # the select at a bench-sized row length (65536) on a sample of rows
    D = datagen.keys(64, 65536, "uniform", seed=9)
    assert_same(gpu_select(D, 32), oracle.select_f32(D, 32))


def test_select_deterministic():
    D = datagen.keys(32, 20000, "dup256", seed=10)
    a, b = gpu_select(D, 100), gpu_select(D, 100)
    assert_same(a, b)


# ------------------------------------------------------------------ merge -----------
def _sorted_lists(G, M, k, seed, dup=False):
    g = np.random.Generator(np.random.Philox(seed))
    vals = (g.integers(0, 50, size=(G, M, k)) / 8.0 if dup else g.random((G, M, k))).astype(np.float32)
    idx = g.integers(0, 10000, size=(G, M, k)).astype(np.int32)
    for a in range(G):
        for r in range(M):
            o = np.lexsort((idx[a, r], vals[a, r]))
            vals[a, r], idx[a, r] = vals[a, r][o], idx[a, r][o]
    return vals, idx


@pytest.mark.parametrize("G,k", [(1, 1), (2, 32), (8, 32), (8, 1024), (3, 1000), (64, 16)])
@pytest.mark.parametrize("dup", [False, True])
def test_merge_parity(G, k, dup):
    M = 40
    vals, idx = _sorted_lists(G, M, k, seed=G * 1000 + k, dup=dup)
    offsets = np.arange(G, dtype=np.int64) * 10000
    ref = oracle.merge(vals, idx, offsets)
    got = knn().merge(torch.from_numpy(vals).cuda(), torch.from_numpy(idx).cuda(), offsets)
    assert_same([t.cpu().numpy() for t in got], ref)


def test_merge_of_column_shards_equals_unsharded_select():
    D = datagen.keys(50, 10000, "dup256", seed=12)
    k = 64
    bounds = [0, 2500, 5000, 7500, 10000]
    pd, pi = [], []
    for a, b in zip(bounds[:-1], bounds[1:]):
        i, d = gpu_select(D[:, a:b], k)
        pd.append(d)
        pi.append(i)
    got = knn().merge(torch.from_numpy(np.stack(pd)).cuda(), torch.from_numpy(np.stack(pi)).cuda(),
                      bounds[:-1])
    assert_same([t.cpu().numpy() for t in got], oracle.select_f32(D, k))


# ------------------------------------------------------------------ warp-per-row path --
# knn_select runs one warp per row when k <= 128 and there are >= 4 rows per SM
# (M >= 592 on B200); these cover that plan with ragged rows and adversarial keys.
@pytest.mark.parametrize("N", [1, 33, 1000, 1024, 1025, 4097, 20000])
@pytest.mark.parametrize("k", [1, 31, 32, 33, 64, 65, 128])
def test_warp_select_uniform(N, k):
    if k > N:
        pytest.skip("k > N")
    D = datagen.keys(700, N, "uniform", seed=N * 13 + k)
    assert_same(gpu_select(D, k), oracle.select_f32(D, k))


@pytest.mark.parametrize("kind", ["dup256", "descending", "ascending", "equal"])
@pytest.mark.parametrize("k", [1, 32, 100, 128])
def test_warp_select_adversarial(kind, k):
    D = datagen.keys(640, 5000, kind, seed=21)
    assert_same(gpu_select(D, k), oracle.select_f32(D, k))


def test_warp_select_special_values():
    g = np.random.Generator(np.random.Philox(23))
    D = g.standard_normal((800, 3000)).astype(np.float32)
    D[:, ::7] = 0.0
    D[:, 3::7] = -0.0
    D[:, 5::11] = np.inf
    D[:, 6::13] = -np.inf
    D[:, 2::17] = np.nan
    D[::3, :] = np.inf  # rows with few / no finite keys
    D[::3, :5] = 1.0
    for k in (1, 17, 128):
        assert_same(gpu_select(D, k), oracle.select_f32(D, k))


# ------------------------------------------------------------------ two-pass warp path --
# k <= 32, 1024 <= N <= 131072, >= 4 rows per SM: pivot = the k-th smallest group minimum
# (a group = one lane's 32 elements of a 1024-element chunk), then only the groups at or
# below it are re-read (select.cu select_warp2p_kernel).
@pytest.mark.parametrize("N", [1024, 1025, 3000, 8192, 65536, 131071])
@pytest.mark.parametrize("k", [1, 16, 32])
def test_two_pass_select_uniform(N, k):
    D = datagen.keys(600, N, "uniform", seed=N * 17 + k)
    got = gpu_select(D, k, ld=(N + 3) // 4 * 4)  # 16-byte aligned rows (the bulk-copy ring)
    assert knn().last_select_kernel()[0] == "two-pass warp per row"
    assert_same(got, oracle.select_f32(D, k))


@pytest.mark.parametrize("kind", ["dup256", "descending", "ascending", "equal"])
@pytest.mark.parametrize("k", [1, 32])
def test_two_pass_select_adversarial(kind, k):
    """Ties at the pivot ("equal": every group minimum is the pivot, all 9000 elements
    survive, in rounds of up to 1024 survivors folded in windows of 256)."""
    D = datagen.keys(600, 9000, kind, seed=31)
    got = gpu_select(D, k)
    assert knn().last_select_kernel()[0] == "two-pass warp per row"
    assert_same(got, oracle.select_f32(D, k))


@pytest.mark.parametrize("N", [4096, 16384])
def test_two_pass_select_heads_exhausted(N):
    """The small keys all sit in one lane's groups (columns with (col // 4) % 32 == 0), so
    that lane's 4 heads run out before k pops and the pivot comes from the other lanes:
    looser, still exact (ring-resident rows and streamed rows)."""
    k = 32
    g = np.random.Generator(np.random.Philox(41))
    D = (g.random((600, N), dtype=np.float32) + np.float32(1.0))
    cols = np.arange(N)
    lane0 = ((cols // 4) % 32) == 0
    D[:, lane0] = g.random((600, int(lane0.sum())), dtype=np.float32) * np.float32(1e-3)
    got = gpu_select(D, k)
    assert knn().last_select_kernel()[0] == "two-pass warp per row"
    assert_same(got, oracle.select_f32(D, k))


def test_two_pass_select_special_values():
    """-0/+0, +-inf, NaN (groups of NaN only: their minimum is the NaN key), rows with
    fewer than k finite keys, ragged N."""
    g = np.random.Generator(np.random.Philox(43))
    N = 5000
    D = g.standard_normal((700, N)).astype(np.float32)
    D[:, ::7] = 0.0
    D[:, 3::7] = -0.0
    D[:, 5::11] = np.inf
    D[:, 6::13] = -np.inf
    D[:, 2::17] = np.nan
    D[::3, :] = np.inf
    D[::3, :5] = 1.0
    D[1::5, :] = np.nan          # rows of NaN only
    D[1::5, 4000:4010] = 2.0
    D[2::7, :2048] = np.nan      # whole NaN groups next to finite ones
    for k in (1, 17, 32):
        got = gpu_select(D, k)
        assert knn().last_select_kernel()[0] == "two-pass warp per row"
        assert_same(got, oracle.select_f32(D, k))


@pytest.mark.parametrize("N,k", [(8192, 1024), (20000, 200), (32768, 1024), (32768, 512),
                                  (65536, 129), (100003, 777)])
def test_select_sampled_pivot(N, k):
    """CTA-per-row select with the pivot sampled from the first chunk (k > 128,
    N >= 2 chunks): uniform rows take the pivot path, sorted rows the redo pass
    (ascending: too few candidates) or the overflow rebuild (descending), mixed in one
    call so the redo row list must map back to the right rows."""
    D = datagen.keys(12, N, "uniform", seed=N + k)
    D[3] = np.arange(N, dtype=np.float32)          # ascending: pivot too low -> redo
    D[7] = np.arange(N, 0, -1, dtype=np.float32)   # descending: overflow -> rebuild
    D[9, : N // 2] = np.float32(5.0)               # sample far above the rest of the row
    D[10] = np.float32(0.25)                        # all equal: index order decides
    D[11, 5::3] = np.inf
    assert_same(gpu_select(D, k), oracle.select_f32(D, k))


def test_select_sampled_pivot_few_finite():
    """Rows with fewer finite keys than k on the sampled-pivot path."""
    N, k = 16384, 600
    D = np.full((4, N), np.inf, np.float32)
    D[0, :100] = np.arange(100, dtype=np.float32)
    D[1, -50:] = 1.0
    D[2, ::40] = np.nan
    D[3, 9000:9600] = -np.arange(600, dtype=np.float32)
    assert_same(gpu_select(D, k), oracle.select_f32(D, k))


@pytest.mark.parametrize("M", [1, 3, 17, 100])
@pytest.mark.parametrize("N,k", [(8192, 1), (20000, 32), (65536, 100), (65536, 1024),
                                  (1 << 20, 64), (1 << 20, 1024), (300001, 333)])
def test_select_few_rows_cluster(M, N, k):
    """Few rows (M < #SMs): a thread-block cluster per row, segments merged over DSMEM
    (NEXT-3).  Adversarial rows exercise the in-kernel re-stream (ascending:
    the segment pivots are too low) and the overflow rebuild (descending)."""
    if M * N > 60_000_000:
        N = 60_000_000 // M // 4 * 4
    D = datagen.keys(M, N, "uniform", seed=M * 1000 + k)
    if M >= 3:
        D[1] = np.arange(N, dtype=np.float32)
        D[2] = np.arange(N, 0, -1, dtype=np.float32)
    if M >= 17:
        D[5] = np.float32(0.5)
        D[6, ::3] = np.inf
        D[7, 1::5] = np.nan
        D[8, N // 2:] = -1.0
    assert_same(gpu_select(D, k), oracle.select_f32(D, k))


def test_cluster_path_is_taken():
    D = datagen.keys(4, 1 << 18, "uniform", seed=77)
    assert_same(gpu_select(D, 64), oracle.select_f32(D, 64))
    kind, splits = knn().last_select_kernel()
    assert kind == "cluster per row" and splits >= 8


@pytest.mark.parametrize("N,k", [(1000, 8), (5000, 1024), (70000, 64), (65536, 512)])
@pytest.mark.parametrize("kind", ["uniform", "dup256", "descending", "equal"])
def test_select_paper_ablation(N, k, kind):
    """The paper's quick multi-select (ablation kernel) is exact too."""
    D = datagen.keys(40, N, kind, seed=N + k)
    ref = oracle.select_f32(D, k)
    Dt = torch.from_numpy(D).cuda()
    got = [t.cpu().numpy() for t in knn().select_paper(Dt, k)]
    assert_same(got, ref)

"""Pin of reading R21: the per-point error bound of the single fp16
product, checked numerically in fp64 on CPU — independent of the CUDA code, which implements
the same formula (prep.cu bound_norms_kernel).

For a point x, prep scales it by s = 2^sh (max|x| s in [2^14, 2^15)) and splits hi = fp16(s x);
e_x = ||s x - hi|| / ||s x||.  With one t > 0 per call and every e <= 2^-11 (1 + 2^-20),
    |2 q.x - 2 (hi_q . hi_x) / (s_q s_x)| <= B_q ||q||^2 + B_x ||x||^2,
    B = (t + e^2 / t)(1 + 2^-10) + 2^-11 (1 + 2^-9) e
(AM-GM on 2|q||x| e, Cauchy-Schwarz on the cross term), i.e. the bound is a sum of per-point
terms.  The tests check it on every pair of seeded point sets of several shapes, and that it
is no weaker than the constant worst-case bound 2^-10 (1 + 2^-10) it replaces when t is the
call's largest e."""
import numpy as np
import pytest

from paper_1309_5478_b200 import datagen


def split(X):
    """prep.cu's scaling and hi split, in fp64 (s x exact; hi = fp16 round to nearest)."""
    X = X.astype(np.float32)
    amax = np.abs(X).max(axis=1)
    e = np.frexp(amax)[1]
    sh = np.where(amax > 0, 15 - e, 0)
    s = np.ldexp(1.0, sh)
    v = X.astype(np.float64) * s[:, None]
    hi = v.astype(np.float16).astype(np.float64)
    nv = np.sqrt((v * v).sum(1))
    eps = np.where(nv > 0, np.sqrt(((v - hi) ** 2).sum(1)) / np.where(nv > 0, nv, 1), 0.0)
    return X.astype(np.float64), s, hi, eps


def bound_terms(eps, t):
    t = max(t, 2.0 ** -13)
    return (t + eps ** 2 / t) * (1 + 2.0 ** -10) + 2.0 ** -11 * (1 + 2.0 ** -9) * eps


CASES = [("uniform", 700, 256), ("gauss", 600, 48), ("clusters", 500, 30), ("grid", 400, 64), ("uniform", 500, 7)]


@pytest.mark.parametrize("dist,n,d", CASES)
@pytest.mark.parametrize("tmode", ["max", "floor", "mixed"])
def test_per_point_split_bound_holds(dist, n, d, tmode):
    X = datagen.points(n, d, dist, seed=n + d)
    if tmode == "mixed":  # fp16-exact points mixed in (e = 0), as the pipelined call's sample
        X[::3] = X[::3].astype(np.float16).astype(np.float32)
    if dist == "gauss":
        X[::5] *= 1e-3  # rows of very different magnitude in one call
    Xd, s, hi, eps = split(X)
    assert np.all(eps <= 2.0 ** -11 * (1 + 2.0 ** -20))
    t = float(np.max(eps)) if tmode != "floor" else 0.0  # "floor": t at its 2^-13 floor
    B = bound_terms(eps, t)
    nq = (Xd * Xd).sum(1)
    exact = 2.0 * (Xd @ Xd.T)
    approx = 2.0 * (hi @ hi.T) / np.outer(s, s)
    err = np.abs(exact - approx)
    allowed = B[:, None] * nq[:, None] + B[None, :] * nq[None, :]
    # the fp64 evaluation itself: products exact, sums of d terms rounded (~d 2^-53 relative)
    slack = 1e-14 * (nq[:, None] + nq[None, :])
    assert np.all(err <= allowed + slack), float(np.max((err - allowed) / (nq[:, None] + nq[None, :])))


@pytest.mark.parametrize("dist,n,d", CASES[:3])
def test_per_point_bound_no_weaker_than_constant(dist, n, d):
    X = datagen.points(n, d, dist, seed=7 * n + d)
    _, _, _, eps = split(X)
    B = bound_terms(eps, float(np.max(eps)))
    const = 2.0 ** -10 * (1 + 2.0 ** -10)  # the round-1 bound (e <= 2^-11 per component)
    # per side each B <= const (1 + small): with t = max e, B <= 2 t (1 + 2^-10) + 2^-22 ...
    assert np.all(B <= const * (1 + 2.0 ** -9))
    # ... and on real data markedly tighter (the point of the reading)
    assert float(np.mean(B)) < 0.6 * const

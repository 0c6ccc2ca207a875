"""Randomised cross-check of the out-of-core call (knn_search_streamed: host corpus streamed in
chunks, partial lists merged) and of the host-buffer block call against the device-resident
search / k-NNG, bit for bit: random shapes, chunk sizes, metrics, k up to 1024.
python scripts/fuzz_stream.py [n] [seed]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1309_5478_b200 import knn, datagen
import oracle
from oracle import checks

if os.environ.get("FUZZ_PLAN") == "exact":  # the FP32-accurate pivot plan everywhere
    knn.set_plan(knn.PLAN_PIVOT_EXACT)


def oracle_ok(Q, X, gi, gd, k, metric, graph, rows):
    """E2E-1/2 of oracle.checks on the given rows (the deciding check when two valid paths
    differ, e.g. fp32 values of different plans)."""
    D64 = oracle.dist_rows(Q, X, rows=rows, metric=0 if metric <= 1 else metric)
    res = checks.check_rows(gi[rows], gd[rows], D64, oracle.sqnorms(Q)[rows], oracle.sqnorms(X), rows, k,
                            metric=metric, graph=graph)
    return res["failures"] == []

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 9)
bad = 0
t0 = time.time()
for case in range(n_cases):
    N = int(rng.integers(1000, 60000))
    M = int(rng.integers(1, 5000))
    d = int(rng.choice([2, 7, 16, 64, 100, 256]))
    k = int(min(N - 1, rng.choice([1, 4, 16, 32, 64, 200, 1024])))
    metric = int(rng.choice([0, 1, 2, 3]))
    dist = str(rng.choice(["uniform", "gauss", "clusters", "grid"]))
    graph = bool(rng.integers(0, 3) == 0)
    X = datagen.points(N, d, dist, seed=7000 + case)
    Q = X if graph else datagen.points(M, d, dist, seed=8000 + case)
    Xt, Qt = torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda()
    ref = knn.graph(Xt, k, metric=metric) if graph else knn.search_block(Qt, Xt, k, metric=metric)
    ref = (ref[0].cpu().numpy(), ref[1].cpu().numpy())
    chunk = int(rng.choice([0, 1000, 4096, 20000]))
    si, sd = knn.search_streamed(Q, X, k, metric=metric, graph=graph, chunk_points=chunk)
    ok_s = np.array_equal(si, ref[0]) and np.array_equal(sd.view(np.uint32), ref[1].view(np.uint32))
    hi, hd = knn.search_block_host(Q, X, k, metric=metric, self_shift=0 if graph else knn.NO_SELF)
    ok_h = np.array_equal(hi, ref[0]) and np.array_equal(hd.view(np.uint32), ref[1].view(np.uint32))
    extra = {}
    if not (ok_s and ok_h):  # which side is wrong: the oracle on the differing rows
        diff = np.flatnonzero((si != ref[0]).any(1) | (sd.view(np.uint32) != ref[1].view(np.uint32)).any(1))
        rows = diff[:16] if len(diff) else np.arange(min(16, Q.shape[0]))
        extra = {"differing_rows": int(len(diff)), "oracle_ref": oracle_ok(Q, X, *ref, k, metric, graph, rows),
                 "oracle_streamed": oracle_ok(Q, X, si, sd, k, metric, graph, rows)}
    # a mismatch is a failure only if the oracle rejects a side (angular k-NNG: symmetric vs
    # blocked orientation rounding; automatic plan: chunks may choose different partitions)
    bad += not (ok_s and ok_h) and not (extra.get("oracle_ref") and extra.get("oracle_streamed"))
    print(json.dumps({"case": case, "N": N, "M": Q.shape[0], "d": d, "k": k, "metric": metric, "dist": dist,
                      "graph": graph, "chunk": chunk, "streamed": bool(ok_s), "host": bool(ok_h), **extra}),
          flush=True)
print(json.dumps({"cases": n_cases, "mismatches": bad, "s": time.time() - t0}))
sys.exit(1 if bad else 0)

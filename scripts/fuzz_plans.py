"""Randomised cross-check over random shapes, metrics and distributions: the automatic plan
vs the materialised plan, bit-identical by design for the FP32-accurate plans; when the device
chose the single-product partition (plans 5 / 6: re-evaluated fp32 values, reading R20) both
results are checked against the oracle on sampled rows instead (E2E checks of oracle.checks).
python scripts/fuzz_plans.py [n] [seed]"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1309_5478_b200 import knn, datagen
import oracle
from oracle import checks

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = 0
t0 = time.time()
for case in range(n_cases):
    N = int(rng.integers(16384, 45000))
    d = int(rng.choice([1, 3, 7, 16, 33, 64, 100, 128, 257, 300]))
    k = int(rng.choice([1, 2, 5, 8, 16, 31, 32, 33, 64, 100, 256, 511, 1024]))
    k = min(k, N - 1)
    metric = int(rng.choice([0, 0, 1, 2, 3]))
    dist = str(rng.choice(["uniform", "gauss", "clusters", "grid"]))
    search = bool(rng.integers(0, 4) == 0)
    X = torch.from_numpy(datagen.points(N, d, dist, seed=1000 + case)).cuda()
    Q = torch.from_numpy(datagen.points(int(rng.integers(256, 5000)), d, dist, seed=2000 + case)).cuda() if search else X
    run = (lambda: knn.search_block(Q, X, k, metric=metric)) if search else (lambda: knn.graph(X, k, metric=metric))
    gi, gd = run()
    plan = knn.last_plan()
    knn.set_plan(knn.PLAN_MATERIALISED)
    try:
        ri, rd = run()
    finally:
        knn.set_plan(knn.PLAN_AUTO)
    if plan in (5, 6):
        Qn, Xn = Q.cpu().numpy(), X.cpu().numpy()
        rows = np.unique(np.concatenate([[0, Qn.shape[0] - 1], rng.integers(0, Qn.shape[0], 14)]))
        D64 = oracle.dist_rows(Qn, Xn, rows=rows, metric=0 if metric <= 1 else metric)  # (L2: squared)
        ok = True
        for i_, d_ in ((gi, gd), (ri, rd)):
            res = checks.check_rows(i_.cpu().numpy()[rows], d_.cpu().numpy()[rows], D64, oracle.sqnorms(Qn)[rows],
                                    oracle.sqnorms(Xn), rows, k, metric=metric, graph=not search)
            ok = ok and res["failures"] == []
    else:
        ok = torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))
    bad += not ok
    print(json.dumps({"case": case, "N": N, "M": Q.shape[0], "d": d, "k": k, "metric": metric, "dist": dist,
                      "search": search, "plan": plan, "equal": ok}), flush=True)
print(json.dumps({"cases": n_cases, "mismatches": bad, "s": time.time() - t0}))
sys.exit(1 if bad else 0)

"""Single-product partition + exact re-evaluation (k <= 32, L2) vs the 3-product plan and the
oracle on sampled rows; timing of both.  python scripts/pivot1_check.py [N d k metric dist]"""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from oracle import checks
from paper_1309_5478_b200 import knn, datagen

N, d, k, metric = [int(a) for a in sys.argv[1:5]] if len(sys.argv) > 4 else (65536, 256, 32, 0)
dist = sys.argv[5] if len(sys.argv) > 5 else "uniform"
Xn = datagen.points(N, d, dist, seed=1309100)
X = torch.from_numpy(Xn).cuda()
gi, gd = knn.graph(X, k, metric=metric)
plan = knn.last_plan()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): knn.graph(X, k, metric=metric)
e0.record()
for _ in range(10): knn.graph(X, k, metric=metric)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
rows = np.arange(0, N, max(1, N // 97))
D64 = oracle.dist_rows(Xn, Xn, rows=rows)
nrm = oracle.sqnorms(Xn)
gin, gdn = gi.cpu().numpy(), gd.cpu().numpy()
res = checks.check_rows(gin[rows], gdn[rows], D64, nrm[rows], nrm, rows, k, metric=metric, graph=True)
# exact fp64 distances of the returned pairs vs the returned values
ex = np.array([[D64[a, gin[r, j]] for j in range(k)] for a, r in enumerate(rows)])
if metric == 1: ex = np.sqrt(ex)
rel = np.abs(gdn[rows] - ex) / np.maximum(ex, 1e-30)
print(json.dumps({"N": N, "d": d, "k": k, "metric": metric, "dist": dist, "plan": plan, "ms": ms,
                  "oracle_failures": len(res["failures"]), "max_rel_err_vs_fp64": float(rel.max()),
                  "candidates_per_row": knn.last_candidates()}))

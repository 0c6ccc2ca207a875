"""Randomised a-S3 parity: knn_distances (the materialised tcgen05 distance GEMM) against the
oracle's fp64 distances within BJ's tolerance (oracle.checks.check_distances), over random
shapes (ragged M, N, d), metrics, distributions and scales.
python scripts/fuzz_dist.py [n] [seed]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from oracle import checks
from paper_1309_5478_b200 import knn, datagen

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
bad = 0
t0 = time.time()
for case in range(n_cases):
    M = int(rng.integers(1, 700))
    N = int(rng.integers(1, 3000))
    d = int(rng.choice([1, 2, 5, 31, 64, 65, 128, 257, 1000]))
    metric = int(rng.choice([0, 1, 2, 3]))
    dist = str(rng.choice(["uniform", "gauss", "clusters", "grid"]))
    scale = float(rng.choice([1.0, 1e-12, 1e12, 3.0]))
    Q = (datagen.points(M, d, dist, seed=100 + case) * scale).astype(np.float32)
    X = (datagen.points(N, d, dist, seed=200 + case) * scale).astype(np.float32)
    D = knn.distances(torch.from_numpy(Q).cuda(), torch.from_numpy(X).cuda(), metric=metric).cpu().numpy()
    D64 = oracle.dist_rows(Q, X, metric=0 if metric <= 1 else metric)
    ratio, nbad = checks.check_distances(D, D64, oracle.sqnorms(Q), oracle.sqnorms(X), metric)
    bad += nbad > 0
    print(json.dumps({"case": case, "M": M, "N": N, "d": d, "metric": metric, "dist": dist, "scale": scale,
                      "max_err_over_tol": ratio, "violations": nbad}), flush=True)
print(json.dumps({"cases": n_cases, "mismatches": bad, "s": time.time() - t0}))
sys.exit(1 if bad else 0)

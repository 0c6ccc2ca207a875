"""Randomised cross-check of the general block call (knn_search_block: a self-exclusion shift
and an index offset, as the sharded drivers use it): the pivot plan with the FP32-accurate
partition (KNN_PLAN_PIVOT_EXACT) against the materialised plan, bit for bit.
python scripts/fuzz_blocks.py [n] [seed]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1309_5478_b200 import knn, datagen

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
t0 = time.time()
for case in range(n_cases):
    N = int(rng.integers(16384, 40000))
    M = int(rng.integers(256, 6000))
    d = int(rng.choice([3, 16, 33, 64, 128]))
    k = int(rng.choice([1, 2, 7, 16, 32, 33, 100, 500]))
    metric = int(rng.choice([0, 1, 2, 3]))
    dist = str(rng.choice(["uniform", "gauss", "clusters", "grid"]))
    shift = int(rng.choice([knn.NO_SELF, 0, int(rng.integers(0, N - M)), int(rng.integers(-M, N))]))
    off = int(rng.choice([0, int(rng.integers(0, 1 << 20))]))
    X = datagen.points(N, d, dist, seed=9000 + case)
    Q = datagen.points(M, d, dist, seed=9500 + case) if shift == knn.NO_SELF else \
        X[max(0, shift):max(0, shift) + M] if shift >= 0 and shift + M <= N else datagen.points(M, d, dist, seed=9600 + case)
    Qt, Xt = torch.from_numpy(np.ascontiguousarray(Q)).cuda(), torch.from_numpy(X).cuda()
    knn.set_plan(knn.PLAN_PIVOT_EXACT)
    gi, gd = knn.search_block(Qt, Xt, k, metric=metric, self_shift=shift, idx_offset=off)
    plan = knn.last_plan()
    knn.set_plan(knn.PLAN_MATERIALISED)
    ri, rd = knn.search_block(Qt, Xt, k, metric=metric, self_shift=shift, idx_offset=off)
    knn.set_plan(knn.PLAN_AUTO)
    ok = torch.equal(gi, ri) and torch.equal(gd.view(torch.int32), rd.view(torch.int32))
    bad += not ok
    print(json.dumps({"case": case, "N": N, "M": M, "d": d, "k": k, "metric": metric, "dist": dist, "shift": shift,
                      "offset": off, "plan": plan, "equal": ok}), flush=True)
print(json.dumps({"cases": n_cases, "mismatches": bad, "s": time.time() - t0}))
sys.exit(1 if bad else 0)

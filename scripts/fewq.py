"""Few-query k-NN search timing (pivot vs materialised plans): M queries vs N = 2^20, d = 128."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1309_5478_b200 import knn, datagen
X = torch.from_numpy(datagen.points(1 << 20, 128, "uniform", seed=5)).cuda()
for M in (8, 128, 1024, 8192):
    Q = torch.from_numpy(datagen.points(M, 128, "uniform", seed=6)).cuda()
    for plan in (knn.PLAN_AUTO, knn.PLAN_MATERIALISED):
        knn.set_plan(plan)
        for k in (10, 100):
            knn.search(Q, X, k); torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(5):
                knn.search(Q, X, k)
            torch.cuda.synchronize()
            print(M, "auto" if plan == 0 else "mat", k, "plan", knn.last_plan(), "%.3f ms" % ((time.perf_counter() - t) / 5 * 1e3), flush=True)
knn.set_plan(knn.PLAN_AUTO)

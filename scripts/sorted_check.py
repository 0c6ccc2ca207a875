import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1309_5478_b200 import knn, datagen
X = datagen.points(65536, 64, "clusters", seed=5)
g = np.random.Generator(np.random.Philox(1))
# sort by nearest centre: recover the cluster order by a coarse key (first coordinate bins)
order = np.argsort(X[:, 0] + 1000 * np.round(X[:, 1]))
Xs = np.ascontiguousarray(X[order])
for name, A in [("shuffled", X), ("sorted", Xs)]:
    Xt = torch.from_numpy(A).cuda()
    for k in (16, 100):
        knn.graph(Xt, k); torch.cuda.synchronize()
        t = time.perf_counter(); knn.graph(Xt, k); torch.cuda.synchronize()
        print(name, k, "plan", knn.last_plan(), "cands/row", knn.last_candidates() / 65536, "%.2f ms" % ((time.perf_counter() - t) * 1e3))

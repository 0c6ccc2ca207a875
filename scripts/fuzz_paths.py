"""Randomised cross-check of the other entry points against the device-resident k-NNG / search
(all under the automatic plan, bit for bit): the host-pipelined call (knn_search_block_host),
Par-3's phases with G = 2..3 emulated ranks, and the one-rank sharded calls (sym / query /
corpus k-NNG, query / corpus search) through their phases.
python scripts/fuzz_paths.py [n] [seed]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1309_5478_b200 import knn, datagen

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
os.environ["KNN_SHARD_G1_PHASES"] = "1"
bad = 0
t0 = time.time()


def same(a, b):
    return torch.equal(a[0].cpu(), torch.as_tensor(b[0]).cpu()) and \
        torch.equal(a[1].cpu().view(torch.int32), torch.as_tensor(b[1]).cpu().view(torch.int32))


for case in range(n_cases):
    N = int(rng.integers(8, 23)) * 2048
    d = int(rng.choice([3, 7, 16, 33, 64, 100, 256]))
    k = int(rng.choice([1, 2, 3, 5, 8, 16, 31, 32]))
    metric = int(rng.choice([0, 1, 2, 3]))
    dist = str(rng.choice(["uniform", "gauss", "clusters", "grid"]))
    X = datagen.points(N, d, dist, seed=5000 + case)
    Xt = torch.from_numpy(X).cuda()
    ref = knn.graph(Xt, k, metric=metric)
    plan = knn.last_plan()
    res = {}
    Xp = torch.from_numpy(X).pin_memory().numpy()
    res["host"] = same(ref, knn.search_block_host(Xp, Xp, k, metric=metric, self_shift=0))
    res["sym1"] = same(ref, knn.graph_sharded(Xt, k, mode="sym", metric=metric))
    res["query1"] = same(ref, knn.graph_sharded(Xt, k, mode="query", metric=metric))
    res["corpus1"] = same(ref, knn.graph_sharded(Xt, k, mode="corpus", metric=metric))
    Qt = torch.from_numpy(datagen.points(int(rng.integers(300, 3000)), d, dist, seed=6000 + case)).cuda()
    sref = knn.search(Qt, Xt, k)  # (knn_search / knn_search_sharded: squared L2, BJ's signature)
    res["search_query1"] = same(sref, knn.search_sharded(Qt, Xt, k, mode="query"))
    res["search_corpus1"] = same(sref, knn.search_sharded(Qt, Xt, k, mode="corpus"))
    G = int(rng.integers(2, 4))
    npad = -(-N // 256) * 256
    thr = torch.full((npad,), float("nan"), device="cuda")
    per = -(-N // G)
    for g in range(G):
        lo, hi = g * per, min(N, (g + 1) * per)
        knn.graph_pivots(Xt, k, lo, hi - lo, thr, metric=metric)
    units, cap = knn.graph_units(N), knn.graph_list_cap(k)
    lists = []
    for g in range(G):
        cnt = torch.zeros(N, dtype=torch.int32, device="cuda")
        ce = torch.empty((N, cap), dtype=torch.int64, device="cuda")
        knn.graph_partition(Xt, k, thr, units * g // G, units * (g + 1) // G, cnt, ce, metric=metric)
        lists.append((cnt, ce))
    torch.cuda.synchronize()
    parts = []
    try:
        for g in range(G):
            lo, hi = g * per, min(N, (g + 1) * per)
            parts.append(knn.graph_gather_select([l[0].data_ptr() for l in lists], [l[1].data_ptr() for l in lists],
                                                 cap, N, k, lo, hi - lo))
        res[f"par3_G{G}"] = same(ref, (torch.cat([p[0] for p in parts]), torch.cat([p[1] for p in parts])))
    except knn.KnnError as e:  # a failed certificate: the sharded call would fall back (not a mismatch)
        res[f"par3_G{G}"] = "fallback"
    ok = all(v is True or v == "fallback" for v in res.values())
    bad += not ok
    print(json.dumps({"case": case, "N": N, "d": d, "k": k, "metric": metric, "dist": dist, "plan": plan, **res}),
          flush=True)
print(json.dumps({"cases": n_cases, "mismatches": bad, "s": time.time() - t0}))
sys.exit(1 if bad else 0)

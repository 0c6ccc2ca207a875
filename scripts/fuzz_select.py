"""Randomised cross-check of the a-S4 selects (knn_select, knn_select_paper) against the
oracle's exact select on the same fp32 matrices, bit for bit: random shapes (1..600 rows,
1..2^17 columns), k up to 1024, ties (quantised values), +-0, +-inf and NaN entries.
python scripts/fuzz_select.py [n] [seed]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from paper_1309_5478_b200 import knn

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
bad = 0
t0 = time.time()
for case in range(n_cases):
    M = int(rng.choice([1, 2, 7, 31, 64, 200, 600]))
    N = int(rng.choice([1, 5, 33, 100, 1000, 4096, 8191, 20000, 65536, 131072]))
    if M * N > 40_000_000:
        M = max(1, 40_000_000 // N)
    k = int(min(N, rng.choice([1, 2, 8, 16, 32, 33, 100, 256, 1000, 1024])))
    kind = str(rng.choice(["uniform", "ties", "special"]))
    D = rng.random((M, N), dtype=np.float32)
    if kind == "ties":
        D = np.floor(D * 64) / 64
    elif kind == "special":
        m = rng.random((M, N))
        D[m < 0.01] = np.inf
        D[(m >= 0.01) & (m < 0.02)] = -0.0
        D[(m >= 0.02) & (m < 0.03)] = 0.0
        D[(m >= 0.03) & (m < 0.035)] = np.nan
    D = np.ascontiguousarray(D.astype(np.float32))
    ri, rd = oracle.select_f32(D, k)
    Dt = torch.from_numpy(D).cuda()
    res = {}
    for name, f in (("select", knn.select), ("paper", knn.select_paper)):
        gi, gd = f(Dt, k)
        res[name] = bool(np.array_equal(gi.cpu().numpy(), ri) and
                         np.array_equal(gd.cpu().numpy().view(np.uint32), rd.view(np.uint32)))
    ok = all(res.values())
    bad += not ok
    print(json.dumps({"case": case, "M": M, "N": N, "k": k, "kind": kind, **res,
                      "kernel": knn.last_select_kernel()[0]}), flush=True)
print(json.dumps({"cases": n_cases, "mismatches": bad, "s": time.time() - t0}))
sys.exit(1 if bad else 0)

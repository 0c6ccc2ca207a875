"""Microbenchmark of knn_select alone on uniform keys (select GB/s)."""
import sys, json
import torch
sys.path.insert(0, '.')
from paper_1309_5478_b200 import knn

def run(M, N, k, reps=5):
    D = torch.rand((M, N), device='cuda', dtype=torch.float32)
    knn.select(D, k); torch.cuda.synchronize()
    knn.profile_enable(True)
    for _ in range(reps):
        knn.select(D, k)
    ms, n = knn.profile_read('select')
    knn.profile_enable(False)
    avg = ms / n
    gbs = (M * N * 4 + M * k * 8) / (avg * 1e-3) / 1e9
    print(json.dumps({"M": M, "N": N, "k": k, "ms": round(avg, 4), "GB/s": round(gbs, 1)}), flush=True)

CASES = [(16384, 65536, 32), (16384, 65536, 1), (16384, 65536, 128), (4096, 32768, 1024), (65536, 4096, 32), (256, 1 << 20, 32), (2048, 1 << 18, 512)]
if len(sys.argv) > 1:
    CASES = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
for (M, N, k) in CASES:
    run(M, N, k)

"""Mainloop-only rate of the distance GEMM (null epilogue) vs the partition GEMM: how much
of the partition's time the epilogue costs.  python scripts/diag_mainloop.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1309_5478_b200 import knn, datagen
for N, d in [(65536, 256), (32768, 1024), (131072, 256)]:
    X = torch.from_numpy(datagen.points(N, d, "uniform", seed=1)).cuda()
    nb = -(-N // 256)
    flop = nb * (nb + 1) / 2 * 256 * 256 * 2 * 3 * (-(-d // 64) * 64)
    ms = knn.diag_mainloop(X, sym=True, reps=10)
    print(json.dumps({"N": N, "d": d, "sym_null_epilogue_ms": ms, "tflops": flop / ms / 1e9}), flush=True)

"""Per-kernel-class device time of the host-pipelined k-NNG (knn_search_block_host) vs the
device-resident call, headline shape: how much the chunked schedule adds to the GPU work."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1309_5478_b200 import knn, datagen
N, d, k = 65536, 256, 32
X = datagen.points(N, d, "uniform", seed=3)
Xh = torch.empty((N, d), dtype=torch.float32, pin_memory=True); Xh.copy_(torch.from_numpy(X)); Xn = Xh.numpy()
oi = torch.empty((N, k), dtype=torch.int32, pin_memory=True).numpy()
od = torch.empty((N, k), dtype=torch.float32, pin_memory=True).numpy()
Xt = torch.from_numpy(X).cuda()
kinds = ["prep", "gemm", "select", "fused", "merge"]
for name, f in [("device", lambda: knn.graph(Xt, k)),
                ("host pipelined", lambda: knn.search_block_host(Xn, Xn, k, self_shift=0, out=(oi, od)))]:
    for _ in range(3): f()
    torch.cuda.synchronize()
    knn.profile_enable(True)
    reps = 10
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e3
    parts = {kk: knn.profile_read(kk)[0] / reps for kk in kinds}
    knn.profile_enable(False)
    print(f"{name:15s} wall {wall:.3f} ms  kernels " + "  ".join(f"{kk} {v:.3f}" for kk, v in parts.items()) +
          f"  sum {sum(parts.values()):.3f}")

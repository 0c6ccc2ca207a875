"""One host-pipelined k-NNG call (headline shape) and one device call, for an ncu launch list
(scripts/e2e_breakdown.py gives the profile-event view)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1309_5478_b200 import knn, datagen
N, d, k = 65536, 256, 32
X = datagen.points(N, d, "uniform", seed=3)
Xh = torch.empty((N, d), dtype=torch.float32, pin_memory=True); Xh.copy_(torch.from_numpy(X)); Xn = Xh.numpy()
oi = torch.empty((N, k), dtype=torch.int32, pin_memory=True).numpy()
od = torch.empty((N, k), dtype=torch.float32, pin_memory=True).numpy()
Xt = torch.from_numpy(X).cuda()
which = sys.argv[1] if len(sys.argv) > 1 else "host"
for _ in range(2):
    if which == "host":
        knn.search_block_host(Xn, Xn, k, self_shift=0, out=(oi, od))
    else:
        knn.graph(Xt, k)
torch.cuda.synchronize()

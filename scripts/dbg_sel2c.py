import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1309_5478_b200 import knn
M, N, k = 700, 1024, 1
g = np.random.default_rng(1)
D = g.random((M, N), dtype=np.float32)
idx, dist = knn.select(torch.from_numpy(D).cuda(), k)
torch.cuda.synchronize()
print(idx[:2].cpu().numpy().ravel(), dist[:2].cpu().numpy().ravel(), 'ref', D[0].argmin(), D[0].min())

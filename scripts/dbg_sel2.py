import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1309_5478_b200 import knn
for (M, N, k) in [(700, 1024, 1), (700, 4096, 32), (700, 16384, 32)]:
    g = np.random.default_rng(1)
    D = g.random((M, N), dtype=np.float32)
    idx, dist = knn.select(torch.from_numpy(D).cuda(), k)
    torch.cuda.synchronize()
    idx = idx.cpu().numpy(); dist = dist.cpu().numpy()
    ref = np.argsort(D, axis=1, kind='stable')[:, :k]
    bad = np.argwhere(idx != ref)
    print(M, N, k, knn.last_select_kernel(), 'bad rows', len(set(bad[:, 0])) if len(bad) else 0, flush=True)
    if len(bad):
        r = bad[0][0]
        print(' row', r, 'got', idx[r][:8], dist[r][:8], 'ref', ref[r][:8], D[r][ref[r][:8]], flush=True)

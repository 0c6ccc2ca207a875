set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
KNN_GEMM=simt timeout -s KILL 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout -s KILL 600 python -m pytest tests/test_gpu_select.py -x -q 2>&1 | tail -15
timeout -s KILL 120 python -c "
import numpy as np, torch, oracle
from oracle import checks
from paper_1309_5478_b200 import knn, datagen
Q = datagen.points(300, 64, 'gauss', seed=1); X = datagen.points(700, 64, 'gauss', seed=2)
D = knn.distances(torch.from_numpy(Q).cuda(), torch.from_numpy(X).cuda()).cpu().numpy()
D64 = oracle.dist_rows(Q, X)
print('max abs err', np.abs(D-D64).max(), 'D sample', D[0,:4], D64[0,:4])
r, bad = checks.check_distances(D, D64, oracle.sqnorms(Q), oracle.sqnorms(X))
print('ratio', r, 'bad', bad)
" 2>&1 | tail -8
timeout -s KILL 900 python -m pytest tests/test_gpu_knn.py -x -q 2>&1 | tail -15

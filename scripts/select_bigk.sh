#!/bin/bash
# Large-k ring select timing on a few shapes (env knobs passed through); "dist" rows are
# N(170, 8^2) like the d = 1024 uniform distances of C4, "unif" rows U[0,1).
python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
from paper_1309_5478_b200 import knn
dev=torch.device('cuda',0); g=torch.Generator(device=dev)
for kind,Q,n,k in [('dist',32768,32768,1024),('unif',32768,32768,1024),('dist',8192,65536,512),('unif',8192,65536,256),('unif',65536,65536,64),('unif',8192,262144,1024),('unif',32768,4096,512)]:
    g.manual_seed(1)
    D=torch.rand((Q,n),generator=g,device=dev) if kind=='unif' else 170+8*torch.randn((Q,n),generator=g,device=dev)
    for _ in range(2): knn.select(D,k)
    torch.cuda.synchronize(); e0,e1=torch.cuda.Event(True),torch.cuda.Event(True); e0.record()
    for _ in range(5): knn.select(D,k)
    e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/5
    print(kind, os.environ.get('KNN_RING_CHUNK','4096'), Q,n,k, knn.last_select_kernel()[0], '%.3f ms %.0f GB/s'%(ms,Q*n*4/ms/1e6), flush=True)
PY

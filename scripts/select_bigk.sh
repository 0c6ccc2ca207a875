#!/bin/bash
# Large-k ring select timing on a few shapes (env knobs passed through).
python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
from paper_1309_5478_b200 import knn
dev=torch.device('cuda',0); g=torch.Generator(device=dev)
for Q,n,k in [(32768,32768,1024),(8192,65536,512),(8192,65536,256),(65536,65536,64),(8192,262144,1024),(32768,4096,512)]:
    g.manual_seed(1); D=torch.rand((Q,n),generator=g,device=dev)
    for _ in range(2): knn.select(D,k)
    torch.cuda.synchronize(); e0,e1=torch.cuda.Event(True),torch.cuda.Event(True); e0.record()
    for _ in range(5): knn.select(D,k)
    e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/5
    print(os.environ.get('KNN_RING_CHUNK','4096'), Q,n,k, knn.last_select_kernel()[0], '%.3f ms %.0f GB/s'%(ms,Q*n*4/ms/1e6), flush=True)
PY

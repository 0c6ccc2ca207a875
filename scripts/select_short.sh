#!/bin/bash
# Short-row select timing (U[0,1) keys), env knobs passed through.
python - <<'PY'
import torch, sys, os
sys.path.insert(0,'.')
from paper_1309_5478_b200 import knn
dev=torch.device('cuda',0); g=torch.Generator(device=dev)
for Q,n,k in [(8192,8192,16),(8192,8192,32),(32768,4096,16),(8192,65536,32),(8192,8192,64),(8192,8192,128),(8192,16384,64),(8192,16384,128),(32768,4096,64),(32768,4096,128),(8192,8192,256),(8192,16384,512)]:
    g.manual_seed(1); D=torch.rand((Q,n),generator=g,device=dev)
    for _ in range(2): knn.select(D,k)
    torch.cuda.synchronize(); e0,e1=torch.cuda.Event(True),torch.cuda.Event(True); e0.record()
    for _ in range(10): knn.select(D,k)
    e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/10
    print(os.environ.get('KNN_WARP_MAXK','128'), Q,n,k, knn.last_select_kernel()[0], '%.3f ms %.0f GB/s'%(ms,Q*n*4/ms/1e6), flush=True)
PY

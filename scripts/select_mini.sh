make -j8 >/dev/null
python - <<'PY'
import torch, json, sys
sys.path.insert(0,'.')
from paper_1309_5478_b200 import knn
import os
dev=torch.device('cuda',0)
g=torch.Generator(device=dev)
for Q,n in [(8192,8192),(8192,32768),(65536,65536),(8192,262144),(32768,4096)]:
  for k in [16,32,64,128]:
    g.manual_seed(1)
    D=torch.rand((Q,n),generator=g,device=dev)
    for _ in range(2): knn.select(D,k)
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(True),torch.cuda.Event(True)
    e0.record()
    for _ in range(5): knn.select(D,k)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/5
    print(os.environ.get('KNN_WARP_MAXK','128'), Q,n,k, knn.last_select_kernel()[0], '%.3f ms %.0f GB/s'%(ms, Q*n*4/ms/1e6))
PY

"""e2e probe: the host-buffer k-NNG call vs its parts (plain H2D of X, strided sample copy,
device-resident call), wall clock around blocking calls, headline shape."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1309_5478_b200 import knn, datagen
N, d, k = 65536, 256, 32
X = datagen.points(N, d, "uniform", seed=3)
Xh = torch.empty((N, d), dtype=torch.float32, pin_memory=True); Xh.copy_(torch.from_numpy(X)); Xn = Xh.numpy()
oi = torch.empty((N, k), dtype=torch.int32, pin_memory=True).numpy()
od = torch.empty((N, k), dtype=torch.float32, pin_memory=True).numpy()
Xd = torch.empty((N, d), dtype=torch.float32, device="cuda")
Sd = torch.empty((N // 8, d), dtype=torch.float32, device="cuda")
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
def t(f, n=10):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
print("H2D 64 MB contiguous  %.3f ms" % t(lambda: Xd.copy_(Xh, non_blocking=True)))
if cudart:
    def s2d():
        cudart.cudaMemcpy2DAsync(ctypes.c_void_p(Sd.data_ptr()), ctypes.c_size_t(d * 4), ctypes.c_void_p(Xh.data_ptr()),
                                 ctypes.c_size_t(8 * d * 4), ctypes.c_size_t(d * 4), ctypes.c_size_t(N // 8), 1,
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    print("H2D 8 MB strided sample %.3f ms" % t(s2d))
Xt = torch.from_numpy(X).cuda()
print("device-resident graph   %.3f ms" % t(lambda: knn.graph(Xt, k)))
print("host pipelined e2e      %.3f ms" % t(lambda: knn.search_block_host(Xn, Xn, k, self_shift=0, out=(oi, od))))
os.environ["KNN_HOST_PIPE"] = "0"
print("host unpipelined e2e    %.3f ms" % t(lambda: knn.search_block_host(Xn, Xn, k, self_shift=0, out=(oi, od))))

"""Host-link copy rates of the pipelined k-NNG's copy shapes (pinned host memory): contiguous
H2D of 8 MB, stride-8 row gathers (1 KB rows, 8 KB pitch) H2D, and D2H of 128-byte rows
scattered with an 1 KB pitch (k = 32 results), CUDA events on one stream."""
import ctypes, os, sys
import torch
N, d, k = 65536, 256, 32
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else \
    ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
s = torch.cuda.current_stream()
Xh = torch.empty((N, d), dtype=torch.float32, pin_memory=True)
Xd = torch.empty((N, d), dtype=torch.float32, device="cuda")
Oh = torch.empty((N, k), dtype=torch.int32, pin_memory=True)
Od = torch.empty((N, k), dtype=torch.int32, device="cuda")
S = N // 8
def cp2d(dst, dp, src, sp, w, h, kind):
    rc = cudart.cudaMemcpy2DAsync(ctypes.c_void_p(dst), ctypes.c_size_t(dp), ctypes.c_void_p(src), ctypes.c_size_t(sp),
                                  ctypes.c_size_t(w), ctypes.c_size_t(h), kind, ctypes.c_void_p(s.cuda_stream))
    assert rc == 0, rc
def timed(f, n=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
t1 = timed(lambda: Xd[:S].copy_(Xh[:S], non_blocking=True))
t2 = timed(lambda: cp2d(Xd.data_ptr(), d * 4, Xh.data_ptr(), 8 * d * 4, d * 4, S, 1))
t3 = timed(lambda: Oh[:S].copy_(Od[:S], non_blocking=True))
t4 = timed(lambda: cp2d(Oh.data_ptr(), 8 * k * 4, Od.data_ptr(), k * 4, k * 4, S, 2))
t5 = timed(lambda: Xd.copy_(Xh, non_blocking=True))
print(f"H2D 8 MB contiguous {t1:.3f} ms ({S*d*4/t1/1e6:.1f} GB/s); stride-8 rows {t2:.3f} ms ({S*d*4/t2/1e6:.1f} GB/s)")
print(f"D2H 1 MB contiguous {t3:.3f} ms ({S*k*4/t3/1e6:.1f} GB/s); 128 B rows, 1 KB pitch {t4:.3f} ms ({S*k*4/t4/1e6:.1f} GB/s)")
print(f"H2D 64 MB contiguous {t5:.3f} ms ({N*d*4/t5/1e6:.1f} GB/s)")

"""DIAGNOSTIC: partition GEMM time with parts of its epilogue disabled (KNN_DBG_EPI, set by
the caller, honoured only by a -DKNN_DIAG_EPI build: make BUILD=build_diag LIB=ablibs/diag.so
NVFLAGS_EXTRA=-DKNN_DIAG_EPI ablibs/diag.so, then KNN_LIB_PATH=ablibs/diag.so); results are
wrong and the call falls back, only the partition launch is read)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1309_5478_b200 import knn, datagen
X = torch.from_numpy(datagen.points(65536, 256, "uniform", seed=1309100)).cuda()
for _ in range(2):
    knn.graph(X, 32)
torch.cuda.synchronize()
knn.profile_enable(True)
for _ in range(10):
    knn.graph(X, 32)
torch.cuda.synchronize()
ms, n = knn.profile_read("fused")
print("dbg", os.environ.get("KNN_DBG_EPI", "0"), "partition ms", ms / max(n, 1))

import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1309_5478_b200 import knn, datagen
X = torch.from_numpy(datagen.points(16384, 64, "uniform", seed=1)).cuda()
knn.graph(X, 16)
torch.cuda.synchronize()
print("ok")

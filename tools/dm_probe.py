import sys, time
sys.path.insert(0, ".")
import torch
from paper_1808_01364_b200.grid import baseline_problem
from paper_1808_01364_b200 import factorization as gf
spec, A, _ = baseline_problem("c5", 0, None)
for _ in range(4):
    A._device = None
    torch.cuda.synchronize(); t = time.perf_counter()
    dm = gf.device_matrix(A, 0)
    torch.cuda.synchronize(); print("device_matrix %.1f ms" % ((time.perf_counter() - t) * 1e3))

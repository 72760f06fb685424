import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1711_10912_b200 as tl
rng = np.random.default_rng(0)
n = 2000
T = tl.DenseTensor.from_memory((n, n), rng.standard_normal(n * n))
u = tl.DenseTensor.from_memory((n,), rng.standard_normal(n))
tl.ttv(T, u, 1); tl.ttv(T, u, 2); torch.cuda.synchronize()
torch.cuda.profiler.start()
tl.ttv(T, u, 1); tl.ttv(T, u, 2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")

import os, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import workloads as W
T, v, M, layout = W.cfg5(0)
A5 = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, layout), layout=layout)
C1 = tl.ttv(A5, tl.DenseTensor.from_memory((9,), v), 5)
Bm = tl.DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)))
rng = np.random.default_rng(1)
X = tl.DenseTensor.from_memory((5, 37, 20001), rng.standard_normal((5, 37, 20001)).reshape(-1, order="F"))
Mx = tl.DenseTensor.from_memory((16, 37), rng.standard_normal((16, 37)).reshape(-1, order="F"))
for _ in range(2):
    tl.ttm(C1, Bm, 2); tl.ttm(X, Mx, 2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
tl.ttm(C1, Bm, 2); tl.ttm(X, Mx, 2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")

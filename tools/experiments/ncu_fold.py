"""One launch of the 400x400 COLS small fold inside a profiler window."""
import os, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R)
import numpy as np, torch
import paper_1711_10912_b200 as tl
rng = np.random.default_rng(0)
A = tl.DenseTensor.from_memory((400, 400), rng.standard_normal(160000))
v = tl.DenseTensor.from_memory((400,), rng.standard_normal(400))
for _ in range(3):
    tl.ttv(A, v, 2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
tl.ttv(A, v, 2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
